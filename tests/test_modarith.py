"""Host check of the device modular reductions (csrc/modarith.cuh compiled
with g++): every Barrett product equals the exact 128-bit remainder."""
import shutil
import subprocess
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parent.parent


@pytest.mark.skipif(shutil.which("g++") is None, reason="needs g++")
def test_barrett_mul_mod_exact(tmp_path):
    exe = tmp_path / "modarith_check"
    subprocess.run(["g++", "-std=c++20", "-O2", f"-I{ROOT / 'paper_2603_04742_b200' / 'csrc'}",
                    str(ROOT / "tests" / "native" / "modarith_check.cpp"), "-o", str(exe)], check=True)
    out = subprocess.run([str(exe)], capture_output=True, text=True)
    assert out.returncode == 0, out.stdout + out.stderr
    assert out.stdout.startswith("0 / ")
