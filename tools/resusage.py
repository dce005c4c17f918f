"""Registers / stack / spills per kernel of the built library (cuobjdump -res-usage).
usage: python tools/resusage.py [substring]"""
import re
import subprocess
import sys
from pathlib import Path

lib = Path(__file__).resolve().parent.parent / "paper_2603_04742_b200" / "lib" / "libcssc_he.so"
out = subprocess.run(["cuobjdump", "-res-usage", str(lib)], capture_output=True, text=True).stdout
name = None
for line in out.splitlines():
    m = re.search(r"Function (\S+):", line)
    if m:
        name = m.group(1)
        continue
    if name and "REG:" in line:
        dem = subprocess.run(["c++filt", name], capture_output=True, text=True).stdout.strip()
        dem = dem.replace("cssc::", "").split("(")[0]
        if len(sys.argv) < 2 or sys.argv[1] in dem:
            reg = re.search(r"REG:(\d+)", line).group(1)
            st = re.search(r"STACK:(\d+)", line).group(1)
            print(f"{dem:60s} REG {reg:>4s} STACK {st}")
        name = None
