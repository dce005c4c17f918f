"""The drop-in boundary from C++ (SURVEY 8(b)): tests/native/backend_check.cpp
is compiled against include/spmv/*.hpp and linked with libcssc_he.so, as a
reference user would; it constructs spmv::GpuBfvBackend and drives every
HeBackend virtual (reference he.hpp:86-115) through the reference's own unit
cases (test_he.cpp:28-207) and the op-by-op aggregation (aggregate.cpp:36-74).
Here the ciphertext words it wrote are compared with the CPU RNS-BFV oracle
(oracle/bfv_oracle.c) and its values/ledgers with the reference semantics."""
import os
import subprocess
from pathlib import Path

import numpy as np
import pytest

import paper_2603_04742_b200 as pk
from oracle_bindings import BfvOracle, sim_spmv_partitioned

ROOT = Path(__file__).resolve().parent.parent
pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def run(tmp_path_factory):
    d = tmp_path_factory.mktemp("backend_check")
    exe = d / "backend_check"
    lib = ROOT / "paper_2603_04742_b200" / "lib"
    subprocess.run(["g++", "-std=c++20", "-O1", "-Wall", "-Wextra", f"-I{ROOT / 'include'}",
                    str(ROOT / "tests" / "native" / "backend_check.cpp"), f"-L{lib}", "-lcssc_he",
                    f"-Wl,-rpath,{lib}", "-o", str(exe)], check=True)
    r = subprocess.run([str(exe), str(d)], capture_output=True, text=True, timeout=600)
    out = {"rc": r.returncode, "stdout": r.stdout, "stderr": r.stderr, "words": {}, "ledger": {}, "slots": {}}
    for line in r.stdout.splitlines():
        f = line.split()
        if f[0] == "words":
            out["words"][f[1]] = np.fromfile(f[2], dtype=np.uint64)
        elif f[0] == "ledger":
            out["ledger"][f[1]] = tuple(int(x) for x in f[2:])
        elif f[0] == "slots":
            out["slots"][f[1]] = [int(x) for x in f[2:]]
    return out


def test_every_virtual_passes_the_reference_cases(run):
    assert run["rc"] == 0 and "failures 0" in run["stdout"], run["stdout"][-3000:] + run["stderr"][-3000:]
    assert "lifetime ok" in run["stdout"]


def test_measured_budget_falls_and_exhausts(run):
    lines = [x for x in run["stdout"].splitlines() if x.startswith("measured after")]
    budgets = [int(x.split()[-1]) for x in lines]
    assert budgets and budgets[-1] <= 0 and all(b > 0 for b in budgets[:-1])


def _chunks():
    r0, c0, r1, c1 = 3, 5, 7, 2
    a0 = np.array([(i % 17) - 8 for i in range(r0 * c0)], np.int64)
    b0 = np.array([(i % 13) - 6 for i in range(r0 * c0)], np.int64)
    a1 = np.array([(i % 11) - 5 for i in range(r1 * c1)], np.int64)
    b1 = np.array([(i % 7) - 3 for i in range(r1 * c1)], np.int64)
    return (r0, c0, a0, b0), (r1, c1, a1, b1)


def test_aggregate_words_equal_the_oracle(run):
    """intra_chunk_sum / inter_chunk_sum op by op over GpuBfvBackend: every
    checked ciphertext equals the oracle's op-by-op evaluation word for word."""
    p = pk.default_params(12)
    orc = BfvOracle(12, p.L, p.K, p.alpha, p.qbits, p.pbits, 65537, 11)
    (r0, c0, a0, b0), (r1, c1, a1, b1) = _chunks()
    ea0, eb0, ea1, eb1 = (orc.encrypt(x, s) for x, s in ((a0, 1), (b0, 2), (a1, 3), (b1, 4)))
    assert np.array_equal(run["words"]["agg_a0"], ea0)
    p0, p1 = orc.mul_relin(ea0, eb0), orc.mul_relin(ea1, eb1)
    assert np.array_equal(run["words"]["agg_p0"], p0)

    def fold(ct, r, c):
        sched = pk.rotation_schedule(r, c)
        for off, _ in sched:
            g = orc.galois_elt(off)
            if g != 1:
                orc.lib.bfvo_add_galois_key(orc.h, g)
        acc = ct
        for off, from_acc in sched:
            acc = orc.add(acc, orc.rotate(acc if from_acc else ct, off))
        return acc

    s0, s1 = fold(p0, r0, c0), fold(p1, r1, c1)
    assert np.array_equal(run["words"]["agg_s0"], s0)
    assert np.array_equal(run["words"]["agg_s1"], s1)
    res = orc.add(orc.mul_plain(s0, np.ones(r0, np.int64)), orc.mul_plain(s1, np.ones(r1, np.int64)))
    assert np.array_equal(run["words"]["agg_res"], res)
    slots, _ = orc.decrypt(res)
    assert list(slots[:16]) == run["slots"]["aggregate"]
    rot = len(pk.rotation_schedule(r0, c0)) + len(pk.rotation_schedule(r1, c1))
    # {cc, cp, rot, add, enc, dec}: aggregate.cpp adds once per rotation and once per part
    assert run["ledger"]["aggregate"] == (2, 2, rot, rot + 2, 4, 1)
    assert run["ledger"]["op_calls"] == (1, 1, 1, 1, 2, 1)


def test_protocol_from_cpp_matches_reference(run):
    m = pk.Csr(5, 4, np.array([0, 2, 2, 5, 6, 7]), np.array([0, 3, 0, 1, 2, 1, 3]),
               np.array([3, -2, 1, 4, -5, 7, 8]))
    want = sim_spmv_partitioned(m, np.array([2, -1, 3, 5]), 2048, 2048)
    led = want["ledger"]
    assert run["ledger"]["protocol"] == tuple(led[k] for k in ("n_mult_cc", "n_mult_cp", "n_rot", "n_add", "n_enc",
                                                              "n_dec"))
