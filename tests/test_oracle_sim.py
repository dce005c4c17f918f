"""Pin the C restatement of the reference path (oracle/sim_oracle.c) against
the reference's OWN golden vectors (proj/tests/test_*.cpp) and against the
fixtures generated from the compiled reference (tests/golden/ref_cases.json)."""
import ctypes as C
import json
from pathlib import Path

import numpy as np
import pytest

import paper_2603_04742_b200 as pk
import synth
from oracle_bindings import _i64, _p, _u64, i64p, ip, oracle_lib, sim_spmv_partitioned, u64p

GOLDEN = json.loads((Path(__file__).parent / "golden" / "ref_cases.json").read_text())["cases"]


def test_signed_residue_golden():  # test_he.cpp:50-59
    L = oracle_lib()
    assert L.simo_to_signed(0, 65537) == 0
    assert L.simo_to_signed(32768, 65537) == 32768
    assert L.simo_to_signed(32769, 65537) == -32768
    assert L.simo_to_signed(65536, 65537) == -1
    assert L.simo_to_residue(-1, 65537) == 65536
    assert L.simo_to_residue(-98, 97) == 96 and L.simo_to_residue(98, 97) == 1
    for v in range(-48, 49):
        assert L.simo_to_signed(L.simo_to_residue(v, 97), 97) == v


def rot(vals, k):
    a = _u64(vals)
    out = np.zeros_like(a)
    oracle_lib().simo_rotate(_p(a, u64p), k, a.size, _p(out, u64p))
    return list(out)


def test_rotation_golden():  # test_he.cpp:152-168
    x = [1, 2, 3, 4]
    assert rot(x, 1) == [2, 3, 4, 1]
    assert rot(x, -1) == [4, 1, 2, 3]
    assert rot(x, 0) == x and rot(x, 4) == x
    assert rot(x, 5) == [2, 3, 4, 1]
    assert rot(rot(x, 3), 1) == x


def sched(r, c):
    off = np.zeros(256, np.uint64)
    fa = (C.c_int * 256)()
    n = oracle_lib().simo_rotation_schedule(r, c, _p(off, u64p), fa)
    return [(int(off[i]), bool(fa[i])) for i in range(n)]


def test_schedule_golden():  # test_aggregate.cpp:45-65
    assert sched(10, 1) == []
    assert [o for o, _ in sched(7, 2)] == [7]
    assert [o for o, _ in sched(3, 4)] == [3, 6]
    for c in range(1, 201):
        for r in (1, 3, 16):
            s = sched(r, c)
            assert len(s) == c.bit_length() + bin(c).count("1") - 2
            assert all(o % r == 0 for o, _ in s)


def cssc(m):
    L = oracle_lib()
    maxn = int(np.max(np.diff(m.row_ptrs))) if m.rows else 0
    rm = np.zeros(max(m.rows, 1), np.int64)
    cp = np.zeros(maxn + 2, np.int64)
    va = np.zeros(max(m.nnz, 1), np.int64)
    ci = np.zeros(max(m.nnz, 1), np.int64)
    Lc = L.simo_csr_to_cssc(m.rows, _p(_i64(m.row_ptrs), i64p), _p(_i64(m.col_indices) if m.nnz else ci, i64p),
                            _p(_i64(m.values) if m.nnz else va, i64p), _p(rm, i64p), _p(cp, i64p), _p(va, i64p),
                            _p(ci, i64p))
    return list(rm[: m.rows]), list(cp[: Lc + 1]), list(va[: m.nnz]), list(ci[: m.nnz])


def test_cssc_golden():  # test_sparse.cpp:55-80
    rm, cp, va, ci = cssc(pk.Csr.from_dense([[1, 0, 0], [0, 1, 0], [0, 0, 1]]))
    assert (rm, cp, va, ci) == ([0, 1, 2], [0, 3], [1, 1, 1], [0, 1, 2])
    rm, cp, va, ci = cssc(pk.Csr.from_dense([[3, 0, 0], [1, 2, 0], [0, 0, 4]]))
    assert rm == [1, 0, 2] and cp == [0, 3, 4] and va == [1, 3, 4, 2]


def heights_matrix(heights):  # test_chunk.cpp:16-26
    rows, cols = heights[0], len(heights)
    d = np.zeros((rows, cols), np.int64)
    for j, h in enumerate(heights):
        for i in range(h):
            d[i, j] = 10 * (j + 1) + i + 1
    return pk.Csr.from_dense(d)


def chunks(m, budget):
    L = oracle_lib()
    rm, cp, va, ci = (_i64(x) for x in cssc(m))
    Lc = len(cp) - 1
    n = L.simo_generate_chunks(Lc, _p(cp, i64p), _p(va, i64p), _p(ci, i64p), budget, None, None, None, None, None)
    if n < 0:
        return None
    r = np.zeros(n + 1, np.int64)
    c = np.zeros(n + 1, np.int64)
    fo = np.zeros(n + 2, np.int64)
    L.simo_generate_chunks(Lc, _p(cp, i64p), _p(va, i64p), _p(ci, i64p), budget, _p(r, i64p), _p(c, i64p),
                           _p(fo, i64p), None, None)
    vf = np.zeros(int(fo[n]) + 1, np.int64)
    cf = np.zeros(int(fo[n]) + 1, np.int64)
    L.simo_generate_chunks(Lc, _p(cp, i64p), _p(va, i64p), _p(ci, i64p), budget, _p(r, i64p), _p(c, i64p),
                           _p(fo, i64p), _p(vf, i64p), _p(cf, i64p))
    return list(r[:n]), list(c[:n]), [list(vf[fo[i]:fo[i + 1]]) for i in range(n)], [list(cf[fo[i]:fo[i + 1]]) for i in range(n)]


def test_chunk_golden():  # test_chunk.cpp:62-104
    r, c, vf, cf = chunks(heights_matrix([4, 2, 1]), 8)
    assert r == [4, 1] and c == [2, 1]
    assert vf[0] == [11, 12, 13, 14, 21, 22, 0, 0] and cf[0] == [0, 0, 0, 0, 1, 1, -1, -1]
    assert vf[1] == [31] and cf[1] == [2]
    r, c, _, _ = chunks(heights_matrix([3, 2, 1]), 6)
    assert c == [2, 1]
    assert chunks(heights_matrix([9]), 8) is None  # ColumnTooTallError


def test_protocol_golden_small():  # test_protocol.cpp:28-70, 138-167
    r = sim_spmv_partitioned(pk.Csr.from_dense([[1, 0], [0, 1]]), [5, -3], 64)
    assert list(r["values"]) == [5, -3] and r["n_ct"] == 1
    assert list(sim_spmv_partitioned(pk.Csr.from_dense([[3]]), [4], 16)["values"]) == [12]
    r = sim_spmv_partitioned(pk.Csr.from_dense([[0, 0], [7, 0], [0, 0]]), [3, 9], 32)
    assert list(r["values"]) == [0, 21, 0]
    z = sim_spmv_partitioned(pk.Csr.from_dense([[0, 0], [0, 0]]), [3, 9], 32)
    assert list(z["values"]) == [0, 0] and z["n_ct"] == 0 and z["noise"] == 146
    m = synth.random_sparse_csr(6, 7, 20, 77)
    r = sim_spmv_partitioned(m, synth.random_vector(7, 77), 64, 16)
    kinds = [x[2] for x in r["messages"]]
    assert kinds == [0, 1, 2, 0, 3]
    assert r["messages"][0][3] == round(r["n_ct"] * 0.52 * 1048576)  # protocol.cpp:51-54
    assert r["messages"][4][3] == 545260  # one 0.52 MB result ciphertext
    assert r["noise"] == 87


@pytest.mark.parametrize("case", GOLDEN, ids=[c["name"] for c in GOLDEN])
def test_restatement_matches_reference_fixtures(case):
    m = pk.Csr(case["rows"], case["cols"], np.array(case["row_ptrs"], np.int64),
               np.array(case["col_indices"], np.int64), np.array(case["values_in"], np.int64))
    r = sim_spmv_partitioned(m, np.array(case["v"], np.int64), case["slot_count"], case["chunk"])
    assert [int(x) for x in r["values"]] == case["values"]
    assert r["ledger"] == case["ledger"]
    assert r["n_ct"] == case["n_ct"] and r["noise"] == case["noise"]
    assert [list(x) for x in r["messages"]] == case["messages"]
