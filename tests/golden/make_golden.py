"""Generate tests/golden/ref_cases.json from the UNMODIFIED reference library
(oracle/_ref/libspmv_ref.so, compiled in place from /root/reference/proj/src by
oracle/Makefile).  Each case stores its inputs explicitly (CSR arrays + vector)
and the reference's SimBackend outputs of spmv_partitioned: values, OpLedger,
transcript (kind, bytes, count) and model noise.  Matrices come from the
reference's own random_sparse_csr (proj/src/synthetic.cpp:32-72).

    python tests/golden/make_golden.py      # rewrites ref_cases.json
"""
import json
import sys
from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent
sys.path.insert(0, str(HERE.parent))
sys.path.insert(0, str(HERE.parent.parent))

from oracle_bindings import _i64, _p, i64p, ref_lib, sim_spmv_partitioned  # noqa: E402
import paper_2603_04742_b200 as pk  # noqa: E402


def ref_csr(L, rows, cols, nnz, seed, lo, hi):
    rp = np.zeros(rows + 1, np.int64)
    ci = np.zeros(max(nnz, 1), np.int64)
    va = np.zeros(max(nnz, 1), np.int64)
    n = L.ref_random_sparse_csr(rows, cols, nnz, seed, lo, hi, _p(rp, i64p), _p(ci, i64p), _p(va, i64p))
    assert n >= 0
    return pk.Csr(rows, cols, rp, ci[:n], va[:n])


def ref_vec(L, n, seed, lo, hi):
    out = np.zeros(max(n, 1), np.int64)
    L.ref_random_vector(n, seed, lo, hi, _p(out, i64p))
    return out[:n]


def case(L, name, m, v, S, chunk):
    r = sim_spmv_partitioned(m, v, S, chunk, lib=L)
    assert "error" not in r, (name, r)
    return {"name": name, "slot_count": S, "chunk": chunk, "rows": m.rows, "cols": m.cols,
            "row_ptrs": [int(x) for x in m.row_ptrs], "col_indices": [int(x) for x in m.col_indices],
            "values_in": [int(x) for x in m.values], "v": [int(x) for x in v],
            "values": [int(x) for x in r["values"]], "ledger": r["ledger"], "n_ct": r["n_ct"],
            "noise": r["noise"], "messages": [list(x) for x in r["messages"]]}


def main():
    L = ref_lib()
    assert L is not None, "build oracle/_ref first (make -C oracle ref)"
    cases = []
    # BASELINE config 1 (reference generator; vector from the reference's
    # random_vector with zeros replaced by 1, values in [-8,8]\{0})
    m = ref_csr(L, 256, 256, 655, 1, -8, 8)
    v = ref_vec(L, 256, 1, -8, 8)
    v[v == 0] = 1
    cases.append(case(L, "config1_256x256_1pct", m, v, 4096, 4096))
    # test_protocol.cpp:44-55 shapes (slot_count 128)
    for seed in range(900, 916):
        rows, cols = 1 + seed % 17, 1 + (seed * 3) % 19
        nnz = (rows * cols) // (1 + seed % 3)
        m = ref_csr(L, rows, cols, nnz, seed, -100, 100)
        cases.append(case(L, f"random_{seed}", m, ref_vec(L, cols, seed, -100, 100), 128, 128))
    # test_protocol.cpp:217-234 partitioned shapes (slot_count 32, budget 8)
    for seed in range(1200, 1210):
        rows, cols = 8 + seed % 70, 1 + (seed * 3) % 12
        m = ref_csr(L, rows, cols, rows * cols // 4, seed, -100, 100)
        cases.append(case(L, f"partitioned_{seed}", m, ref_vec(L, cols, seed, -100, 100), 32, 8))
    # edge cases (test_protocol.cpp:28-70)
    cases.append(case(L, "identity", pk.Csr.from_dense([[1, 0], [0, 1]]), np.array([5, -3]), 64, 64))
    cases.append(case(L, "one_cell", pk.Csr.from_dense([[3]]), np.array([4]), 16, 16))
    cases.append(case(L, "zero_rows", pk.Csr.from_dense([[0, 0], [7, 0], [0, 0]]), np.array([3, 9]), 32, 32))
    cases.append(case(L, "all_zero", pk.Csr.from_dense([[0, 0], [0, 0]]), np.array([3, 9]), 32, 32))
    # dense-ish matrix forcing multi-column chunks and deep schedules
    m = ref_csr(L, 40, 60, 900, 77, -8, 8)
    cases.append(case(L, "dense_40x60", m, ref_vec(L, 60, 77, -8, 8), 256, 256))
    (HERE / "ref_cases.json").write_text(json.dumps({"generator": "tests/golden/make_golden.py",
                                                     "reference": "oracle/_ref (SimBackend)",
                                                     "cases": cases}, separators=(",", ":")))
    print(len(cases), "cases")


if __name__ == "__main__":
    main()
