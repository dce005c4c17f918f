"""C-ABI boundary and host-side logic, CPU only (no compute call needs a GPU):
the native library loads, exports every symbol include/spmvgpu.h declares, and
its host algorithms (CSSC pack, chunker, rotation plan, generators, parameter
derivation) agree with the reference / the oracle."""
import ctypes as C
import re
from pathlib import Path

import numpy as np
import pytest

import paper_2603_04742_b200 as pk
import synth
from oracle_bindings import BfvOracle, _i64, _p, i64p, ip, ref_lib, sim_spmv_partitioned, u64p

ROOT = Path(__file__).resolve().parent.parent


def declared_symbols():
    text = (ROOT / "include" / "spmvgpu.h").read_text()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"\b((?:spmvgpu|cssc)_[a-z0-9_]+)\s*\(", text)))


def test_library_exports_every_declared_symbol():
    lib = pk.lib()
    syms = declared_symbols()
    assert len(syms) >= 45
    for s in syms:
        assert hasattr(lib, s), s
    assert set(syms) == set(pk._SIGS), set(syms) ^ set(pk._SIGS)


def test_no_oracle_in_product():
    """The product never links or loads the checkers."""
    banned = ("liboracle", "libspmv_ref", "oracle_bindings", "bfvo_", "simo_", "ref_spmv", "bfv_oracle.h")
    for f in list((ROOT / "paper_2603_04742_b200").rglob("*")) + list((ROOT / "include").rglob("*")):
        if f.suffix in (".py", ".cu", ".cpp", ".cuh", ".hpp", ".h") and f.name != "build.py":
            t = f.read_text()
            for b in banned:
                assert b not in t, (f, b)
    nm = __import__("subprocess").run(["nm", "-D", str(pk.LIB_PATH)], capture_output=True, text=True).stdout
    assert "bfvo_" not in nm and "simo_" not in nm and "ref_spmv" not in nm


def test_default_params_and_security_budget():
    for logn, maxbits in ((13, 218), (14, 438), (15, 881)):
        p = pk.default_params(logn)
        assert p.L * p.qbits + p.K * p.pbits <= maxbits
        assert p.K >= p.alpha


@pytest.mark.skipif(ref_lib() is None, reason="reference library not built")
def test_generators_match_reference():
    L = ref_lib()
    for rows, cols, nnz, seed in ((256, 256, 655, 1), (4096, 4096, 16777, 2), (2048, 2048, 20972, 500),
                                  (2048, 2048, 20972, 563), (30, 40, 700, 9), (5, 5, 20, 3), (7, 9, 0, 4)):
        m = synth.random_sparse_csr(rows, cols, nnz, seed, -8, 8)
        rp = np.zeros(rows + 1, np.int64)
        ci = np.zeros(max(nnz, 1), np.int64)
        va = np.zeros(max(nnz, 1), np.int64)
        assert L.ref_random_sparse_csr(rows, cols, nnz, seed, -8, 8, _p(rp, i64p), _p(ci, i64p), _p(va, i64p)) == nnz
        assert np.array_equal(m.row_ptrs, rp) and np.array_equal(m.col_indices, ci[:nnz])
        assert np.array_equal(m.values, va[:nnz])
    out = np.zeros(100, np.int64)
    L.ref_random_vector(100, 5, -8, 8, _p(out, i64p))
    assert np.array_equal(synth.random_vector(100, 5, -8, 8), out)


def test_product_carries_no_generator():
    """Input generation is bench/test data (synth.py), not part of the library."""
    nm = __import__("subprocess").run(["nm", "-D", "--defined-only", str(pk.LIB_PATH)], capture_output=True,
                                      text=True).stdout
    for bad in ("random_sparse_csr", "random_vector", "power_law", "stencil27", "mt19937"):
        assert bad not in nm, bad
    assert "import synth" not in (ROOT / "paper_2603_04742_b200" / "__init__.py").read_text()


def test_batch_vector_count_mismatch_raises():
    m = synth.random_sparse_csr(6, 5, 10, 1, -8, 8)
    with pytest.raises(pk.SpmvError) as e:
        pk._vectors([m, m], [np.ones(5)], [])
    assert e.value.kind == "DimensionMismatchError"


def test_config_generators_shapes():
    assert synth.stencil27_csr(32, 4).nnz == 830584  # 94^3, boundary-truncated 27-point stencil
    p = synth.power_law_csr(16384, 12.0, 2.0, 3)
    assert 150_000 < p.nnz < 250_000
    v = synth.random_vector(1000, 3, -8, 8, nonzero=True)
    assert (v != 0).all() and v.min() >= -8 and v.max() <= 8


def ref_chunks(m, budget):
    L = ref_lib()
    tot = C.c_uint64()
    rp, ci, va = _i64(m.row_ptrs), _i64(m.col_indices), _i64(m.values)
    if va.size == 0:
        ci = va = np.zeros(1, np.int64)
    n = L.ref_chunks(m.rows, m.cols, _p(rp, i64p), _p(ci, i64p), _p(va, i64p), budget, None, None, None, None,
                     None, C.byref(tot))
    if n < 0:
        return n
    r = np.zeros(max(n, 1), np.int64)
    c = np.zeros(max(n, 1), np.int64)
    vf = np.zeros(max(tot.value, 1), np.int64)
    cf = np.zeros(max(tot.value, 1), np.int64)
    rm = np.zeros(max(m.rows, 1), np.int64)
    L.ref_chunks(m.rows, m.cols, _p(rp, i64p), _p(ci, i64p), _p(va, i64p), budget, _p(r, i64p), _p(c, i64p),
                 _p(vf, i64p), _p(cf, i64p), _p(rm, i64p), C.byref(tot))
    return {"n_ct": n, "r": r[:n], "c": c[:n], "vflat": vf[: tot.value], "cflat": cf[: tot.value],
            "row_map": rm[: m.rows]}


@pytest.mark.skipif(ref_lib() is None, reason="reference library not built")
@pytest.mark.parametrize("shape", [(256, 256, 655, 1, 4096), (4096, 4096, 16777, 2, 8192), (60, 70, 900, 3, 64),
                                   (8, 8, 64, 4, 8), (100, 3, 150, 5, 128)])
def test_pack_matches_reference(shape):
    rows, cols, nnz, seed, budget = shape
    m = synth.random_sparse_csr(rows, cols, nnz, seed, -8, 8)
    got = pk.pack_chunks(m, budget)
    want = ref_chunks(m, budget)
    for k in ("r", "c", "vflat", "cflat", "row_map"):
        assert np.array_equal(got[k], want[k]), k


def test_pack_large_configs_consistent():
    """C3 (power law, 2 slices) and C4 (stencil) pack invariants at full size."""
    for m, S in ((synth.power_law_csr(16384, 12.0, 2.0, 3), 8192), (synth.stencil27_csr(32, 4), 16384)):
        for r0 in range(0, m.rows, S):
            r1 = min(m.rows, r0 + S)
            b, e = int(m.row_ptrs[r0]), int(m.row_ptrs[r1])
            sl = pk.Csr(r1 - r0, m.cols, m.row_ptrs[r0: r1 + 1] - b, m.col_indices[b:e], m.values[b:e])
            pc = pk.pack_chunks(sl, S)
            assert (pc["r"] * pc["c"] <= S).all()
            assert int((pc["cflat"] >= 0).sum()) == sl.nnz
            assert sorted(pc["row_map"].tolist()) == list(range(sl.rows))


@pytest.mark.skipif(ref_lib() is None, reason="reference library not built")
def test_rotation_schedule_matches_reference():
    L = ref_lib()
    off = np.zeros(128, np.uint64)
    fa = (C.c_int * 128)()
    for r in (1, 3, 243, 4096):
        for c in list(range(1, 70)) + [2713, 8191, 8192]:
            if r * c > 16384:
                continue
            n = L.ref_rotation_schedule(r, c, _p(off, u64p), fa)
            assert pk.rotation_schedule(r, c) == [(int(off[i]), bool(fa[i])) for i in range(n)]


def test_error_codes_map_to_reference_exceptions():
    m = pk.Csr.from_dense([[1], [2], [3]])
    with pytest.raises(pk.SpmvError) as e:
        pk.pack_chunks(m, 2)
    assert e.value.kind == "ColumnTooTallError"
    with pytest.raises(pk.SpmvError) as e:
        pk.rotation_schedule(0, 3)
    assert e.value.kind == "ValueError"


def test_context_creation_fails_loudly_without_gpu():
    import torch
    if torch.cuda.is_available():
        pytest.skip("GPU present")
    with pytest.raises(pk.SpmvError) as e:
        pk.Context(logn=10)
    assert e.value.kind == "RuntimeError"
