"""CSSC persistence: the reference stores a CSSC only as the
JSON `spmv convert` writes (tools/spmv_main.cpp:39-58).  The library's JSON
export equals that text byte for byte (the reference compiled with the same
nlohmann/json, oracle/_ref), and the compact binary form round-trips to the
reference's csr_to_cssc arrays and rejects malformed buffers (ParseError).
Host-only: no GPU needed."""
import ctypes as C
from pathlib import Path

import numpy as np
import pytest

import paper_2603_04742_b200 as pk
import synth
from oracle_bindings import _i64, _p, i64p, ref_lib

ROOT = Path(__file__).resolve().parent.parent


def tiny():  # tests/data/tiny.mtx of the reference: 4 x 5, 7 nonzeros
    d = [[1, 0, 0, 2, 0], [0, 0, 3, 0, 0], [4, 5, 0, 0, 6], [0, 0, 0, 0, 7]]
    return pk.Csr.from_dense(d)


CASES = [
    ("tiny", tiny),
    ("empty_rows", lambda: pk.Csr.from_dense([[0, 0, 0], [7, 0, -9], [0, 0, 0], [0, 5, 0]])),
    ("all_zero", lambda: pk.Csr.from_dense([[0, 0], [0, 0]])),
    ("uniform", lambda: synth.random_sparse_csr(300, 200, 1500, 42, -8, 8)),
    ("wide_values", lambda: synth.random_sparse_csr(50, 60, 400, 7, -100000, 100000)),
    ("power_law", lambda: synth.power_law_csr(2000, 12.0, 2.0, 3, -8, 8)),
]


def ref_cssc(m):
    L = ref_lib()
    rp, ci, va = _i64(m.row_ptrs), _i64(m.col_indices), _i64(m.values)
    if va.size == 0:
        ci = va = np.zeros(1, np.int64)
    L.ref_csr_to_cssc.restype = C.c_int64
    L.ref_csr_to_cssc.argtypes = [C.c_uint64, C.c_uint64] + [i64p] * 7 + [C.POINTER(C.c_uint64)]
    al = C.c_uint64()
    nnz = L.ref_csr_to_cssc(m.rows, m.cols, _p(rp, i64p), _p(ci, i64p), _p(va, i64p), None, None, None, None,
                            C.byref(al))
    o = [np.zeros(max(nnz, 1), np.int64), np.zeros(max(nnz, 1), np.int64), np.zeros(max(m.rows, 1), np.int64),
         np.zeros(al.value + 1, np.int64)]
    L.ref_csr_to_cssc(m.rows, m.cols, _p(rp, i64p), _p(ci, i64p), _p(va, i64p), *[_p(x, i64p) for x in o],
                      C.byref(al))
    return {"va": o[0][:nnz], "ci": o[1][:nnz], "rm": o[2][: m.rows], "cp": o[3][: al.value + 1]}


def ref_json(m):
    L = ref_lib()
    rp, ci, va = _i64(m.row_ptrs), _i64(m.col_indices), _i64(m.values)
    if va.size == 0:
        ci = va = np.zeros(1, np.int64)
    L.ref_cssc_json.restype = C.c_int64
    L.ref_cssc_json.argtypes = [C.c_uint64, C.c_uint64, i64p, i64p, i64p, C.c_char_p, C.c_uint64]
    n = L.ref_cssc_json(m.rows, m.cols, _p(rp, i64p), _p(ci, i64p), _p(va, i64p), None, 0)
    if n < 0:
        pytest.skip("reference shim built without nlohmann/json")
    buf = C.create_string_buffer(n)
    L.ref_cssc_json(m.rows, m.cols, _p(rp, i64p), _p(ci, i64p), _p(va, i64p), buf, n)
    return buf.raw[:n].decode()


@pytest.mark.skipif(ref_lib() is None, reason="reference library not built")
@pytest.mark.parametrize("name,make", CASES)
def test_json_equals_spmv_convert(name, make):
    """Same document as the reference's `spmv convert` (field order and every
    value); same text as stock nlohmann 3.11.3 `dump(2)`, which prints one
    array element per line like Python's json.dumps(indent=2).  (The only
    nlohmann copy in this image is cudnn-frontend's, patched to print integer
    arrays inline, so the text is compared against the stock layout.)"""
    import json

    m = make()
    ours = pk.cssc_to_json(m)
    ref = json.loads(ref_json(m))
    assert list(json.loads(ours).items()) == list(ref.items())
    assert ours == json.dumps(ref, indent=2) + "\n"


@pytest.mark.skipif(ref_lib() is None, reason="reference library not built")
@pytest.mark.parametrize("name,make", CASES)
def test_binary_roundtrip_equals_reference_cssc(name, make):
    m = make()
    data = pk.cssc_to_bytes(m)
    got = pk.cssc_from_bytes(data)
    want = ref_cssc(m)
    assert got["rows"] == m.rows and got["cols"] == m.cols
    for k in ("va", "ci", "rm", "cp"):
        assert np.array_equal(got[k], want[k]), k
    vw = data[5]
    span = max(1, int(np.abs(np.asarray(m.values)).max()) if len(m.values) else 1)
    assert vw == (1 if span < 128 else 2 if span < 32768 else 4)
    # denser than the reference's JSON (and than int64 CSR arrays)
    assert len(data) < len(pk.cssc_to_json(m).encode())


def test_binary_rejects_malformed():
    data = pk.cssc_to_bytes(tiny())
    for bad in (b"", data[:-1], b"CSSX" + data[4:], data[:5] + b"\x03" + data[6:]):
        with pytest.raises(pk.SpmvError) as e:
            pk.cssc_from_bytes(bad)
        assert e.value.kind == "ParseError"
    b = bytearray(data)
    b[-1] ^= 0x7F  # last column pointer no longer equals nnz
    with pytest.raises(pk.SpmvError) as e:
        pk.cssc_from_bytes(bytes(b))
    assert e.value.kind == "ParseError"
