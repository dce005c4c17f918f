"""The diagonal-method baseline (reference diagonal.cpp) batched on the GPU
backend vs the reference's own diag_spmv on SimBackend (oracle/_ref): values,
ledger, transcript and model noise; plus the exact matvec."""
import numpy as np
import pytest

import paper_2603_04742_b200 as pk
import synth
from oracle_bindings import diag_reference

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def ctx11():
    return pk.Context(logn=11, seed=4)


def exact(m, v, t=65537):
    d = m.dense() @ np.asarray(v, np.int64)
    r = np.mod(d, t)
    return np.where(r > t // 2, r - t, r)


@pytest.mark.parametrize("n,nnz,seed", [(8, 20, 1), (64, 300, 2), (512, 2000, 3), (1024, 1500, 4), (500, 9000, 5)])
def test_diag_matches_reference(ctx11, n, nnz, seed):
    m = synth.random_sparse_csr(n, n, nnz, seed, -8, 8)
    v = synth.random_vector(n, seed, -8, 8, nonzero=True)
    got = pk.diag_spmv(ctx11, m, v)
    want = diag_reference(m, v, ctx11.slots)
    assert np.array_equal(got["values"], want["values"])
    assert np.array_equal(got["values"], exact(m, v))
    assert got["ledger"] == want["ledger"] and got["n_ct"] == want["n_ct"] and got["noise"] == want["noise"]
    assert [tuple(x) for x in got["messages"]] == [tuple(x) for x in want["messages"]]
    assert got["measured_noise"] > 0


def test_diag_edge_cases(ctx11):
    S = ctx11.slots
    z = pk.Csr.from_dense([[0, 0], [0, 0]])
    r = pk.diag_spmv(ctx11, z, [1, 2])
    assert list(r["values"]) == [0, 0] and r["n_ct"] == 0 and r["noise"] == 146
    full = synth.random_sparse_csr(S, S, 3 * S, 9, -8, 8)  # n == slot_count: natural wrap
    v = synth.random_vector(S, 9, -8, 8, nonzero=True)
    assert np.array_equal(pk.diag_spmv(ctx11, full, v)["values"], exact(full, v))
    with pytest.raises(pk.SpmvError) as e:  # non-square
        pk.diag_spmv(ctx11, pk.Csr.from_dense([[1, 2, 3], [4, 5, 6]]), [1, 2, 3])
    assert e.value.kind == "NonSquareError"
    m = synth.random_sparse_csr(S // 2 + 1, S // 2 + 1, 10, 1, -8, 8)
    with pytest.raises(pk.SpmvError) as e:  # S/2 < n < S
        pk.diag_spmv(ctx11, m, np.ones(S // 2 + 1, np.int64))
    assert e.value.kind == "OverLengthError"
    with pytest.raises(pk.SpmvError) as e:  # dimension
        pk.diag_spmv(ctx11, pk.Csr.from_dense([[1, 0], [0, 1]]), [1, 2, 3])
    assert e.value.kind == "DimensionMismatchError"
