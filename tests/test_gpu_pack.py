"""Device packing (spmvgpu_encrypt_cssc, k_pack_cssc) against the host packing
that mirrors the reference (csr_to_cssc + generate_chunks + reorg_vector,
checked against the compiled reference in test_capi.py): decrypting the
packed ciphertexts must give exactly the reference's chunk plaintexts."""
import numpy as np
import pytest

import paper_2603_04742_b200 as pk
import synth

pytestmark = pytest.mark.gpu
T = 65537


def descriptors(m, budget):
    """Python restatement of BatchedSpmv::add_slice for one slice."""
    rp = m.row_ptrs
    lens = np.diff(rp)
    order = sorted(range(m.rows), key=lambda i: (-lens[i], i))  # stable, longest first
    max_len = int(lens.max()) if m.rows else 0
    height = [int((lens > j).sum()) for j in range(max_len)]
    cols, r_list, c_list = [], [], []
    first = 0
    while first < max_len:
        h = height[first]
        fit = min(budget // h, max_len - first)
        for k in range(fit):
            cols.append((len(r_list), k, h, 0))
        r_list.append(h)
        c_list.append(fit)
        first += fit
    rows = [(int(rp[i]), int(lens[i]), p, 0) for p, i in enumerate(order) if lens[i]]
    return (np.array(rows, np.int32).reshape(-1, 4), np.array([[0, 0]], np.int32),
            np.array(cols, np.int32).reshape(-1, 4), r_list, c_list)


@pytest.fixture(scope="module")
def ctx():
    return pk.Context(logn=11, seed=9)


@pytest.mark.parametrize("seed", [1, 2, 3, 4])
def test_device_pack_equals_reference_chunks(ctx, seed):
    rng = np.random.default_rng(seed)
    rows, ncols = int(rng.integers(20, 300)), int(rng.integers(20, 300))
    nnz = int(rng.integers(1, rows * 4))
    m = synth.random_sparse_csr(rows, ncols, min(nnz, rows * ncols), seed, -9, 9)
    v = synth.random_vector(ncols, seed, -9, 9)
    budget = ctx.slots if seed % 2 else max(int(np.diff(m.row_ptrs).astype(bool).sum()), 64)
    ref = pk.pack_chunks(m, budget)
    rows_d, slices_d, cols_d, r_list, c_list = descriptors(m, budget)
    assert r_list == list(ref["r"]) and c_list == list(ref["c"])
    n = len(r_list)
    cts = ctx.encrypt_cssc(m.col_indices, m.values, v, rows_d, slices_d, cols_d, n)
    slots, _ = ctx.decrypt(cts)
    ctx.free(cts)
    off = 0
    for i in range(n):
        size = r_list[i] * c_list[i]
        vf = ref["vflat"][off:off + size]
        cf = ref["cflat"][off:off + size]
        off += size
        want_a = np.zeros(ctx.slots, np.int64)
        want_a[:size] = np.mod(vf, T)
        want_b = np.zeros(ctx.slots, np.int64)
        want_b[:size] = np.where(cf >= 0, np.mod(v[np.maximum(cf, 0)], T), 0)
        assert np.array_equal(slots[i].astype(np.int64), want_a)
        assert np.array_equal(slots[n + i].astype(np.int64), want_b)


def test_device_pack_rejects_bad_descriptors(ctx):
    m = synth.random_sparse_csr(30, 30, 90, 5, -9, 9)
    v = synth.random_vector(30, 5, -9, 9)
    rows_d, slices_d, cols_d, r_list, _ = descriptors(m, ctx.slots)
    n = len(r_list)
    bad = rows_d.copy()
    bad[0, 0] = m.values.size  # entry range past nnz
    with pytest.raises(pk.SpmvError):
        ctx.encrypt_cssc(m.col_indices, m.values, v, bad, slices_d, cols_d, n)
    bad = cols_d.copy()
    bad[0, 2] = ctx.slots + 1  # chunk taller than the slots
    with pytest.raises(pk.SpmvError):
        ctx.encrypt_cssc(m.col_indices, m.values, v, rows_d, slices_d, bad, n)
    ci = m.col_indices.copy()
    ci[0] = 30  # column outside the vector
    with pytest.raises(pk.SpmvError):
        ctx.encrypt_cssc(ci, m.values, v, rows_d, slices_d, cols_d, n)
    with pytest.raises(pk.SpmvError):
        ctx.encrypt_cssc(m.col_indices, m.values, v, rows_d, slices_d, cols_d, 0)


@pytest.mark.parametrize("logn,seed", [(11, 1), (14, 2)])
def test_forked_encryption_gives_the_staged_words(logn, seed):
    """The two-branch encryption of the cached whole-evaluation graph (upload +
    pack beside the message-independent part, bfv_context.cu
    encrypt_cssc_forked) produces the staged path's ciphertext words: two
    contexts with the same seed hand out the same stream ids."""
    a, b = pk.Context(logn=logn, seed=4), pk.Context(logn=logn, seed=4)
    b.set_option("forked_encrypt", 1)
    m = synth.random_sparse_csr(200, 150, 900, seed, -8, 8)
    v = synth.random_vector(150, seed, -8, 8)
    rows_d, slices_d, cols_d, r_list, _ = descriptors(m, a.slots)
    n = len(r_list)
    ca = a.encrypt_cssc(m.col_indices, m.values, v, rows_d, slices_d, cols_d, n)
    cb = b.encrypt_cssc(m.col_indices, m.values, v, rows_d, slices_d, cols_d, n)
    for x, y in zip(ca, cb):
        assert np.array_equal(a.download(int(x)), b.download(int(y)))
    a.close()
    b.close()
