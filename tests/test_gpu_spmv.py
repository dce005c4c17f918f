"""End-to-end encrypted SpMV on the GPU backend vs the reference semantics (P1-P4).

The checker is the reference library itself (oracle/_ref, compiled from
/root/reference) when present, else the C restatement (oracle/sim_oracle.c);
both run SimBackend with slot_count = S = N/2."""
import numpy as np
import pytest

import paper_2603_04742_b200 as pk
import synth
from oracle_bindings import ref_lib, sim_spmv_partitioned

pytestmark = pytest.mark.gpu


def checker(m, v, S, chunk):
    lib = ref_lib()
    return sim_spmv_partitioned(m, v, S, chunk, lib=lib)


@pytest.fixture(scope="module")
def ctx10():
    return pk.Context(logn=10, seed=3)


@pytest.fixture(scope="module")
def ctx13():
    return pk.Context(logn=13, seed=1)


def assert_same(got, want):
    assert np.array_equal(got["values"], want["values"])
    assert got["ledger"] == want["ledger"]
    assert got["n_ct"] == want["n_ct"]
    assert got["noise"] == want["noise"]
    if "messages" in got:
        assert got["messages"] == want["messages"]


@pytest.mark.parametrize("seed", range(900, 912))
def test_random_small_instances(ctx10, seed):
    rows, cols = 1 + seed % 17, 1 + (seed * 3) % 19
    nnz = (rows * cols) // (1 + seed % 3)
    m = synth.random_sparse_csr(rows, cols, nnz, seed)
    v = synth.random_vector(cols, seed)
    got = pk.spmv_partitioned(ctx10, m, v, ctx10.slots)
    assert_same(got, checker(m, v, ctx10.slots, ctx10.slots))
    assert got["measured_noise"] > 0 or got["n_ct"] == 0


@pytest.mark.parametrize("seed", range(1200, 1206))
def test_partitioned_small_budget(ctx10, seed):
    rows, cols = 8 + seed % 70, 1 + (seed * 3) % 12
    m = synth.random_sparse_csr(rows, cols, rows * cols // 4, seed)
    v = synth.random_vector(cols, seed)
    got = pk.spmv_partitioned(ctx10, m, v, 8)
    assert_same(got, checker(m, v, ctx10.slots, 8))


def test_edge_cases(ctx10):
    S = ctx10.slots
    zeros = pk.Csr.from_dense([[0, 0], [0, 0]])
    r = pk.spmv_partitioned(ctx10, zeros, [3, 9], S)
    assert list(r["values"]) == [0, 0] and r["n_ct"] == 0 and r["noise"] == 146
    m = pk.Csr.from_dense([[0, 0], [7, 0], [0, 0]])
    assert list(pk.spmv_partitioned(ctx10, m, [3, 9], S)["values"]) == [0, 21, 0]
    ident = pk.Csr.from_dense([[1, 0], [0, 1]])
    r = pk.spmv_partitioned(ctx10, ident, [5, -3], S)
    assert list(r["values"]) == [5, -3] and r["noise"] == 87
    empty = pk.Csr(0, 4, np.zeros(1, np.int64), np.zeros(0, np.int64), np.zeros(0, np.int64))
    assert pk.spmv_partitioned(ctx10, empty, [1, 2, 3, 4], 8)["values"].size == 0
    with pytest.raises(pk.SpmvError) as e:
        pk.spmv_partitioned(ctx10, ident, [1, 2, 3], S)
    assert e.value.kind == "DimensionMismatchError"
    with pytest.raises(pk.SpmvError) as e:
        pk.spmv_partitioned(ctx10, ident, [1, 2], S + 1)
    assert e.value.kind == "ValueError"


def test_config1_matches_reference(ctx13):
    """BASELINE config 1: 256x256, 1% density, values in [-8,8]\\{0}, N=8192."""
    m = synth.random_sparse_csr(256, 256, 655, 1, -8, 8)
    v = synth.random_vector(256, 1, -8, 8, nonzero=True)
    got = pk.spmv_partitioned(ctx13, m, v)
    want = checker(m, v, ctx13.slots, ctx13.slots)
    assert_same(got, want)
    dense = m.dense()
    exact = (dense @ v) % 65537
    exact = np.where(exact > 32768, exact - 65537, exact)
    assert np.array_equal(got["values"], exact)


def test_batch_equals_individual_runs(ctx10):
    ms = [synth.random_sparse_csr(40, 40, 120, s, -8, 8) for s in range(500, 506)]
    vs = [synth.random_vector(40, s, -8, 8, nonzero=True) for s in range(500, 506)]
    batch = pk.spmv_batch(ctx10, ms, vs, 32)
    for m, v, b in zip(ms, vs, batch):
        want = checker(m, v, ctx10.slots, 32)
        assert np.array_equal(b["values"], want["values"])
        assert b["ledger"] == want["ledger"]


def test_job_graph_replay(ctx10):
    ms = [synth.random_sparse_csr(60, 50, 300, s, -8, 8) for s in range(7, 10)]
    vs = [synth.random_vector(50, s, -8, 8, nonzero=True) for s in range(7, 10)]
    job = pk.Job(ctx10, ms, vs)
    job.encrypt()
    for _ in range(3):
        job.cloud(graph=True)
    res = job.finish()
    for m, v, r in zip(ms, vs, res):
        assert np.array_equal(r["values"], checker(m, v, ctx10.slots, ctx10.slots)["values"])
    st = job.stats()
    assert st["chunks"] > 0 and st["limb_ntts_per_run"] > 0
    ph = job.profile()
    assert ph[0]["name"] == "multiply+relin" and ph[-1]["name"] == "mask accumulate"
    assert len([p for p in ph if p["name"].startswith("rotate level")]) == st["levels"]
    assert all(p["us"] > 0 and p["bytes"] > 0 for p in ph)
    # the profiled replay leaves the same result behind
    res = job.finish()
    for m, v, r in zip(ms, vs, res):
        assert np.array_equal(r["values"], checker(m, v, ctx10.slots, ctx10.slots)["values"])


@pytest.mark.parametrize("capacity", [4, 1, 0])
def test_plan_cache_reuse_with_new_values(capacity):
    """Repeated calls over one sparsity structure reuse the cached plan (and its
    graph from the second use); every call still encrypts its own values."""
    ctx = pk.Context(logn=10, seed=5)
    ctx.set_option("plan_cache", capacity)
    rng = np.random.default_rng(capacity)
    shapes = [synth.random_sparse_csr(70, 60, 400, 31, -8, 8), synth.random_sparse_csr(50, 90, 200, 32, -8, 8)]
    for it in range(6):
        base = shapes[it % 2] if it < 4 else shapes[0]
        vals = rng.integers(1, 9, base.values.size) * rng.choice([-1, 1], base.values.size)
        m = pk.Csr(base.rows, base.cols, base.row_ptrs, base.col_indices, vals.astype(np.int64))
        v = rng.integers(-8, 9, base.cols).astype(np.int64)
        got = pk.spmv_partitioned(ctx, m, v, ctx.slots)
        assert_same(got, checker(m, v, ctx.slots, ctx.slots))
    ctx.close()


GOLDEN = __import__("json").loads(
    (__import__("pathlib").Path(__file__).parent / "golden" / "ref_cases.json").read_text())["cases"]


@pytest.mark.parametrize("case", GOLDEN, ids=[c["name"] for c in GOLDEN])
def test_matches_reference_fixtures(ctx10, ctx13, case):
    """Committed outputs of the compiled reference (tests/golden/make_golden.py);
    values are independent of slot_count once chunk_size is fixed."""
    ctx = ctx13 if case["chunk"] > ctx10.slots else ctx10
    m = pk.Csr(case["rows"], case["cols"], np.array(case["row_ptrs"], np.int64),
               np.array(case["col_indices"], np.int64), np.array(case["values_in"], np.int64))
    got = pk.spmv_partitioned(ctx, m, np.array(case["v"], np.int64), case["chunk"])
    assert [int(x) for x in got["values"]] == case["values"]
    assert got["ledger"] == case["ledger"] and got["n_ct"] == case["n_ct"] and got["noise"] == case["noise"]
    assert [list(x) for x in got["messages"]] == case["messages"]


@pytest.mark.parametrize("world", [2, 3])
def test_chunk_split_shards_sum_to_the_full_result(world):
    """the chunks of one matrix split over `world` shards (evaluated
    here one after another on one GPU); the summed partial results, folded mod
    q, decrypt to the reference's values, ledger, transcript and noise."""
    ctx = pk.Context(logn=10, seed=8)
    m = synth.random_sparse_csr(1300, 700, 6000, 77, -8, 8)  # 3 slices of 512 rows, several chunks each
    v = synth.random_vector(700, 77, -8, 8, nonzero=True)
    from paper_2603_04742_b200 import shard
    total = None
    jobs = []
    for r in range(world):
        job = pk.Job(ctx, [m], [v], rank=r, world=world)
        job.encrypt()
        job.cloud(graph=r == 0)
        w = job.result_words()
        total = w if total is None else total + w
        jobs.append(job)
    folded = shard.fold_mod(total, ctx.primes, ctx.L, ctx.n)
    got = jobs[0].finish_words(folded)[0]
    want = checker(m, v, ctx.slots, ctx.slots)
    assert np.array_equal(got["values"], want["values"])
    assert got["ledger"] == want["ledger"] and got["n_ct"] == want["n_ct"] and got["noise"] == want["noise"]
    with pytest.raises(pk.SpmvError):  # a shard alone cannot decrypt its partial slices
        jobs[1].finish()
    for j in jobs:
        j.close()
    ctx.close()


@pytest.mark.parametrize("world", [2, 3])
def test_chunk_split_device_reduction(world):
    """The device path of the chunk split: each shard copies its partial result
    ciphertexts into a device buffer (what NCCL all-reduces across GPUs), the
    buffers are summed on the device, and the library folds mod q on the GPU and
    decrypts; equals the reference, and the fold equals the host fold."""
    import torch

    ctx = pk.Context(logn=10, seed=8)
    m = synth.random_sparse_csr(1300, 700, 6000, 78, -8, 8)
    v = synth.random_vector(700, 78, -8, 8, nonzero=True)
    from paper_2603_04742_b200 import shard
    total, host_total, jobs = None, None, []
    for r in range(world):
        job = pk.Job(ctx, [m], [v], rank=r, world=world)
        job.encrypt()
        job.cloud(graph=False)
        d = job.result_words_dev()
        total = d if total is None else total + d  # the all-reduce's int64 sum
        w = job.result_words()
        host_total = w if host_total is None else host_total + w
        jobs.append(job)
    torch.cuda.synchronize()
    assert np.array_equal(total.cpu().numpy().view(np.uint64).reshape(host_total.shape), host_total)
    got = jobs[0].finish_words_dev(total)[0]
    folded = shard.fold_mod(host_total, ctx.primes, ctx.L, ctx.n)
    assert np.array_equal(total.cpu().numpy().view(np.uint64).reshape(folded.shape), folded)
    want = checker(m, v, ctx.slots, ctx.slots)
    assert np.array_equal(got["values"], want["values"])
    assert got["ledger"] == want["ledger"] and got["noise"] == want["noise"]
    for j in jobs:
        j.close()
    ctx.close()


def test_context_shared_across_host_threads():
    """a backend may be shared by host threads; calls on one
    context serialise and every result stays the reference's."""
    from concurrent.futures import ThreadPoolExecutor

    ctx = pk.Context(logn=10, seed=12)
    cases = [(synth.random_sparse_csr(90, 70, 500, s, -8, 8), synth.random_vector(70, s, -8, 8, nonzero=True))
             for s in range(40, 52)]

    def run(i):
        m, v = cases[i % len(cases)]
        return i, pk.spmv_partitioned(ctx, m, v, ctx.slots)

    with ThreadPoolExecutor(max_workers=6) as ex:
        results = list(ex.map(run, range(36)))
    for i, got in results:
        m, v = cases[i % len(cases)]
        assert_same(got, checker(m, v, ctx.slots, ctx.slots))
    ctx.close()


def test_plain_spmv_is_one_slice(ctx10):
    """spmv (protocol.cpp:74-153): one slice; equals spmv_partitioned when the
    rows fit one chunk budget, ColumnTooTallError when a column does not."""
    m = synth.random_sparse_csr(300, 80, 900, 61, -8, 8)
    v = synth.random_vector(80, 61, -8, 8, nonzero=True)
    got = pk.spmv(ctx10, m, v)
    assert_same(got, checker(m, v, ctx10.slots, ctx10.slots))
    with pytest.raises(pk.SpmvError) as e:
        pk.spmv(ctx10, m, v, 16)  # 300 rows: aligned column 0 is taller than 16
    assert e.value.kind == "ColumnTooTallError"


def test_job_run_uses_the_pipeline_and_compact_download():
    """Job.run (cssc_job_run) = encrypt + cloud + decrypt; from the second job
    over one chunk-shape structure it is the cached graph, whose download holds
    only each slice's first max-height slots (u32) and the deviations."""
    ctx = pk.Context(logn=12, seed=8)
    base = synth.random_sparse_csr(300, 250, 1800, 77, -8, 8)
    rng = np.random.default_rng(3)
    for it in range(3):
        vals = (rng.integers(1, 9, base.values.size) * rng.choice([-1, 1], base.values.size)).astype(np.int64)
        m = pk.Csr(base.rows, base.cols, base.row_ptrs, base.col_indices, vals)
        v = rng.integers(-8, 9, base.cols).astype(np.int64)
        j = pk.Job(ctx, [m], [v])
        got = j.run()[0]
        h2d, d2h = j.io_bytes()
        j.close()
        assert_same(got, checker(m, v, ctx.slots, ctx.slots))
        if it:  # pipeline: rows of the tallest chunk as u32, padded to 16 B, + one u64
            tallest = int((np.diff(base.row_ptrs) > 0).sum())
            assert d2h == ((4 * tallest + 15) // 16) * 16 + 8
    ctx.close()


@pytest.mark.parametrize("logn", [10, 11, 12, 13])
@pytest.mark.parametrize("fused,pipe", [(1, 0), (1, 1), (1, 2), (1, 3), (0, 0)])
def test_pipeline_over_ring_sizes_and_chunk_depths(logn, fused, pipe):
    """Repeated spmv_batch calls (the cached whole-evaluation graph from the
    second one: depth-ordered multiply items, compact download; party-separated
    by default, pipe = 1/2/3 fuses the encryption finish / the decryption into
    the cloud kernels) equal the reference semantics; chunks of different tree
    depths make the plan reorder its items."""
    ctx = pk.Context(logn=logn, seed=8)
    ctx.set_option("fused_key_switch", fused)
    ctx.set_option("pipeline_fuse", pipe)
    base = synth.random_sparse_csr(300, 250, 1800, 77, -8, 8)
    rng = np.random.default_rng(3)
    for _ in range(3):
        vals = (rng.integers(1, 9, base.values.size) * rng.choice([-1, 1], base.values.size)).astype(np.int64)
        m = pk.Csr(base.rows, base.cols, base.row_ptrs, base.col_indices, vals)
        v = rng.integers(-8, 9, base.cols).astype(np.int64)
        got = pk.spmv_batch(ctx, [m], [v])[0]
        assert_same(got, checker(m, v, ctx.slots, ctx.slots))
    ctx.close()


@pytest.mark.parametrize("where", ["first", "middle", "last"])
def test_large_batch_validation_on_the_host_pool(where):
    """Batches of >= 2^18 nonzeros scan the CSR arrays on the host pool; a bad
    column index anywhere is still reported as the sequential check reports it,
    and a valid large batch evaluates exactly."""
    ctx = pk.Context(logn=13, seed=2)
    ms = [synth.random_sparse_csr(2048, 2048, 70000, 100 + i, -8, 8) for i in range(4)]
    vs = [synth.random_vector(2048, 100 + i, -8, 8, nonzero=True) for i in range(4)]
    k = {"first": 0, "middle": 35000, "last": 69999}[where]
    bad = ms[2].col_indices.copy()
    bad[k] = 2048 + 5
    mbad = pk.Csr(2048, 2048, ms[2].row_ptrs, bad, ms[2].values)
    with pytest.raises(pk.SpmvError) as e:
        pk.spmv_batch(ctx, [ms[0], ms[1], mbad, ms[3]], vs, chunk_size=ctx.slots)
    assert e.value.kind == "IndexOutOfRangeError" and "2053" in str(e.value)
    got = pk.spmv_batch(ctx, ms, vs, chunk_size=ctx.slots)
    for m, v, g in zip(ms, vs, got):
        assert np.array_equal(g["values"], checker(m, v, ctx.slots, ctx.slots)["values"])
    ctx.close()


def test_large_batch_error_order():
    """Large batches check column ranges inside the image pass; when several
    matrices are bad, the error raised is still the one the sequential
    evaluation meets first (per matrix: row_ptrs, columns, then chunking), and
    a failed call leaves the cached plan usable."""
    ctx = pk.Context(logn=13, seed=2)
    ms = [synth.random_sparse_csr(2048, 2048, 70000, 100 + i, -8, 8) for i in range(4)]
    vs = [synth.random_vector(2048, 100 + i, -8, 8, nonzero=True) for i in range(4)]

    def badcol(i):
        c = ms[i].col_indices.copy()
        c[123] = 2048 + 7
        return pk.Csr(2048, 2048, ms[i].row_ptrs, c, ms[i].values)

    def badrows(i):
        rp = ms[i].row_ptrs.copy()
        rp[10] = rp[11] + 1
        return pk.Csr(2048, 2048, rp, ms[i].col_indices, ms[i].values)

    def run(batch, chunk=None):
        with pytest.raises(pk.SpmvError) as e:
            pk.spmv_batch(ctx, batch, vs, chunk_size=chunk or ctx.slots)
        return e.value

    good = pk.spmv_batch(ctx, ms, vs, chunk_size=ctx.slots)  # caches the plan
    e = run([ms[0], badcol(1), ms[2], badrows(3)])
    assert e.kind == "IndexOutOfRangeError" and "2055" in str(e)
    e = run([ms[0], badrows(1), badcol(2), ms[3]])
    assert "non-decreasing" in str(e)
    e = run([badcol(0), ms[1], ms[2], ms[3]], ctx.slots + 1)
    assert e.kind == "IndexOutOfRangeError"
    e = run([ms[0], ms[1], badcol(2), ms[3]], ctx.slots + 1)
    assert "chunk_size" in str(e)
    e = run([ms[0], ms[1], ms[2], badcol(3)])  # same shapes as the cached plan
    assert e.kind == "IndexOutOfRangeError"
    again = pk.spmv_batch(ctx, ms, vs, chunk_size=ctx.slots)
    for m, v, g, h in zip(ms, vs, good, again):
        want = checker(m, v, ctx.slots, ctx.slots)["values"]
        assert np.array_equal(g["values"], want) and np.array_equal(h["values"], want)
    ctx.close()


@pytest.mark.parametrize("capacity", [1, 4])
def test_alternating_plans_with_speculative_early_encryption(capacity):
    """Each spmv_batch call enqueues the previous call's early encryption graph
    before packing (pipeline_speculate).  Alternating sparsity structures makes
    every guess wrong (the graph is re-run for the selected plan), a cache of
    one plan evicts the guessed plan while its early graph may still run, and
    repeats of one structure make the guess right; every result must equal the
    reference semantics."""
    ctx = pk.Context(logn=10, seed=5)
    ctx.set_option("plan_cache", capacity)
    a = synth.random_sparse_csr(200, 180, 900, 11, -8, 8)
    b = synth.random_sparse_csr(120, 260, 700, 12, -8, 8)
    rng = np.random.default_rng(9)
    for m in [a, b, a, b, a, a, a, b, b, a]:
        v = rng.integers(-8, 9, m.cols).astype(np.int64)
        got = pk.spmv_batch(ctx, [m], [v])[0]
        assert_same(got, checker(m, v, ctx.slots, ctx.slots))
    ctx.close()


def test_batch_vector_length_checked_at_the_c_abi():
    """cssc_spmv_batch takes each vector's length and raises DimensionMismatchError
    (reference protocol.cpp:77-81) instead of reading past a short vector."""
    ctx = pk.Context(logn=10, seed=3)
    m = synth.random_sparse_csr(20, 30, 50, 1, -8, 8)
    keep = []
    csrs = pk._csr_table([m], keep)
    vptr, vlens = pk._vectors([m], [np.ones(29, np.int64)], keep)  # one entry short
    _, _, _, optr, res = pk._outputs([m], keep)
    assert pk.lib().cssc_spmv_batch(ctx.h, pk._addr(csrs), vptr, vlens, 1, ctx.slots, 0, optr, pk._addr(res)) == -4
    assert b"does not match" in pk.lib().spmvgpu_last_error()
    with pytest.raises(pk.SpmvError) as e:
        pk.spmv_batch(ctx, [m], [np.ones(31, np.int64)])
    assert e.value.kind == "DimensionMismatchError"
    ctx.close()


def test_exhausted_noise_budget_raises():
    """A modulus too small for the path's depth (Q = one 54-bit prime): the
    product's measured invariant-noise budget is gone, so the batched path
    raises NoiseExhaustedError (reference he.cpp:84-91 semantics) instead of
    returning wrong values; the model counter alone (87 bits) would pass it."""
    ctx = pk.Context(logn=12, seed=3, L=1, K=1, alpha=1, qbits=54, pbits=54)
    m = synth.random_sparse_csr(64, 64, 300, 5, -8, 8)
    v = synth.random_vector(64, 5, -8, 8, nonzero=True)
    with pytest.raises(pk.SpmvError) as e:
        pk.spmv_partitioned(ctx, m, v)
    assert e.value.kind == "NoiseExhaustedError"
    ctx.close()


@pytest.mark.parametrize("vals,vec,cols,big", [(8, 8, 300, False), (1000, 8, 300, False), (8, 1 << 40, 300, False),
                                               (200, 300, 70000, False), (8, 8, 300, True), (1 << 40, 8, 300, True)])
def test_compact_client_image_widths(vals, vec, cols, big):
    """The client upload image narrows column indices to 16 bits (<= 2^16
    columns, else 32) and values / vector entries to int8 when every one fits,
    int64 otherwise; every combination, small batches and host-pool batches
    (>= 2^18 nonzeros), evaluates exactly."""
    ctx = pk.Context(logn=11, seed=4)
    rng = np.random.default_rng(vals % 97 + cols)
    n_m = 8 if big else 1
    ms, vs = [], []
    for i in range(n_m):
        nnz = 40000 if big else 900
        base = synth.random_sparse_csr(600, cols, nnz, 300 + i, -8, 8)
        va = rng.integers(-vals, vals + 1, base.values.size)
        va[va == 0] = 1
        ms.append(pk.Csr(base.rows, cols, base.row_ptrs, base.col_indices, va.astype(np.int64)))
        vs.append(rng.integers(-vec, vec + 1, cols).astype(np.int64))
    got = pk.spmv_batch(ctx, ms, vs, chunk_size=ctx.slots)
    for m, v, g in zip(ms, vs, got):
        assert np.array_equal(g["values"], checker(m, v, ctx.slots, ctx.slots)["values"])
    ctx.close()
