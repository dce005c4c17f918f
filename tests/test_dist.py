"""Multi-process host logic for BASELINE config 5 (row-slice / matrix
sharding), run with torch.distributed gloo, world size 2, on
CPU.  The per-rank compute is stood in by the reference-semantics checker so
the test exercises only the sharding + gather path of paper_2603_04742_b200.shard."""
import os

import numpy as np
import torch.distributed as dist
import torch.multiprocessing as mp

import paper_2603_04742_b200 as pk
import synth
from paper_2603_04742_b200 import shard


def _worker(rank, world, port, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    import sys
    sys.path.insert(0, os.path.dirname(__file__))
    from oracle_bindings import sim_spmv_partitioned

    ms = [synth.random_sparse_csr(64, 64, 200, s, -8, 8) for s in range(500, 507)]
    vs = [synth.random_vector(64, s, -8, 8, nonzero=True) for s in range(500, 507)]
    mine = shard.units_for_rank(len(ms), rank, world)
    local = {i: sim_spmv_partitioned(ms[i], vs[i], 64, 64)["values"] for i in mine}
    full = shard.gather_values(local, len(ms), [m.rows for m in ms])
    if rank == 0:
        q.put([v.tolist() for v in full])
    dist.destroy_process_group()


def test_sharded_batch_gathers_in_order():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = 29500 + os.getpid() % 1000
    ps = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in ps:
        p.start()
    got = q.get(timeout=120)
    for p in ps:
        p.join(timeout=60)
        assert p.exitcode == 0
    import sys
    sys.path.insert(0, os.path.dirname(__file__))
    from oracle_bindings import sim_spmv_partitioned
    for i, s in enumerate(range(500, 507)):
        m = synth.random_sparse_csr(64, 64, 200, s, -8, 8)
        v = synth.random_vector(64, s, -8, 8, nonzero=True)
        assert got[i] == sim_spmv_partitioned(m, v, 64, 64)["values"].tolist()


def test_units_partition_is_exact():
    for n in range(0, 20):
        for w in range(1, 5):
            parts = [shard.units_for_rank(n, r, w) for r in range(w)]
            assert sorted(sum(parts, [])) == list(range(n))


Q4 = [288230376151748609, 288230376151760897, 288230376151777281, 288230376151789569]  # < 2^58


def _fold_worker(rank, world, port, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    L, n, R = 4, 16, 3
    rng = np.random.default_rng(rank)
    qs = np.array(Q4, np.uint64).reshape(1, 1, L, 1)
    words = (rng.integers(0, 2**62, (R, 2, L, n), dtype=np.uint64) % qs).reshape(R, -1)
    out = shard.reduce_partials(words, Q4, L, n)
    if rank == 0:
        q.put(out.tolist())
    dist.destroy_process_group()


def test_chunk_split_partials_reduce_mod_q():
    """The chunk-split all-reduce of partial result words equals
    the per-limb modular sum, for world size 3 over gloo."""
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = 30500 + os.getpid() % 1000
    world = 3
    ps = [ctx.Process(target=_fold_worker, args=(r, world, port, q)) for r in range(world)]
    for p in ps:
        p.start()
    got = np.array(q.get(timeout=120), dtype=np.uint64)
    for p in ps:
        p.join(timeout=60)
        assert p.exitcode == 0
    L, n, R = 4, 16, 3
    qs = np.array(Q4, np.uint64).reshape(1, 1, L, 1)
    want = np.zeros((R, 2, L, n), np.uint64)
    for r in range(world):
        rng = np.random.default_rng(r)
        w = rng.integers(0, 2**62, (R, 2, L, n), dtype=np.uint64) % qs
        want = (want + w) % qs
    assert np.array_equal(got, want.reshape(R, -1))
    assert np.array_equal(shard.fold_mod(want.reshape(R, -1) + want.reshape(R, -1), Q4, L, n),
                          ((2 * want) % qs).reshape(R, -1))
