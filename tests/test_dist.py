"""Multi-process host logic for BASELINE config 5 (row-slice / matrix
sharding), run with torch.distributed gloo, world size 2, on
CPU.  The per-rank compute is stood in by the reference-semantics checker so
the test exercises only the sharding + gather path of paper_2603_04742_b200.shard."""
import os

import numpy as np
import torch.distributed as dist
import torch.multiprocessing as mp

import paper_2603_04742_b200 as pk
from paper_2603_04742_b200 import shard


def _worker(rank, world, port, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    import sys
    sys.path.insert(0, os.path.dirname(__file__))
    from oracle_bindings import sim_spmv_partitioned

    ms = [pk.random_sparse_csr(64, 64, 200, s, -8, 8) for s in range(500, 507)]
    vs = [pk.random_vector(64, s, -8, 8, nonzero=True) for s in range(500, 507)]
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
        m = pk.random_sparse_csr(64, 64, 200, s, -8, 8)
        v = pk.random_vector(64, s, -8, 8, nonzero=True)
        assert got[i] == sim_spmv_partitioned(m, v, 64, 64)["values"].tolist()


def test_units_partition_is_exact():
    for n in range(0, 20):
        for w in range(1, 5):
            parts = [shard.units_for_rank(n, r, w) for r in range(w)]
            assert sorted(sum(parts, [])) == list(range(n))
