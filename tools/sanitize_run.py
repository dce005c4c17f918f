"""Small workload for compute-sanitizer (memcheck / racecheck / synccheck, one
tool per run): every kernel family of the path at small sizes -- key
generation, device pack + encryption (staged and the whole-evaluation graph,
party-separated and fused), the cloud plan (multiply + relinearisation,
rotate-and-add levels, mask), decryption, op-by-op rotate / mul_plain, the
chunk-split device fold.  usage: compute-sanitizer --tool X python tools/sanitize_run.py"""
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))

import numpy as np  # noqa: E402

import bench  # noqa: E402
import paper_2603_04742_b200 as pk  # noqa: E402
import synth  # noqa: E402

ok = True
ctx = pk.Context(logn=12, seed=5)
m = synth.random_sparse_csr(700, 500, 4000, 9, -8, 8)  # one slice (S = 2048), several chunks
v = synth.random_vector(500, 9, -8, 8, nonzero=True)
for fuse in (0, 3):
    ctx.set_option("pipeline_fuse", fuse)
    for _ in range(2):  # staged path, then the cached graph
        r = pk.spmv_batch(ctx, [m], [v])[0]
        ok &= bool(np.array_equal(r["values"], bench.exact_values(m, v)))
(a, b) = ctx.encrypt([np.arange(50), np.arange(50) % 7], [1, 2])
(p,) = ctx.mul_relin([a], [b])
(q,) = ctx.rotate([p], [5])
(s,) = ctx.mul_plain([q], [np.ones(20, np.int64)])
slots, _ = ctx.decrypt([s])
job = pk.Job(ctx, [m], [v], rank=0, world=2)
job.encrypt()
job.cloud(graph=False)
d = job.result_words_dev()
job.close()
ctx.close()
cfg = bench.make_config(2)  # one C2 cloud step at full parameters
ctx = pk.Context(logn=cfg["logn"], seed=1)
job = pk.Job(ctx, cfg["ms"], cfg["vs"])
job.encrypt()
job.cloud(graph=False)
res = job.finish()
ok &= all(np.array_equal(x["values"], bench.exact_values(mm, vv)) for mm, vv, x in zip(cfg["ms"], cfg["vs"], res))
job.close()
ctx.close()
print("sanitize_run ok" if ok else "sanitize_run MISMATCH")
sys.exit(0 if ok else 1)
