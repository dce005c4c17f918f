"""Wall-clock breakdown of one end-to-end spmv_batch call of a BASELINE config
(pack -> encrypt -> plan + cloud -> decrypt), stage by stage through the Job API.
usage: python tools/e2e_breakdown.py [config] [reps]"""
import statistics
import sys
import time
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))

import bench  # noqa: E402
import paper_2603_04742_b200 as pk  # noqa: E402

cfgno = int(sys.argv[1]) if len(sys.argv) > 1 else 2
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 20
cfg = bench.make_config(cfgno)
ctx = pk.Context(logn=cfg["logn"], seed=1)
ms, vs = cfg["ms"], cfg["vs"]
for _ in range(3):
    pk.spmv_batch(ctx, ms, vs)
ctx.sync()

stages = {"pack": [], "encrypt": [], "cloud(plan+run)": [], "finish(decrypt)": [], "close": [], "total": []}
whole = []
for _ in range(reps):
    ctx.sync()
    t0 = time.perf_counter()
    job = pk.Job(ctx, ms, vs)
    t1 = time.perf_counter()
    job.encrypt()
    ctx.sync()
    t2 = time.perf_counter()
    job.cloud(graph=False)
    ctx.sync()
    t3 = time.perf_counter()
    job.finish()
    t4 = time.perf_counter()
    job.close()
    t5 = time.perf_counter()
    for k, a, b in (("pack", t0, t1), ("encrypt", t1, t2), ("cloud(plan+run)", t2, t3),
                    ("finish(decrypt)", t3, t4), ("close", t4, t5), ("total", t0, t5)):
        stages[k].append((b - a) * 1e3)
    ctx.sync()
    t0 = time.perf_counter()
    pk.spmv_batch(ctx, ms, vs)
    whole.append((time.perf_counter() - t0) * 1e3)
if "--profile" in sys.argv:
    import torch
    ctx.sync()
    torch.cuda.profiler.start()
    pk.spmv_batch(ctx, ms, vs)
    ctx.sync()
    torch.cuda.profiler.stop()
for k, v in stages.items():
    print(f"{k:18s} median {statistics.median(v):8.4f} ms  min {min(v):8.4f}")
print(f"{'spmv_batch':18s} median {statistics.median(whole):8.4f} ms  min {min(whole):8.4f}")
