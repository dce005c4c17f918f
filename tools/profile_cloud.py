"""Run one cloud phase of a BASELINE config between cudaProfilerStart/Stop so
`ncu --profile-from-start off` captures exactly the launches of one step.
usage: python tools/profile_cloud.py [config] [graph:0|1]"""
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))

import torch  # noqa: E402

import bench  # noqa: E402
import paper_2603_04742_b200 as pk  # noqa: E402

cfgno = int(sys.argv[1]) if len(sys.argv) > 1 else 2
graph = len(sys.argv) > 2 and sys.argv[2] == "1"
cfg = bench.make_config(cfgno)
ctx = pk.Context(logn=cfg["logn"], seed=1)
job = pk.Job(ctx, cfg["ms"], cfg["vs"])
job.encrypt()
for _ in range(3):
    job.cloud(graph=graph)
ctx.sync()
torch.cuda.profiler.start()
job.cloud(graph=graph)
ctx.sync()
torch.cuda.profiler.stop()
res = job.finish()
ok = all((r["values"] == bench.exact_values(m, v)).all() for m, v, r in zip(cfg["ms"], cfg["vs"], res))
print("config", cfgno, "verified", ok, job.stats())
