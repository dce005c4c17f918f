"""Run one end-to-end spmv_batch call of a BASELINE config (from the cached
pipeline graph: upload, pack, encrypt, cloud, decrypt, download) between
cudaProfilerStart/Stop so `ncu --profile-from-start off` lists its launches.
usage: python tools/profile_e2e.py [config]"""
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))

import torch  # noqa: E402

import bench  # noqa: E402
import paper_2603_04742_b200 as pk  # noqa: E402

cfgno = int(sys.argv[1]) if len(sys.argv) > 1 else 2
cfg = bench.make_config(cfgno)
ctx = pk.Context(logn=cfg["logn"], seed=1)
for _ in range(3):
    pk.spmv_batch(ctx, cfg["ms"], cfg["vs"])
ctx.sync()
torch.cuda.profiler.start()
res = pk.spmv_batch(ctx, cfg["ms"], cfg["vs"])
ctx.sync()
torch.cuda.profiler.stop()
ok = all((r["values"] == bench.exact_values(m, v)).all() for m, v, r in zip(cfg["ms"], cfg["vs"], res))
print("config", cfgno, "verified", ok)
