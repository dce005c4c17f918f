"""spmv_batch wall-clock statistics (min / median / mean over reps) for one config.
usage: python tools/e2e_stats.py [config] [reps]"""
import statistics
import sys
import time
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))

import torch  # noqa: E402

import bench  # noqa: E402
import paper_2603_04742_b200 as pk  # noqa: E402

cfgno = int(sys.argv[1]) if len(sys.argv) > 1 else 5
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 30
cfg = bench.make_config(cfgno)
ctx = pk.Context(logn=cfg["logn"])
for _ in range(5):
    pk.spmv_batch(ctx, cfg["ms"], cfg["vs"])
ts = []
for _ in range(reps):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    pk.spmv_batch(ctx, cfg["ms"], cfg["vs"])
    ts.append((time.perf_counter() - t0) * 1e3)
print(f"C{cfgno} e2e ms: min {min(ts):.3f} median {statistics.median(ts):.3f} mean {statistics.mean(ts):.3f} "
      f"max {max(ts):.3f}", flush=True)
