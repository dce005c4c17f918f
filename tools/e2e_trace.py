"""Per-call host/device split of spmv_batch (CSSC_TRACE_E2E=1 prints the
C++ stage times to stderr).  usage: CSSC_TRACE_E2E=1 python tools/e2e_trace.py [config] [reps]"""
import sys
import time
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))

import bench  # noqa: E402
import paper_2603_04742_b200 as pk  # noqa: E402

cfgno = int(sys.argv[1]) if len(sys.argv) > 1 else 2
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 10
cfg = bench.make_config(cfgno)
ctx = pk.Context(logn=cfg["logn"], seed=1)
for _ in range(3):
    pk.spmv_batch(ctx, cfg["ms"], cfg["vs"])
ctx.sync()
for _ in range(reps):
    t0 = time.perf_counter()
    pk.spmv_batch(ctx, cfg["ms"], cfg["vs"])
    print(f"python wall {(time.perf_counter() - t0) * 1e6:.1f} us", file=sys.stderr, flush=True)
