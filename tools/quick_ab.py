"""Cloud-step A/B timing: for each config, the mean ms of K graph replays
(L2 flushed before each) and the exactness of the decrypted result.  Knobs
are env vars read once per process, so run one process per variant.
usage: python tools/quick_ab.py [configs=5,3,2] [steps=20]"""
import json
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))

import numpy as np  # noqa: E402
import torch  # noqa: E402

import bench  # noqa: E402
import paper_2603_04742_b200 as pk  # noqa: E402

cfgs = [int(c) for c in (sys.argv[1] if len(sys.argv) > 1 else "5,3,2").split(",")]
steps = int(sys.argv[2]) if len(sys.argv) > 2 else 20
out = {}
for c in cfgs:
    cfg = bench.make_config(c)
    ctx = pk.Context(logn=cfg["logn"])
    job = pk.Job(ctx, cfg["ms"], cfg["vs"])
    job.encrypt()
    job.cloud(graph=True)
    res = job.finish()
    ok = all(np.array_equal(r["values"], bench.exact_values(m, v)) for m, v, r in zip(cfg["ms"], cfg["vs"], res))
    stream = torch.cuda.ExternalStream(ctx.stream_ptr())
    flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
    times, _ = bench.time_cloud(job, stream, flush, steps, 5)
    out[f"C{c}"] = {"ms": round(float(np.mean(times)), 4), "min": round(float(np.min(times)), 4), "exact": bool(ok)}
    del job, ctx
print(json.dumps(out), flush=True)
