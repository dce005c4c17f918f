"""Host-side latency of the client calls (C-ABI, preallocated buffers).
usage: python tools/dec_timing.py"""
import ctypes as C
import statistics
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import numpy as np  # noqa: E402

import paper_2603_04742_b200 as pk  # noqa: E402
from paper_2603_04742_b200 import _p, i32p, lib, u64p  # noqa: E402

ctx = pk.Context(logn=14, seed=1)
for n in (1, 8):
    cts = ctx.encrypt([np.arange(100)] * n)
    slots = np.zeros((n, ctx.slots), np.uint64)
    b = np.zeros(n, np.int32)
    for _ in range(5):
        lib().spmvgpu_decrypt(ctx.h, _p(cts, u64p), n, _p(slots, u64p), _p(b, i32p))
    ts = []
    for _ in range(100):
        t = time.perf_counter()
        lib().spmvgpu_decrypt(ctx.h, _p(cts, u64p), n, _p(slots, u64p), _p(b, i32p))
        ts.append((time.perf_counter() - t) * 1e3)
    print(f"decrypt x{n}: median {statistics.median(ts):.4f} ms min {min(ts):.4f}")
    ctx.sync()
    ts = []
    for _ in range(100):
        t = time.perf_counter()
        lib().spmvgpu_sync(ctx.h)
        ts.append((time.perf_counter() - t) * 1e3)
    print(f"sync: {statistics.median(ts):.4f} ms")
