import time, statistics, sys
sys.path.insert(0, "/root/repo")
import numpy as np, paper_2603_04742_b200 as pk
ctx = pk.Context(logn=14, seed=1)
cts = ctx.encrypt([np.arange(100)])
for n in (1, 8):
    cs = ctx.encrypt([np.arange(100)] * n)
    for _ in range(5): ctx.decrypt(cs)
    ts = []
    for _ in range(50):
        t = time.perf_counter(); ctx.decrypt(cs); ts.append((time.perf_counter() - t) * 1e3)
    print("decrypt", n, statistics.median(ts))
    ts = []
    for _ in range(50):
        ctx.sync(); t = time.perf_counter(); ctx.encrypt([np.arange(100)] * n); ctx.sync(); ts.append((time.perf_counter() - t) * 1e3)
    print("encrypt", n, statistics.median(ts))
