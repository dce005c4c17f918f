import sys, os
sys.path.insert(0, '/root/repo'); sys.path.insert(0, '/root/repo/tests')
import numpy as np, bench, paper_2603_04742_b200 as pk
cfg = bench.make_config(int(sys.argv[1]))
ctx = pk.Context(logn=cfg["logn"], seed=7)
job = pk.Job(ctx, cfg["ms"], cfg["vs"])
job.encrypt()
job.cloud(graph=False)
res = job.finish()
print("ok", all(np.array_equal(r["values"], bench.exact_values(m, v)) for m, v, r in zip(cfg["ms"], cfg["vs"], res)))
