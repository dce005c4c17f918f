"""Summarise an ncu --metrics gpu__time_duration.sum launch list (csv)."""
import collections
import csv
import sys

lines = open(sys.argv[1]).read().splitlines()
i = [k for k, l in enumerate(lines) if l.startswith('"ID"')][0]
rows = list(csv.DictReader(lines[i:]))
tot = collections.defaultdict(float)
cnt = collections.Counter()
for r in rows:
    name = r["Kernel Name"]
    k = name.split("(")[0].replace("void ", "")
    if len(sys.argv) > 2:
        k += " grid" + r["Grid Size"]
    tot[k] += float(r["Metric Value"]) / 1e3
    cnt[k] += 1
T = sum(tot.values())
for k, v in sorted(tot.items(), key=lambda x: -x[1]):
    print(f"{v:9.1f} us {100 * v / T:5.1f}%  x{cnt[k]:<3d} {k}")
print(f"total {T:.1f} us over {len(rows)} launches")
