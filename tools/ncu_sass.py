"""Per-instruction SASS profile of one kernel from an .ncu-rep (source page):
opcode histogram weighted by executed instructions, plus the hottest lines.
usage: python tools/ncu_sass.py report.ncu-rep kernel_regex [top]"""
import collections
import csv
import io
import subprocess
import sys

rep, kern = sys.argv[1], sys.argv[2]
top = int(sys.argv[3]) if len(sys.argv) > 3 else 30
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass", "-k", f"regex:{kern}",
                      "-c", "1"], capture_output=True, text=True).stdout
lines = out.splitlines()
i = [k for k, l in enumerate(lines) if l.startswith('"Address"')][0]
rows = list(csv.DictReader(io.StringIO("\n".join(lines[i:]))))
hist = collections.Counter()
stall = collections.Counter()
tot = 0
for r in rows:
    if not (r["Instructions Executed"] or "0").isdigit():
        continue
    n = int(r["Instructions Executed"] or 0)
    op = r["Source"].split()[0] if r["Source"].split() else "?"
    if op.startswith("@"):
        op = r["Source"].split()[1]
    op = op.split(".")[0]
    hist[op] += n
    stall[op] += int(r["Warp Stall Sampling (All Samples)"] or 0)
    tot += n
print(f"total warp instructions {tot}")
for op, n in hist.most_common(top):
    print(f"{op:12s} {n:12d} {100 * n / tot:5.1f}%  stall-samples {stall[op]}")
