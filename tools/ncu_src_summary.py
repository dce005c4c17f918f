"""Opcode histogram and hottest SASS lines of one kernel from an exported
`ncu -i rep --page source --csv --print-source sass` file.
usage: python tools/ncu_src_summary.py src.csv [top]"""
import collections
import csv
import io
import sys


def load(path):
    lines = open(path).read().splitlines()
    i = [n for n, l in enumerate(lines) if l.startswith('"Address"')][0]
    out = []
    for r in csv.DictReader(io.StringIO("\n".join(lines[i:]))):
        try:
            r["n"] = int(r["Instructions Executed"] or 0)
            r["s"] = int(r["Warp Stall Sampling (All Samples)"] or 0)
        except ValueError:
            continue
        out.append(r)
    return out


def op_of(src):
    t = src.split()
    if not t:
        return "?"
    return (t[1] if t[0].startswith("@") and len(t) > 1 else t[0]).split(".")[0]


if __name__ == "__main__":
    rows = load(sys.argv[1])
    top = int(sys.argv[2]) if len(sys.argv) > 2 else 12
    hist, st = collections.Counter(), collections.Counter()
    for r in rows:
        hist[op_of(r["Source"])] += r["n"]
        st[op_of(r["Source"])] += r["s"]
    tot, stot = sum(hist.values()), sum(st.values())
    print(f"instructions {tot}, stall samples {stot}")
    for op, n in hist.most_common(14):
        print(f"  {op:10s} {n / tot * 100:5.1f}% instr {st[op] / stot * 100:5.1f}% stalls")
    for k, r in enumerate(sorted(range(len(rows)), key=lambda i: -rows[i]["s"])[:top]):
        x = rows[r]
        print(f"  #{r:5d} {x['s']:6d} {x['Source'][:90]}")
