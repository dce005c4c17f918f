"""DRAM traffic per kernel launch of one cloud step from an ncu raw-page CSV
(`ncu -i step.ncu-rep --page raw --csv`, the capture of tools/profile_cloud.py):
writes profiles/r02_traffic_c<cfg>.json, which bench.py reads as the
`roofline.traffic` of the same launch (launches in plan order).
usage: python tools/ncu_traffic.py raw.csv <cfg> [out.json]"""
import csv
import json
import sys
from pathlib import Path

SCALE = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "ns": 1e-3, "nsecond": 1e-3, "usecond": 1,
         "us": 1, "msecond": 1e3, "ms": 1e3}

rows = list(csv.reader(open(sys.argv[1])))
h, units = rows[0], rows[1]
u = dict(zip(h, units))


def val(d, k):
    return float(d[k].replace(",", "")) * SCALE.get(u.get(k, ""), 1)


out = []
for r in rows[2:]:
    d = dict(zip(h, r))
    out.append({"kernel": d["Kernel Name"].split("(")[0].replace("void ", "").replace("cssc::", ""),
                "grid": d["Grid Size"], "us_ncu": round(val(d, "gpu__time_duration.sum"), 2),
                "dram_bytes": int(val(d, "dram__bytes_read.sum") + val(d, "dram__bytes_write.sum"))})
dst = Path(sys.argv[3]) if len(sys.argv) > 3 else Path(__file__).resolve().parent.parent / "profiles" / f"r02_traffic_c{sys.argv[2]}.json"
dst.write_text(json.dumps({"source": Path(sys.argv[1]).name, "config": int(sys.argv[2]),
                           "note": "ncu --set full --clock-control none of one cloud step (tools/profile_cloud.py), "
                                   "dram__bytes_read.sum + dram__bytes_write.sum per launch, launches in plan order",
                           "launches": out}, indent=1))
print(dst, len(out), "launches")
