"""Write profiles/r01_ntt_traffic_<limbs>.json from an ncu csv of tools/probe.py
(metrics dram__bytes_read.sum, dram__bytes_write.sum, gpu__time_duration.sum):
the DRAM traffic of one forward NTT launch (column + block kernels).
usage: python tools/ntt_traffic.py ncu.csv limbs logn"""
import collections
import csv
import json
import sys
from pathlib import Path

path, limbs, logn = sys.argv[1], int(sys.argv[2]), int(sys.argv[3])
lines = open(path).read().splitlines()
i = [k for k, l in enumerate(lines) if l.startswith('"ID"')][0]
per = collections.defaultdict(dict)
order = []
for r in csv.DictReader(lines[i:]):
    name = r["Kernel Name"].split("(")[0].replace("void ", "").replace("cssc::", "")
    key = (r["ID"], name)
    if key not in order:
        order.append(key)
    per[key][r["Metric Name"]] = float(r["Metric Value"].replace(",", ""))
# first forward column + block launches of the profiled range
fwd = [k for k in order if k[1] in (f"k_ntt_cols<{logn}, 0>", f"k_ntt_blocks<{logn}, 0>")][:2]
traffic = sum(per[k].get("dram__bytes_read.sum", 0) + per[k].get("dram__bytes_write.sum", 0) for k in fwd)
out = {"source": f"ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum on "
                 f"tools/probe.py {logn} {limbs} (forward NTT launch = cols + blocks kernels)",
       "limbs": limbs, "logn": logn, "traffic_bytes_per_launch": traffic,
       "algorithmic_bytes_per_launch": 2 * limbs * (1 << logn) * 8,
       "per_kernel": {f"{k[1]} #{k[0]}": per[k] for k in order},
       "note": "DRAM writes of the launch may be absorbed by L2 within the kernel (write-back), so dram__bytes_write can read 0"}
Path(f"profiles/r01_ntt_traffic_{limbs}.json").write_text(json.dumps(out, indent=1))
print(json.dumps({k: out[k] for k in ("limbs", "traffic_bytes_per_launch", "algorithmic_bytes_per_launch")}))
