"""One line per kernel of an .ncu-rep: time, grid, regs, warps active, issue
active, fmaheavy busy and the top stall ratios.
usage: python tools/ncu_table.py report.ncu-rep | raw.csv (ncu --page raw --csv)"""
import csv
import io
import subprocess
import sys

if sys.argv[1].endswith(".csv"):
    raw = open(sys.argv[1]).read()
else:
    raw = subprocess.run(["ncu", "-i", sys.argv[1], "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(raw)))
h = rows[0]
units = dict(zip(h, rows[1]))
SCALE = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "ns": 1e-3, "usecond": 1, "us": 1, "msecond": 1e3,
         "ms": 1e3, "second": 1e6, "s": 1e6}
S = "smsp__average_warps_issue_stalled_%s_per_issue_active.ratio"
stalls = ["long_scoreboard", "barrier", "math_pipe_throttle", "wait", "short_scoreboard", "dispatch_stall",
          "not_selected", "mio_throttle"]
print(f"{'kernel':34s} {'grid':>14s} {'us':>7s} {'dramMB':>7s} {'reg':>4s} {'warps%':>6s} {'issue%':>6s} {'fmaH%':>6s} " +
      " ".join(f"{s[:6]:>6s}" for s in stalls))
for r in rows[2:]:
    d = dict(zip(h, r))
    name = d["Kernel Name"].split("(")[0].replace("void ", "").replace("cssc::", "")[:34]

    def f(k):  # times in us, bytes in bytes
        try:
            return float(d.get(k, "nan").replace(",", "")) * SCALE.get(units.get(k, ""), 1)
        except ValueError:
            return float("nan")
    dram = (f('dram__bytes_read.sum') + f('dram__bytes_write.sum')) / 1e6
    print(f"{name:34s} {d['Grid Size']:>14s} {f('gpu__time_duration.sum'):7.2f} {dram:7.1f} "
          f"{f('launch__registers_per_thread'):4.0f} {f('sm__warps_active.avg.pct_of_peak_sustained_active'):6.1f} "
          f"{f('smsp__issue_active.avg.pct_of_peak_sustained_active'):6.1f} "
          f"{f('sm__pipe_fmaheavy_cycles_active.avg.pct_of_peak_sustained_elapsed'):6.1f} " +
          " ".join(f"{f(S % s):6.2f}" for s in stalls))
