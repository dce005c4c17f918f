"""BASELINE.md section 4 table from a bench.py line and the reference arm's line.
usage: python tools/baseline_table.py bench.json reference.json"""
import json
import sys

d = json.loads(open(sys.argv[1]).read().strip().splitlines()[-1])
ref = json.loads(open(sys.argv[2]).read().strip().splitlines()[-1]) if len(sys.argv) > 2 else None
print("| cfg | GPU cloud (ms) | GPU e2e, party-separated (ms) | SpMV/s · nnz/s (cloud) | key-switch: % of HBM · int frac | "
      "top kernel: int frac | whole-step int frac | exact (P1, P5) | measured noise (bits) | "
      "B1 reference 1 core: cloud / whole (ms) | B3 RNS-BFV CPU: 1 thread / all threads (ms, extrapolated) | "
      "B2 estimate (ms) |")
print("|---|---|---|---|---|---|---|---|---|---|---|---|")
nnz = {"C1": 655, "C2": 16777, "C3": 192949, "C4": 830584, "C5": 64 * 20972}
for c in ("C1", "C2", "C3", "C4", "C5"):
    r = d["configs"].get(c)
    if not r or "error" in r:
        print(f"| {c} | error | | | | | | | | | | |")
        continue
    ks = r.get("key_switch")
    kss = f"{100 * ks['hbm_frac']:.1f} % · {ks['int_frac']:.2f}" if ks else "no rotations"
    b1, b3 = r.get("cpu_baseline") or {}, r.get("cpu_bfv_baseline") or {}
    rf = r.get("roofline") or {}
    per_s = 1e3 / r["ms"]
    print(f"| {c} | {r['ms']:.3f} | {r['e2e']['value']:.3f} | {per_s:.0f} · {per_s * nnz[c] / 1e9:.2f} G | {kss} | "
          f"{rf.get('kernel', '')[:24]}: {rf.get('frac', 0):.2f} | {r['whole_step_int_frac']:.2f} | "
          f"{'yes' if r['verified'] else 'NO'} | {r['measured_noise_bits']} | "
          f"{b1.get('value', '-')} / {b1.get('e2e_value', '-')} | "
          f"{b3.get('extrapolated_ms_1_thread', '-')} / {b3.get('extrapolated_ms_all_threads', '-')} | "
          f"{r.get('paper_cost_model', {}).get('cloud_ms', '-')} |")
if ref:
    print()
    print(f"Reference arm (`bench.py --impl reference`, {ref['config']['parallelism']}, {ref['config']['workload'][:2]}): "
          f"cloud section {ref['value']} ms, whole spmv_partitioned {ref['e2e']['value']} ms.")
