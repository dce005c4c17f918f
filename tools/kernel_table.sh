# per-launch CUDA-event table of one config's cloud step (bench.py's kernel profile)
mkdir -p gpurun_out
CFG=${1:-5}
timeout 600 python bench.py --only --config $CFG --no-cpu-baseline --steps 10 > gpurun_out/kt_c$CFG.json 2> gpurun_out/kt_c$CFG.err
python - "$CFG" <<'PY'
import json, sys
c = sys.argv[1]
l = [x for x in open(f"gpurun_out/kt_c{c}.json") if x.strip().startswith("{")][-1]
d = json.loads(l)["configs"][f"C{c}"]
print("ms", d["ms"], "e2e", d["e2e"]["value"], "int_frac", d["whole_step_int_frac"])
for g in d["groups"]: print(f"{g['group']:22s} {g['items']:5d} {g['us']:9.1f} us  int {g['int_frac']:.3f}")
for k in d["kernels"]: print(f"  {k['kernel'][:42]:42s} {k['group'][:16]:16s} {k['us']:8.1f} {k['int_frac']:.3f}")
PY
