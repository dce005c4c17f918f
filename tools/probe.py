"""Run the roofline probes (plan-shaped NTT launch + register-resident butterfly
peak) between cudaProfilerStart/Stop, for ncu --profile-from-start off."""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import torch  # noqa: E402
import paper_2603_04742_b200 as pk  # noqa: E402

logn = int(sys.argv[1]) if len(sys.argv) > 1 else 14
limbs = int(sys.argv[2]) if len(sys.argv) > 2 else 1152
ctx = pk.Context(logn=logn, seed=1)
print("warm", ctx.probe_ntt_us(limbs, False, 3), ctx.probe_ntt_us(limbs, True, 3))
n = 1 << logn
for _ in range(3):
    f20, i20 = ctx.probe_ntt_us(limbs, False, 20), ctx.probe_ntt_us(limbs, True, 20)
    print(f"reps20 fwd {f20:.2f} us ({limbs * n // 2 * logn / (f20 * 1e-6) / 1e9:.1f} Gbfly/s) inv {i20:.2f} us")
torch.cuda.profiler.start()
f = ctx.probe_ntt_us(limbs, False, 1)
i = ctx.probe_ntt_us(limbs, True, 1)
p = ctx.probe_butterfly_peak()
torch.cuda.profiler.stop()
n = 1 << logn
print(f"fwd {f:.1f} us inv {i:.1f} us; {limbs * n // 2 * logn / (f * 1e-6) / 1e9:.1f} Gbfly/s fwd; peak {p / 1e9:.1f}")
