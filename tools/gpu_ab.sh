# parity tests of the key-switch / multiply paths, then A/B cloud timings
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/pytest_gpu.log
for v in "$@"; do
  echo "== $v"; env $v timeout 300 python tools/quick_ab.py ${CFGS:-5,4,3,2} 20 2>&1 | tail -1
done
