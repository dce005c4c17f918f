# ncu --set full of one cloud step per config (current code): per-launch table and
# DRAM-traffic json (bench.py's roofline.traffic) into gpurun_out/; reports dropped
mkdir -p gpurun_out
for CFG in "$@"; do
  timeout 1200 ncu --set full --import-source on --clock-control none --profile-from-start off \
    -o /tmp/cfull$CFG -f python tools/profile_cloud.py $CFG > gpurun_out/ncu_c$CFG.log 2>&1
  echo "c$CFG ncu rc=$?"; tail -1 gpurun_out/ncu_c$CFG.log
  ncu -i /tmp/cfull$CFG.ncu-rep --page raw --csv > gpurun_out/c${CFG}_raw.csv
  python tools/ncu_table.py gpurun_out/c${CFG}_raw.csv > gpurun_out/r02_ncu_c${CFG}_step_table.txt
  python tools/ncu_traffic.py gpurun_out/c${CFG}_raw.csv $CFG gpurun_out/r02_traffic_c$CFG.json
  rm -f /tmp/cfull$CFG.ncu-rep gpurun_out/c${CFG}_raw.csv
done
