# ncu --set full of one C5 cloud step (current code), with source; exports text and drops the report
CFG=${1:-5}
mkdir -p gpurun_out
timeout 900 ncu --set full --import-source on --clock-control none --profile-from-start off \
  -o /tmp/cfull -f python tools/profile_cloud.py $CFG > gpurun_out/ncu_c$CFG.log 2>&1
echo "ncu rc=$?"; tail -3 gpurun_out/ncu_c$CFG.log
ncu -i /tmp/cfull.ncu-rep --page raw --csv > gpurun_out/c${CFG}_raw.csv
python tools/ncu_table.py gpurun_out/c${CFG}_raw.csv > gpurun_out/c${CFG}_table.txt
for k in k_ks_modup_cols k_ks_blocks_inner k_ks_cols_moddown k_mul_blocks_tensor k_mul_scale_k k_mul_extend_k k_ntt_cols; do
  ncu -i /tmp/cfull.ncu-rep --page source --csv --print-source sass --kernel-name regex:$k --launch-count 1 > gpurun_out/c${CFG}_src_$k.csv 2>&1
done
ls -la gpurun_out
