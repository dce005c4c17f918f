# ncu --set full of selected kernels (regex $2, first $3 launches) of one config's cloud step; text exports only
CFG=${1:-5}; KR=${2:-cols_moddown}; CNT=${3:-1}
mkdir -p gpurun_out
timeout 900 ncu --set full --import-source on --clock-control none --profile-from-start off \
  -k regex:"$KR" -c $CNT -o /tmp/kfull -f python tools/profile_cloud.py $CFG > gpurun_out/ncuk.log 2>&1
echo "ncu rc=$?"; tail -2 gpurun_out/ncuk.log
ncu -i /tmp/kfull.ncu-rep --page raw --csv > gpurun_out/k_raw.csv
python tools/ncu_table.py gpurun_out/k_raw.csv > gpurun_out/k_table.txt
i=0
for id in $(seq 0 $((CNT-1))); do
  ncu -i /tmp/kfull.ncu-rep --page source --csv --print-source sass --launch-skip $id --launch-count 1 > gpurun_out/k_src_$id.csv 2>&1
done
ncu -i /tmp/kfull.ncu-rep --page details --csv > gpurun_out/k_details.csv 2>&1
cat gpurun_out/k_table.txt
