# ncu evidence for profiles/ (one GPU; run only after the same commands
# exited 0 without ncu):
#  1. launch list of the bench command (per-launch durations, serialised)
#  2. per-family DRAM traffic of one Inception-BN pass (-> traffic json)
#  3. --set full of the first GEMMs and cluster BatchNorms of a pass
set -e
python bench.py --steps 2 --warmup 3 --no-extra --kv-bytes 1048576 > /dev/null 2>&1
python tools/ncu_step.py inception_bn > /dev/null 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none -c 3000 --csv \
    --log-file gpurun_out/ncu_launches_raw.csv \
    python bench.py --steps 2 --warmup 3 --no-extra --kv-bytes 1048576 > gpurun_out/ncu_launches.log 2>&1
ncu --profile-from-start off --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum \
    --clock-control none --csv --log-file gpurun_out/ncu_step_raw.csv \
    python tools/ncu_step.py inception_bn > gpurun_out/ncu_step.log 2>&1
ncu --set full --clock-control none --import-source on --profile-from-start off \
    -k regex:'tc_gemm|bn_fwd_fused|bn_bwd_fused' -c 12 -o gpurun_out/ncu_full -f \
    python tools/ncu_step.py inception_bn > gpurun_out/ncu_full.log 2>&1
ncu -i gpurun_out/ncu_full.ncu-rep --page details --csv > gpurun_out/ncu_full_details.csv
ncu -i gpurun_out/ncu_full.ncu-rep --page raw --csv > gpurun_out/ncu_full_raw.csv
rm -f gpurun_out/ncu_full.ncu-rep
echo done
