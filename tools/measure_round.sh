set -x
timeout 1200 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/pytest_gpu_all.log 2>&1; echo PYTEST $? >> gpurun_out/pytest_gpu_all.log
timeout 900 python bench.py > gpurun_out/bench_full.json 2> gpurun_out/bench_full.err; echo BENCH $?
ncu --profile-from-start off --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/ncu_step_raw.csv python tools/ncu_step.py inception_bn > gpurun_out/ncu_step.log 2>&1; echo NCUSTEP $?
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/ncu_launch_raw.csv python bench.py --no-extra --steps 3 --warmup 3 > gpurun_out/ncu_launch.log 2>&1; echo NCULAUNCH $?
ncu --profile-from-start off --set full --import-source on -k regex:tc_gemm --launch-skip 12 -c 1 -o gpurun_out/gemm_step -f python tools/ncu_step.py inception_bn > gpurun_out/ncu_gemm.log 2>&1; echo NCUGEMM $?
