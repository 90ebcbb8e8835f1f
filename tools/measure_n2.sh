set -x
python -m pytest tests/test_kv_dist_gpu.py -q 2>&1 | tail -5 > gpurun_out/r02_dist2.log
for cfg in alexnet inception_bn; do
  for ov in 1 0; do
    MGX_OVERLAP=$ov timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29511 bench.py --gpus 2 --steps 20 --warmup 5 --config $cfg --no-extra --kv-bytes 67108864 > gpurun_out/r02_n2_${cfg}_ov${ov}.json 2> gpurun_out/r02_n2_${cfg}_ov${ov}.err
  done
done
for cfg in alexnet; do
  timeout 600 python bench.py --steps 20 --warmup 5 --config $cfg --no-extra --kv-bytes 67108864 > gpurun_out/r02_n1_${cfg}.json 2> gpurun_out/r02_n1_${cfg}.err
done
