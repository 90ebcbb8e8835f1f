# round-2 multi-GPU evidence on one box: distributed tests, weak scaling
# (Inception-BN headline, AlexNet-style aggregation-bound) and the config-2
# KVStore sweep, at N = 2 and 4 (plus N = 1 on the same box for the ratio)
python -m pytest tests/test_kv_dist_gpu.py -q 2>&1 | tail -3 > gpurun_out/r02_dist4.log
for cfg in inception_bn alexnet; do
  python bench.py --steps 30 --warmup 5 --config $cfg --no-extra --kv-bytes 1048576 > gpurun_out/r02_scale_${cfg}_n1.json 2>/dev/null
  for n in 2 4; do
    timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 --master-port 2952$n bench.py --gpus $n --steps 30 --warmup 5 --config $cfg --no-extra --kv-bytes 1048576 > gpurun_out/r02_scale_${cfg}_n$n.json 2>/dev/null
  done
done
for n in 2 4; do
  timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 --master-port 2953$n bench.py --gpus $n --steps 20 --warmup 3 --config lenet --no-extra > gpurun_out/r02_kvsweep_n$n.json 2>/dev/null
done
