# push/backward overlap: KV blocks per embedded round vs step time at N=2
for cfg in alexnet inception_bn; do
  for nb in 0 64 32 16; do
    MGX_KV_OVERLAP_BLOCKS=$nb timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29513 bench.py --gpus 2 --steps 30 --warmup 5 --config $cfg --no-extra --kv-bytes 67108864 > gpurun_out/ovl_${cfg}_${nb}.json 2> gpurun_out/ovl_${cfg}_${nb}.err
  done
done
