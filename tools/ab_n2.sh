# A/B of env settings on a bench config at N=2 (torchrun): CFG=<config> $@ = settings
CFG=${CFG:-inception_bn}
run() { env "$@" timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port $((29500 + RANDOM % 400)) bench.py --gpus 2 --steps 30 --warmup 5 --config $CFG --no-extra --kv-bytes 1048576 2>/dev/null | tail -1; }
for i in 1 2; do
  echo "base $(run MGX_NONE=1 | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(round(d["value"]), round(d["ms_per_step"],4))')"
  for e in "$@"; do
    echo "$e $(run $e | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(round(d["value"]), round(d["ms_per_step"],4))')"
  done
done
