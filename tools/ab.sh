# A/B of an environment switch on the Inception-BN bench (N=1): $1 = VAR=value
for i in 1 2; do
  python bench.py --steps 30 --warmup 5 --no-extra --kv-bytes 1048576 > gpurun_out/ab_base_$i.json 2>/dev/null
  env $1 python bench.py --steps 30 --warmup 5 --no-extra --kv-bytes 1048576 > gpurun_out/ab_exp_$i.json 2>/dev/null
done
for f in gpurun_out/ab_base_*.json gpurun_out/ab_exp_*.json; do
  python -c "import json; d=json.loads(open('$f').read().strip().splitlines()[-1]); print('$f', round(d['value']), round(d['ms_per_step'],4))"
done
