# A/B/C of env settings on the Inception-BN bench (N=1): $@ = VAR=value settings (one per run)
for i in 1 2; do
  python bench.py --steps 30 --warmup 5 --no-extra --kv-bytes 1048576 > gpurun_out/abc_base_$i.json 2>/dev/null
  n=0
  for e in "$@"; do
    n=$((n+1))
    env $e python bench.py --steps 30 --warmup 5 --no-extra --kv-bytes 1048576 > gpurun_out/abc_${n}_$i.json 2>/dev/null
  done
done
for f in gpurun_out/abc_*.json; do
  python -c "import json; d=json.loads(open('$f').read().strip().splitlines()[-1]); print('$f', round(d['value']), round(d['ms_per_step'],4))"
done
