# A/B of env settings on one bench config at N=1: CFG=<config> $@ = settings
CFG=${CFG:-inception_bn}
run() { env "$@" python bench.py --config $CFG --steps 30 --warmup 5 --no-extra --kv-bytes 1048576 2>/dev/null | tail -1 | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(round(d["value"]), round(d["ms_per_step"],4))'; }
for i in 1 2; do
  echo "base $(run MGX_NONE=1)"
  for e in "$@"; do echo "$e $(run $e)"; done
done
