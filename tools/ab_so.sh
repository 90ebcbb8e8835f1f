# A/B of two builds of libmgx.so on the Inception-BN bench (N=1): the tree's
# build vs paper_1512_01274_b200/libmgx_base.so, alternating
L=paper_1512_01274_b200
cp $L/libmgx.so /tmp/libmgx_new.so
for i in 1 2; do
  for v in new base; do
    cp /tmp/libmgx_$v.so $L/libmgx.so 2>/dev/null || cp $L/libmgx_base.so $L/libmgx.so
    [ $v = base ] && cp $L/libmgx_base.so $L/libmgx.so
    echo "$v $(python bench.py --steps 30 --warmup 5 --no-extra --kv-bytes 1048576 2>/dev/null | tail -1 | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(round(d["value"]), round(d["ms_per_step"],4))')"
  done
done
cp /tmp/libmgx_new.so $L/libmgx.so
