for cfg in "2 148 112" "4 148 112" "4 96 112" "4 64 200" "8 32 200"; do
  set -- $cfg
  MGX_BNF_MINW=$1 MGX_BNF_MINCTAS=$2 MGX_BNF_SMEM_KB=$3 ncu --metrics gpu__time_duration.sum --clock-control none --cache-control none --csv --log-file gpurun_out/bnf_sweep_$1_$2_$3.csv python tools/kbench.py bnf > /dev/null 2>&1
  echo "cfg $cfg -> $?"
done
