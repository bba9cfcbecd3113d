# v7 (default) vs v5 (DSC_KERNEL=tc) across configs
mkdir -p gpurun_out
OUT=gpurun_out/cmp_${1:-x}.txt; : > $OUT
for cfg in ${CFGS:-c5 c3 c4 c2}; do
for k in fa tc; do
  v=$(DSC_KERNEL=$k timeout -s KILL 300 python bench.py --config $cfg --no-cpu-baseline --steps 30 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['value'], d['roofline']['achieved'], d['roofline']['frac'], d['clocks']['sm_mhz'])")
  echo "$cfg $k | $v" | tee -a $OUT
done; done
