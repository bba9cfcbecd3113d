# full GPU suite on the default library + interleaved A/B vs every variant on the given configs
mkdir -p gpurun_out
OUT=gpurun_out/ab_${1:-x}.txt; : > $OUT
shift || true
CFGS=${@:-c5}
echo "default suite: $(timeout -s KILL 1200 python -m pytest tests -m gpu -q -p no:cacheprovider 2>&1 | tail -1)" | tee -a $OUT
for round in 1 2; do
for cfg in $CFGS; do
for lib in paper_2605_01858_b200/libdscache.so paper_2605_01858_b200/variants/*.so; do
  v=$(DSCACHE_LIB=$PWD/$lib timeout -s KILL 300 python bench.py --config $cfg --no-cpu-baseline --steps 30 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['value'], d['roofline']['achieved'])")
  echo "round $round $cfg $(basename $lib) | $v" | tee -a $OUT
done; done; done
