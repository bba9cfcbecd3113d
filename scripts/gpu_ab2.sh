# interleaved A/B (2 rounds) of the default library and every variant: c5 fused bench
mkdir -p gpurun_out
OUT=gpurun_out/ab_${1:-x}.txt; : > $OUT
for round in 1 2; do
for lib in paper_2605_01858_b200/libdscache.so paper_2605_01858_b200/variants/*.so; do
  v=$(DSCACHE_LIB=$PWD/$lib timeout -s KILL 300 python bench.py --no-cpu-baseline --steps 30 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['value'], d['roofline']['achieved'])")
  echo "round $round $(basename $lib) | $v" | tee -a $OUT
done; done
