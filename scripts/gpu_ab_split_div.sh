mkdir -p gpurun_out; OUT=gpurun_out/ab_div.txt; : > $OUT
for round in 1 2; do
for args in "--config c2 --steps 200" "--config c4 --steps 200" "--mode kvsplit --steps 200" "--mode context --steps 200"; do
for lib in $(ls paper_2605_01858_b200/variants/libdscache_div*.so); do
  v=$(DSCACHE_LIB=$PWD/$lib timeout -s KILL 300 python bench.py $args --no-cpu-baseline --no-extras 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['value'], d['roofline']['achieved'], d['clocks']['sm_mhz'])")
  echo "r$round $args $(basename $lib) | $v" | tee -a $OUT
done; done; done
