# interleaved A/B of the product library and every variant on the single-stream configs
# (c2, c4, kvsplit) and c5: value, ms/step, attention TFLOP/s
mkdir -p gpurun_out
T=${1:-small}
for round in 1 2; do for args in "--config c2" "--config c4" "--mode kvsplit" "--config c5"; do
for lib in paper_2605_01858_b200/libdscache.so $(ls paper_2605_01858_b200/variants/*.so | grep -v trace | grep -v checked); do
  v=$(DSCACHE_LIB=$PWD/$lib timeout -s KILL 300 python bench.py $args --no-cpu-baseline --no-extras --steps 60 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['value'], d['ms_per_step'], d['roofline']['achieved'])")
  echo "r$round $args $(basename $lib) | $v" | tee -a gpurun_out/ab_$T.txt
done; done; done
