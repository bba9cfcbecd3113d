# ablation timing: default vs variants (c5 bench, split api so build/attend are separate launches), + traces
mkdir -p gpurun_out
OUT=gpurun_out/abl.txt; : > $OUT
for lib in paper_2605_01858_b200/libdscache.so paper_2605_01858_b200/variants/*.so; do
  v=$(DSCACHE_LIB=$PWD/$lib timeout -s KILL 300 python bench.py --no-cpu-baseline --steps 30 --api split 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['value'], d['roofline']['achieved'])")
  echo "$(basename $lib) | $v" | tee -a $OUT
  DSCACHE_LIB=$PWD/$lib timeout -s KILL 300 python scripts/trace_attn.py --ctas 2 > gpurun_out/trace_$(basename $lib .so).txt 2>&1
done
