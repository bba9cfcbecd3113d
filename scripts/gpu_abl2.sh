# ablation timing of the attention kernel: default vs knob variants (results wrong when set), traces
mkdir -p gpurun_out
OUT=gpurun_out/abl_${1:-x}.txt; : > $OUT
for lib in paper_2605_01858_b200/libdscache.so paper_2605_01858_b200/variants/*.so; do
  v=$(DSCACHE_LIB=$PWD/$lib timeout -s KILL 300 python bench.py --no-cpu-baseline --steps 30 --api split 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['value'], d['roofline']['achieved'])")
  echo "$(basename $lib) | $v" | tee -a $OUT
  DSCACHE_LIB=$PWD/$lib timeout -s KILL 300 python scripts/trace_attn.py --ctas 2 > gpurun_out/trace_${1:-x}_$(basename $lib .so).txt 2>&1
  grep -E "==|summary" gpurun_out/trace_${1:-x}_$(basename $lib .so).txt | tee -a $OUT
done
