# A/B of v7 variant libraries (all but the trace variant) + a trace of the default
mkdir -p gpurun_out
T=${1:-x}; shift || true
CFGS=${@:-c5}
OUT=gpurun_out/ab_${T}.txt; : > $OUT
for round in 1 2; do
for cfg in $CFGS; do
for lib in paper_2605_01858_b200/libdscache.so $(ls paper_2605_01858_b200/variants/*.so | grep -v trace); do
  v=$(DSCACHE_LIB=$PWD/$lib timeout -s KILL 300 python bench.py --config $cfg --no-cpu-baseline --steps 30 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['value'], d['roofline']['achieved'], d['clocks']['sm_mhz'])")
  echo "r$round $cfg $(basename $lib) | $v" | tee -a $OUT
done; done; done
TR=$(ls paper_2605_01858_b200/variants/*trace*.so 2>/dev/null | head -1)
if [ -n "$TR" ]; then
timeout -s KILL 120 python scripts/trace_fa.py --lib $TR --ctas 2 --items 10 > gpurun_out/${T}_trace.txt 2>&1; grep -E "===|latency|period|switch|prep" gpurun_out/${T}_trace.txt
fi
if [ -n "$NCU" ]; then
CMD="python bench.py --no-cpu-baseline --steps 2 --warmup 3"
$CMD > gpurun_out/ncu_plain_${T}.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:attn_fa -s 4 -c 1 -o gpurun_out/prof_${T} $CMD > gpurun_out/ncu_${T}.log 2>&1
echo "ncu rc=$?"; tail -2 gpurun_out/ncu_${T}.log
fi
