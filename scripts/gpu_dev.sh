# dev loop: GPU parity (fail fast), c5 bench, traces of default + variants
mkdir -p gpurun_out
TAG=${1:-d}
timeout -s KILL 900 python -m pytest tests/test_gpu_parity.py -q -x -m gpu --timeout 600 -p no:cacheprovider > gpurun_out/test_$TAG.log 2>&1
RC=$?; echo rc=$RC >> gpurun_out/test_$TAG.log; tail -3 gpurun_out/test_$TAG.log
if [ $RC -ne 0 ]; then grep -E "Error|error|assert|FAIL" gpurun_out/test_$TAG.log | head -30; exit $RC; fi
OUT=gpurun_out/dev_$TAG.txt; : > $OUT
for lib in paper_2605_01858_b200/libdscache.so paper_2605_01858_b200/variants/*.so; do
  [ -f "$lib" ] || continue
  for api in fused split; do
  v=$(DSCACHE_LIB=$PWD/$lib timeout -s KILL 300 python bench.py --no-cpu-baseline --steps 30 --api $api 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['value'], d['roofline']['achieved'], d['roofline'].get('traffic'))")
  echo "$(basename $lib) $api | $v" | tee -a $OUT
  done
done
# event timeline of the default build (trace variant compiled by the script)
timeout -s KILL 300 python scripts/trace_attn.py --ctas 2 --streams 64 > gpurun_out/trace_${TAG}.txt 2>&1
grep -E "==|summary|switch" gpurun_out/trace_${TAG}.txt | tee -a $OUT
