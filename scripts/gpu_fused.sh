# fused-step parity + A/B of --api fused vs split on every bench config
mkdir -p gpurun_out
OUT=gpurun_out/fused.txt; : > $OUT
timeout -s KILL 900 python -m pytest tests/test_gpu_parity.py -x -q -k "fused or c2_bf16_tcgen05 or edge" 2>&1 | tail -5 | tee -a $OUT
for round in 1 2; do
for cfg in c5 c2 c3 c4; do
for api in split fused; do
  v=$(timeout -s KILL 300 python bench.py --no-cpu-baseline --config $cfg --api $api --steps 40 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['value'], d['roofline']['achieved'], d['gpu_launches'], d['e2e']['value'])")
  echo "round $round $cfg $api | $v" | tee -a $OUT
done; done; done
