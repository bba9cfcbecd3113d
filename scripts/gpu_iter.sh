# iteration: fast parity subset, c5 bench, trace of the fused step
mkdir -p gpurun_out
T=${1:-it}
timeout -s KILL 600 python -m pytest tests/test_gpu_parity.py -q -m gpu -x --timeout 300 -p no:cacheprovider ${PARITY_K:+-k "$PARITY_K"} > gpurun_out/${T}_test.log 2>&1
echo "pytest rc=$?"; tail -3 gpurun_out/${T}_test.log | cut -c1-300
for c in ${CFGS:-c5}; do
timeout -s KILL 300 python bench.py --config $c --no-cpu-baseline --steps 30 > gpurun_out/${T}_bench_$c.json 2> gpurun_out/${T}_bench_$c.err; echo "bench $c rc=$?"; python -c "import json; d=json.load(open('gpurun_out/${T}_bench_$c.json')); print('$c', d['value'], d['roofline']['achieved'], d['roofline']['frac'], d['clocks'])"
done
[ -f paper_2605_01858_b200/variants/libdscache_trace.so ] && timeout -s KILL 120 python scripts/trace_fa.py --lib paper_2605_01858_b200/variants/libdscache_trace.so --ctas 2 --items 10 > gpurun_out/${T}_trace.txt 2>&1; grep -E "===|latency|period|switch|prep" gpurun_out/${T}_trace.txt
