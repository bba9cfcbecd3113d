# parity (all GPU tests), trace, bench c5 + c2
mkdir -p gpurun_out
TAG=${1:-r}
timeout -s KILL 900 python -m pytest tests/test_gpu_parity.py -q -s -m gpu --timeout 600 -p no:cacheprovider -x > gpurun_out/test_$TAG.log 2>&1
RC=$?; echo rc=$RC >> gpurun_out/test_$TAG.log; tail -3 gpurun_out/test_$TAG.log
if [ $RC -ne 0 ]; then grep -E "Error|error|assert" gpurun_out/test_$TAG.log | head -20; exit $RC; fi
timeout -s KILL 300 python scripts/trace_attn.py --ctas 2 > gpurun_out/trace_$TAG.txt 2>&1
python bench.py --no-cpu-baseline > gpurun_out/bench_c5_$TAG.json 2> gpurun_out/bench_c5_$TAG.err; cat gpurun_out/bench_c5_$TAG.json
python bench.py --config c2 --steps 50 --no-cpu-baseline > gpurun_out/bench_c2_$TAG.json 2> gpurun_out/bench_c2_$TAG.err; head -c 700 gpurun_out/bench_c2_$TAG.json
echo done
