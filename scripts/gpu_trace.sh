mkdir -p gpurun_out
timeout -s KILL 600 python -m pytest tests/test_gpu_parity.py -q -m gpu --timeout 300 -p no:cacheprovider -x -k "c2_bf16_tcgen05 or edge or debug or c5" > gpurun_out/test_trace.log 2>&1; echo rc=$? >> gpurun_out/test_trace.log; tail -2 gpurun_out/test_trace.log
timeout -s KILL 300 python scripts/trace_attn.py --ctas 2 > gpurun_out/trace.txt 2>&1
python bench.py --no-cpu-baseline > gpurun_out/bench_trace.json 2>&1; cat gpurun_out/bench_trace.json | head -c 600
