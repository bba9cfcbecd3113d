# P2 fused all-gather epilogue: GPU tests (single process + CUDA IPC across processes), full GPU suite, c5 bench
mkdir -p gpurun_out
T=${1:-x}
timeout -s KILL 600 python -m pytest tests/test_gpu_peers.py -m gpu -x -q 2>&1 | tail -15 > gpurun_out/peers_$T.log
timeout -s KILL 900 python -m pytest tests -m gpu -q 2>&1 | tail -5 > gpurun_out/gpu_all_$T.log
for i in 1 2; do timeout -s KILL 300 python bench.py --no-cpu-baseline --steps 30 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['value'], d['roofline']['achieved'])" >> gpurun_out/peers_bench_$T.txt; done
