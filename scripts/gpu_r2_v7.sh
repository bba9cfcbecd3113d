# v7 kernel bring-up: smoke, GPU parity (-x), c5 bench; v5 bench for comparison
mkdir -p gpurun_out
T=${1:-v7}
timeout -s KILL 120 python __graft_entry__.py --smoke > gpurun_out/${T}_smoke.log 2>&1; echo "smoke rc=$?"; tail -4 gpurun_out/${T}_smoke.log
timeout -s KILL 900 python -m pytest tests/test_gpu_parity.py -q -m gpu -x --timeout 300 -p no:cacheprovider > gpurun_out/${T}_test.log 2>&1
echo "pytest rc=$?"; tail -15 gpurun_out/${T}_test.log | cut -c1-300
timeout -s KILL 300 python bench.py --no-cpu-baseline > gpurun_out/${T}_bench_c5.json 2> gpurun_out/${T}_bench_c5.err; echo "bench rc=$?"; head -c 900 gpurun_out/${T}_bench_c5.json; tail -3 gpurun_out/${T}_bench_c5.err
