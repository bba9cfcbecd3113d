# round 2, first call: tcgen05 micro numbers, GPU tests, c5 bench (baseline of this round)
mkdir -p gpurun_out
timeout -s KILL 120 ./scripts/micro/mma_bench > gpurun_out/r2_mma_bench.txt 2>&1; cat gpurun_out/r2_mma_bench.txt
timeout -s KILL 900 python -m pytest tests -q -m gpu -x --timeout 600 -p no:cacheprovider > gpurun_out/r2_test0.log 2>&1
echo "pytest rc=$?"; tail -3 gpurun_out/r2_test0.log
python bench.py --no-cpu-baseline > gpurun_out/r2_bench0.json 2> gpurun_out/r2_bench0.err; head -c 1500 gpurun_out/r2_bench0.json
