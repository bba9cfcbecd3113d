# NEXT-4 boost: GPU parity (boost tests + errors) and bench lines for the boost mode
mkdir -p gpurun_out
T=${1:-x}
timeout -s KILL 900 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "boost or zz" -s 2>&1 | grep -v "^PARITY" | tail -5 > gpurun_out/boost_test_$T.log
timeout -s KILL 900 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "boost or zz" -s 2>&1 | grep "^PARITY" > gpurun_out/boost_parity_$T.log
for b in 2.25 4; do
  timeout -s KILL 300 python bench.py --boost $b --no-cpu-baseline --steps 30 > gpurun_out/bench_boost${b}_$T.json 2> gpurun_out/bench_boost${b}_$T.err
done
timeout -s KILL 300 python bench.py --api split --no-cpu-baseline --steps 30 > gpurun_out/bench_split_$T.json 2>&1
