# parity tests, then (only if green) bench c5/c2 and an ncu capture of the attention kernel
mkdir -p gpurun_out
TAG=${1:-r}
timeout -s KILL 900 python -m pytest tests/test_gpu_parity.py -q -s -m gpu --timeout 600 -p no:cacheprovider > gpurun_out/test_$TAG.log 2>&1
RC=$?; echo rc=$RC >> gpurun_out/test_$TAG.log; tail -3 gpurun_out/test_$TAG.log
if [ $RC -ne 0 ]; then exit $RC; fi
python bench.py > gpurun_out/bench_c5_$TAG.json 2> gpurun_out/bench_c5_$TAG.err; cat gpurun_out/bench_c5_$TAG.json
python bench.py --config c2 --steps 50 --no-cpu-baseline > gpurun_out/bench_c2_$TAG.json 2> gpurun_out/bench_c2_$TAG.err; cat gpurun_out/bench_c2_$TAG.json
if [ "$2" = "ncu" ]; then
python bench.py --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/plain_$TAG.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:attn_tc -s 4 -c 2 -o gpurun_out/prof_c5_$TAG python bench.py --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/ncu_$TAG.log 2>&1
fi
echo done
