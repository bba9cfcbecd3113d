# round evidence (r06 = r04 + the peer-epilogue / IPC tests and the boost bench lines): GPU parity (with the per-case error report), every config's bench line (N=1),
# kvsplit, the default bench (with cpu_baseline), the reference arm, an ncu launch list,
# --set full captures (fused step + split build / attend) and the append kernel's DRAM rate
mkdir -p gpurun_out
TAG=${1:-r12}
timeout -s KILL 1200 python -m pytest tests/test_gpu_parity.py -q -s -m gpu --timeout 1000 -p no:cacheprovider > gpurun_out/parity_$TAG.log 2>&1
echo "parity rc=$?"; tail -2 gpurun_out/parity_$TAG.log
timeout -s KILL 600 python -m pytest tests/test_gpu_peers.py -q -m gpu -p no:cacheprovider > gpurun_out/peers_$TAG.log 2>&1
echo "peers rc=$?"; tail -1 gpurun_out/peers_$TAG.log
for b in 2.25 4; do
  python bench.py --boost $b --no-cpu-baseline --steps 40 > gpurun_out/bench_${TAG}_boost$b.json 2> gpurun_out/bench_${TAG}_boost$b.err
  head -c 120 gpurun_out/bench_${TAG}_boost$b.json; echo
done
for c in c1 c2 c3 c4 c5; do
  python bench.py --config $c --no-cpu-baseline --steps 40 > gpurun_out/bench_${TAG}_$c.json 2> gpurun_out/bench_${TAG}_$c.err
  head -c 160 gpurun_out/bench_${TAG}_$c.json; echo
done
python bench.py --mode kvsplit --no-cpu-baseline --steps 40 > gpurun_out/bench_${TAG}_kvsplit.json 2>&1; head -c 160 gpurun_out/bench_${TAG}_kvsplit.json; echo
python bench.py > gpurun_out/bench_$TAG.json 2> gpurun_out/bench_$TAG.err; head -c 300 gpurun_out/bench_$TAG.json; echo
python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/bench_${TAG}_ref.json 2>&1; head -c 200 gpurun_out/bench_${TAG}_ref.json; echo
python bench.py --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/plain_$TAG.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_$TAG.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/ncu_launch_$TAG.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:attn_tc -s 4 -c 1 -o gpurun_out/prof_$TAG python bench.py --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/ncu_full_$TAG.log 2>&1
echo "ncu rc=$?"
python bench.py --steps 2 --warmup 3 --no-cpu-baseline --api split > gpurun_out/plain_split_$TAG.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:attn_tc -s 8 -c 2 -o gpurun_out/prof_split_$TAG python bench.py --steps 2 --warmup 3 --no-cpu-baseline --api split > gpurun_out/ncu_full_split_$TAG.log 2>&1
echo "ncu split rc=$?"
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed --clock-control none -k regex:"append_kernel|stage_instant" -s 40 -c 6 --csv --log-file gpurun_out/append_$TAG.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/ncu_append_$TAG.log 2>&1
echo "ncu append rc=$?"
