# round 2 evidence: GPU tests, bench lines of every config/mode, ncu launch list (c5) and
# ncu --set full captures of the fused launch for c5 / c2 / c3 / c4
mkdir -p gpurun_out
T=${1:-r2a}
timeout -s KILL 1200 python -m pytest tests -q -m gpu -x -p no:cacheprovider --timeout 900 > gpurun_out/${T}_test.log 2>&1
echo "pytest rc=$?"; tail -2 gpurun_out/${T}_test.log
grep PARITY gpurun_out/${T}_test.log | wc -l
run() {  # name, args...
  n=$1; shift
  timeout -s KILL 600 python bench.py "$@" > gpurun_out/${T}_bench_$n.json 2> gpurun_out/${T}_bench_$n.err
  echo "bench $n rc=$? $(head -c 300 gpurun_out/${T}_bench_$n.json | cut -c1-200)"
}
run c5
run c2 --config c2 --steps 200 --no-cpu-baseline
run c3 --config c3 --steps 20 --no-cpu-baseline
run c3seq --config c3 --steps 10 --layer-seq --no-cpu-baseline
run c4 --config c4 --steps 200 --no-cpu-baseline
run c1 --config c1 --steps 200 --no-cpu-baseline
run kvsplit --mode kvsplit --steps 200 --no-cpu-baseline
run context --mode context --steps 200 --no-cpu-baseline
run ref --impl reference --steps 3
CMD="python bench.py --no-cpu-baseline --steps 2 --warmup 3"
$CMD > gpurun_out/ncu_plain_${T}.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_${T}.csv $CMD > gpurun_out/ncu_l_${T}.log 2>&1
echo "ncu launches rc=$?"
for c in c5 c2 c3 c4; do
  CMD="python bench.py --config $c --no-cpu-baseline --steps 2 --warmup 3"
  $CMD > gpurun_out/ncu_plain_${T}_$c.log 2>&1 && \
  ncu --set full --clock-control none --import-source on -k regex:attn_fa -s 4 -c 1 -o gpurun_out/prof_${T}_$c $CMD > gpurun_out/ncu_${T}_$c.log 2>&1
  echo "ncu full $c rc=$?"
done
