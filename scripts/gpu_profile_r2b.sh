# round 2 final evidence: GPU tests, bench lines of every config / mode, per-config ncu launch
# lists and ncu --set full captures of the fused step (c5/c2/c3/c4) and of the decode kernel
mkdir -p gpurun_out
T=${1:-r2b}
timeout -s KILL 1500 python -m pytest tests -q -m gpu -p no:cacheprovider --timeout 900 > gpurun_out/${T}_test.log 2>&1
echo "pytest rc=$?"; tail -2 gpurun_out/${T}_test.log
run() {  # name, args...
  n=$1; shift
  timeout -s KILL 600 python bench.py "$@" > gpurun_out/${T}_bench_$n.json 2> gpurun_out/${T}_bench_$n.err
  echo "bench $n rc=$? $(head -c 400 gpurun_out/${T}_bench_$n.json | cut -c1-160)"
}
run c5
run c5split --api split --no-cpu-baseline
run c2 --config c2 --steps 200 --no-cpu-baseline
run c3 --config c3 --steps 20 --no-cpu-baseline
run c3seq --config c3 --steps 10 --layer-seq --no-cpu-baseline
run c4 --config c4 --steps 200 --no-cpu-baseline
run c1 --config c1 --steps 200 --no-cpu-baseline
run kvsplit --mode kvsplit --steps 200 --no-cpu-baseline
run context --mode context --steps 200 --no-cpu-baseline
run boost4 --boost 4 --no-cpu-baseline
run approx8 --instant-frames 8 --approx 8 --no-cpu-baseline
run exact8 --instant-frames 8 --no-cpu-baseline
run dec_c5 --mode decode --steps 50
run dec_c5s2 --mode decode --decode-stride 2 --steps 50
run dec_c2 --mode decode --config c2 --steps 200
run dec_c4 --mode decode --config c4 --steps 200
run ref --impl reference --steps 3
for c in c5 c2 c3 c4; do
  CMD="python bench.py --config $c --no-cpu-baseline --steps 2 --warmup 3"
  $CMD > gpurun_out/ncu_plain_${T}_$c.log 2>&1 && \
  ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_${T}_$c.csv $CMD > gpurun_out/ncu_l_${T}_$c.log 2>&1 && \
  ncu --set full --clock-control none --import-source on -k regex:attn_fa -s 4 -c 1 -o gpurun_out/prof_${T}_$c $CMD > gpurun_out/ncu_${T}_$c.log 2>&1
  echo "ncu $c rc=$?"
done
for c in c5 c2; do
  CMD="python bench.py --mode decode --config $c --steps 2 --warmup 3"
  $CMD > gpurun_out/ncu_plain_${T}_dec_$c.log 2>&1 && \
  ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_${T}_dec_$c.csv $CMD > gpurun_out/ncu_l_${T}_dec_$c.log 2>&1 && \
  ncu --set full --clock-control none --import-source on -k regex:decode -s 3 -c 1 -o gpurun_out/prof_${T}_dec_$c $CMD > gpurun_out/ncu_${T}_dec_$c.log 2>&1
  echo "ncu decode $c rc=$?"
done
