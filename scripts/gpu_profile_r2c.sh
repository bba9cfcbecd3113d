# round 2 (v8 pair kernel) evidence: bench lines of every config / mode (+ v7 for comparison),
# per-config ncu launch lists and ncu --set full captures of the fused step (c5/c2/c3/c4), and
# the GPU suite under the bounds-checked (DSC_CHECK) build
mkdir -p gpurun_out
T=${1:-r2c}
run() {  # name, args...
  n=$1; shift
  timeout -s KILL 600 python bench.py "$@" > gpurun_out/${T}_bench_$n.json 2> gpurun_out/${T}_bench_$n.err
  echo "bench $n rc=$? $(head -c 300 gpurun_out/${T}_bench_$n.json | cut -c1-150)"
}
run c5
DSC_FA=7 run c5_v7 --no-cpu-baseline --no-extras
run c5split --api split --no-cpu-baseline
run c2 --config c2 --steps 200 --no-cpu-baseline
DSC_FA=7 run c2_v7 --config c2 --steps 200 --no-cpu-baseline --no-extras
run c3 --config c3 --steps 20 --no-cpu-baseline
run c3seq --config c3 --steps 10 --layer-seq --no-cpu-baseline
run c4 --config c4 --steps 200 --no-cpu-baseline
DSC_FA=7 run c4_v7 --config c4 --steps 200 --no-cpu-baseline --no-extras
run c1 --config c1 --steps 200 --no-cpu-baseline
run kvsplit --mode kvsplit --steps 200 --no-cpu-baseline
run context --mode context --steps 200 --no-cpu-baseline
run boost4 --boost 4 --no-cpu-baseline
run approx8 --instant-frames 8 --approx 8 --no-cpu-baseline
run exact8 --instant-frames 8 --no-cpu-baseline
run ref --impl reference --steps 3
for c in c5 c2 c3 c4; do
  CMD="python bench.py --config $c --no-cpu-baseline --no-extras --steps 2 --warmup 3"
  $CMD > gpurun_out/ncu_plain_${T}_$c.log 2>&1 && \
  ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_${T}_$c.csv $CMD > gpurun_out/ncu_l_${T}_$c.log 2>&1 && \
  ncu --set full --clock-control none --import-source on -k regex:attn_pair -s 4 -c 1 -o gpurun_out/prof_${T}_$c $CMD > gpurun_out/ncu_${T}_$c.log 2>&1
  echo "ncu $c rc=$?"
done
timeout -s KILL 1500 env DSCACHE_LIB=$PWD/paper_2605_01858_b200/variants/libdscache_checked.so python -m pytest tests -q -m gpu -p no:cacheprovider > gpurun_out/${T}_checked_suite.log 2>&1
echo "checked suite rc=$? $(tail -1 gpurun_out/${T}_checked_suite.log)"
