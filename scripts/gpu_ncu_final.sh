# ncu launch lists + --set full of the pair kernel's fused-step launch, c5/c2/c3/c4 (final library)
mkdir -p gpurun_out
T=${1:-r2e}
for c in c5 c2 c3 c4; do
  CMD="python bench.py --config $c --no-cpu-baseline --no-extras --steps 2 --warmup 3"
  $CMD > gpurun_out/bench_${T}_$c.json 2> gpurun_out/ncu_plain_${T}_$c.log && \
  ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_${T}_$c.csv $CMD > gpurun_out/ncu_l_${T}_$c.log 2>&1 && \
  ncu --set full --clock-control none --import-source on -k regex:attn_pair -s 4 -c 1 -o gpurun_out/prof_${T}_$c $CMD > gpurun_out/ncu_${T}_$c.log 2>&1
  echo "ncu $c rc=$?"
done
