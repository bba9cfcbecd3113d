# NEXT-3 sweep: exact (fused / split) vs approximate instant cache (periods 4/8/16) at l_I 4/8/16
mkdir -p gpurun_out
T=${1:-apx}
for L in 4 8 16; do
  for M in fused split 4 8 16; do
    if [ "$M" = fused ] || [ "$M" = split ]; then A="--api $M"; else A="--approx $M"; fi
    timeout -s KILL 300 python bench.py --config ${CFG:-c5} --instant-frames $L $A --no-cpu-baseline --steps 30 \
      > gpurun_out/${T}_L${L}_${M}.json 2> gpurun_out/${T}_L${L}_${M}.err
    python -c "import json; d=json.load(open('gpurun_out/${T}_L${L}_${M}.json')); print('lI=$L mode=$M', d['value'], d['ms_per_step'], d['roofline']['achieved'], d['clocks']['sm_mhz'], d['clocks']['reasons'])" || tail -3 gpurun_out/${T}_L${L}_${M}.err
  done
done
