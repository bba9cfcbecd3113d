# A/B of the attention kernels: v8 pair (default) vs v7 (DSC_FA=7) on c5, c3, c4, c2, interleaved
mkdir -p gpurun_out/ab
for rep in 1 2; do
for c in c5 c3 c4 c2; do
  for v in 8 7; do
    DSC_FA=$v timeout -s KILL 240 python bench.py --config $c --no-extras --no-cpu-baseline --steps 30 > gpurun_out/ab/${c}_v${v}_$rep.json 2> gpurun_out/ab/${c}_v${v}_$rep.err
    python -c "import json; d=json.load(open('gpurun_out/ab/${c}_v${v}_$rep.json')); r=d['roofline']; print('$c v$v', d['value'], r['achieved'], r['frac'], d['clocks']['sm_mhz'], d['clocks']['reasons'])" 2>&1 | tail -1
  done
done
done
