# A/B: lazy-rescale threshold of the v8 softmax (PR_RESCALE_T, log2 units) 8 (default) vs 12 / 16, interleaved
mkdir -p gpurun_out/abr
timeout -s KILL 300 env DSCACHE_LIB=paper_2605_01858_b200/variants/libdscache_rs16.so python -m pytest tests/test_gpu_parity.py -q -m gpu -x --timeout 250 -p no:cacheprovider -k "c5 or c3 or c2" > gpurun_out/abr/parity_rs16.log 2>&1; echo "parity rs16 rc=$?"; tail -1 gpurun_out/abr/parity_rs16.log
for rep in 1 2; do
for c in c5 c3; do
  for v in base rs12 rs16; do
    if [ $v = base ]; then L=paper_2605_01858_b200/libdscache.so; else L=paper_2605_01858_b200/variants/libdscache_$v.so; fi
    DSCACHE_LIB=$L timeout -s KILL 240 python bench.py --config $c --no-extras --no-cpu-baseline --steps 30 > gpurun_out/abr/${c}_${v}_$rep.json 2> gpurun_out/abr/${c}_${v}_$rep.err
    python -c "import json; d=json.load(open('gpurun_out/abr/${c}_${v}_$rep.json')); r=d['roofline']; print('$c $v', d['value'], r['achieved'], r['frac'], d['clocks']['sm_mhz'], d['clocks']['reasons'])" 2>&1 | tail -1
  done
done
done
