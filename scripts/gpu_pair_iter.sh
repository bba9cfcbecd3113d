# one iteration of the pair kernel: parity, c5/c3/c4/c2 bench (v8 and v7), a trace
mkdir -p gpurun_out/it
export DSC_WATCHDOG=1 DSC_WATCHDOG_CLK=4000000000
T=${1:-x}
DSC_FA=8 timeout 600 python -m pytest tests/test_gpu_parity.py -x -q -m gpu > gpurun_out/it/${T}_parity.txt 2>&1; echo "parity rc=$? $(tail -1 gpurun_out/it/${T}_parity.txt)"
for c in ${CFGS:-c5 c3 c4 c2}; do
  for v in 8 ${V7:-}; do
    DSC_FA=$v timeout -s KILL 240 python bench.py --config $c --no-extras --no-cpu-baseline --steps 30 > gpurun_out/it/${T}_${c}_v${v}.json 2> gpurun_out/it/${T}_${c}_v${v}.err
    python -c "import json; d=json.load(open('gpurun_out/it/${T}_${c}_v${v}.json')); r=d['roofline']; print('$c v$v', d['value'], r['achieved'], r['frac'], d['clocks']['sm_mhz'], d['clocks']['reasons'])" 2>&1 | tail -1
  done
done
DSC_FA=8 timeout 200 python scripts/trace_pair.py --lib paper_2605_01858_b200/variants/libdscache_ptrace.so --items 3 --tiles 4 > gpurun_out/it/${T}_trace.txt 2>&1
DSC_FA=8 timeout 200 python scripts/trace_pair.py --lib paper_2605_01858_b200/variants/libdscache_ptrace.so --items 3 --tiles 4 --first-item 40 > gpurun_out/it/${T}_trace2.txt 2>&1
