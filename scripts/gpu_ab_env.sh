# A/B of an environment switch on the product library: VAR=name VALS="0 1" bash scripts/gpu_ab_env.sh TAG cfgs...
mkdir -p gpurun_out
T=${1:-env}; shift || true
CFGS=${@:-c5}
OUT=gpurun_out/ab_${T}.txt; : > $OUT
for round in 1 2; do
for cfg in $CFGS; do
for v in ${VALS:-0 1}; do
  r=$(env $VAR=$v timeout -s KILL 300 python bench.py --config $cfg --no-cpu-baseline --steps ${STEPS:-60} 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['value'], d['ms_per_step'], d['roofline']['achieved'], d['clocks']['sm_mhz'])")
  echo "r$round $cfg $VAR=$v | $r" | tee -a $OUT
done; done; done
