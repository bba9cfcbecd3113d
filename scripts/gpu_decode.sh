# decode kernel: parity tests + bench lines (c5 / c2 / c4, strides 1 and 2)
mkdir -p gpurun_out
T=${1:-dec}
timeout -s KILL 600 python -m pytest tests/test_gpu_decode.py -q -m gpu -x --timeout 300 -p no:cacheprovider > gpurun_out/${T}_test.log 2>&1
echo "pytest rc=$?"; tail -3 gpurun_out/${T}_test.log | cut -c1-300
for c in c5 c2 c4; do for st in 1 2; do
  timeout -s KILL 300 python bench.py --mode decode --config $c --decode-stride $st --steps 50 > gpurun_out/${T}_${c}_s$st.json 2> gpurun_out/${T}_${c}_s$st.err
  python -c "import json; d=json.load(open('gpurun_out/${T}_${c}_s$st.json')); print('$c stride $st', d['value'], d['ms_per_step'], d['roofline']['achieved'], d['roofline']['frac'], d['clocks']['sm_mhz'])" || tail -5 gpurun_out/${T}_${c}_s$st.err
done; done
