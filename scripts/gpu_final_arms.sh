# final-session arms: reference (oracle) arm, and the torchrun launch the driver uses for N > 1 (here N = 1)
mkdir -p gpurun_out
S=$(date +%s); timeout -s KILL 600 python bench.py --impl reference > gpurun_out/fa_ref.json 2> gpurun_out/fa_ref.err; echo "ref rc=$? $(( $(date +%s) - S ))s"; cut -c1-400 gpurun_out/fa_ref.json
S=$(date +%s); timeout -s KILL 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 1 --master-addr 127.0.0.1 --master-port 29517 bench.py --gpus 1 --steps 20 --warmup 3 > gpurun_out/fa_torchrun1.json 2> gpurun_out/fa_torchrun1.err; echo "torchrun rc=$? $(( $(date +%s) - S ))s"; cut -c1-300 gpurun_out/fa_torchrun1.json
for m in kvsplit context decode; do
timeout -s KILL 300 python bench.py --mode $m --no-cpu-baseline --steps 30 > gpurun_out/fa_$m.json 2> gpurun_out/fa_$m.err; echo "$m rc=$?"; python -c "import json; d=json.load(open('gpurun_out/fa_$m.json')); print('$m', d['value'], d['unit'], d['roofline']['achieved'], d['roofline']['unit'], d['roofline']['frac'], d['clocks']['sm_mhz'], d['clocks']['reasons'])"
done
