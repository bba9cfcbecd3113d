# one --set full capture (with source counters) of the split build / attend launches (c5)
mkdir -p gpurun_out
TAG=${1:-s}
python bench.py --steps 2 --warmup 3 --no-cpu-baseline --api split > gpurun_out/plain_$TAG.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:attn_tc -s 4 -c 2 -o gpurun_out/prof_src_$TAG python bench.py --steps 2 --warmup 3 --no-cpu-baseline --api split > gpurun_out/ncu_$TAG.log 2>&1
echo rc=$?
