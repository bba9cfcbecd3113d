bash scripts/gpu_variants.sh ${1:-x}
timeout -s KILL 300 python scripts/trace_attn.py --ctas 1 > gpurun_out/trace_${1:-x}.txt 2>&1
