bash scripts/gpu_variants.sh ${1:-x}
timeout -s KILL 300 python scripts/trace_attn.py --ctas 1 > gpurun_out/trace_${1:-x}.txt 2>&1
DSCACHE_LIB=$PWD/paper_2605_01858_b200/variants/libdscache_sm1.so timeout -s KILL 300 python scripts/trace_attn.py --ctas 1 > gpurun_out/trace_${1:-x}_sm1.txt 2>&1
