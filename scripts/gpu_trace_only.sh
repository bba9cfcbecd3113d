mkdir -p gpurun_out
timeout -s KILL 300 python scripts/trace_attn.py --ctas 2 > gpurun_out/trace_${1:-t}.txt 2>&1; tail -3 gpurun_out/trace_${1:-t}.txt
