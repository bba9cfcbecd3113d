mkdir -p gpurun_out
for v in "" ord0; do
  if [ -z "$v" ]; then L=$PWD/paper_2605_01858_b200/libdscache.so; else L=$PWD/paper_2605_01858_b200/variants/libdscache_$v.so; fi
  DSCACHE_LIB=$L python bench.py --steps 2 --warmup 3 --no-cpu-baseline --api split > /dev/null 2>&1 && \
  DSCACHE_LIB=$L ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sector_hit_rate.pct --clock-control none -k regex:attn_tc -s 8 -c 2 python bench.py --steps 2 --warmup 3 --no-cpu-baseline --api split 2>&1 | grep -E "attn_tc|duration|dram__|lts__" | tee gpurun_out/ord_$v.txt
done
