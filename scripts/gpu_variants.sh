# A/B the tuning variants under paper_2605_01858_b200/variants/ on the c5 bench (+ a parity smoke per variant)
mkdir -p gpurun_out
OUT=gpurun_out/variants_${1:-x}.txt; : > $OUT
for lib in paper_2605_01858_b200/libdscache.so paper_2605_01858_b200/variants/*.so; do
  export DSCACHE_LIB=$PWD/$lib
  ok=$(timeout -s KILL 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1)
  v=$(timeout -s KILL 300 python bench.py --no-cpu-baseline --steps 40 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['value'], d['roofline']['achieved'], d['roofline']['frac'])")
  echo "$(basename $lib) | $v | $ok" | tee -a $OUT
done
