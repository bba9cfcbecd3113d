mkdir -p gpurun_out
timeout -s KILL 1500 python -m pytest tests -q -m gpu -x --timeout 600 -p no:cacheprovider > gpurun_out/val_gputests.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/val_gputests.log
timeout -s KILL 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/val_smoke.log 2>&1; echo "smoke rc=$?"; tail -2 gpurun_out/val_smoke.log
timeout -s KILL 600 python bench.py > gpurun_out/val_bench.json 2> gpurun_out/val_bench.err; echo "bench rc=$?"; cat gpurun_out/val_bench.json | cut -c1-600
