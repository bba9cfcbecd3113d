mkdir -p gpurun_out
timeout -s KILL 600 python -m pytest tests/test_gpu_checkpoint.py -q -m gpu --timeout 300 -p no:cacheprovider > gpurun_out/ckpt_test.log 2>&1; echo "pytest rc=$?"; tail -25 gpurun_out/ckpt_test.log | cut -c1-400
