# The in-house sanitizer pass (compute-sanitizer is closed on the GPU pool): the whole GPU
# test suite and scripts/sanitize_run.py against the DSC_CHECK=1 build, whose kernels trap
# on any out-of-range global row / TMA box / workspace index (paper_2605_01858_b200/csrc,
# DSC_ASSERT).  Build first: python -m paper_2605_01858_b200._build --checked
mkdir -p gpurun_out
export DSCACHE_LIB=$PWD/paper_2605_01858_b200/variants/libdscache_checked.so
python scripts/sanitize_run.py > gpurun_out/chk_run.txt 2>&1; echo "sanitize_run rc=$?"; tail -6 gpurun_out/chk_run.txt
timeout -s KILL 1500 python -m pytest tests -q -m gpu -p no:cacheprovider --timeout 900 > gpurun_out/chk_tests.log 2>&1
echo "pytest (checked build) rc=$?"; tail -3 gpurun_out/chk_tests.log
grep -c "DSC_CHECK failed" gpurun_out/chk_tests.log gpurun_out/chk_run.txt
