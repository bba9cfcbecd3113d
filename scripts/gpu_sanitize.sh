# compute-sanitizer over scripts/sanitize_run.py, one tool per run (memcheck, racecheck,
# synccheck, initcheck); summaries under gpurun_out/san_<tool>.txt
mkdir -p gpurun_out
python scripts/sanitize_run.py > gpurun_out/san_plain.txt 2>&1; echo "plain rc=$?"
for tool in ${TOOLS:-memcheck racecheck synccheck initcheck}; do
  DSC_WATCHDOG_CLK=0 timeout -s KILL ${SAN_TIMEOUT:-900} compute-sanitizer --tool $tool --print-limit 50 --error-exitcode 9 \
    python scripts/sanitize_run.py > gpurun_out/san_$tool.txt 2>&1
  echo "$tool rc=$?"; grep -E "ERROR SUMMARY|RACECHECK SUMMARY|ok$" gpurun_out/san_$tool.txt | tail -8
done
