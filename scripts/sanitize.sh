# compute-sanitizer over the small driver, one tool per pass (reports under gpurun_out/)
CS=/usr/local/cuda/bin/compute-sanitizer
for tool in ${TOOLS:-memcheck racecheck synccheck}; do
  timeout 1500 $CS --tool $tool --print-limit 20 --error-exitcode 9 python scripts/sanitize_driver.py > gpurun_out/sanitize_$tool.log 2>&1
  echo "$tool exit $?" | tee -a gpurun_out/sanitize_summary.txt
done
