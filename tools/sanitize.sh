# compute-sanitizer over tools/sanitize_cases.py: graph path and direct path
# (TS_NO_GRAPH=1), memcheck / racecheck / synccheck.  Summary -> gpurun_out/sanitize/
mkdir -p gpurun_out/sanitize
for tool in memcheck racecheck synccheck; do
  for mode in graph direct; do
    env=""; [ $mode = direct ] && env="TS_NO_GRAPH=1"
    env $env timeout 1200 /usr/local/cuda/bin/compute-sanitizer --tool $tool --error-exitcode 9 \
      --print-limit 20 python tools/sanitize_cases.py > gpurun_out/sanitize/${tool}_${mode}.log 2>&1
    echo "$tool $mode rc=$?" | tee -a gpurun_out/sanitize/summary.txt
    tail -3 gpurun_out/sanitize/${tool}_${mode}.log
  done
done
