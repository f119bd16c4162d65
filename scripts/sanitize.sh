# compute-sanitizer over every kernel family (scripts/sanitize_cases.py); logs to gpurun_out/
mkdir -p gpurun_out
CS=/usr/local/cuda/bin/compute-sanitizer
for tool in memcheck racecheck synccheck initcheck; do
  NLSE_CUDA_MALLOC=1 timeout 1500 $CS --tool $tool --print-limit 50 --error-exitcode 9 \
    python scripts/sanitize_cases.py > gpurun_out/sanitizer_$tool.log 2>&1
  echo "$tool rc=$?"
  tail -3 gpurun_out/sanitizer_$tool.log
done
