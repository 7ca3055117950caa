# compute-sanitizer memcheck / racecheck / synccheck on small cases of every
# kernel family (GPU box):  bash tools/sanitize.sh  -> gpurun_out/sanitize_*.log
CS=/usr/local/cuda/bin/compute-sanitizer
PY="python tools/sanitize_cases.py"
for tool in memcheck racecheck synccheck; do
  for case in f32_sorted_cluster f32_unsorted f32_minibatch f32_exact_tma f64 joint letkf; do
    timeout 900 $CS --tool $tool --error-exitcode 99 --print-limit 20 $PY $case \
      > gpurun_out/sanitize_${tool}_${case}.log 2>&1
    echo "$tool $case rc=$? $(grep -E 'ERROR SUMMARY|RACECHECK SUMMARY' gpurun_out/sanitize_${tool}_${case}.log | tail -1)"
  done
done
