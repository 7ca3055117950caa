# compute-sanitizer stand-in (the tool is closed on the GPU pool): rebuild the
# library with device-side bounds assertions (make CHECKED=1), then run the
# small per-family cases and the parity / determinism suites under it.  Any
# out-of-bounds index traps (cudaErrorAssert) and fails the run.
set -o pipefail
make -C paper_2407_12168_b200/csrc clean > /dev/null
timeout 900 make -C paper_2407_12168_b200/csrc -j16 CHECKED=1 PY=python3 > gpurun_out/checked_build.log 2>&1 || { echo "checked build failed"; exit 1; }
for case in f32_sorted_multi_cta f32_unsorted f32_unsorted_generic f32_minibatch f32_exact_tma f64 joint joint_big letkf; do
  timeout 600 python tools/checked_cases.py $case > gpurun_out/checked_$case.log 2>&1; echo "checked case $case rc=$?"
done
timeout 1800 python -m pytest tests/test_gpu_parity.py tests/test_gpu_determinism.py tests/test_gpu_letkf.py \
  -q -p no:cacheprovider -m "gpu and not slow" > gpurun_out/checked_tests.log 2>&1; echo "checked pytest rc=$?"
tail -3 gpurun_out/checked_tests.log
