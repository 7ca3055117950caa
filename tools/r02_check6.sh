bash tools/r02_check5.sh
timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_gpu_determinism.py -q -p no:cacheprovider -x > gpurun_out/r02_gputests6.log 2>&1; echo "pytest rc=$?"
grep -E "passed|failed|FAILED|Error" gpurun_out/r02_gputests6.log | tail -8
