# correctness after the fused-path threshold + staging-pool exit fix; then sanitizers
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/r02_gputests8.log 2>&1; echo "pytest rc=$?"
grep -E "passed|failed|FAILED|Error" gpurun_out/r02_gputests8.log | tail -12
timeout 300 python bench.py --config cfg1 --steps 20 --no-cpu-baseline --no-fp64 > gpurun_out/r02_cfg1.json 2>/dev/null; echo "cfg1 rc=$?"
timeout 1500 bash tools/sanitize.sh
