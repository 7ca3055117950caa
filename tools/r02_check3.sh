timeout 1500 python tests/golden/make_cycle_golden.py short gpurun_out/cycle_cfg2_short_reference.json > gpurun_out/r02_golden_short.log 2>&1; echo "golden rc=$?"; tail -2 gpurun_out/r02_golden_short.log
cp gpurun_out/cycle_cfg2_short_reference.json tests/golden/ 2>/dev/null
timeout 1800 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/r02_gputests3.log 2>&1; echo "pytest rc=$?"
grep -E "passed|failed|FAILED|Error" gpurun_out/r02_gputests3.log | tail -25
python tools/hostreg_probe.py 2>&1 | tail -8
