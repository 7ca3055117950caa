# GPU: config-2 cycled golden from the reference driver, then the GPU suite
timeout 2400 python tests/golden/make_cycle_golden.py gpurun_out/cycle_cfg2_reference.json > gpurun_out/r02_golden.log 2>&1; echo "golden rc=$?"; tail -2 gpurun_out/r02_golden.log
cp gpurun_out/cycle_cfg2_reference.json tests/golden/ 2>/dev/null
timeout 2400 python -m pytest tests -m gpu -x -q -p no:cacheprovider > gpurun_out/r02_gputests2.log 2>&1; echo "pytest rc=$?"
tail -15 gpurun_out/r02_gputests2.log
