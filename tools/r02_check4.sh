for cfg in cfg3 cfg2 cfg5; do for rcp in 0 1; do
  TURBDA_F32_RCP=$rcp python bench.py --config $cfg --no-cpu-baseline --no-fp64 --no-e2e-variants --steps ${STEPS:-5} > gpurun_out/sw.json 2>gpurun_out/sw.err
  python -c "
import json; d=json.loads(open('gpurun_out/sw.json').read()); r=d['roofline']
print('$cfg rcp $rcp', 'ms/step %.3f'%d['ms_per_step'], 'kernel %.3f'%r['kernel_ms'], 'sfu %.3f'%r['binding_roofline']['frac'], 'launches', d['gpu_launches'], 'clk', d['clocks']['sm_mhz'], flush=True)" || tail -3 gpurun_out/sw.err
done; done
timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_gpu_letkf.py tests/test_reference_unit_tests.py tests/test_gpu_determinism.py -q -p no:cacheprovider > gpurun_out/r02_gputests4.log 2>&1; echo "pytest rc=$?"
grep -E "passed|failed|FAILED" gpurun_out/r02_gputests4.log | tail -12
