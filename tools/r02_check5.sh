for cfg in cfg5 cfg2 cfg3; do for unf in 0 1; do
  TURBDA_F32_UNFUSED=$unf python bench.py --config $cfg --no-cpu-baseline --no-fp64 --no-e2e-variants --steps ${STEPS:-4} > gpurun_out/sw.json 2>gpurun_out/sw.err
  python -c "
import json; d=json.loads(open('gpurun_out/sw.json').read()); r=d['roofline']
print('$cfg unfused $unf', 'ms/step %.3f'%d['ms_per_step'], 'kernel %.3f'%r['kernel_ms'], 'sfu %.3f'%r['binding_roofline']['frac'], 'launches', d['gpu_launches'], 'clk', d['clocks']['sm_mhz'], flush=True)" || tail -3 gpurun_out/sw.err
done; done
