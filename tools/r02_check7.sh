for cfg in cfg4 cfg1; do for unf in 0 1; do
  TURBDA_F32_UNFUSED=$unf python bench.py --config $cfg --no-cpu-baseline --no-fp64 --no-e2e-variants --steps ${STEPS:-3} > gpurun_out/sw.json 2>gpurun_out/sw.err
  python -c "
import json; d=json.loads(open('gpurun_out/sw.json').read()); r=d['roofline']
print('$cfg unfused $unf', 'ms/step %.3f'%d['ms_per_step'], 'kernel %.3f'%r['kernel_ms'], 'sfu %.3f'%r['binding_roofline']['frac'], 'launches', d['gpu_launches'], 'e2e', d['e2e']['value'], 'clk', d['clocks']['sm_mhz'], flush=True)" || tail -3 gpurun_out/sw.err
done; done
python bench.py --no-cpu-baseline --no-fp64 --steps 3 > gpurun_out/r02_e2e.json 2>/dev/null; python -c "
import json; d=json.loads(open('gpurun_out/r02_e2e.json').read()); print('cfg3 e2e', d['e2e']['value'], {k: v['s_per_step'] for k, v in d['e2e']['variants'].items()})"
timeout 600 python -m pytest tests/test_gpu_determinism.py -q -p no:cacheprovider -k pageable 2>&1 | tail -2
