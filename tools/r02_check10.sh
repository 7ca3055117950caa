for cfg in cfg1 cfg3 cfg2; do
  timeout 600 python bench.py --config $cfg --no-cpu-baseline --no-fp64 --no-e2e-variants --steps 10 > gpurun_out/sw.json 2>gpurun_out/sw.err
  python -c "
import json; d=json.loads(open('gpurun_out/sw.json').read()); r=d['roofline']
print('$cfg', 'ms/step %.4f'%d['ms_per_step'], 'kernel %.4f'%r['kernel_ms'], 'sfu %.3f'%r['binding_roofline']['frac'], 'e2e %.4g'%d['e2e']['value'], flush=True)" || tail -3 gpurun_out/sw.err
done
timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_gpu_determinism.py -q -p no:cacheprovider -x 2>&1 | tail -2
