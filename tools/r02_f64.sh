for cfg in cfg3 cfg2; do
  timeout 600 python bench.py --config $cfg --precision fp64 --no-cpu-baseline --no-fp64 --no-e2e-variants --steps 3 > gpurun_out/sw.json 2>gpurun_out/sw.err
  python -c "
import json; d=json.loads(open('gpurun_out/sw.json').read()); r=d['roofline']
print('$cfg fp64', 'ms/step %.2f'%d['ms_per_step'], 'kernel %.2f'%r['kernel_ms'], flush=True)" || tail -3 gpurun_out/sw.err
done
timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_gpu_determinism.py -q -p no:cacheprovider -k "fp64 or golden or far_from or windows or cfg1 or cfg2_shape or deterministic or window or philox or long_step" 2>&1 | tail -3
