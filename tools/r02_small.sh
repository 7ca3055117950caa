for mb in 5 2; do
  TURBDA_F32_J20_MINB=$mb timeout 300 python bench.py --config cfg1 --no-cpu-baseline --no-fp64 --no-e2e-variants --steps 20 > gpurun_out/sw.json 2>gpurun_out/sw.err
  python -c "
import json; d=json.loads(open('gpurun_out/sw.json').read()); r=d['roofline']
print('cfg1 minb $mb', 'ms/step %.4f'%d['ms_per_step'], 'kernel %.4f'%r['kernel_ms'], 'frac %.3f'%r['binding_roofline']['frac'], 'launches', d['gpu_launches'], flush=True)" || tail -3 gpurun_out/sw.err
  TURBDA_F32_J20_MINB=$mb timeout 200 python tools/steps_slope.py 8192 20 | tail -1
done
timeout 900 python -m pytest tests -m gpu -q -p no:cacheprovider -x -k "parity or determinism" 2>&1 | tail -3
