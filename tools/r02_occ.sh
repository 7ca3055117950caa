for occ in 0 7 8 0; do
  TURBDA_F32_OCC=$occ timeout 300 python bench.py --config cfg3 --no-cpu-baseline --no-fp64 --no-e2e-variants --steps 5 > gpurun_out/sw.json 2>gpurun_out/sw.err
  python -c "
import json; d=json.loads(open('gpurun_out/sw.json').read()); r=d['roofline']
print('cfg3 occ $occ', 'ms/step %.3f'%d['ms_per_step'], 'kernel %.3f'%r['kernel_ms'], 'xu %.3f'%r['binding_roofline']['xu_pipe_frac'], flush=True)" || tail -3 gpurun_out/sw.err
done
