# programmatic dependent launch of the fused kernel after the observation prep: on / off
for cfg in cfg1 cfg2; do for pdl in 1 0; do
  TURBDA_PDL=$pdl timeout 300 python bench.py --config $cfg --no-cpu-baseline --no-fp64 --no-e2e-variants --steps 20 > gpurun_out/sw.json 2>gpurun_out/sw.err
  python -c "
import json; d=json.loads(open('gpurun_out/sw.json').read()); r=d['roofline']
print('$cfg pdl $pdl', 'ms/step %.4f'%d['ms_per_step'], 'kernel %.4f'%r['kernel_ms'], 'e2e %.4g'%d['e2e']['value'], flush=True)" || tail -3 gpurun_out/sw.err
done; done
TURBDA_PDL=1 timeout 200 python tools/steps_slope.py 8192 20 | tail -1
TURBDA_PDL=0 timeout 200 python tools/steps_slope.py 8192 20 | tail -1
timeout 900 python -m pytest tests -m gpu -q -p no:cacheprovider -x -k "parity or determinism or cycle" 2>&1 | tail -2
