#!/bin/bash
# sweep kernel variants x particles-per-warp on one config (GPU box)
cfg=$1
for v in ${VARIANTS:-0 2}; do for pp in ${PS:-0}; do
  TURBDA_F32_VARIANT=$v TURBDA_F32_P=$pp python bench.py --config $cfg --no-cpu-baseline --steps ${STEPS:-3} > gpurun_out/sw.json 2>/dev/null
  python -c "
import json; d=json.load(open('gpurun_out/sw.json')); r=d['roofline']
print('$cfg variant $v P $pp', 'ms/step %.3f'%d['ms_per_step'], 'kernel %.3f'%r['kernel_ms'], 'sfu %.3f'%r['binding_roofline']['frac'])" || echo "$cfg $v $pp failed"
done; done
