#!/bin/bash
# CTAs/SM register budget (TURBDA_F32_CTAS = 3: 80 regs, 4: 64 regs) x configs
for cfg in ${CFGS:-cfg2 cfg3 cfg1}; do for c in ${CTAS:-3 4}; do
  TURBDA_F32_CTAS=$c python bench.py --config $cfg --no-cpu-baseline --steps ${STEPS:-5} > gpurun_out/sw.json 2>/dev/null
  python -c "
import json; d=json.load(open('gpurun_out/sw.json')); r=d['roofline']
print('$cfg ctas $c', 'ms/step %.3f'%d['ms_per_step'], 'kernel %.3f'%r['kernel_ms'], 'sfu %.3f'%r['binding_roofline']['frac'])" || echo "$cfg $c failed"
done; done
