#!/bin/bash
# time every fp32 kernel variant on the bench workload (run on the GPU box)
cfg=${1:-cfg2}
for v in ${VARIANTS:-0 1 2 3 4 5}; do
  TURBDA_F32_VARIANT=$v python bench.py --config $cfg --no-cpu-baseline --steps 5 > gpurun_out/var_$v.json 2>/dev/null
  python -c "
import json,sys; d=json.load(open('gpurun_out/var_$v.json')); r=d['roofline']
print('variant $v', '$cfg', 'ms/step %.3f'%d['ms_per_step'], 'kernel ms %.3f'%r['kernel_ms'], 'sfu frac %.3f'%r['binding_roofline']['frac'], 'clk', d['clocks']['sm_mhz'])" || echo "variant $v failed"
done
