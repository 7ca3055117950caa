#!/bin/bash
# host-buffer pipeline chunk size (TURBDA_CHUNK_MB) vs the e2e leg of bench.py
for cfg in ${CFGS:-cfg2}; do for mb in ${MBS:-2 4 8 16 32}; do
  TURBDA_CHUNK_MB=$mb python bench.py --config $cfg --no-cpu-baseline --steps ${STEPS:-10} > gpurun_out/sw.json 2>/dev/null
  python -c "
import json; d=json.load(open('gpurun_out/sw.json'))
print('$cfg chunk_mb $mb', 'ms/step %.3f'%d['ms_per_step'], 'e2e %.4g'%d['e2e']['value'], 'value %.4g'%d['value'], 'e2e ms %.3f'%(d['ms_per_step']*d['value']/d['e2e']['value']))" || echo "$cfg $mb failed"
done; done
