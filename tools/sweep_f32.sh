# fp32 kernel tuning sweep on one config (GPU box):
#   CFG=cfg3 bash tools/sweep_f32.sh "POLY:MINB:P ..."
cfg=${CFG:-cfg3}
for v in $1; do
  IFS=: read poly minb pp <<< "$v"
  env TURBDA_F32_POLY=$poly TURBDA_F32_MINB=$minb ${pp:+TURBDA_F32_P=$pp} python bench.py --config $cfg \
      --no-cpu-baseline --no-fp64 --no-e2e-variants --steps ${STEPS:-5} > gpurun_out/sw.json 2>gpurun_out/sw.err
  python -c "
import json; d=json.loads(open('gpurun_out/sw.json').read()); r=d['roofline']
print('$cfg poly $poly minb $minb P ${pp:-auto}', 'ms/step %.3f'%d['ms_per_step'], 'kernel %.3f'%r['kernel_ms'], 'sfu %.3f'%r['binding_roofline']['frac'], 'clk', d['clocks']['sm_mhz'], flush=True)" || { echo "$cfg $v failed"; tail -3 gpurun_out/sw.err; }
done
