# fp32 kernel sweep on one config (GPU box):  CFG=cfg3 bash tools/sweep_f32.sh "POLY ..."
# POLY: 0 = all-MUFU sorted kernel, -1 = default.  The round-2 sweep's other
# axes (register budgets, particles per warp, FMA-pipe Box-Muller) were
# temporary instantiations, removed from the product after the measurement
# (profiles/r02_sweeps.md).
cfg=${CFG:-cfg3}
for poly in $1; do
  env TURBDA_F32_POLY=$poly python bench.py --config $cfg --no-cpu-baseline --no-fp64 \
      --no-e2e-variants --steps ${STEPS:-5} > gpurun_out/sw.json 2>gpurun_out/sw.err
  python -c "
import json; d=json.loads(open('gpurun_out/sw.json').read()); r=d['roofline']
print('$cfg poly $poly', 'ms/step %.3f'%d['ms_per_step'], 'kernel %.3f'%r['kernel_ms'], 'sfu %.3f'%r['binding_roofline']['frac'], 'clk', d['clocks']['sm_mhz'], flush=True)" || { echo "$cfg $poly failed"; tail -3 gpurun_out/sw.err; }
done
