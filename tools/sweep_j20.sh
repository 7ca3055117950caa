# compile-time-J (N = 20) kernel sweep: "CFG:FORCE_P:J20 ..." (GPU box)
for spec in $1; do
  IFS=: read cfg fp j <<< "$spec"
  env TURBDA_F32_FORCE_P=$fp TURBDA_F32_J20=$j timeout 300 python bench.py --config $cfg --no-cpu-baseline --no-fp64 \
      --no-e2e-variants --steps ${STEPS:-5} > gpurun_out/sw.json 2>gpurun_out/sw.err
  python -c "
import json; d=json.loads(open('gpurun_out/sw.json').read()); r=d['roofline']
print('$spec', 'ms/step %.4f'%d['ms_per_step'], 'kernel %.4f'%r['kernel_ms'], 'frac %.3f'%r['binding_roofline']['frac'], 'clk', d['clocks']['sm_mhz'], flush=True)" || { echo "$spec failed"; tail -3 gpurun_out/sw.err; }
done
