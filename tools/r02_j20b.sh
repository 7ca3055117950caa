for spec in "8:0:0" "8:0:3" "4:1:3" "2:1:3" "1:1:3" "4:1:0" "2:1:0" "2:1:2"; do
  IFS=: read wm fa j <<< "$spec"
  env TURBDA_F32_WMAX=$wm TURBDA_F32_FUSE_ALL=$fa TURBDA_F32_J20=$j timeout 300 python bench.py --config cfg1 --no-cpu-baseline --no-fp64 \
      --no-e2e-variants --steps 20 > gpurun_out/sw.json 2>gpurun_out/sw.err
  python -c "
import json; d=json.loads(open('gpurun_out/sw.json').read()); r=d['roofline']
print('wmax:fuseall:j20 $spec', 'ms/step %.4f'%d['ms_per_step'], 'kernel %.4f'%r['kernel_ms'], 'frac %.3f'%r['binding_roofline']['frac'], 'clk', d['clocks']['sm_mhz'], flush=True)" || { echo "$spec failed"; tail -3 gpurun_out/sw.err; }
done
