# fp64 kernel: 5-warp CTAs when they leave fewer padding warps (config 3 / 1 fp64) + fp64 parity
for cfg in cfg3 cfg1; do
  timeout 600 python bench.py --config $cfg --precision fp64 --steps 3 --warmup 3 --no-cpu-baseline --no-fp64 --no-e2e-variants > gpurun_out/f64$cfg.json 2> gpurun_out/f64$cfg.err
  python -c "
import json; d=json.loads(open('gpurun_out/f64$cfg.json').read().strip().splitlines()[-1]); print('$cfg fp64 ms %.4f'%d['ms_per_step'], 'val %.4g'%d['value'])" || tail -3 gpurun_out/f64$cfg.err
done
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider -x -k "(parity or determinism) and not joint" 2>&1 | tail -2
