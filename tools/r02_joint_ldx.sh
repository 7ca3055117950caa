# joint apply with the conflict-free X-tile stride: config 4 and config 2 joint lines + joint tests
bash tools/r02_joint_cfg4.sh
timeout 600 python bench.py --config cfg2 --score joint --precision fp64 --steps 5 --warmup 3 --no-cpu-baseline --no-e2e-variants > gpurun_out/jc2.json 2> gpurun_out/jc2.err
python -c "
import json; d=json.loads(open('gpurun_out/jc2.json').read().strip().splitlines()[-1]); print('cfg2 joint ms %.3f'%d['ms_per_step'])" || tail -3 gpurun_out/jc2.err
