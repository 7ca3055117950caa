# joint mode over N ranks: per-step allreduce on NCCL symmetric memory vs plain
N=$(nvidia-smi -L | wc -l)
for sym in 1 0; do
  TURBDA_NCCL_SYMMETRIC=$sym timeout 600 python bench.py --gpus $N --config cfg2 --score joint --precision fp64 --steps 5 --warmup 3 --no-e2e-variants --no-cpu-baseline > gpurun_out/r02_joint_sym${sym}_n$N.json 2> gpurun_out/r02_joint_sym${sym}_n$N.err
  python -c "
import json; d=json.loads(open('gpurun_out/r02_joint_sym${sym}_n$N.json').read().strip().splitlines()[-1]); print('joint n$N sym $sym', 'ms/step %.3f'%d['ms_per_step'], 'value %.4g'%d['value'])" || tail -5 gpurun_out/r02_joint_sym${sym}_n$N.err
done
NCCL_DEBUG=INFO TURBDA_NCCL_SYMMETRIC=1 timeout 300 python bench.py --gpus $N --config cfg2 --score joint --precision fp64 --steps 3 --warmup 3 --no-e2e-variants --no-cpu-baseline 2>&1 >/dev/null | grep -iE "symmetric|nvls|window|Algo" | head -20
timeout 900 python -m pytest tests -m gpu -q -p no:cacheprovider -k "multi_process or multi_device" 2>&1 | tail -2
