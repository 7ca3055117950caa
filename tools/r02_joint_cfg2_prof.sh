# config-2 joint-norm launch list (direct launches so ncu sees every kernel)
TURBDA_JOINT_GRAPH=0 timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -s 300 -c 60 --csv --log-file gpurun_out/r02_joint_cfg2_launches.csv python bench.py --config cfg2 --score joint --precision fp64 --steps 1 --warmup 3 --no-cpu-baseline --no-fp64 --no-e2e-variants > /dev/null 2>&1; echo ncu rc=$?
