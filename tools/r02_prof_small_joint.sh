# ncu: the small-grid config-1 kernel, and config 4's joint-norm Gram / apply kernels

J="python bench.py --config cfg4 --score joint --precision fp64 --steps 1 --warmup 3 --no-cpu-baseline --no-fp64 --no-e2e-variants"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:gram_partial -s 5 -c 1 -o gpurun_out/r02_ncu_full_joint_gram $J > gpurun_out/r02_ncu_jg.log 2>&1; echo rc=$?
timeout 900 ncu --set full --clock-control none --import-source on -k regex:joint_apply -s 5 -c 1 -o gpurun_out/r02_ncu_full_joint_apply $J > gpurun_out/r02_ncu_ja.log 2>&1; echo rc=$?
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -s 600 -c 12 --csv --log-file gpurun_out/r02_joint_cfg4_launches.csv $J > /dev/null 2>&1; echo rc=$?
