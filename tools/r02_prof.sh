# ncu evidence for the round-2 kernels (run only after the same commands exit 0 without ncu)
set -x
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 60 --csv \
  --log-file gpurun_out/r02_launches_cfg3.csv python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-fp64 --no-e2e-variants > gpurun_out/r02_ncu_l3.log 2>&1
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 80 --csv \
  --log-file gpurun_out/r02_launches_cfg2.csv python bench.py --config cfg2 --steps 3 --warmup 3 --no-cpu-baseline --no-fp64 --no-e2e-variants > gpurun_out/r02_ncu_l2.log 2>&1
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:ensf_f32_kernel -s 3 -c 1 \
  -o gpurun_out/r02_ncu_full_cfg3 python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-fp64 --no-e2e-variants > gpurun_out/r02_ncu_f3.log 2>&1
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:ensf_f32_kernel -s 3 -c 1 \
  -o gpurun_out/r02_ncu_full_cfg2 python bench.py --config cfg2 --steps 1 --warmup 3 --no-cpu-baseline --no-fp64 --no-e2e-variants > gpurun_out/r02_ncu_f2.log 2>&1
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:ensf_f64_kernel -c 1 \
  -o gpurun_out/r02_ncu_full_cfg3_f64 python bench.py --precision fp64 --steps 1 --warmup 3 --no-cpu-baseline --no-fp64 --no-e2e-variants > gpurun_out/r02_ncu_f64.log 2>&1
echo done
