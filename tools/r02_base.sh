set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
python bench.py --config cfg3 --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/r02b_cfg3.json 2> gpurun_out/r02b_cfg3.err
python bench.py --config cfg1 --steps 20 --warmup 3 --no-cpu-baseline > gpurun_out/r02b_cfg1.json 2> gpurun_out/r02b_cfg1.err
timeout 900 ncu --set full --clock-control none --import-source on -k regex:ensf_f32_kernel -s 3 -c 1 -o gpurun_out/r02b_ncu_cfg3 python bench.py --config cfg3 --steps 1 --warmup 3 --no-cpu-baseline > gpurun_out/r02b_ncu.log 2>&1
echo done
