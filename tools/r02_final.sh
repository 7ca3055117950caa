# round-2 final evidence on one B200: every config's bench line, the joint
# extension, the reference arm; then the whole GPU suite and smoke()
set -x
for cfg in cfg3 cfg2 cfg5 cfg1; do
  timeout 900 python bench.py --config $cfg --steps 10 --warmup 3 > gpurun_out/r02_final_bench_$cfg.json 2> gpurun_out/r02_final_bench_$cfg.err
done
timeout 1200 python bench.py --config cfg4 --steps 3 --warmup 3 --no-fp64 > gpurun_out/r02_final_bench_cfg4.json 2> gpurun_out/r02_final_bench_cfg4.err
timeout 600 python bench.py --config cfg2 --score joint --precision fp64 --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/r02_final_bench_cfg2_joint.json 2> gpurun_out/r02_final_bench_cfg2_joint.err
timeout 1200 python bench.py --config cfg4 --score joint --precision fp64 --steps 2 --warmup 3 --no-cpu-baseline --no-e2e-variants > gpurun_out/r02_final_bench_cfg4_joint.json 2> gpurun_out/r02_final_bench_cfg4_joint.err
timeout 900 python bench.py --impl reference --steps 20 --warmup 5 > gpurun_out/r02_final_bench_ref.json 2> gpurun_out/r02_final_bench_ref.err
timeout 2400 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/r02_final_gpu_tests.log 2>&1; echo "pytest rc=$?"
tail -3 gpurun_out/r02_final_gpu_tests.log
timeout 600 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r02_final_smoke.log 2>&1; echo "smoke rc=$?"
