# the whole GPU suite + smoke() on one B200 (final code)
timeout 2400 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/r02_final_gpu_tests.log 2>&1; echo "pytest rc=$?"
tail -3 gpurun_out/r02_final_gpu_tests.log
timeout 600 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r02_final_smoke.log 2>&1; echo "smoke rc=$?"
tail -2 gpurun_out/r02_final_smoke.log
timeout 900 python bench.py --steps 10 --warmup 3 > gpurun_out/r02_final_bench_default.json 2> gpurun_out/r02_final_bench_default.err; echo "bench rc=$?"
