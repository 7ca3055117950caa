# 2-GPU checks: self-spawned weak-scaling bench (config 3) + the multi-rank tests
nvidia-smi -L
timeout 900 python bench.py --gpus 2 --steps 5 --warmup 3 > gpurun_out/r02_bench_n2.json 2> gpurun_out/r02_bench_n2.err; echo "bench n2 rc=$?"
tail -3 gpurun_out/r02_bench_n2.err
timeout 1200 python -m pytest tests -m gpu -q -p no:cacheprovider -k "multi_process or multi_device or multi_gpu or sharded" > gpurun_out/r02_multi_tests.log 2>&1; echo "pytest rc=$?"
tail -5 gpurun_out/r02_multi_tests.log
