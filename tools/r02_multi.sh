# multi-GPU checks (run with gpurun --gpus N): self-spawned weak-scaling bench
# (config 3), the joint mode's per-step NCCL allreduce, the multi-rank tests
nvidia-smi -L
N=$(nvidia-smi -L | wc -l)
timeout 900 python bench.py --gpus $N --steps 5 --warmup 3 > gpurun_out/r02_bench_n$N.json 2> gpurun_out/r02_bench_n$N.err; echo "bench n$N rc=$?"
timeout 600 python bench.py --gpus $N --config cfg2 --score joint --precision fp64 --steps 3 --warmup 3 --no-e2e-variants > gpurun_out/r02_bench_joint_n$N.json 2> gpurun_out/r02_bench_joint_n$N.err; echo "joint n$N rc=$?"
timeout 1200 python -m pytest tests -m gpu -q -p no:cacheprovider -k "multi_process or multi_device or multi_gpu or sharded" > gpurun_out/r02_multi_tests_n$N.log 2>&1; echo "pytest rc=$?"
tail -5 gpurun_out/r02_multi_tests_n$N.log
