# GPU check: full gpu test suite + default bench line (+ free -g for host RAM)
free -g | head -2; nproc
timeout 2400 python -m pytest tests -m gpu -x -q -p no:cacheprovider > gpurun_out/r02_gputests.log 2>&1; echo "pytest rc=$?"
tail -5 gpurun_out/r02_gputests.log
timeout 900 python bench.py > gpurun_out/r02_bench_default.json 2> gpurun_out/r02_bench_default.err; echo "bench rc=$?"
tail -3 gpurun_out/r02_bench_default.err
