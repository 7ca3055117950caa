for cfg in cfg3 cfg1; do
  timeout 900 python bench.py --config $cfg --steps 10 --warmup 3 > gpurun_out/r02_final_bench_$cfg.json 2> gpurun_out/r02_final_bench_$cfg.err; echo "$cfg rc=$?"
done
