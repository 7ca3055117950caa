#!/bin/bash
# round-end evidence: GPU tests, smoke, bench lines of every config, the
# reference arm, 2-GPU weak scaling, the ncu launch list and one full capture
python -m pytest tests -m gpu -q -x > gpurun_out/final_gpu_tests.log 2>&1; echo "pytest rc=$?"
tail -3 gpurun_out/final_gpu_tests.log
python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" 2>&1 | tail -2
python bench.py > gpurun_out/final_bench_cfg2.json 2> gpurun_out/final_bench_cfg2.err; echo "bench rc=$?"
for c in cfg1 cfg3 cfg5 cfg4; do
  python bench.py --config $c > gpurun_out/final_bench_$c.json 2>/dev/null; echo "$c rc=$?"
done
python bench.py --score joint > gpurun_out/final_bench_joint.json 2>/dev/null; echo "joint rc=$?"
python bench.py --impl reference > gpurun_out/final_bench_ref.json 2>/dev/null; echo "ref rc=$?"
if [ "$(nvidia-smi -L | wc -l)" -ge 2 ]; then
  python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29531 bench.py --gpus 2 > gpurun_out/final_bench_n2.json 2>/dev/null; echo "n2 rc=$?"
fi
CUDA_VISIBLE_DEVICES=0 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/final_launches.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/ncu_l.log 2>&1; echo "ncu1 rc=$?"
CUDA_VISIBLE_DEVICES=0 ncu --set full --clock-control none --import-source on -k regex:ensf_f32 -c 1 -o gpurun_out/final_full -f python bench.py --steps 1 --warmup 3 --no-cpu-baseline > gpurun_out/ncu_f.log 2>&1; echo "ncu2 rc=$?"
