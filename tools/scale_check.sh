#!/bin/bash
# weak-scaling evidence on every visible GPU: componentwise at N = 1, 2, 4
# and the joint-norm mode (per-step NCCL allreduce) at N = 1 and the max N
n=$(nvidia-smi -L | wc -l)
python bench.py --no-cpu-baseline > gpurun_out/scale_n1.json 2>/dev/null; echo "n1 rc=$?"
for g in 2 4; do
  [ "$g" -le "$n" ] || continue
  python -m torch.distributed.run --nnodes=1 --nproc-per-node $g --master-addr 127.0.0.1 --master-port 2953$g bench.py --gpus $g > gpurun_out/scale_n$g.json 2>gpurun_out/scale_n$g.err; echo "n$g rc=$?"
done
python bench.py --score joint --no-cpu-baseline > gpurun_out/scale_j1.json 2>/dev/null; echo "j1 rc=$?"
python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 --master-port 29539 bench.py --gpus $n --score joint > gpurun_out/scale_j$n.json 2>gpurun_out/scale_j$n.err; echo "j$n rc=$?"
