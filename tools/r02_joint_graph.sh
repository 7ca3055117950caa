# joint mode: captured pseudo-steps (CUDA graph, communicator-free calls) vs direct launches
for g in 1 0; do
  CUDA_VISIBLE_DEVICES=0 TURBDA_JOINT_GRAPH=$g timeout 300 python bench.py --config cfg2 --score joint --steps 5 --warmup 3 --no-cpu-baseline --no-e2e-variants > gpurun_out/jg$g.json 2>gpurun_out/jg$g.err
  python -c "import json; d=json.loads(open('gpurun_out/jg$g.json').read().strip().splitlines()[-1]); print('joint 1gpu graph $g', 'ms %.3f'%d['ms_per_step'], 'e2e %.4g'%d['e2e']['value'])" || tail -3 gpurun_out/jg$g.err
done
timeout 300 python bench.py --gpus 2 --config cfg2 --score joint --steps 5 --warmup 3 --no-cpu-baseline --no-e2e-variants > gpurun_out/jg2.json 2>gpurun_out/jg2.err
python -c "import json; d=json.loads(open('gpurun_out/jg2.json').read().strip().splitlines()[-1]); print('joint 2gpu', 'ms %.3f'%d['ms_per_step'], 'e2e %.4g'%d['e2e']['value'])" || tail -3 gpurun_out/jg2.err
timeout 700 python -m pytest tests -m gpu -q -p no:cacheprovider -k "joint" 2>&1 | tail -2
