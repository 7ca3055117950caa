# joint mode after the W X GEMM became the N > 64 apply: config-4 line, launch list, joint tests
timeout 1200 python bench.py --config cfg4 --score joint --precision fp64 --steps 2 --warmup 3 --no-cpu-baseline --no-e2e-variants > gpurun_out/r02_final_bench_cfg4_joint.json 2> gpurun_out/r02_final_bench_cfg4_joint.err
python -c "
import json; d=json.loads(open('gpurun_out/r02_final_bench_cfg4_joint.json').read().strip().splitlines()[-1]); r=d['roofline']
print('cfg4 joint ms %.1f'%d['ms_per_step'], 'fp64 frac %.3f'%r['binding_roofline']['frac'], 'e2e %.4g'%d['e2e']['value'])" || tail -3 gpurun_out/r02_final_bench_cfg4_joint.err
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -s 600 -c 12 --csv --log-file gpurun_out/r02_joint_cfg4_launches_final.csv python bench.py --config cfg4 --score joint --precision fp64 --steps 1 --warmup 3 --no-cpu-baseline --no-fp64 --no-e2e-variants > /dev/null 2>&1; echo ncu rc=$?
timeout 900 python -m pytest tests -m gpu -q -p no:cacheprovider -k "joint" 2>&1 | tail -2
