# joint mode N <= 64: fused 64x64 apply vs the W X GEMM (64-row tiles) + elementwise update
for wx in 1 0; do
  TURBDA_JOINT_WX_SMALL=$wx timeout 900 python bench.py --config cfg2 --score joint --precision fp64 --steps 5 --warmup 3 --no-cpu-baseline --no-fp64 --no-e2e-variants > gpurun_out/jws$wx.json 2> gpurun_out/jws$wx.err
  python -c "
import json; d=json.loads(open('gpurun_out/jws$wx.json').read().strip().splitlines()[-1])
print('cfg2 joint wx_small $wx ms %.3f'%d['ms_per_step'])" || tail -3 gpurun_out/jws$wx.err
done
TURBDA_JOINT_WX_SMALL=1 TURBDA_JOINT_GRAPH=0 timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -s 300 -c 60 --csv --log-file gpurun_out/r02_joint_cfg2_launches_wx.csv python bench.py --config cfg2 --score joint --precision fp64 --steps 1 --warmup 3 --no-cpu-baseline --no-fp64 --no-e2e-variants > /dev/null 2>&1; echo ncu rc=$?
TURBDA_JOINT_WX_SMALL=1 timeout 900 python -m pytest tests -m gpu -q -p no:cacheprovider -x -k "joint" 2>&1 | tail -2
python - <<'PY'
import subprocess, sys, os, numpy as np
for m, d in ((64, 3000), (20, 1000), (33, 257)):
    code = ("import numpy as np, sys; sys.path.insert(0, '.'); from paper_2407_12168_b200 import capi; "
            f"from oracle.oracle import conditioned_inputs; x, y, i, _ = conditioned_inputs({m}, {d}, stride=3); "
            "np.save(sys.argv[1], capi.analyze_host(0.05 * x, y, 4.0, i, n_steps=20, joint=True, precision=capi.FP64))")
    outs = []
    for wx in ("0", "1"):
        subprocess.run([sys.executable, "-c", code, f"gpurun_out/jws_bits{wx}.npy"], check=True, env=dict(os.environ, TURBDA_JOINT_WX_SMALL=wx))
        outs.append(np.load(f"gpurun_out/jws_bits{wx}.npy"))
    print(f"m={m} WX_SMALL bit-identical:", np.array_equal(outs[0], outs[1]), "max abs diff", float(np.abs(outs[0] - outs[1]).max()))
PY
