# joint apply: fused tensor-core apply vs the W X GEMM + elementwise update (TURBDA_JOINT_WX=1)
for wx in 1 0; do
  TURBDA_JOINT_WX=$wx timeout 900 python bench.py --config cfg4 --score joint --precision fp64 --steps 2 --warmup 3 --no-cpu-baseline --no-fp64 --no-e2e-variants > gpurun_out/jwx$wx.json 2> gpurun_out/jwx$wx.err
  python -c "
import json; d=json.loads(open('gpurun_out/jwx$wx.json').read().strip().splitlines()[-1])
print('cfg4 joint wx $wx ms %.1f'%d['ms_per_step'])" || tail -3 gpurun_out/jwx$wx.err
done
TURBDA_JOINT_WX=1 timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -s 600 -c 12 --csv --log-file gpurun_out/r02_joint_cfg4_launches_wx.csv python bench.py --config cfg4 --score joint --precision fp64 --steps 1 --warmup 3 --no-cpu-baseline --no-fp64 --no-e2e-variants > /dev/null 2>&1; echo ncu rc=$?
TURBDA_JOINT_WX=1 timeout 900 python -m pytest tests -m gpu -q -p no:cacheprovider -x -k "joint" 2>&1 | tail -2
python - <<'PY'
# bit-identity of the two apply paths (N = 160 > 64), fresh processes
import subprocess, sys, os, numpy as np
code = ("import numpy as np, sys; sys.path.insert(0, '.'); from paper_2407_12168_b200 import capi; "
        "from oracle.oracle import conditioned_inputs; x, y, i, _ = conditioned_inputs(160, 1000, stride=3); "
        "np.save(sys.argv[1], capi.analyze_host(0.05 * x, y, 4.0, i, n_steps=20, joint=True, precision=capi.FP64))")
outs = []
for wx in ("0", "1"):
    subprocess.run([sys.executable, "-c", code, f"gpurun_out/jwx_bits{wx}.npy"], check=True, env=dict(os.environ, TURBDA_JOINT_WX=wx))
    outs.append(np.load(f"gpurun_out/jwx_bits{wx}.npy"))
print("WX bit-identical:", np.array_equal(outs[0], outs[1]), "max abs diff", float(np.abs(outs[0] - outs[1]).max()))
PY
