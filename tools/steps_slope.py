"""Fixed vs per-step cost of a small analysis: device-resident
turbda_ensf_analyze at n_steps = 10, 25, 50, 100 (CUDA events, 200 repeats),
so time(S) = a + b S separates launch / prologue / epilogue from the
pseudo-step loop.   python tools/steps_slope.py [d] [m]"""
import sys
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2407_12168_b200 import capi  # noqa: E402

d = int(sys.argv[1]) if len(sys.argv) > 1 else 8192
m = int(sys.argv[2]) if len(sys.argv) > 2 else 20
dev = torch.device("cuda", 0)
st = torch.cuda.Stream(dev)
torch.cuda.set_stream(st)
g = torch.Generator(device=dev)
g.manual_seed(5)
x = torch.randn((m, d), generator=g, device=dev, dtype=torch.float64)
y = torch.randn((d,), generator=g, device=dev, dtype=torch.float64)
r = torch.ones_like(y)
out = torch.empty_like(x)
res = []
for s in (10, 25, 50, 100):
    p = capi.params(d_total=d, d_local=d, obs_dim=d, n_members=m, n_steps=s, device=0,
                    flags=capi.INPUTS_ON_DEVICE | capi.ASYNC)
    for _ in range(20):
        capi.analyze(p, x, y, r, None, out, stream=st.cuda_stream)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    e0.record(st)
    for _ in range(200):
        capi.analyze(p, x, y, r, None, out, stream=st.cuda_stream)
    e1.record(st)
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / 200
    res.append((s, ms))
    print(f"d={d} m={m} S={s} ms={ms:.4f}", flush=True)
n = len(res)
sx = sum(s for s, _ in res); sy = sum(t for _, t in res)
sxx = sum(s * s for s, _ in res); sxy = sum(s * t for s, t in res)
b = (n * sxy - sx * sy) / (n * sxx - sx * sx)
a = (sy - b * sx) / n
print(f"fit: fixed {a * 1000:.1f} us + {b * 1000:.3f} us/step")
