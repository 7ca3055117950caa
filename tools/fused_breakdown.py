"""Where does the fused kernel's extra time go at 4 CTAs per tile? Device-
resident analyses of config 5's shape (d = 2.1M, N = 128, S = 100) with
relax_factor 1 and 0 (0 skips the forecast statistics and the epilogue's
relax) and TURBDA_F32_FUSE_ALL=1 / TURBDA_F32_UNFUSED=1 set by the caller."""
import os
import sys
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2407_12168_b200 import capi  # noqa: E402

d, m = int(sys.argv[1]) if len(sys.argv) > 1 else 2_097_152, int(sys.argv[2]) if len(sys.argv) > 2 else 128
dev = torch.device("cuda", 0)
g = torch.Generator(device=dev)
g.manual_seed(1)
x = torch.randn((m, d), generator=g, device=dev, dtype=torch.float64)
y = torch.randn((d,), generator=g, device=dev, dtype=torch.float64)
r = torch.ones_like(y)
out = torch.empty_like(x)
st = torch.cuda.Stream(dev)
torch.cuda.set_stream(st)
for relax in (1.0, 0.0):
    p = capi.params(d_total=d, d_local=d, obs_dim=d, n_members=m, n_steps=100, relax_factor=relax,
                    device=0, flags=capi.INPUTS_ON_DEVICE | capi.ASYNC)
    capi.analyze(p, x, y, r, None, out, stream=st.cuda_stream)
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record(st)
    for _ in range(3):
        capi.analyze(p, x, y, r, None, out, stream=st.cuda_stream)
    b.record(st)
    b.synchronize()
    print(f"d={d} m={m} relax={relax} fuse_all={os.environ.get('TURBDA_F32_FUSE_ALL', '0')} "
          f"unfused={os.environ.get('TURBDA_F32_UNFUSED', '0')}: {a.elapsed_time(b) / 3:.2f} ms", flush=True)
