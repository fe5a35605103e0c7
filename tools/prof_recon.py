"""C2 reconstruction on the GPU (h-dome under tile (0,0)'s H plane, h = 32):
per-call CUDA-event time and the IWPP counters (for ncu launch lists)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from oracle import pyoracle  # noqa: E402
from paper_1405_7958_b200 import rtg  # noqa: E402

conn = int(os.environ.get("CONN", "8"))
H = W = 4096
rgb = pyoracle.synth_tile_host(0, 0, H, W)
hema, _, _ = pyoracle.colordeconv(rgb, pyoracle.default_params())
marker = np.maximum(hema.astype(np.int16) - 32, 0).astype(np.uint8)
ctx = rtg.Context(0, H, W, 1 << 12)
s = torch.cuda.Stream()
ctx.set_stream(s.cuda_stream)
with torch.cuda.stream(s):
    d_mk, d_ms = torch.from_numpy(marker).cuda(), torch.from_numpy(hema).cuda()
    out = torch.empty((H, W), dtype=torch.uint8, device="cuda")
s.synchronize()
ctx.stats()
reps = int(os.environ.get("REPS", "3"))
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record(s)
for _ in range(reps):
    ctx.recon_dev(d_mk, d_ms, H, W, conn, out)
e1.record(s)
s.synchronize()
st = ctx.stats()
print(f"conn {conn}: {e0.elapsed_time(e1) / reps:.3f} ms per call; visits {st[4] / reps:.0f}, "
      f"sweep iterations {st[5] / reps:.0f} per call")
