"""One 4096^2 tile through the stage with params.texture = 1 (for ncu launch
lists of the f4 texture kernels)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_1405_7958_b200 import rtg  # noqa: E402

h = w = 4096
ctx = rtg.Context(0, h, w, 32768)
p = rtg.default_params()
p.texture = 1
t = torch.empty((h, w, 3), dtype=torch.uint8, device="cuda")
ctx.synth_tile_dev(t, 0, 0, h, w)
feat = torch.empty((32768, rtg.NUM_FEATURES + rtg.NUM_TEXTURE), dtype=torch.float32, device="cuda")
n = torch.zeros(1, dtype=torch.int32, device="cuda")
ctx.sync()
ctx.set_option(rtg.OPT_USE_GRAPHS, 0)
ctx.process_tile_dev(t, h, w, p, None, None, None, feat, n)  # warm-up (first-call costs)
ctx.sync()
ctx.profile(True)
ctx.process_tile_dev(t, h, w, p, None, None, None, feat, n)
prof = ctx.profile_read()
print({k: round(v[0], 4) for k, v in prof.items()})
