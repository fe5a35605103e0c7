"""Debug driver: one small tile through the stage and a few operators, with a
line printed after each step (bisects a crash on the GPU box)."""
import faulthandler
import os
import sys

faulthandler.enable()
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_1405_7958_b200 import rtg  # noqa: E402

print("start", flush=True)
rgb = rtg.synth_tile_host(0, 0, 512, 512)
with rtg.Context(0, 512, 512, 1 << 14) as ctx:
    ctx.set_option(rtg.OPT_USE_GRAPHS, 0)
    ctx.set_option(rtg.OPT_STREAM_IMPL, int(os.environ.get("SI", "1")))
    d = torch.from_numpy(rgb).cuda()
    hema = torch.empty((512, 512), dtype=torch.uint8, device="cuda")
    tis = torch.empty_like(hema)
    torch.cuda.synchronize()
    ctx.colordeconv_dev(d, 512, 512, rtg.default_params(), hema, None, tis)
    ctx.sync()
    print("colordeconv ok", flush=True)
    m = (hema > 100).to(torch.uint8)
    lab = torch.empty((512, 512), dtype=torch.int32, device="cuda")
    n = torch.zeros(1, dtype=torch.int32, device="cuda")
    torch.cuda.synchronize()
    ctx.bwlabel_dev(m, 512, 512, 8, lab, n)
    ctx.sync()
    print("bwlabel ok", int(n.cpu()[0]), flush=True)
    out = ctx.process_tile(rgb)
    print("process ok", out[4], flush=True)
print("done", flush=True)
