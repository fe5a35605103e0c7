"""Profiling driver: runs the stage on N device-resident 4096^2 tiles through
rtg_process_tile_dev (for ncu launch lists / --set full captures).  Prints
per-stage CUDA-event times of the last pass (not under ncu)."""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_1405_7958_b200 import rtg  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--tiles", type=int, default=2)
ap.add_argument("--passes", type=int, default=2)
ap.add_argument("--size", type=int, default=4096)
ap.add_argument("--pdl", action="store_true")
ap.add_argument("--time", action="store_true",
                help="graph-mode wall time of the passes on one stream (no stage events)")
a = ap.parse_args()
h = w = a.size
cap = 32768 * max(1, (h * w) // (4096 * 4096))
ctx = rtg.Context(0, h, w, cap)
if a.pdl:
    ctx.set_option(rtg.OPT_PDL, 1)
p = rtg.default_params()
rgbs = []
for k in range(a.tiles):
    t = torch.empty((h, w, 3), dtype=torch.uint8, device="cuda")
    ctx.synth_tile_dev(t, k, 0, h, w)
    rgbs.append(t)
feat = torch.empty((cap, 20), dtype=torch.float32, device="cuda")
n = torch.zeros(1, dtype=torch.int32, device="cuda")
ctx.sync()
if a.time:
    for t in rgbs:  # warm-up (graph capture)
        ctx.process_tile_dev(t, h, w, p, None, None, None, feat, n)
    ctx.sync()
    import time
    t0 = time.perf_counter()
    for ps in range(a.passes):
        for t in rgbs:
            ctx.process_tile_dev(t, h, w, p, None, None, None, feat, n)
    ctx.sync()
    dt = (time.perf_counter() - t0) / (a.passes * a.tiles)
    print(f"{h}x{w}: {dt * 1e3:.4f} ms/tile -> {h * w / dt / 1e6:.0f} Mpixel/s (objects {int(n.item())})")
    sys.exit(0)
for ps in range(a.passes):
    if ps == a.passes - 1:
        ctx.profile(True)
    for t in rgbs:
        ctx.process_tile_dev(t, h, w, p, None, None, None, feat, n)
    ctx.sync()
prof = ctx.profile_read()
tot = sum(v[0] for v in prof.values())
print("objects", int(n.item()))
for s, (ms, c) in prof.items():
    print(f"{s:12s} {ms / max(c, 1):8.4f} ms/tile  {100 * ms / tot:5.1f}%")
print(f"total {tot / a.tiles:.4f} ms/tile -> {h * w / (tot / a.tiles / 1e3) / 1e6:.0f} Mpixel/s")
print("stats", ctx.stats())
