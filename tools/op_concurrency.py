"""Per-operator throughput at 1 and S concurrent streams (one rtg_ctx per
stream) through the C-ABI device entry points, on resident 4096^2 inputs
produced by the stage itself.  An operator whose aggregate throughput does not
grow with S saturates a shared GPU resource on its own; one that scales was
latency-bound.  Prints one line per operator (not under ncu)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_1405_7958_b200 import rtg  # noqa: E402

H = W = 4096
S = int(sys.argv[1]) if len(sys.argv) > 1 else 3
K = 8  # tiles (inputs) cycled per stream
p = rtg.default_params()
ctxs = [rtg.Context(0, H, W, 32768) for _ in range(S)]
streams = [torch.cuda.Stream() for _ in range(S)]
for c, s in zip(ctxs, streams):
    c.set_stream(s.cuda_stream)
u8 = lambda: torch.empty((H, W), dtype=torch.uint8, device="cuda")  # noqa: E731
i32 = lambda: torch.empty((H, W), dtype=torch.int32, device="cuda")  # noqa: E731
rgb, mask, labels, hema, nobj = [], [], [], [], []
feat = torch.empty((32768, rtg.NUM_FEATURES), dtype=torch.float32, device="cuda")
for k in range(K):
    t = torch.empty((H, W, 3), dtype=torch.uint8, device="cuda")
    ctxs[0].synth_tile_dev(t, k, 0, H, W)
    m, lb, hm = u8(), i32(), u8()
    n = torch.zeros(1, dtype=torch.int32, device="cuda")
    ctxs[0].process_tile_dev(t, H, W, p, m, lb, hm, feat, n)
    rgb.append(t); mask.append(m); labels.append(lb); hema.append(hm); nobj.append(n)
torch.cuda.synchronize()
outs = [dict(a=u8(), b=u8(), c=u8(), l=i32(), n=torch.zeros(1, dtype=torch.int32, device="cuda"),
             f=torch.empty((32768, rtg.NUM_FEATURES), dtype=torch.float32, device="cuda"))
        for _ in range(S)]

OPS = {
    "colordeconv": lambda c, o, k: c.colordeconv_dev(rgb[k], H, W, p, o["a"], None, o["b"]),
    "fill_holes": lambda c, o, k: c.fill_holes_dev(mask[k], H, W, o["a"]),
    "bwlabel": lambda c, o, k: c.bwlabel_dev(mask[k], H, W, 8, o["l"], o["n"]),
    "edt": lambda c, o, k: c.edt_dev(mask[k], H, W, o["l"]),
    "watershed": lambda c, o, k: c.watershed_dev(mask[k], H, W, p.ws_h, o["a"]),
    "features": lambda c, o, k: c.features_dev(labels[k], hema[k], H, W, nobj[k], o["f"]),
    "stage": lambda c, o, k: c.process_tile_dev(rgb[k], H, W, p, o["a"], o["l"], o["c"], o["f"],
                                                o["n"]),
}


def run(op, ns, reps):
    fn = OPS[op]
    for i in range(ns):  # warm-up (graph capture for the stage)
        fn(ctxs[i], outs[i], i % K)
    torch.cuda.synchronize()
    e0 = torch.cuda.Event(enable_timing=True)
    e1 = torch.cuda.Event(enable_timing=True)
    e0.record()
    for s in streams[:ns]:
        s.wait_event(e0)
    for r in range(reps):
        for i in range(ns):
            fn(ctxs[i], outs[i], (r * ns + i) % K)
    for s in streams[:ns]:
        e = torch.cuda.Event()
        e.record(s)
        torch.cuda.current_stream().wait_event(e)
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / (reps * ns)


print(f"{'op':12s} {'1 stream us':>12s} {S} streams us/call {'gain':>6s}")
for op in OPS:
    t1 = run(op, 1, 24)
    ts = run(op, S, 24)
    print(f"{op:12s} {t1 * 1e3:12.1f} {ts * 1e3:18.1f} {t1 / ts:6.2f}x")
