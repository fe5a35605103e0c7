import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from scipy import ndimage as ndi
from paper_1405_7958_b200 import rtg
from oracle import pyoracle as O
ctx = rtg.Context(0, 4096, 4096, 1 << 17)
ctx.set_stream(torch.cuda.current_stream().cuda_stream)
for (h, w, conn, dens, sm) in [(4096, 4096, 4, 0.3, 1.0), (4096, 4096, 8, 0.3, 1.0), (1024, 1024, 4, 0.3, 1.0), (2048, 2048, 4, 0.3, 1.0), (4096, 4096, 4, 0.7, 1.0), (2048, 2048, 4, 0.7, 1.0)]:
    rng = np.random.default_rng(h + conn)
    f = ndi.gaussian_filter(rng.random((h, w)), sm)
    m = (f > np.quantile(f, 1 - dens)).astype(np.uint8)
    ref, nref = O.bwlabel(m, conn)
    lab = torch.empty((h, w), dtype=torch.int32, device="cuda")
    n = torch.zeros(1, dtype=torch.int32, device="cuda")
    res = []
    for rep in range(3):
        ctx.bwlabel_dev(torch.from_numpy(m).cuda(), h, w, conn, lab, n)
        torch.cuda.synchronize()
        g = lab.cpu().numpy()
        bad = g != ref
        res.append((int(n.item()), int(bad.sum())))
    print(h, w, conn, dens, 'ref n', nref, 'gpu (n, mismatches) x3', res, flush=True)
    if bad.any():
        ys, xs = np.nonzero(bad)
        print('  first bad', ys[:5], xs[:5], 'gpu', g[ys[:5], xs[:5]], 'ref', ref[ys[:5], xs[:5]])
        print('  bad rows mod 32', np.bincount(ys % 32, minlength=32)[:8], 'cols mod 32', np.bincount(xs % 32, minlength=32)[:8])
