"""One small stage call (and the per-operator entry points it is built from)
for compute-sanitizer (memcheck / racecheck / synccheck / initcheck):

  compute-sanitizer --tool racecheck python tools/sanitize_stage.py

Eager launches (no CUDA graph), one 1024^2 tile, results checked against the
oracle so a clean sanitizer log is also a correct run."""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from oracle import pyoracle  # noqa: E402
from paper_1405_7958_b200 import rtg  # noqa: E402


def main():
    h = w = int(os.environ.get("RTG_SAN_TILE", "1024"))
    rgb = rtg.synth_tile_host(2, 3, h, w)
    p = rtg.default_params()
    ref = pyoracle.process_tile(rgb, p)
    with rtg.Context(0, h, w, 1 << 15) as ctx:
        ctx.set_option(rtg.OPT_USE_GRAPHS, 0)
        mask, labels, hema, feats, n = ctx.process_tile(rgb, p)
        assert n == ref["n"] and np.array_equal(mask, ref["mask"])
        assert np.array_equal(labels, ref["labels"])
        np.testing.assert_allclose(feats, ref["features"], rtol=1e-5, atol=1e-6)
        # the option paths: IWPP reconstruction / fill, IWPP HMAX, object-parallel watershed
        for opt, val in ((rtg.OPT_RECON_IMPL, 1), (rtg.OPT_FILL_HOLES_IMPL, 1),
                         (rtg.OPT_HMAX_IMPL, 1), (rtg.OPT_WATERSHED_IMPL, 1)):
            ctx.set_option(opt, val)
            m2, l2, _, f2, n2 = ctx.process_tile(rgb, p)
            assert n2 == n and np.array_equal(l2, labels), opt
            ctx.set_option(opt, 0)
        # async 3-phase entry point
        t = ctx.process_tile_async(rgb, p, mask=np.empty_like(mask),
                                   labels=np.empty_like(labels))
        assert ctx.wait(t) == n
        tex = ctx.texture(labels, hema, n)
        assert tex.shape == (n, rtg.NUM_TEXTURE)
    print(f"sanitize_stage ok: {h}x{w}, {n} objects")


if __name__ == "__main__":
    main()
