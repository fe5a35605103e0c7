"""GPU parity under the bench's own conditions and the round-2 entry points:

* the asynchronous 3-phase host entry point (rtg_process_tile_async) against
  the synchronous one, pinned and pageable, pitched slide views, out-of-order
  waits, more tickets than slots, overflow;
* four contexts on separate streams over the 80 tiles of one rank's WSI shard
  (the bench's configuration), every mask / label / feature row vs the oracle;
* BASELINE config C3 at full size: a 4096^2 mask of dense touching nuclei
  (>= 35 % foreground, >= 50 % of nuclei touching) through area threshold +
  watershed + canonical labelling, and through the whole stage near the
  context's max_objects;
* two devices in one process (per-device shared-memory opt-in).
Bar: masks / labels bit-exact, features within rtol 1e-5 (atol 1e-6)."""
from concurrent.futures import ThreadPoolExecutor

import numpy as np
import pytest

torch = pytest.importorskip("torch")

pytestmark = pytest.mark.gpu

FEAT_RTOL = 1e-5
FEAT_ATOL = 1e-6


def _need_gpu(n=1):
    if not torch.cuda.is_available() or torch.cuda.device_count() < n:
        pytest.skip(f"needs {n} CUDA device(s)")


def _pinned(shape, dtype):
    t = torch.empty(shape, dtype=dtype, pin_memory=True)
    return t, t.numpy()


def _check_tile(got, ref):
    mask, labels, feats, n = got
    assert n == ref["n"]
    assert np.array_equal(mask, ref["mask"])
    assert np.array_equal(labels, ref["labels"])
    np.testing.assert_allclose(feats[:n], ref["features"], rtol=FEAT_RTOL, atol=FEAT_ATOL)


# ---------------------------------------------------------------- async entry

def test_async_matches_sync(rtg):
    _need_gpu()
    shapes = [(4096, 4096, 0, 0), (4096, 1696, 3, 24), (1696, 1696, 24, 24), (1024, 1333, 5, 5),
              (97, 203, 9, 9)]
    keep = []
    with rtg.Context(0, 4096, 4096, 1 << 16) as ctx:
        ref = {}
        for h, w, r, c in shapes:
            rgb = rtg.synth_tile_host(r, c, h, w)
            mask, labels, _, feats, n = ctx.process_tile(rgb)
            ref[(h, w)] = (rgb, mask, labels, feats, n)
        for pinned in (True, False):
            tickets = []
            for h, w, r, c in shapes:
                rgb = ref[(h, w)][0]
                if pinned:
                    tr, rgb_p = _pinned((h, w, 3), torch.uint8)
                    rgb_p[...] = rgb
                    tm, mask = _pinned((h, w), torch.uint8)
                    tl, labels = _pinned((h, w), torch.int32)
                    tf, feats = _pinned((1 << 16, rtg.NUM_FEATURES), torch.float32)
                    keep += [tr, tm, tl, tf]
                else:
                    rgb_p = rgb
                    mask = np.empty((h, w), np.uint8)
                    labels = np.empty((h, w), np.int32)
                    feats = np.empty((1 << 16, rtg.NUM_FEATURES), np.float32)
                t = ctx.process_tile_async(rgb_p, mask=mask, labels=labels, feats=feats)
                tickets.append((t, (h, w), mask, labels, feats))
            # more tickets than slots were submitted; wait in reverse order
            for t, key, mask, labels, feats in reversed(tickets):
                n = ctx.wait(t)
                _, m_ref, l_ref, f_ref, n_ref = ref[key]
                assert n == n_ref
                assert np.array_equal(mask, m_ref) and np.array_equal(labels, l_ref)
                assert np.array_equal(feats[:n], f_ref)
            with pytest.raises(rtg.NotFoundError):
                ctx.wait(tickets[0][0])


def test_async_pitched_slide_view(rtg, oracle):
    """A tile read straight out of a larger slide (row pitch = slide row
    bytes, cudaMemcpy2DAsync) equals the contiguous tile."""
    _need_gpu()
    slide = rtg.synth_tile_host(1, 1, 1536, 2560)
    with rtg.Context(0, 1024, 1024, 1 << 15) as ctx:
        view = slide[256:1280, 512:1536]
        mask = np.empty((1024, 1024), np.uint8)
        labels = np.empty((1024, 1024), np.int32)
        feats = np.empty((1 << 15, rtg.NUM_FEATURES), np.float32)
        t = ctx.process_tile_async(view, mask=mask, labels=labels, feats=feats,
                                   pitch=slide.strides[0])
        n = ctx.wait(t)
    _check_tile((mask, labels, feats, n), oracle.process_tile(np.ascontiguousarray(view)))


def test_async_overflow_and_query(rtg):
    _need_gpu()
    rgb = rtg.synth_tile_host(0, 0, 1024, 1024)
    with rtg.Context(0, 1024, 1024, 1 << 15) as ctx:
        _, _, _, f_ref, n_ref = ctx.process_tile(rgb)
        assert n_ref > 8
        feats = np.zeros((8, rtg.NUM_FEATURES), np.float32)
        t = ctx.process_tile_async(rgb, feats=feats, max_rows=8)
        with pytest.raises(rtg.OverflowError_):
            ctx.wait(t)
        assert np.array_equal(feats, f_ref[:8])
        t = ctx.process_tile_async(rgb)
        torch.cuda.synchronize()
        n = ctx.wait(t)
        assert n == n_ref
        assert not hasattr(ctx, "_no_such") and len(ctx._inflight) == 0


# ---------------------------------------------------------------- bench mirror

def test_concurrent_contexts_wsi_shard(rtg, oracle):
    """The bench's configuration: 4 contexts, each on its own stream, share
    one GPU over the 80 tiles of rank 0's WSI shard (edge tiles included);
    every tile's mask, labels and features equal the oracle's."""
    _need_gpu()
    from paper_1405_7958_b200.wsi import rank_tiles
    tiles = rank_tiles(0, 80)
    assert any(h != 4096 or w != 4096 for (_, _, h, w) in tiles)
    S = 4
    ctxs = [rtg.Context(0, 4096, 4096, 1 << 15) for _ in range(S)]
    try:
        p = rtg.default_params()
        dev = []
        for k, (r, c, h, w) in enumerate(tiles):
            d_rgb = torch.empty((h, w, 3), dtype=torch.uint8, device="cuda")
            ctxs[0].synth_tile_dev(d_rgb, r, c, h, w)
            dev.append((d_rgb,
                        torch.empty((h, w), dtype=torch.uint8, device="cuda"),
                        torch.empty((h, w), dtype=torch.int32, device="cuda"),
                        torch.empty((1 << 15, rtg.NUM_FEATURES), dtype=torch.float32, device="cuda"),
                        torch.zeros(1, dtype=torch.int32, device="cuda")))
        ctxs[0].sync()
        torch.cuda.synchronize()  # torch's zero fills vs the ctx streams
        for k, (r, c, h, w) in enumerate(tiles):
            d_rgb, d_mask, d_lab, d_feat, d_n = dev[k]
            ctxs[k % S].process_tile_dev(d_rgb, h, w, p, d_mask, d_lab, None, d_feat, d_n)
        for cx in ctxs:
            cx.sync()
        got = []
        for k, (r, c, h, w) in enumerate(tiles):
            _, d_mask, d_lab, d_feat, d_n = dev[k]
            n = int(d_n.cpu()[0])
            got.append((d_mask.cpu().numpy(), d_lab.cpu().numpy(), d_feat[:n].cpu().numpy(), n))
        del dev
    finally:
        for cx in ctxs:
            cx.close()

    def ref(k):
        r, c, h, w = tiles[k]
        return oracle.process_tile(oracle.synth_tile_host(r, c, h, w), p)

    with ThreadPoolExecutor(max_workers=16) as ex:
        for k, rk in enumerate(ex.map(ref, range(len(tiles)))):
            _check_tile(got[k], rk)


# ---------------------------------------------------------------- C3 dense nuclei

from synthetic_inputs import dense_touching as _dense_touching  # noqa: E402


@pytest.fixture(scope="module")
def c3_mask():
    return _dense_touching(3, 4096, 4096)


def test_c3_dense_touching_4k_operators(rtg, oracle, c3_mask):
    _need_gpu()
    from scipy import ndimage as ndi
    mask, discs = c3_mask
    comps = ndi.label(mask, np.ones((3, 3)))[1]
    assert mask.mean() >= 0.35
    assert comps <= discs // 2  # >= 50 % of nuclei touch another one
    p = rtg.default_params()
    h, w = mask.shape
    with rtg.Context(0, h, w, 1 << 17) as ctx:
        d_in = torch.from_numpy(mask).cuda()
        torch.cuda.synchronize()  # the ctx stream does not order with torch's
        d_area = torch.empty_like(d_in)
        d_sep = torch.empty_like(d_in)
        d_basin = torch.empty((h, w), dtype=torch.int32, device="cuda")
        d_lab = torch.empty((h, w), dtype=torch.int32, device="cuda")
        d_n = torch.zeros(1, dtype=torch.int32, device="cuda")
        ctx.area_threshold_dev(d_in, h, w, 8, p.min_area, p.max_area, d_area)
        ctx.watershed_dev(d_area, h, w, p.ws_h, d_sep, d_basin)
        ctx.bwlabel_dev(d_sep, h, w, 8, d_lab, d_n)
        ctx.sync()
        area = d_area.cpu().numpy()
        sep, basin = d_sep.cpu().numpy(), d_basin.cpu().numpy()
        lab, n = d_lab.cpu().numpy(), int(d_n.cpu()[0])
    r_area = oracle.area_threshold(mask, 8, p.min_area, p.max_area)
    assert np.array_equal(area, r_area)
    r_sep, r_basin = oracle.watershed(r_area, p.ws_h)
    assert np.array_equal(sep, r_sep)
    assert np.array_equal(basin, r_basin)
    r_lab, r_n = oracle.bwlabel(r_sep, 8)
    assert n == r_n and n > 15000
    assert np.array_equal(lab, r_lab)


def _render_he(mask, seed):
    """An H&E-like RGB rendering of a nucleus mask (hematoxylin nuclei on
    eosin stroma, +-8 noise)."""
    rng = np.random.default_rng(seed)
    h, w = mask.shape
    rgb = np.empty((h, w, 3), np.int16)
    rgb[...] = (225, 160, 200)
    rgb[mask > 0] = (80, 60, 150)
    rgb += rng.integers(-8, 9, size=(h, w, 3), dtype=np.int16)
    return np.clip(rgb, 0, 255).astype(np.uint8)


def test_c3_dense_whole_stage_near_capacity(rtg, oracle, c3_mask):
    """The dense tile through the whole stage with max_objects just above its
    object count (bit-exact), and just below it (RTG_ERR_OVERFLOW)."""
    _need_gpu()
    mask, _ = c3_mask
    rgb = _render_he(mask, 5)
    p = rtg.default_params()
    ref = oracle.process_tile(rgb, p)
    n_ref = ref["n"]
    assert n_ref > 15000
    with rtg.Context(0, 4096, 4096, n_ref + 8) as ctx:
        m, lab, _, feats, n = ctx.process_tile(rgb, p)
    _check_tile((m, lab, feats, n), ref)
    with rtg.Context(0, 4096, 4096, n_ref - 1) as ctx:
        with pytest.raises(rtg.OverflowError_):
            ctx.process_tile(rgb, p)


# ---------------------------------------------------------------- two devices

def test_two_devices_one_process(rtg):
    """Contexts on two devices in one process: every kernel's dynamic
    shared-memory opt-in is per device (k_colordeconv_vec uses ~100 KB)."""
    _need_gpu(2)
    rgb = rtg.synth_tile_host(4, 4, 2048, 2048)
    outs = []
    ctxs = [rtg.Context(d, 2048, 2048, 1 << 15) for d in (0, 1, 0)]
    try:
        for cx in ctxs:
            outs.append(cx.process_tile(rgb))
    finally:
        for cx in ctxs:
            cx.close()
    for o in outs[1:]:
        assert o[4] == outs[0][4]
        assert np.array_equal(o[0], outs[0][0]) and np.array_equal(o[1], outs[0][1])
        assert np.array_equal(o[3], outs[0][3])


# ---------------------------------------------------------------- memory-safety / race evidence
# compute-sanitizer is not available on the GPU pool, so out-of-bounds writes
# into caller buffers are caught with guard bands, and races with repeated
# concurrent runs that must stay bit-identical.

_GUARD = 4096


def _guarded(n_bytes, fill=0xA5):
    buf = torch.full((_GUARD * 2 + n_bytes,), fill, dtype=torch.uint8, device="cuda")
    return buf, buf[_GUARD:_GUARD + n_bytes]


def _guards_intact(buf, fill=0xA5):
    g = torch.cat([buf[:_GUARD], buf[-_GUARD:]])
    return bool((g == fill).all())


@pytest.mark.parametrize("shape", [(1, 1), (7, 5), (33, 31), (97, 203), (1000, 1333),
                                   (4096, 1696)])
def test_entry_points_write_inside_their_outputs(rtg, oracle, shape):
    _need_gpu()
    h, w = shape
    rgb = rtg.synth_tile_host(3, 3, h, w)
    p = rtg.default_params()
    with rtg.Context(0, 4096, 4096, 1 << 15) as ctx:
        bufs = {}
        for name, nbytes in (("rgb", 3 * h * w), ("mask", h * w), ("labels", 4 * h * w),
                             ("hema", h * w), ("feats", (1 << 15) * rtg.NUM_FEATURES * 4),
                             ("n", 4), ("tissue", h * w), ("marker", h * w), ("rec", h * w),
                             ("fill", h * w), ("area", h * w), ("dist", 4 * h * w),
                             ("sep", h * w), ("basin", 4 * h * w), ("lab2", 4 * h * w),
                             ("n2", 4), ("tex", (1 << 15) * rtg.NUM_TEXTURE * 4),
                             ("edges", h * w)):
            bufs[name] = _guarded(nbytes)
        v = {k: b[1] for k, b in bufs.items()}
        v["rgb"].copy_(torch.from_numpy(rgb.reshape(-1)))
        torch.cuda.synchronize()  # the ctx's own stream does not order with torch's
        u8 = lambda k: v[k].view(h, w)  # noqa: E731
        i32 = lambda k: v[k].view(torch.int32).view(h, w)  # noqa: E731
        ctx.process_tile_dev(v["rgb"], h, w, p, v["mask"], v["labels"].view(torch.int32),
                             v["hema"], v["feats"].view(torch.float32), v["n"].view(torch.int32))
        ctx.colordeconv_dev(v["rgb"], h, w, p, v["hema"], v["marker"], v["tissue"])
        ctx.recon_dev(u8("marker"), u8("hema"), h, w, 8, v["rec"])
        ctx.fill_holes_dev(u8("mask"), h, w, v["fill"])
        ctx.area_threshold_dev(u8("mask"), h, w, 8, p.min_area, p.max_area, v["area"])
        ctx.edt_dev(u8("mask"), h, w, i32("dist"))
        ctx.watershed_dev(u8("area"), h, w, p.ws_h, v["sep"], i32("basin"))
        ctx.bwlabel_dev(u8("sep"), h, w, 8, i32("lab2"), v["n2"].view(torch.int32))
        ctx.features_dev(i32("labels"), u8("hema"), h, w, v["n"].view(torch.int32),
                         v["feats"].view(torch.float32))
        ctx.texture_dev(i32("labels"), u8("hema"), h, w, v["n"].view(torch.int32),
                        v["tex"].view(torch.float32))
        ctx.canny_dev(u8("hema"), h, w, v["edges"])
        ctx.sync()
        torch.cuda.synchronize()
        bad = [k for k, (buf, _) in bufs.items() if not _guards_intact(buf)]
        assert not bad, f"writes outside the output buffers: {bad}"
        ref = oracle.process_tile(rgb, p)
        assert np.array_equal(u8("mask").cpu().numpy(), ref["mask"])
        assert np.array_equal(i32("labels").cpu().numpy(), ref["labels"])


@pytest.mark.parametrize("shape", [(4096, 4096), (97, 203), (1696, 1696)])
def test_internal_scratch_guard_bands(rtg, oracle, shape, monkeypatch):
    """Every internal scratch buffer of the context followed by a canary band
    (RTG_GUARD_BYTES): the whole stage under every implementation option and
    with texture columns, then every per-operator entry point, must leave all
    bands intact (rtg_ctx_guard_check) and the stage must still match the
    oracle."""
    _need_gpu()
    h, w = shape
    monkeypatch.setenv("RTG_GUARD_BYTES", "65536")
    rgb = rtg.synth_tile_host(5, 2, h, w)
    p = rtg.default_params()
    ref = oracle.process_tile(rgb, p)
    with rtg.Context(0, 4096, 4096, 1 << 15) as ctx:
        assert ctx.guard_check() > 30
        for opts in ({}, {rtg.OPT_LABEL_RUNS: 0}, {rtg.OPT_USE_GRAPHS: 0, rtg.OPT_PDL: 1},
                     {rtg.OPT_WATERSHED_IMPL: 1}, {rtg.OPT_HMAX_IMPL: 1},
                     {rtg.OPT_FILL_HOLES_IMPL: 1}, {rtg.OPT_RECON_IMPL: 1},
                     {rtg.OPT_STREAM_IMPL: 0}):
            for k, val in opts.items():
                ctx.set_option(k, val)
            mask, labels, hema_np, feats, n = ctx.process_tile(rgb, p)
            for k in opts:
                ctx.set_option(k, {rtg.OPT_USE_GRAPHS: 1, rtg.OPT_STREAM_IMPL: 1,
                                   rtg.OPT_LABEL_RUNS: 1}.get(k, 0))
            ctx.guard_check()
            assert n == ref["n"] and np.array_equal(labels, ref["labels"]), opts
        pt = rtg.default_params()
        pt.texture = 1
        ctx.process_tile(rgb, pt)
        ctx.guard_check()
        # the per-operator entry points on device buffers
        d = lambda a: torch.from_numpy(np.ascontiguousarray(a)).cuda()  # noqa: E731
        hema = d(hema_np)
        m = d(ref["mask"])
        o8 = torch.empty((h, w), dtype=torch.uint8, device="cuda")
        o32 = torch.empty((h, w), dtype=torch.int32, device="cuda")
        n1 = torch.empty(1, dtype=torch.int32, device="cuda")
        torch.cuda.synchronize()
        ctx.fill_holes_dev(m, h, w, o8)
        ctx.area_threshold_dev(m, h, w, 8, p.min_area, p.max_area, o8)
        ctx.edt_dev(m, h, w, o32)
        ctx.watershed_dev(m, h, w, p.ws_h, o8, o32)
        ctx.bwlabel_dev(m, h, w, 8, o32, n1)
        ctx.recon_dev(hema, hema, h, w, 8, o8)
        ctx.canny_dev(hema, h, w, o8)
        ctx.sync()
        assert ctx.guard_check() > 30


def test_internal_scratch_guard_check_detects(rtg, monkeypatch):
    """The checker's control: a context whose arena band is corrupted at
    creation (RTG_GUARD_SELFTEST) must fail the check, naming the buffer."""
    _need_gpu()
    monkeypatch.setenv("RTG_GUARD_BYTES", "4096")
    monkeypatch.setenv("RTG_GUARD_SELFTEST", "1")
    with rtg.Context(0, 256, 256, 1 << 10) as ctx:
        with pytest.raises(rtg.Error, match="arena' overwritten at \\+5"):
            ctx.guard_check()


def test_concurrent_runs_are_deterministic(rtg):
    """The same two tiles on four contexts at once, five rounds, with and
    without CUDA graphs and programmatic dependent launch: every run must be
    bit-identical (a race in the union-find / queue / look-back kernels would
    show up as run-to-run differences)."""
    _need_gpu()
    tiles = [rtg.synth_tile_host(0, 0, 2048, 2048), rtg.synth_tile_host(24, 24, 1696, 1696)]
    p = rtg.default_params()
    ctxs = [rtg.Context(0, 2048, 2048, 1 << 15) for _ in range(4)]
    try:
        d = [torch.from_numpy(t).cuda() for t in tiles]
        torch.cuda.synchronize()
        first = None
        for rnd in range(5):
            for k, cx in enumerate(ctxs):
                cx.set_option(rtg.OPT_USE_GRAPHS, (rnd + k) % 2)
                cx.set_option(rtg.OPT_PDL, (rnd // 2 + k) % 2)
            outs = []
            for k, cx in enumerate(ctxs):
                for ti, t in enumerate(tiles):
                    h, w = t.shape[:2]
                    lab = torch.empty((h, w), dtype=torch.int32, device="cuda")
                    f = torch.empty((1 << 15, rtg.NUM_FEATURES), dtype=torch.float32, device="cuda")
                    n = torch.empty(1, dtype=torch.int32, device="cuda")
                    cx.process_tile_dev(d[ti], h, w, p, None, lab, None, f, n)
                    outs.append((ti, lab, f, n))
            for cx in ctxs:
                cx.sync()
            got = {}
            for ti, lab, f, n in outs:
                nn = int(n.cpu()[0])
                key = (lab.cpu().numpy().tobytes(), f[:nn].cpu().numpy().tobytes(), nn)
                got.setdefault(ti, set()).add(key)
            assert all(len(s) == 1 for s in got.values()), f"round {rnd}: runs differ"
            if first is None:
                first = got
            assert got == first, f"round {rnd} differs from round 0"
    finally:
        for cx in ctxs:
            cx.close()


# ---------------------------------------------------------------- C2 reconstruction paths

@pytest.mark.parametrize("conn", [4, 8])
def test_recon_maze_4k_level_decomposition(rtg, oracle, conn):
    """C2's adversarial input at full size: a 1-px serpentine corridor through
    every other row of a 4096^2 tile, one seed.  Two values -> the level
    path (one seeded labelling); bit-exact with the oracle and the wave
    reaches the far end."""
    _need_gpu()
    from synthetic_inputs import serpentine_maze
    maze, seed = serpentine_maze(4096, 4096)
    ref = oracle.recon(seed, maze, conn)
    with rtg.Context(0, 4096, 4096, 1 << 12) as ctx:
        out = torch.empty((4096, 4096), dtype=torch.uint8, device="cuda")
        d_seed, d_maze = torch.from_numpy(seed).cuda(), torch.from_numpy(maze).cuda()
        torch.cuda.synchronize()  # the ctx's own stream does not order with torch's
        ctx.recon_dev(d_seed, d_maze, 4096, 4096, conn, out)
        ctx.sync()
        got = out.cpu().numpy()
    assert np.array_equal(got, ref)
    assert (got == 200).sum() == (maze > 0).sum()


@pytest.mark.parametrize("levels", [1, 3, 4, 5, 9])
@pytest.mark.parametrize("conn", [4, 8])
def test_recon_few_levels_vs_iwpp(rtg, oracle, levels, conn):
    """Quantised masks / markers with `levels` distinct non-zero values: up to
    4 take the level-decomposition path, more the IWPP queue; both paths and
    the forced-IWPP option are bit-exact with the oracle."""
    _need_gpu()
    rng = np.random.default_rng(100 * levels + conn)
    h, w = 777, 1025
    vals = np.sort(rng.choice(np.arange(1, 256), size=levels, replace=False)).astype(np.uint8)
    from scipy import ndimage as ndi
    f = ndi.gaussian_filter(rng.random((h, w)), 3)
    q = np.digitize(f, np.quantile(f, np.linspace(0.2, 1, levels + 1)[:-1]))
    mask = np.where(q > 0, vals[np.clip(q - 1, 0, levels - 1)], 0).astype(np.uint8)
    marker = (mask * (rng.random((h, w)) < 0.001)).astype(np.uint8)
    ref = oracle.recon(marker, mask, conn)
    with rtg.Context(0, h, w, 1 << 12) as ctx:
        d_mk, d_ms = torch.from_numpy(marker).cuda(), torch.from_numpy(mask).cuda()
        for impl in (0, 1):
            ctx.set_option(rtg.OPT_RECON_ENTRY_IMPL, impl)
            out = torch.empty((h, w), dtype=torch.uint8, device="cuda")
            torch.cuda.synchronize()  # the ctx's own stream does not order with torch's
            ctx.recon_dev(d_mk, d_ms, h, w, conn, out)
            ctx.sync()
            assert np.array_equal(out.cpu().numpy(), ref), impl


# ---------------------------------------------------------------- f4 in the stage product

TEX_RTOL, TEX_ATOL = 1e-5, 1e-6


@pytest.mark.parametrize("shape,rc", [((4096, 4096), (0, 0)), ((1696, 4096), (24, 3)),
                                      ((333, 517), (2, 2))])
def test_stage_with_texture_columns(rtg, oracle, shape, rc):
    """params.texture = 1: every feature row carries the 14 texture columns
    after the 20 shape / intensity ones, through the synchronous, batch and
    asynchronous host entry points; equal to the oracle's rows."""
    _need_gpu()
    h, w = shape
    rgb = rtg.synth_tile_host(rc[0], rc[1], h, w)
    p = rtg.default_params()
    p.texture = 1
    assert rtg.feature_columns(p) == rtg.NUM_FEATURES + rtg.NUM_TEXTURE
    from oracle import pyoracle
    op = pyoracle.default_params()
    op.texture = 1
    ref = oracle.process_tile(rgb, op)
    assert ref["features"].shape[1] == 34
    with rtg.Context(0, 4096, 4096, 1 << 15) as ctx:
        mask, labels, _, feats, n = ctx.process_tile(rgb, p)
        assert n == ref["n"] and np.array_equal(labels, ref["labels"])
        np.testing.assert_allclose(feats[:, :20], ref["features"][:, :20], rtol=FEAT_RTOL,
                                   atol=FEAT_ATOL)
        np.testing.assert_allclose(feats[:, 20:], ref["features"][:, 20:], rtol=TEX_RTOL,
                                   atol=TEX_ATOL)
        got, ns = ctx.process_tiles([rgb, rgb], p)
        assert ns == [n, n] and all(np.array_equal(g, feats) for g in got)
        f2 = np.empty((1 << 15, 34), np.float32)
        t = ctx.process_tile_async(rgb, p, feats=f2)
        assert ctx.wait(t) == n and np.array_equal(f2[:n], feats)
        # the same context without texture still gives 20-column rows
        _, _, _, f20, n20 = ctx.process_tile(rgb)
        assert n20 == n and f20.shape[1] == 20 and np.array_equal(f20, feats[:, :20])


@pytest.mark.parametrize("shape", [(4096, 4096), (1696, 4096), (1000, 1333), (64, 48)])
def test_colordeconv_tma_ring_matches_stream(rtg, oracle, shape):
    """RTG_OPT_STREAM_IMPL = 1 (cp.async.bulk ring) gives the same planes as
    the LDG.128 stream kernel and the oracle, and the same stage output."""
    _need_gpu()
    h, w = shape
    rgb = rtg.synth_tile_host(8, 2, h, w)
    p = rtg.default_params()
    want = oracle.colordeconv(rgb, oracle.default_params())
    with rtg.Context(0, 4096, 4096, 1 << 15) as ctx:
        d_rgb = torch.from_numpy(rgb).cuda()
        outs = []
        for impl in (0, 1):
            ctx.set_option(rtg.OPT_STREAM_IMPL, impl)
            planes = [torch.empty((h, w), dtype=torch.uint8, device="cuda") for _ in range(3)]
            torch.cuda.synchronize()
            ctx.colordeconv_dev(d_rgb, h, w, p, planes[0], planes[1], planes[2])
            ctx.sync()
            got = [t.cpu().numpy() for t in planes]
            for g, wnt in zip(got, want):
                assert np.array_equal(g, wnt), impl
            outs.append(ctx.process_tile(rgb, p))
        assert outs[0][4] == outs[1][4] and np.array_equal(outs[0][1], outs[1][1])
        assert np.array_equal(outs[0][3], outs[1][3])


# ------------------------------------------------- run-table labellings (RTG_OPT_LABEL_RUNS)

@pytest.mark.parametrize("shape,rc,conn", [((4096, 4096), (5, 7), 8), ((1000, 1024), (3, 9), 8),
                                           ((777, 1696), (24, 1), 4), ((96, 64), (1, 1), 8),
                                           ((33, 32), (2, 5), 8), ((1000, 1000), (4, 4), 8)])
def test_label_runs_match_per_pixel_roots(rtg, oracle, shape, rc, conn):
    """The run-table labellings (row masks + run tables + border roots, per-
    tile output passes) give the same mask, labels and feature rows as the
    per-pixel-root form, and both equal the oracle (w % 32 != 0 runs the
    per-pixel form either way)."""
    _need_gpu()
    h, w = shape
    rgb = rtg.synth_tile_host(rc[0], rc[1], h, w)
    p = rtg.default_params()
    p.recon_conn = conn
    outs = []
    with rtg.Context(0, 4096, 4096, 1 << 15) as ctx:
        for runs in (1, 0):
            ctx.set_option(rtg.OPT_LABEL_RUNS, runs)
            outs.append(ctx.process_tile(rgb, p))
            # the device entry point (graph replay) and the async one agree
            d_rgb = torch.from_numpy(rgb).cuda()
            d_mask = torch.empty((h, w), dtype=torch.uint8, device="cuda")
            d_lab = torch.empty((h, w), dtype=torch.int32, device="cuda")
            d_feat = torch.empty((1 << 15, 20), dtype=torch.float32, device="cuda")
            d_n = torch.zeros(1, dtype=torch.int32, device="cuda")
            torch.cuda.synchronize()
            for _ in range(2):
                ctx.process_tile_dev(d_rgb, h, w, p, d_mask, d_lab, None, d_feat, d_n)
            ctx.sync()
            assert int(d_n.item()) == outs[-1][4]
            assert np.array_equal(d_mask.cpu().numpy(), outs[-1][0])
            assert np.array_equal(d_lab.cpu().numpy(), outs[-1][1])
    a, b = outs
    assert a[4] == b[4] and np.array_equal(a[0], b[0]) and np.array_equal(a[1], b[1])
    assert np.array_equal(a[3], b[3])
    if h * w <= 1 << 20:
        op = oracle.default_params()
        op.recon_conn = conn
        ref = oracle.process_tile(rgb, op)
        assert a[4] == ref["n"] and np.array_equal(a[1], ref["labels"])
        np.testing.assert_allclose(a[3], ref["features"], rtol=FEAT_RTOL, atol=FEAT_ATOL)


@pytest.mark.parametrize("nuc,rh", [(250, 10), (300, 0), (1, 0), (40, 300), (0, 5), (-3, 2)])
def test_label_runs_threshold_planes_params(rtg, oracle, nuc, rh):
    """The streaming kernel's threshold / seed / tissue bit planes (run-table
    path) across the corners of the ReconToNuclei parameters: seed threshold
    above 255 (no seeds), foreground threshold above 255 (nothing), a
    threshold of 1, and t <= 0 (the candidates are the tissue mask, bytes
    path).  Same output as the per-pixel form and as the oracle."""
    _need_gpu()
    h, w = 512, 768
    rgb = rtg.synth_tile_host(6, 3, h, w)
    p = rtg.default_params()
    p.nuc_thresh, p.recon_h = nuc, rh
    op = oracle.default_params()
    op.nuc_thresh, op.recon_h = nuc, rh
    ref = oracle.process_tile(rgb, op)
    outs = []
    with rtg.Context(0, 1024, 1024, 1 << 15) as ctx:
        for runs in (1, 0):
            ctx.set_option(rtg.OPT_LABEL_RUNS, runs)
            outs.append(ctx.process_tile(rgb, p))
    for mask, labels, _, feats, n in outs:
        assert n == ref["n"]
        assert np.array_equal(mask, ref["mask"]) and np.array_equal(labels, ref["labels"])
        np.testing.assert_allclose(feats, ref["features"], rtol=FEAT_RTOL, atol=FEAT_ATOL)


def test_stage_outputs_at_unaligned_addresses(rtg):
    """process_tile_dev into a mask buffer at an odd byte offset and a label
    buffer 4 bytes off a 16-byte boundary: the run-table path takes its
    scalar-store / byte-plane variants, with the same results as aligned
    outputs."""
    _need_gpu()
    h, w = 1024, 1024
    rgb = torch.from_numpy(rtg.synth_tile_host(3, 5, h, w)).cuda()
    p = rtg.default_params()
    with rtg.Context(0, h, w, 1 << 14) as ctx:
        outs = []
        for off_m, off_l in ((0, 0), (1, 1)):
            mbuf = torch.zeros(h * w + 16, dtype=torch.uint8, device="cuda")
            lbuf = torch.zeros(h * w + 16, dtype=torch.int32, device="cuda")
            m = mbuf[off_m:off_m + h * w].view(h, w)
            lab = lbuf[off_l:off_l + h * w].view(h, w)
            feat = torch.zeros((1 << 14, 20), dtype=torch.float32, device="cuda")
            n = torch.zeros(1, dtype=torch.int32, device="cuda")
            torch.cuda.synchronize()
            ctx.process_tile_dev(rgb, h, w, p, m, lab, None, feat, n)
            ctx.sync()
            k = int(n.item())
            outs.append((k, m.cpu().numpy(), lab.cpu().numpy(), feat[:k].cpu().numpy()))
    (na, ma, la, fa), (nb, mb, lb, fb) = outs
    assert na == nb and np.array_equal(ma, mb) and np.array_equal(la, lb) and np.array_equal(fa, fb)
