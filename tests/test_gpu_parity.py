"""GPU parity: every operator of the stage, called through the C-ABI, against
the CPU oracle on the same seeded inputs.  Bar: bit-exact for masks, labels,
distances, reconstructions; features within rtol 1e-5 (atol 1e-6 for values
that can be ~0, e.g. orientation)."""
import numpy as np
import pytest

torch = pytest.importorskip("torch")

pytestmark = pytest.mark.gpu

FEAT_RTOL = 1e-5
FEAT_ATOL = 1e-6


def _np_dev(a):
    a = np.ascontiguousarray(a)
    if a.dtype == np.uint16:
        a = a.view(np.int16)
    return torch.from_numpy(a).cuda()


def _dev_np(t, dtype=None):
    torch.cuda.synchronize()
    a = t.cpu().numpy()
    if dtype is not None:
        a = a.view(dtype)
    return a


@pytest.fixture(scope="module")
def ctx(rtg):
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    c = rtg.Context(0, 4096, 4096, 1 << 17)
    # one stream for torch's copies and the ctx's kernels (the default stream
    # handle 0 would select the ctx's own stream, unordered with torch's)
    s = torch.cuda.Stream()
    prev = torch.cuda.current_stream()
    torch.cuda.set_stream(s)
    c.set_stream(s.cuda_stream)
    yield c
    torch.cuda.synchronize()
    torch.cuda.set_stream(prev)
    c.close()


@pytest.fixture(scope="module")
def tile4k(rtg):
    return rtg.synth_tile_host(0, 0, 4096, 4096)


def _rand_blobs(rng, h, w, density=0.3, smooth=2):
    from scipy import ndimage as ndi
    f = ndi.gaussian_filter(rng.random((h, w)), smooth)
    return (f > np.quantile(f, 1 - density)).astype(np.uint8)


def _maze(h, w):
    """Single-pixel-wide serpentine corridor: worst-case IWPP wavefront."""
    m = np.zeros((h, w), np.uint8)
    for y in range(0, h, 2):
        m[y, :] = 1
    for k, y in enumerate(range(1, h, 2)):
        m[y, (w - 1) if k % 2 == 0 else 0] = 1
    return m


# ---------------------------------------------------------------- generator

def test_synth_dev_matches_host(rtg, ctx):
    for (h, w, r, c) in [(512, 640, 0, 0), (4096, 4096, 3, 7), (1696, 4096, 24, 5)]:
        host = rtg.synth_tile_host(r, c, h, w)
        d = torch.empty((h, w, 3), dtype=torch.uint8, device="cuda")
        ctx.synth_tile_dev(d, r, c, h, w)
        assert np.array_equal(_dev_np(d), host)


# ---------------------------------------------------------------- o1/o2

@pytest.mark.parametrize("shape", [(4096, 4096), (1000, 1333), (7, 5), (1, 1)])
def test_colordeconv(rtg, ctx, oracle, shape):
    h, w = shape
    rgb = rtg.synth_tile_host(1, 2, h, w)
    p = rtg.default_params()
    ref = oracle.colordeconv(rgb, p)
    d_rgb = _np_dev(rgb)
    outs = [torch.empty((h, w), dtype=torch.uint8, device="cuda") for _ in range(3)]
    ctx.colordeconv_dev(d_rgb, h, w, p, *outs)
    for o, r in zip(outs, ref):
        assert np.array_equal(_dev_np(o), r)


@pytest.mark.parametrize("variant", ["default", "params"])
def test_colordeconv_random_bytes(rtg, ctx, oracle, variant):
    """Uniform random RGB (every LUT entry, bg/RBC boundaries) through the
    vector kernel, with and without the marker plane (the default stage path
    writes hematoxylin + tissue only)."""
    h, w = 2048, 1536
    rgb = np.random.default_rng(7).integers(0, 256, (h, w, 3), dtype=np.uint8)
    p = rtg.default_params()
    if variant == "params":
        p.bg_thresh, p.rbc_rg10, p.rbc_rb10, p.recon_h = 128, 11, 29, 300
    ref = oracle.colordeconv(rgb, p)
    d_rgb = _np_dev(rgb)
    hema, marker, tissue = (torch.empty((h, w), dtype=torch.uint8, device="cuda")
                            for _ in range(3))
    ctx.colordeconv_dev(d_rgb, h, w, p, hema, None, tissue)
    assert np.array_equal(_dev_np(hema), ref[0])
    assert np.array_equal(_dev_np(tissue), ref[2])
    ctx.colordeconv_dev(d_rgb, h, w, p, hema, marker, tissue)
    for o, r in zip((hema, marker, tissue), ref):
        assert np.array_equal(_dev_np(o), r)


def test_colordeconv_pitched(rtg, ctx, oracle):
    h, w, pitch = 333, 517, 3 * 517 + 13
    rgb = rtg.synth_tile_host(4, 4, h, w)
    buf = np.zeros((h, pitch), np.uint8)
    buf[:, : 3 * w] = rgb.reshape(h, 3 * w)
    p = rtg.default_params()
    ref = oracle.colordeconv(rgb, p)
    outs = [torch.empty((h, w), dtype=torch.uint8, device="cuda") for _ in range(3)]
    ctx.colordeconv_dev(_np_dev(buf), h, w, p, *outs, pitch=pitch)
    for o, r in zip(outs, ref):
        assert np.array_equal(_dev_np(o), r)


# ---------------------------------------------------------------- o3

@pytest.mark.parametrize("conn", [4, 8])
def test_recon_hdome_4k(rtg, ctx, oracle, tile4k, conn):
    p = rtg.default_params()
    hema, marker, _ = oracle.colordeconv(tile4k, p)
    ref = oracle.recon(marker, hema, conn)
    out = torch.empty((4096, 4096), dtype=torch.uint8, device="cuda")
    ctx.recon_dev(_np_dev(marker), _np_dev(hema), 4096, 4096, conn, out)
    assert np.array_equal(_dev_np(out), ref)


@pytest.mark.parametrize("conn", [4, 8])
@pytest.mark.parametrize("shape", [(257, 391), (64, 64), (1, 100), (100, 1), (33, 31)])
def test_recon_random(ctx, oracle, conn, shape):
    rng = np.random.default_rng(shape[0] * 1000 + shape[1] + conn)
    h, w = shape
    mask = rng.integers(0, 256, (h, w), dtype=np.uint8)
    marker = (mask * (rng.random((h, w)) < 0.02)).astype(np.uint8)
    ref = oracle.recon(marker, mask, conn)
    out = torch.empty((h, w), dtype=torch.uint8, device="cuda")
    ctx.recon_dev(_np_dev(marker), _np_dev(mask), h, w, conn, out)
    assert np.array_equal(_dev_np(out), ref)


@pytest.mark.parametrize("conn", [4, 8])
def test_recon_maze_long_wavefront(ctx, oracle, conn):
    h, w = 512, 512
    mask = (_maze(h, w) * 200).astype(np.uint8)
    marker = np.zeros_like(mask)
    marker[0, 0] = 200
    ref = oracle.recon(marker, mask, conn)
    out = torch.empty((h, w), dtype=torch.uint8, device="cuda")
    ctx.recon_dev(_np_dev(marker), _np_dev(mask), h, w, conn, out)
    got = _dev_np(out)
    assert np.array_equal(got, ref)
    assert (got == 200).sum() == (mask > 0).sum()  # the wave reached the far end


def test_recon_u16(ctx, oracle):
    rng = np.random.default_rng(7)
    h, w = 300, 420
    mask = rng.integers(0, 60000, (h, w)).astype(np.uint16)
    marker = np.maximum(mask.astype(np.int64) - 5000, 0).astype(np.uint16)
    ref = oracle.recon(marker, mask, 8)
    out = torch.empty((h, w), dtype=torch.int16, device="cuda")
    ctx.recon_dev(_np_dev(marker), _np_dev(mask), h, w, 8, out, bits=16)
    assert np.array_equal(_dev_np(out, np.uint16), ref)


# ---------------------------------------------------------------- o4

@pytest.mark.parametrize("impl", [0, 1])
@pytest.mark.parametrize("shape", [(512, 512), (4096, 4096), (31, 77)])
def test_fill_holes(rtg, ctx, oracle, shape, impl):
    rng = np.random.default_rng(shape[0])
    h, w = shape
    m = 1 - _rand_blobs(rng, h, w, 0.45, 1.5)
    ref = oracle.fill_holes(m)
    out = torch.empty((h, w), dtype=torch.uint8, device="cuda")
    ctx.set_option(rtg.OPT_FILL_HOLES_IMPL, impl)
    try:
        ctx.fill_holes_dev(_np_dev(m), h, w, out)
        assert np.array_equal(_dev_np(out), ref)
    finally:
        ctx.set_option(rtg.OPT_FILL_HOLES_IMPL, 0)


@pytest.fixture(scope="module")
def ref2048(rtg, oracle):
    rgb = rtg.synth_tile_host(7, 7, 2048, 2048)
    return rgb, oracle.process_tile(rgb)


@pytest.mark.parametrize("ws", [0, 1, 2])
@pytest.mark.parametrize("recon", [0, 1])
@pytest.mark.parametrize("impl", [0, 1])
@pytest.mark.parametrize("graphs", [0, 1])
def test_pipeline_impl_options(rtg, ctx, ref2048, impl, graphs, recon, ws):
    """Every implementation option of the stage (fill-holes union-find vs
    IWPP, ReconToNuclei threshold decomposition vs grayscale IWPP,
    object-parallel vs tiled watershed, graph replay vs eager) gives the
    oracle's result bit for bit."""
    rgb, ref = ref2048
    ctx.set_option(rtg.OPT_FILL_HOLES_IMPL, impl)
    ctx.set_option(rtg.OPT_USE_GRAPHS, graphs)
    ctx.set_option(rtg.OPT_RECON_IMPL, recon)
    ctx.set_option(rtg.OPT_WATERSHED_IMPL, 1 if ws == 1 else 0)
    ctx.set_option(rtg.OPT_HMAX_IMPL, 1 if ws == 2 else 0)  # ws 2: tiled with IWPP HMAX
    try:
        mask, labels, _, feats, n = ctx.process_tile(rgb)
    finally:
        ctx.set_option(rtg.OPT_FILL_HOLES_IMPL, 0)
        ctx.set_option(rtg.OPT_USE_GRAPHS, 1)
        ctx.set_option(rtg.OPT_RECON_IMPL, 0)
        ctx.set_option(rtg.OPT_WATERSHED_IMPL, 0)
        ctx.set_option(rtg.OPT_HMAX_IMPL, 0)
    assert n == ref["n"]
    assert np.array_equal(mask, ref["mask"])
    assert np.array_equal(labels, ref["labels"])


# ---------------------------------------------------------------- o5 / o8

@pytest.mark.parametrize("conn", [4, 8])
@pytest.mark.parametrize("shape", [(4096, 4096), (1000, 1333), (1, 1), (5, 70)])
def test_bwlabel(ctx, oracle, conn, shape):
    rng = np.random.default_rng(sum(shape) + conn)
    h, w = shape
    m = _rand_blobs(rng, h, w, 0.3, 1.0) if min(h, w) > 4 else (rng.random((h, w)) < 0.5).astype(np.uint8)
    ref, nref = oracle.bwlabel(m, conn)
    lab = torch.empty((h, w), dtype=torch.int32, device="cuda")
    n = torch.zeros(1, dtype=torch.int32, device="cuda")
    ctx.bwlabel_dev(_np_dev(m), h, w, conn, lab, n)
    assert int(_dev_np(n)[0]) == nref
    assert np.array_equal(_dev_np(lab), ref)


def test_bwlabel_full_and_empty(ctx, oracle):
    for v in (0, 1):
        m = np.full((300, 300), v, np.uint8)
        lab = torch.empty((300, 300), dtype=torch.int32, device="cuda")
        n = torch.zeros(1, dtype=torch.int32, device="cuda")
        ctx.bwlabel_dev(_np_dev(m), 300, 300, 8, lab, n)
        assert int(_dev_np(n)[0]) == v
        assert np.array_equal(_dev_np(lab), oracle.bwlabel(m, 8)[0])


@pytest.mark.parametrize("conn", [4, 8])
def test_area_threshold(ctx, oracle, conn):
    rng = np.random.default_rng(11)
    h, w = 2048, 1536
    m = _rand_blobs(rng, h, w, 0.25, 1.2)
    ref = oracle.area_threshold(m, conn, 24, 300)
    out = torch.empty((h, w), dtype=torch.uint8, device="cuda")
    ctx.area_threshold_dev(_np_dev(m), h, w, conn, 24, 300, out)
    assert np.array_equal(_dev_np(out), ref)


# ---------------------------------------------------------------- o6

@pytest.mark.parametrize("case", ["blobs", "sparse_zeros", "no_zeros", "one_zero", "thin"])
def test_edt(ctx, oracle, case):
    rng = np.random.default_rng(3)
    h, w = 777, 1024
    if case == "blobs":
        m = _rand_blobs(rng, h, w, 0.4, 3)
    elif case == "sparse_zeros":
        m = (rng.random((h, w)) > 0.0002).astype(np.uint8)  # exercises the exact fallback
    elif case == "no_zeros":
        m = np.ones((h, w), np.uint8)
    elif case == "one_zero":
        m = np.ones((h, w), np.uint8)
        m[h // 3, w - 5] = 0
    else:
        m = np.ones((h, w), np.uint8)
        m[:, ::7] = 0
    ref = oracle.edt_sq(m)
    out = torch.empty((h, w), dtype=torch.int32, device="cuda")
    ctx.edt_dev(_np_dev(m), h, w, out)
    assert np.array_equal(_dev_np(out), ref)


# ---------------------------------------------------------------- o6/o7

@pytest.mark.parametrize("ws_h", [0, 3, 8])
@pytest.mark.parametrize("impl,hmax", [(0, 0), (0, 1), (1, 0)])
def test_watershed(rtg, ctx, oracle, ws_h, impl, hmax):
    """Tiled watershed with sparse-component HMAX (default) or IWPP HMAX, and
    the object-parallel watershed, against the oracle."""
    rng = np.random.default_rng(ws_h + 100)
    h, w = 1024, 1280
    m = _rand_blobs(rng, h, w, 0.35, 2.5)
    sep_ref, basin_ref = oracle.watershed(m, ws_h)
    sep = torch.empty((h, w), dtype=torch.uint8, device="cuda")
    basin = torch.empty((h, w), dtype=torch.int32, device="cuda")
    ctx.set_option(rtg.OPT_WATERSHED_IMPL, impl)
    ctx.set_option(rtg.OPT_HMAX_IMPL, hmax)
    try:
        ctx.watershed_dev(_np_dev(m), h, w, ws_h, sep, basin)
    finally:
        ctx.set_option(rtg.OPT_WATERSHED_IMPL, 0)
        ctx.set_option(rtg.OPT_HMAX_IMPL, 0)
    assert np.array_equal(_dev_np(basin), basin_ref)
    assert np.array_equal(_dev_np(sep), sep_ref)


@pytest.mark.parametrize("ws_h", [1, 5])
def test_watershed_4k(rtg, ctx, oracle, ws_h):
    """The default watershed (sparse-component HMAX, compact plateau forests,
    masked-code basin chains) on a full 4096^2 tile of touching blobs."""
    rng = np.random.default_rng(ws_h + 4096)
    h = w = 4096
    m = _rand_blobs(rng, h, w, 0.4, 3.0)
    sep_ref, basin_ref = oracle.watershed(m, ws_h)
    sep = torch.empty((h, w), dtype=torch.uint8, device="cuda")
    basin = torch.empty((h, w), dtype=torch.int32, device="cuda")
    ctx.watershed_dev(_np_dev(m), h, w, ws_h, sep, basin)
    assert np.array_equal(_dev_np(basin), basin_ref)
    assert np.array_equal(_dev_np(sep), sep_ref)


@pytest.mark.parametrize("impl", [0, 1])
@pytest.mark.parametrize("case", ["big_blob", "thin_diagonal", "border_touching", "all_fg",
                                  "bands", "squares"])
def test_watershed_objects_size_classes(rtg, ctx, oracle, case, impl):
    """Both watershed implementations (tiled default, object-parallel) on
    objects beyond the object-parallel path's 12 KB per-warp class: a large
    blob (227 KB CTA class), a long diagonal thread whose bbox region is huge
    (global-arena class), objects cut by the tile border, a tile with no
    background at all, and plateau-heavy shapes (thick bands and squares:
    long flat EDT ridges, i.e. large plateau components in the compact
    plateau forest)."""
    h, w = 600, 700
    m = np.zeros((h, w), np.uint8)
    if case == "big_blob":
        yy, xx = np.mgrid[0:h, 0:w]
        m[((yy - 250) / 110.0) ** 2 + ((xx - 300) / 70.0) ** 2 <= 1] = 1
        m[((yy - 250) / 60.0) ** 2 + ((xx - 420) / 60.0) ** 2 <= 1] = 1
    elif case == "thin_diagonal":
        for k in range(560):
            m[20 + k, 30 + k] = 1
            m[20 + k, 31 + k] = 1
        m[300:330, 100:140] = 1
    elif case == "border_touching":
        yy, xx = np.mgrid[0:h, 0:w]
        m[(yy ** 2 + xx ** 2) < 120 ** 2] = 1
        m[((yy - h) ** 2 + (xx - 350) ** 2) < 90 ** 2] = 1
    elif case == "bands":
        m[40:71, 10:690] = 1
        m[120:160, 50:650] = 1
        m[200:400, 300:340] = 1
        m[420:451, :] = 1
    elif case == "squares":
        for y0 in range(10, 560, 70):
            for x0 in range(10, 660, 70):
                m[y0:y0 + 41 + (x0 % 3), x0:x0 + 41 + (y0 % 5)] = 1
        m[100:140, 45:90] = 1  # joins two squares
    else:
        m[:] = 1
    sep_ref, basin_ref = oracle.watershed(m, 3)
    sep = torch.empty((h, w), dtype=torch.uint8, device="cuda")
    basin = torch.empty((h, w), dtype=torch.int32, device="cuda")
    ctx.set_option(rtg.OPT_WATERSHED_IMPL, impl)
    try:
        ctx.watershed_dev(_np_dev(m), h, w, 3, sep, basin)
    finally:
        ctx.set_option(rtg.OPT_WATERSHED_IMPL, 0)
    assert np.array_equal(_dev_np(basin), basin_ref)
    assert np.array_equal(_dev_np(sep), sep_ref)


def test_sparse_edt_whole_tile_fallback(rtg, ctx, oracle):
    """A blob far wider than the sparse EDT's 32-row window: the gated
    whole-tile pass (one cooperative launch) must run (need_full flag) and
    the watershed still equals the oracle."""
    h, w = 512, 640
    yy, xx = np.mgrid[0:h, 0:w]
    m = (((yy - 250) / 150.0) ** 2 + ((xx - 300) / 120.0) ** 2 <= 1).astype(np.uint8)
    m[400:430, 500:530] = 1
    sep_ref, basin_ref = oracle.watershed(m, 3)
    sep = torch.empty((h, w), dtype=torch.uint8, device="cuda")
    basin = torch.empty((h, w), dtype=torch.int32, device="cuda")
    ctx.stats()  # clear the counters
    ctx.watershed_dev(_np_dev(m), h, w, 3, sep, basin)
    assert ctx.stats()[3] == 1  # the sparse EDT raised need_full
    assert np.array_equal(_dev_np(basin), basin_ref)
    assert np.array_equal(_dev_np(sep), sep_ref)


# ---------------------------------------------------------------- o9

def test_features(ctx, oracle, tile4k):
    ref = oracle.process_tile(tile4k[:1024, :1024])
    labels, n = ref["labels"], ref["n"]
    hema = oracle.colordeconv(tile4k[:1024, :1024], oracle.default_params())[0]
    got = ctx.features(labels, hema, n)
    np.testing.assert_allclose(got, ref["features"], rtol=FEAT_RTOL, atol=FEAT_ATOL)


# ---------------------------------------------------------------- whole stage

@pytest.mark.parametrize("shape,rc", [((1024, 1024), (0, 0)), ((4096, 4096), (0, 0)),
                                      ((4096, 1696), (3, 24)), ((1696, 1696), (24, 24)),
                                      ((97, 203), (9, 9))])
def test_pipeline(rtg, ctx, oracle, shape, rc):
    h, w = shape
    rgb = rtg.synth_tile_host(rc[0], rc[1], h, w)
    p = rtg.default_params()
    mask, labels, hema, feats, n = ctx.process_tile(rgb, p)
    ref = oracle.process_tile(rgb, p)
    assert n == ref["n"]
    assert np.array_equal(mask, ref["mask"])
    assert np.array_equal(labels, ref["labels"])
    np.testing.assert_allclose(feats, ref["features"], rtol=FEAT_RTOL, atol=FEAT_ATOL)


def test_pipeline_dev_async_matches_host_entry(rtg, ctx):
    h = w = 2048
    p = rtg.default_params()
    d_rgb = torch.empty((h, w, 3), dtype=torch.uint8, device="cuda")
    ctx.synth_tile_dev(d_rgb, 5, 6, h, w)
    d_mask = torch.empty((h, w), dtype=torch.uint8, device="cuda")
    d_lab = torch.empty((h, w), dtype=torch.int32, device="cuda")
    d_feat = torch.empty((ctx.max_objects, rtg.NUM_FEATURES), dtype=torch.float32, device="cuda")
    d_n = torch.zeros(1, dtype=torch.int32, device="cuda")
    ctx.process_tile_dev(d_rgb, h, w, p, d_mask, d_lab, None, d_feat, d_n)
    ctx.sync()
    n = int(_dev_np(d_n)[0])
    mask, labels, _, feats, n2 = ctx.process_tile(_dev_np(d_rgb), p)
    assert n == n2
    assert np.array_equal(_dev_np(d_mask), mask)
    assert np.array_equal(_dev_np(d_lab), labels)
    assert np.array_equal(_dev_np(d_feat)[:n], feats)


def test_graph_replay_matches_eager(rtg, ctx):
    """process_tile_dev: first call captures a CUDA graph, later calls replay
    it; both must equal the kernel-by-kernel path."""
    h, w = 1536, 2048
    p = rtg.default_params()
    d_rgb = torch.empty((h, w, 3), dtype=torch.uint8, device="cuda")
    ctx.synth_tile_dev(d_rgb, 9, 1, h, w)
    outs = []
    for graphs in (1, 1, 0):
        ctx.set_option(rtg.OPT_USE_GRAPHS, graphs)
        d_lab = torch.zeros((h, w), dtype=torch.int32, device="cuda")
        d_feat = torch.zeros((ctx.max_objects, rtg.NUM_FEATURES), dtype=torch.float32, device="cuda")
        d_n = torch.zeros(1, dtype=torch.int32, device="cuda")
        ctx.process_tile_dev(d_rgb, h, w, p, None, d_lab, None, d_feat, d_n)
        ctx.sync()
        n = int(_dev_np(d_n)[0])
        outs.append((n, _dev_np(d_lab), _dev_np(d_feat)[:n]))
    ctx.set_option(rtg.OPT_USE_GRAPHS, 1)
    for o in outs[1:]:
        assert o[0] == outs[0][0] and np.array_equal(o[1], outs[0][1]) and np.array_equal(o[2], outs[0][2])


def test_repeatable(rtg, ctx):
    rgb = rtg.synth_tile_host(2, 2, 1024, 1024)
    a = ctx.process_tile(rgb)
    b = ctx.process_tile(rgb)
    for x, y in zip(a, b):
        if isinstance(x, np.ndarray):
            assert np.array_equal(x, y)
        else:
            assert x == y


def test_stage_state_interleaved_with_operators(rtg, ctx, oracle):
    """The stage clears its counters inside its own launches (the streaming
    kernel's first CTA, the watershed's zeroing launch, the ranking pass);
    per-operator entry points on the same context in between must not leak
    state into it: every stage call stays bit-exact with the oracle."""
    h, w = 1024, 1280
    rng = np.random.default_rng(11)
    blobs = _rand_blobs(rng, h, w, density=0.3)
    d_mask = _np_dev(blobs)
    lab = torch.empty((h, w), dtype=torch.int32, device="cuda")
    n = torch.zeros(1, dtype=torch.int32, device="cuda")
    sep = torch.empty((h, w), dtype=torch.uint8, device="cuda")
    for k, (r, c) in enumerate([(3, 1), (5, 2), (7, 3)]):
        rgb = rtg.synth_tile_host(r, c, h, w)
        ref = oracle.process_tile(rgb, rtg.default_params())
        mask, labels, hema, feats, nobj = ctx.process_tile(rgb)
        assert nobj == ref["n"]
        assert np.array_equal(mask, ref["mask"])
        assert np.array_equal(labels, ref["labels"])
        np.testing.assert_allclose(feats, ref["features"], rtol=FEAT_RTOL, atol=FEAT_ATOL)
        # operators in between leave counters / bitmaps in arbitrary states
        ctx.bwlabel_dev(d_mask, h, w, 8 if k % 2 else 4, lab, n)
        ctx.watershed_dev(d_mask, h, w, rtg.default_params().ws_h, sep)
        ctx.fill_holes_dev(d_mask, h, w, sep)


def test_process_tiles_batch(rtg, ctx):
    """rtg_process_tiles (double-buffered batch) returns exactly what
    rtg_process_tile returns per tile, with pinned (zero-copy rows) and
    pageable feature buffers."""
    h, w = 1024, 1536
    rgbs = [rtg.synth_tile_host(r, 2 * r + 1, h, w) for r in range(5)]
    ref = [ctx.process_tile(t) for t in rgbs]
    pinned = [torch.empty((ctx.max_objects, rtg.NUM_FEATURES), dtype=torch.float32,
                          pin_memory=True).numpy() for _ in rgbs]
    for feats in (None, pinned):
        got, ns = ctx.process_tiles(rgbs, feats=feats)
        for (mask, labels, hema, f_ref, n_ref), f, n in zip(ref, got, ns):
            assert n == n_ref
            assert np.array_equal(f, f_ref)


# ---------------------------------------------------------------- f4 texture

@pytest.mark.parametrize("case", ["tile", "noise", "step", "tiny"])
def test_canny(rtg, ctx, oracle, tile4k, case):
    """Canny edges (smoothing, Sobel, NMS, hysteresis on the CCL) bit-exact
    vs the oracle's BFS hysteresis."""
    rng = np.random.default_rng(5)
    if case == "tile":
        inten = oracle.colordeconv(tile4k[:1200, :1000], oracle.default_params())[0]
    elif case == "noise":
        inten = rng.integers(0, 256, (333, 517)).astype(np.uint8)
    elif case == "step":
        inten = np.zeros((64, 96), np.uint8)
        inten[:, 40:] = 200
        inten[30:, :] = 90
    else:
        inten = rng.integers(0, 256, (3, 7)).astype(np.uint8)
    h, w = inten.shape
    want = oracle.canny(inten)
    out = torch.empty((h, w), dtype=torch.uint8, device="cuda")
    ctx.canny_dev(_np_dev(inten), h, w, out)
    got = _dev_np(out)
    assert np.array_equal(got, want)


TEX_RTOL, TEX_ATOL = 1e-5, 1e-6


@pytest.mark.parametrize("case", ["pipeline", "blobs", "single_pixels"])
def test_texture(rtg, ctx, oracle, tile4k, case):
    """f4 texture table (histogram + co-occurrence statistics) vs the oracle:
    labels of a real tile, random 8-connected blobs, and 1-pixel objects (no
    co-occurrence pairs)."""
    rng = np.random.default_rng(11)
    if case == "pipeline":
        ref = oracle.process_tile(tile4k[:1024, :1536])
        labels, n = ref["labels"], ref["n"]
        inten = oracle.colordeconv(tile4k[:1024, :1536], oracle.default_params())[0]
    elif case == "blobs":
        m = _rand_blobs(rng, 700, 900, 0.3, 3)
        labels = np.zeros(m.shape, np.int32)
        n = oracle.load().orc_bwlabel(m.ctypes.data, 700, 900, 8, labels.ctypes.data)
        inten = rng.integers(0, 256, m.shape).astype(np.uint8)
    else:
        labels = np.zeros((64, 80), np.int32)
        n = 0
        for y in range(0, 64, 3):
            for x in range(0, 80, 3):
                n += 1
                labels[y, x] = n
        inten = rng.integers(0, 256, labels.shape).astype(np.uint8)
    want = oracle.texture(labels, inten, n)
    got = ctx.texture(labels, inten, n)
    assert got.shape == want.shape == (n, rtg.NUM_TEXTURE)
    np.testing.assert_allclose(got, want, rtol=TEX_RTOL, atol=TEX_ATOL)


def test_texture_dev_matches_host(rtg, ctx, oracle, tile4k):
    """rtg_texture_features_dev on device buffers equals the host variant."""
    ref = oracle.process_tile(tile4k[:512, :768])
    labels, n = ref["labels"], ref["n"]
    inten = oracle.colordeconv(tile4k[:512, :768], oracle.default_params())[0]
    host = ctx.texture(labels, inten, n)
    d_out = torch.zeros((ctx.max_objects, rtg.NUM_TEXTURE), dtype=torch.float32, device="cuda")
    d_n = torch.tensor([n], dtype=torch.int32, device="cuda")
    ctx.texture_dev(_np_dev(labels), _np_dev(inten), 512, 768, d_n, d_out)
    ctx.sync()
    assert np.array_equal(d_out[:n].cpu().numpy(), host)


def test_canny_thresholds_validated(rtg, ctx):
    d = torch.zeros((16, 16), dtype=torch.uint8, device="cuda")
    e = torch.zeros((16, 16), dtype=torch.uint8, device="cuda")
    with pytest.raises(rtg.Error):
        ctx.canny_dev(d, 16, 16, e, low=100, high=50)
    with pytest.raises(rtg.Error):
        ctx.canny_dev(d, 16, 16, e, low=-1, high=50)


def test_process_tiles_edge_cases(rtg, ctx):
    """Empty batch is a no-op; a feature table too small for a tile reports
    RTG_ERR_OVERFLOW while still filling the counts."""
    feats, ns = ctx.process_tiles([])
    assert feats == [] and ns == []
    rgb = rtg.synth_tile_host(0, 0, 512, 512)
    with pytest.raises(rtg.Error):
        ctx.process_tiles([rgb], max_rows=3)
