"""Independent pins of the self-defined operators (CPU; no GPU).

The reference ships no pixel arithmetic, so colour
deconvolution, the watershed and the feature table are pinned here against
code the oracle does not share: the published Ruifrok-Johnston stain vectors
with float64 deconvolution, OpenCV's connected-component statistics and
image moments, scipy.ndimage's Sobel and labelled statistics, and a Meyer
priority-flood watershed (a different algorithm from the oracle's arrowing).
The GPU path is bit-exact against the oracle (tests/test_gpu_*.py), so these
pins carry over to it.  PAPER.md:1133-1137 (colour deconvolution,
watershed), :1152-1177 (features).
"""
import heapq

import numpy as np
import pytest

cv2 = pytest.importorskip("cv2")
ndi = pytest.importorskip("scipy.ndimage")

# Ruifrok & Johnston (2001) H&E(+DAB) optical-density stain vectors.
STAIN_H = (0.65, 0.70, 0.29)
STAIN_E = (0.07, 0.99, 0.11)
STAIN_DAB = (0.27, 0.57, 0.78)


def test_h_coefficients_are_the_inverse_stain_matrix(oracle):
    m = np.stack([np.asarray(v) / np.linalg.norm(v) for v in (STAIN_H, STAIN_E, STAIN_DAB)])
    col = np.linalg.inv(m)[:, 0]
    p = oracle.default_params()
    np.testing.assert_allclose(list(p.h_coef), col, rtol=1e-12)


def test_hematoxylin_vs_float_deconvolution(oracle):
    """Every one of the 2^24 RGB values: the oracle's 16.16 fixed-point LUT
    hematoxylin is within 1 LSB of float64 Ruifrok-Johnston deconvolution,
    and equal for all but a sliver of values (ties at .5 after rounding)."""
    p = oracle.default_params()
    v = np.arange(1 << 24, dtype=np.uint32)
    rgb = np.stack([(v >> 16) & 255, (v >> 8) & 255, v & 255], axis=-1).astype(np.uint8)
    rgb = rgb.reshape(4096, 4096, 3)
    hema, _, _ = oracle.colordeconv(rgb, p)
    hema = hema.reshape(-1).astype(np.int32)
    coef = np.asarray(p.h_coef)
    od = -np.log10((np.arange(256, dtype=np.float64) + 1.0) / 256.0)
    worst, exact = 0, 0
    for s in range(0, 1 << 24, 1 << 20):
        c = rgb.reshape(-1, 3)[s:s + (1 << 20)].astype(np.int64)
        ch = coef[0] * od[c[:, 0]] + coef[1] * od[c[:, 1]] + coef[2] * od[c[:, 2]]
        ref = np.clip(np.rint(ch * 255.0 / p.h_scale), 0, 255).astype(np.int32)
        d = np.abs(hema[s:s + (1 << 20)] - ref)
        worst = max(worst, int(d.max()))
        exact += int((d == 0).sum())
    assert worst <= 1
    assert exact / float(1 << 24) > 0.999


def _stage(oracle, r, c, h, w):
    from oracle.pyoracle import synth_tile_host
    rgb = synth_tile_host(r, c, h, w)
    p = oracle.default_params()
    out = oracle.process_tile(rgb, p, want_planes=True)
    return rgb, out


@pytest.fixture(scope="module")
def stage1k(oracle):
    return _stage(oracle, 0, 0, 1024, 1024)


def _canon(lab):
    """Renumbers a labelling 1..n by each object's minimum linear index."""
    flat = lab.reshape(-1)
    ids = np.unique(flat[flat > 0])
    first = np.array([np.flatnonzero(flat == i)[0] for i in ids]) if len(ids) else np.array([])
    order = ids[np.argsort(first)]
    lut = np.zeros(int(flat.max()) + 1, np.int32)
    lut[order] = np.arange(1, len(order) + 1)
    return lut[lab]


def test_labels_vs_opencv(stage1k):
    _, out = stage1k
    n, lab = cv2.connectedComponents(out["mask"], connectivity=8, ltype=cv2.CV_32S)
    assert n - 1 == out["n"]
    assert np.array_equal(_canon(lab), out["labels"])


def test_shape_features_vs_opencv(stage1k):
    """Area, bounding box and centroid from cv2.connectedComponentsWithStats;
    second moments (axes, eccentricity, orientation) from cv2.moments of each
    object's mask; perimeter as a numpy count of 4-neighbour edges."""
    _, out = stage1k
    labels, f, n = out["labels"], out["features"], out["n"]
    _, lab_cv, stats, cent = cv2.connectedComponentsWithStats(
        (labels > 0).astype(np.uint8), connectivity=8, ltype=cv2.CV_32S)
    canon = _canon(lab_cv)
    # map cv2 ids onto canonical ids
    m = np.zeros(n + 1, np.int64)
    m[canon.reshape(-1)] = lab_cv.reshape(-1)
    st, ce = stats[m[1:]], cent[m[1:]]
    rt = dict(rtol=1e-5, atol=1e-6)
    np.testing.assert_allclose(f[:, 0], st[:, cv2.CC_STAT_AREA], **rt)
    np.testing.assert_allclose(f[:, 2], st[:, cv2.CC_STAT_TOP], **rt)
    np.testing.assert_allclose(f[:, 3], st[:, cv2.CC_STAT_LEFT], **rt)
    np.testing.assert_allclose(f[:, 4], st[:, cv2.CC_STAT_TOP] + st[:, cv2.CC_STAT_HEIGHT] - 1, **rt)
    np.testing.assert_allclose(f[:, 5], st[:, cv2.CC_STAT_LEFT] + st[:, cv2.CC_STAT_WIDTH] - 1, **rt)
    np.testing.assert_allclose(f[:, 6], ce[:, 1], **rt)
    np.testing.assert_allclose(f[:, 7], ce[:, 0], **rt)
    pad = np.pad(labels, 1)
    checked = 0
    for k in range(1, n + 1):
        y0, x0, y1, x1 = (int(v) for v in f[k - 1, 2:6])
        obj = (labels[y0:y1 + 1, x0:x1 + 1] == k).astype(np.uint8)
        mo = cv2.moments(obj, binaryImage=True)
        a = mo["m00"]
        mxx = mo["mu20"] / a + 1.0 / 12.0
        myy = mo["mu02"] / a + 1.0 / 12.0
        mxy = mo["mu11"] / a
        root = np.sqrt(0.25 * (mxx - myy) ** 2 + mxy ** 2)
        l1, l2 = 0.5 * (mxx + myy) + root, max(0.5 * (mxx + myy) - root, 0.0)
        exp = [4 * np.sqrt(l1), 4 * np.sqrt(l2), np.sqrt(1 - l2 / l1)]
        np.testing.assert_allclose(f[k - 1, 14:17], exp, rtol=1e-5, atol=2e-5)
        if l1 - l2 > 1e-4 * l1:  # orientation is undefined for isotropic objects
            # an axis angle: equal modulo pi (+pi/2 and -pi/2 are one axis)
            d = f[k - 1, 17] - 0.5 * np.arctan2(2 * mxy, mxx - myy)
            assert abs((d + np.pi / 2) % np.pi - np.pi / 2) <= 2e-5, (k, d)
        sub = pad[y0:y1 + 3, x0:x1 + 3] == k
        perim = sum(int((sub & ~np.roll(sub, s, axis=ax)).sum()) for ax in (0, 1) for s in (1, -1))
        assert f[k - 1, 1] == perim
        np.testing.assert_allclose(f[k - 1, 18], 4 * np.pi * a / perim ** 2, rtol=1e-5)
        np.testing.assert_allclose(f[k - 1, 19], a / ((y1 - y0 + 1) * (x1 - x0 + 1)), rtol=1e-5)
        checked += 1
    assert checked == n and n > 100


def test_intensity_and_gradient_vs_scipy(stage1k, oracle):
    """Mean / std / min / max of the hematoxylin plane and of the Sobel
    magnitude floor(4|g|)/4 (replicated border) per object, from
    scipy.ndimage.sobel and scipy.ndimage's labelled statistics."""
    rgb, out = stage1k
    hema = out["hema"].astype(np.float64)
    labels, f, n = out["labels"], out["features"], out["n"]
    idx = np.arange(1, n + 1)
    rt = dict(rtol=1e-5, atol=1e-5)
    np.testing.assert_allclose(f[:, 8], ndi.mean(hema, labels, idx), **rt)
    np.testing.assert_allclose(f[:, 9], ndi.standard_deviation(hema, labels, idx), rtol=1e-4, atol=1e-4)
    np.testing.assert_allclose(f[:, 10], ndi.minimum(hema, labels, idx), **rt)
    np.testing.assert_allclose(f[:, 11], ndi.maximum(hema, labels, idx), **rt)
    gx = ndi.sobel(hema, axis=1, mode="nearest")
    gy = ndi.sobel(hema, axis=0, mode="nearest")
    g = np.floor(4.0 * np.sqrt(gx * gx + gy * gy)) / 4.0
    np.testing.assert_allclose(f[:, 12], ndi.mean(g, labels, idx), **rt)
    np.testing.assert_allclose(f[:, 13], ndi.standard_deviation(g, labels, idx), rtol=1e-4, atol=1e-4)


def _meyer_flood(f, markers, mask):
    """Meyer's priority-flood watershed (highest f first, FIFO among equal f):
    a different algorithm from the oracle's steepest-ascent arrowing."""
    h, w = f.shape
    lab = markers.astype(np.int64).copy()
    queued = markers > 0
    heap, cnt = [], 0
    nb = [(-1, -1), (-1, 0), (-1, 1), (0, -1), (0, 1), (1, -1), (1, 0), (1, 1)]

    def push_neighbours(y, x):
        nonlocal cnt
        for dy, dx in nb:
            yy, xx = y + dy, x + dx
            if 0 <= yy < h and 0 <= xx < w and mask[yy, xx] and not queued[yy, xx]:
                queued[yy, xx] = True
                heapq.heappush(heap, (-int(f[yy, xx]), cnt, yy, xx))
                cnt += 1

    for y, x in zip(*np.nonzero(markers)):
        push_neighbours(y, x)
    while heap:
        _, _, y, x = heapq.heappop(heap)
        best = None
        for dy, dx in nb:
            yy, xx = y + dy, x + dx
            if 0 <= yy < h and 0 <= xx < w and lab[yy, xx] > 0 and (
                    best is None or f[yy, xx] > f[best]):
                best = (yy, xx)
        lab[y, x] = lab[best]
        push_neighbours(y, x)
    return lab


def _separate(basin, mask):
    h, w = basin.shape
    out = mask.copy()
    pad = np.pad(basin, 1)
    for dy in (-1, 0, 1):
        for dx in (-1, 0, 1):
            out[pad[1 + dy:1 + dy + h, 1 + dx:1 + dx + w] > basin] = 0
    return out


def _dense_touching_mask(rng, h, w, fg=0.35):
    """Clusters of overlapping discs (radius 4-8): ~fg foreground, most
    nuclei touching a neighbour (the C3 workload)."""
    m = np.zeros((h, w), np.uint8)
    yy, xx = np.mgrid[-9:10, -9:10]
    while m.mean() < fg:
        cy, cx = rng.integers(10, h - 10), rng.integers(10, w - 10)
        for _ in range(rng.integers(2, 5)):
            r = rng.integers(4, 9)
            oy, ox = cy + rng.integers(-r, r + 1), cx + rng.integers(-r, r + 1)
            if 9 <= oy < h - 9 and 9 <= ox < w - 9:
                m[oy - 9:oy + 10, ox - 9:ox + 10] |= (yy * yy + xx * xx <= r * r).astype(np.uint8)
    return m


@pytest.mark.parametrize("case", ["tile", "dense"])
def test_watershed_vs_meyer_flooding(oracle, case):
    """Same function Fw and markers, different flooding rule: the basins and
    the separated masks agree on >= 99.5 % of the foreground and give the
    same object count."""
    if case == "tile":
        _, out = _stage(oracle, 3, 5, 512, 512)
        mask = out["area"]
    else:
        mask = _dense_touching_mask(np.random.default_rng(7), 384, 384)
    p = oracle.default_params()
    sep, basin, pl = oracle.watershed(mask, p.ws_h, want_planes=True)
    fw = pl["fw"].astype(np.int64)
    markers = np.where(pl["rmax"] > 0, basin, 0)
    lab = _meyer_flood(fw, markers, mask > 0)
    fg = mask > 0
    assert (lab[fg] == basin[fg]).mean() >= 0.995
    s2 = _separate(lab, mask)
    assert (s2 == sep).mean() >= 0.999
    n_ours = ndi.label(sep, np.ones((3, 3)))[1]
    n_meyer = ndi.label(s2, np.ones((3, 3)))[1]
    assert abs(n_ours - n_meyer) <= max(1, n_ours // 200), (n_ours, n_meyer)
