"""Generates the golden vectors that pin the CPU oracle (tests/golden/*.npz).

The reference (/root/reference) has no image-analysis code, so
the oracle is pinned against INDEPENDENT implementations available in this
container, never against itself:
  - scipy.ndimage 1.18.1: grey_dilation (iterated to convergence = morphological
    reconstruction), binary_fill_holes, label, distance_transform_edt;
  - OpenCV 4.13: connectedComponents (4-conn cross-check of scipy);
  - numpy restatements (written here, not sharing code with oracle/) of the
    colour-deconvolution LUT arithmetic, the per-object features and the
    arrowing watershed spec of DESIGN.md §3.
Run:  python tests/golden/make_golden.py   (writes next to this file)
The inputs are stored inside each .npz so the tests need neither this script
nor the generator library.
"""
from __future__ import annotations

import math
import os
import sys
from collections import deque

import numpy as np
from scipy import ndimage as ndi

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))

FP8 = np.ones((3, 3), bool)
FP4 = ndi.generate_binary_structure(2, 1)

# same numbers as rtg_params_default (include/rtg.h docs)
PARAMS = dict(h_coef=(1.874787447891341, -0.06579592311838535, -0.6008832496835673),
              h_scale=1.25, bg_thresh=215, rbc_rg10=25, rbc_rb10=22, recon_h=24,
              recon_conn=8, nuc_thresh=70, min_area=24, max_area=2500, ws_h=3)


# ------------------------------------------------------------------ restatements

def colordeconv(rgb, p=PARAMS):
    """LUT colour deconvolution (DESIGN.md §3 o1/o2) restated with numpy."""
    v = np.arange(256, dtype=np.float64)
    od = -np.log10((v + 1.0) / 256.0)
    scale255 = 255.0 / p["h_scale"]
    luts = [np.array([int(round_half_away(c * o * scale255 * 65536.0)) for o in od], np.int64)
            for c in p["h_coef"]]
    r = rgb[..., 0].astype(np.int64)
    g = rgb[..., 1].astype(np.int64)
    b = rgb[..., 2].astype(np.int64)
    s = luts[0][r] + luts[1][g] + luts[2][b]
    hv = np.where(s > 0, np.minimum((s + 32768) >> 16, 255), 0).astype(np.uint8)
    marker = np.where(hv > p["recon_h"], hv.astype(np.int32) - p["recon_h"], 0).astype(np.uint8)
    t = p["bg_thresh"]
    bg = (r > t) & (g > t) & (b > t)
    rbc = (10 * r > p["rbc_rg10"] * g) & (10 * r > p["rbc_rb10"] * b)
    tissue = (~bg & ~rbc).astype(np.uint8)
    return hv, marker, tissue


def round_half_away(x):
    # C llround semantics
    return math.floor(x + 0.5) if x >= 0 else -math.floor(-x + 0.5)


def recon(marker, mask, conn):
    """Reconstruction by dilation: iterate min(dilate(J), mask) to stability."""
    fp = FP8 if conn == 8 else FP4
    J = np.minimum(marker, mask).astype(np.int64)
    M = mask.astype(np.int64)
    while True:
        nJ = np.minimum(ndi.grey_dilation(J, footprint=fp, mode="constant", cval=0), M)
        if np.array_equal(nJ, J):
            return J.astype(mask.dtype)
        J = nJ


def fill_holes(m):
    return ndi.binary_fill_holes(m.astype(bool)).astype(np.uint8)


def label(m, conn):
    lab, n = ndi.label(m.astype(bool), structure=FP8 if conn == 8 else FP4)
    return lab.astype(np.int32), int(n)


def area_threshold(m, conn, lo, hi):
    lab, n = label(m, conn)
    cnt = np.bincount(lab.ravel(), minlength=n + 1)
    keep = (cnt >= lo) & (cnt <= hi)
    keep[0] = False
    return keep[lab].astype(np.uint8)


def edt_sq(m):
    if not (m == 0).any():
        return np.full(m.shape, np.iinfo(np.int32).max, np.int32)
    d = ndi.distance_transform_edt(m.astype(bool))
    return np.rint(d * d).astype(np.int32)


def watershed(m, ws_h):
    """Arrowing watershed (DESIGN.md §3 o6/o7), restated with plain loops."""
    h, w = m.shape
    d2 = edt_sq(m).astype(np.int64)
    dq = np.empty((h, w), np.int64)
    for i, v in np.ndenumerate(d2):
        q = 65535 if v >= np.iinfo(np.int32).max else math.isqrt(16 * int(v))
        dq[i] = min(q, 65534)
    mk = np.where(dq > ws_h, dq - ws_h, 0)
    F = recon(mk.astype(np.uint16), dq.astype(np.uint16), 8).astype(np.int64)
    Fw = np.where(m > 0, F + 1, 0)
    G = recon(np.where(Fw > 0, Fw - 1, 0).astype(np.uint16), Fw.astype(np.uint16), 8).astype(np.int64)
    rm = (Fw > G) & (m > 0)
    mlab, _ = label(rm.astype(np.uint8), 8)
    first = {}
    for idx in range(h * w):
        l = mlab.flat[idx]
        if l and l not in first:
            first[l] = idx
    nb = [(-1, -1), (-1, 0), (-1, 1), (0, -1), (0, 1), (1, -1), (1, 0), (1, 1)]
    ptr = -np.ones(h * w, np.int64)
    delta = -np.ones(h * w, np.int64)
    q = deque()
    for y in range(h):
        for x in range(w):
            i = y * w + x
            if Fw[y, x] == 0:
                continue
            if rm[y, x]:
                ptr[i] = i
                continue
            best, arg = Fw[y, x], -1
            for dy, dx in nb:
                yy, xx = y + dy, x + dx
                if 0 <= yy < h and 0 <= xx < w and Fw[yy, xx] > best:
                    best, arg = Fw[yy, xx], yy * w + xx
            if arg >= 0:
                ptr[i] = arg
                delta[i] = 0
                q.append(i)
    while q:
        i = q.popleft()
        y, x = divmod(i, w)
        for dy, dx in nb:
            yy, xx = y + dy, x + dx
            if 0 <= yy < h and 0 <= xx < w:
                j = yy * w + xx
                if Fw[yy, xx] == Fw[y, x] and not rm[yy, xx] and delta[j] < 0:
                    delta[j] = delta[i] + 1
                    q.append(j)
    for i in range(h * w):
        y, x = divmod(i, w)
        if Fw[y, x] == 0 or rm[y, x] or delta[i] <= 0:
            continue
        cands = [yy * w + xx for dy, dx in nb
                 for yy, xx in [(y + dy, x + dx)]
                 if 0 <= yy < h and 0 <= xx < w and Fw[yy, xx] == Fw[y, x]
                 and not rm[yy, xx] and delta[yy * w + xx] == delta[i] - 1]
        ptr[i] = min(cands) if cands else -1
    basin = np.zeros(h * w, np.int64)
    for i in range(h * w):
        if Fw.flat[i] == 0:
            continue
        j, steps = i, 0
        while ptr[j] >= 0 and ptr[j] != j and steps < h * w:
            j, steps = ptr[j], steps + 1
        basin[i] = first[mlab.flat[j]] + 1 if ptr[j] == j else 0
    basin = basin.reshape(h, w)
    sep = np.zeros((h, w), np.uint8)
    for y in range(h):
        for x in range(w):
            b = basin[y, x]
            if b <= 0:
                continue
            nbr = basin[max(y - 1, 0):y + 2, max(x - 1, 0):x + 2]
            sep[y, x] = 0 if (nbr > b).any() else 1
    return sep, basin.astype(np.int32)


def features(labels, I, n):
    """Per-object features (DESIGN.md §3 o9) restated with numpy."""
    h, w = labels.shape
    Ii = I.astype(np.int64)
    P = np.pad(Ii, 1, mode="edge")
    gx = (P[:-2, 2:] + 2 * P[1:-1, 2:] + P[2:, 2:]) - (P[:-2, :-2] + 2 * P[1:-1, :-2] + P[2:, :-2])
    gy = (P[2:, :-2] + 2 * P[2:, 1:-1] + P[2:, 2:]) - (P[:-2, :-2] + 2 * P[:-2, 1:-1] + P[:-2, 2:])
    gq = np.vectorize(math.isqrt)(16 * (gx * gx + gy * gy)).astype(np.int64)
    L = np.pad(labels, 1, constant_values=-1)
    out = np.zeros((n, 20), np.float32)
    ys, xs = np.mgrid[0:h, 0:w]
    for l in range(1, n + 1):
        sel = labels == l
        A = int(sel.sum())
        if A == 0:
            continue
        y = ys[sel].astype(np.int64)
        x = xs[sel].astype(np.int64)
        v = Ii[sel]
        g = gq[sel]
        core = L[1:-1, 1:-1] == l
        per = int((core & (L[:-2, 1:-1] != l)).sum() + (core & (L[2:, 1:-1] != l)).sum()
                  + (core & (L[1:-1, :-2] != l)).sum() + (core & (L[1:-1, 2:] != l)).sum())
        Af = float(A)
        cy, cx = float(y.sum()) / Af, float(x.sum()) / Af
        mi = float(v.sum()) / Af
        vi = float((v * v).sum()) / Af - mi * mi
        mg = float(g.sum()) / (4.0 * Af)
        vg = float((g * g).sum()) / (16.0 * Af) - mg * mg
        mxx = float((x * x).sum()) / Af - cx * cx + 1.0 / 12.0
        myy = float((y * y).sum()) / Af - cy * cy + 1.0 / 12.0
        mxy = float((x * y).sum()) / Af - cx * cy
        half, dd = 0.5 * (mxx + myy), 0.5 * (mxx - myy)
        root = math.sqrt(dd * dd + mxy * mxy)
        l1, l2 = half + root, max(half - root, 0.0)
        y0, y1, x0, x1 = int(y.min()), int(y.max()), int(x.min()), int(x.max())
        out[l - 1] = [Af, per, y0, x0, y1, x1, cy, cx, mi, math.sqrt(max(vi, 0.0)),
                      int(v.min()), int(v.max()), mg, math.sqrt(max(vg, 0.0)),
                      4.0 * math.sqrt(l1), 4.0 * math.sqrt(l2),
                      math.sqrt(1.0 - l2 / l1) if l1 > 0 else 0.0,
                      0.5 * math.atan2(2.0 * mxy, mxx - myy),
                      4.0 * math.pi * Af / (per * per),
                      Af / ((y1 - y0 + 1) * (x1 - x0 + 1))]
    return out


def pipeline(rgb, p=PARAMS):
    hema, marker, tissue = colordeconv(rgb, p)
    rec = recon(marker, hema, p["recon_conn"])
    m1 = ((rec >= p["nuc_thresh"]) & (tissue > 0)).astype(np.uint8)
    m2 = fill_holes(m1)
    m3 = area_threshold(m2, 8, p["min_area"], p["max_area"])
    sep, basin = watershed(m3, p["ws_h"])
    lab, n = label(sep, 8)
    return dict(hema=hema, recon=rec, cand=m1, filled=m2, area=m3, sep=sep, basin=basin,
                labels=lab, n=n, features=features(lab, hema, n))


# ------------------------------------------------------------------ cases

def blobs(rng, h, w, density, smooth):
    f = ndi.gaussian_filter(rng.random((h, w)), smooth)
    return (f > np.quantile(f, 1 - density)).astype(np.uint8)


def main():
    rng = np.random.default_rng(1405)
    out = {}
    # o1/o2
    rgb = rng.integers(0, 256, (37, 53, 3), dtype=np.uint8)
    out["cd"] = dict(rgb=rgb, **dict(zip(("hema", "marker", "tissue"), colordeconv(rgb))))
    # o3 reconstruction, 4/8-connectivity, incl. degenerate shapes
    for k, (h, w) in enumerate([(24, 37), (50, 50), (1, 40), (40, 1)]):
        mask = rng.integers(0, 256, (h, w), dtype=np.uint8)
        marker = (mask * (rng.random((h, w)) < 0.05)).astype(np.uint8)
        for conn in (4, 8):
            out[f"recon{k}_{conn}"] = dict(marker=marker, mask=mask, conn=np.int32(conn),
                                           out=recon(marker, mask, conn))
    # o4 fill holes: random blobs + hole touching the border + nested holes
    fh = [1 - blobs(rng, 60, 70, 0.5, 1.3)]
    ring = np.zeros((20, 20), np.uint8)
    ring[2:18, 2:18] = 1
    ring[5:15, 5:15] = 0
    ring[8:12, 8:12] = 1
    ring[0:10, 9] = 0  # hole opened to the border
    fh.append(ring)
    for k, m in enumerate(fh):
        out[f"fill{k}"] = dict(m=m, out=fill_holes(m))
    # o8 labels (cross-checked against OpenCV for 4-conn)
    import cv2
    for k, (h, w) in enumerate([(64, 80), (1, 50), (33, 1)]):
        m = blobs(rng, h, w, 0.35, 1.0) if min(h, w) > 1 else (rng.random((h, w)) < 0.5).astype(np.uint8)
        for conn in (4, 8):
            lab, n = label(m, conn)
            if conn == 4 and min(h, w) > 1:
                n_cv, lab_cv = cv2.connectedComponents(m, connectivity=4, ltype=cv2.CV_32S)
                assert n_cv - 1 == n and np.array_equal(lab_cv, lab)
            out[f"label{k}_{conn}"] = dict(m=m, conn=np.int32(conn), labels=lab, n=np.int32(n))
    # o5 area threshold
    m = blobs(rng, 90, 100, 0.3, 1.0)
    for conn in (4, 8):
        out[f"area_{conn}"] = dict(m=m, conn=np.int32(conn), lo=np.int32(5), hi=np.int32(60),
                                   out=area_threshold(m, conn, 5, 60))
    # o6 EDT
    for k, m in enumerate([blobs(rng, 70, 90, 0.6, 2.0), np.ones((9, 9), np.uint8),
                           (rng.random((40, 40)) > 0.01).astype(np.uint8)]):
        out[f"edt{k}"] = dict(m=m, d2=edt_sq(m))
    # o6/o7 watershed
    for k, ws_h in enumerate([0, 3]):
        m = blobs(rng, 48, 56, 0.45, 2.2)
        sep, basin = watershed(m, ws_h)
        out[f"ws{k}"] = dict(m=m, ws_h=np.int32(ws_h), sep=sep, basin=basin)
    # o9 features on scipy labels
    m = blobs(rng, 64, 64, 0.35, 1.5)
    lab, n = label(m, 8)
    I = rng.integers(0, 256, (64, 64), dtype=np.uint8)
    out["feat"] = dict(labels=lab, I=I, n=np.int32(n), features=features(lab, I, n))
    # whole stage on a synthetic tile crop (generator from the built library)
    sys.path.insert(0, ROOT)
    from paper_1405_7958_b200 import rtg
    tile = rtg.synth_tile_host(0, 0, 160, 176)
    pl = pipeline(tile)
    out["stage"] = dict(rgb=tile, **{k: (np.int32(v) if k == "n" else v) for k, v in pl.items()})

    for name, arrs in out.items():
        np.savez_compressed(os.path.join(HERE, f"{name}.npz"), **arrs)
    print(f"wrote {len(out)} golden files to {HERE}")


if __name__ == "__main__":
    main()
