"""Pins the CPU oracle against the golden vectors made by independent
implementations (scipy.ndimage / OpenCV / numpy restatements; generator:
tests/golden/make_golden.py).  CPU only."""
import glob
import os

import numpy as np
import pytest

GOLDEN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")


def g(name):
    return np.load(os.path.join(GOLDEN, name + ".npz"))


def names(prefix):
    return sorted(os.path.basename(p)[:-4] for p in glob.glob(os.path.join(GOLDEN, prefix + "*.npz")))


def test_golden_present():
    assert len(glob.glob(os.path.join(GOLDEN, "*.npz"))) >= 20


def test_params_default_match_product(oracle, rtg):
    a, b = oracle.default_params().as_dict(), rtg.default_params().as_dict()
    assert a == b


def test_colordeconv(oracle):
    d = g("cd")
    hema, marker, tissue = oracle.colordeconv(d["rgb"], oracle.default_params())
    assert np.array_equal(hema, d["hema"])
    assert np.array_equal(marker, d["marker"])
    assert np.array_equal(tissue, d["tissue"])


@pytest.mark.parametrize("name", names("recon"))
def test_recon(oracle, name):
    d = g(name)
    assert np.array_equal(oracle.recon(d["marker"], d["mask"], int(d["conn"])), d["out"])


@pytest.mark.parametrize("name", names("fill"))
def test_fill_holes(oracle, name):
    d = g(name)
    assert np.array_equal(oracle.fill_holes(d["m"]), d["out"])


@pytest.mark.parametrize("name", names("label"))
def test_bwlabel(oracle, name):
    d = g(name)
    lab, n = oracle.bwlabel(d["m"], int(d["conn"]))
    assert n == int(d["n"])
    assert np.array_equal(lab, d["labels"])


@pytest.mark.parametrize("name", names("area"))
def test_area_threshold(oracle, name):
    d = g(name)
    out = oracle.area_threshold(d["m"], int(d["conn"]), int(d["lo"]), int(d["hi"]))
    assert np.array_equal(out, d["out"])


@pytest.mark.parametrize("name", names("edt"))
def test_edt(oracle, name):
    d = g(name)
    assert np.array_equal(oracle.edt_sq(d["m"]), d["d2"])


@pytest.mark.parametrize("name", names("ws"))
def test_watershed(oracle, name):
    d = g(name)
    sep, basin = oracle.watershed(d["m"], int(d["ws_h"]))
    assert np.array_equal(basin, d["basin"])
    assert np.array_equal(sep, d["sep"])


def test_features(oracle):
    d = g("feat")
    out = oracle.features(d["labels"], d["I"], int(d["n"]))
    np.testing.assert_allclose(out, d["features"], rtol=1e-5, atol=1e-6)


def test_stage(oracle):
    d = g("stage")
    r = oracle.process_tile(d["rgb"], want_planes=True)
    for k in ("hema", "recon", "cand", "filled", "area", "sep", "basin", "labels"):
        assert np.array_equal(r[k], d[k]), k
    assert r["n"] == int(d["n"])
    np.testing.assert_allclose(r["features"], d["features"], rtol=1e-5, atol=1e-6)


def test_recon_properties(oracle):
    """Idempotence and monotonicity (hypothesis-style seeded sweep)."""
    rng = np.random.default_rng(5)
    for _ in range(20):
        h, w = rng.integers(1, 40, 2)
        mask = rng.integers(0, 256, (h, w), dtype=np.uint8)
        marker = (mask * (rng.random((h, w)) < 0.1)).astype(np.uint8)
        r = oracle.recon(marker, mask, 8)
        assert (r <= mask).all() and (r >= np.minimum(marker, mask)).all()
        assert np.array_equal(oracle.recon(r, mask, 8), r)
        # 8-connectivity reconstruction dominates 4-connectivity
        assert (oracle.recon(marker, mask, 4) <= r).all()


@pytest.mark.parametrize("conn", [4, 8])
def test_threshold_decomposition_of_recon(oracle, conn):
    """The identity the GPU stage's default ReconToNuclei path relies on:
    recon(max(H-h,0), H) >= t  <=>  the pixel's conn-component of {H >= t}
    holds a pixel with H >= t + h (flat connectivity commutes with
    thresholding).  Checked against the oracle's grayscale reconstruction."""
    from scipy import ndimage as ndi
    rng = np.random.default_rng(77 + conn)
    st = np.ones((3, 3), bool) if conn == 8 else ndi.generate_binary_structure(2, 1)
    for trial in range(12):
        hh, ww = rng.integers(8, 90, 2)
        H = ndi.gaussian_filter(rng.integers(0, 256, (hh, ww)).astype(float), 1.2).astype(np.uint8)
        hd = int(rng.integers(0, 40))
        marker = np.maximum(H.astype(int) - hd, 0).astype(np.uint8)
        R = oracle.recon(marker, H, conn)
        for t in (1, 30, 70, 120, 200):
            lab, _ = ndi.label(H >= t, structure=st)
            seeded = np.unique(lab[(H.astype(int) >= t + hd) & (lab > 0)])
            got = np.isin(lab, seeded) & (lab > 0)
            assert np.array_equal(R >= t, got), (trial, t)


def test_watershed_properties(oracle):
    """Every basin carries exactly one marker id, basins stay inside the mask,
    and the separated mask has no 8-adjacent pixels of different basins."""
    from scipy import ndimage as ndi
    rng = np.random.default_rng(9)
    f = ndi.gaussian_filter(rng.random((96, 96)), 2.5)
    m = (f > np.quantile(f, 0.6)).astype(np.uint8)
    sep, basin = oracle.watershed(m, 3)
    assert ((basin > 0) == (m > 0)).all()
    assert (sep <= m).all()
    lab, n = oracle.bwlabel(sep, 8)
    for l in range(1, n + 1):
        assert len(np.unique(basin[lab == l])) == 1



def test_texture_known_answer(oracle):
    """f4 texture row of a hand-checked 2x2 object with grey levels 0, 1, 2, 3
    (intensities 0, 32, 64, 96): 6 co-occurrence pairs (T = 12 symmetric
    counts), uniform 4-bin histogram."""
    lab = np.zeros((4, 4), np.int32)
    lab[1:3, 1:3] = 1
    inten = np.zeros((4, 4), np.uint8)
    inten[1, 1], inten[1, 2], inten[2, 1], inten[2, 2] = 0, 32, 64, 96
    t = oracle.texture(lab, inten, 1)[0]
    np.testing.assert_allclose(t[0], 2.0)            # histogram entropy (4 equal bins)
    np.testing.assert_allclose(t[1], 0.25)           # histogram energy
    np.testing.assert_allclose(t[2], 0.0, atol=1e-7)  # skewness
    np.testing.assert_allclose(t[3], -1.36, rtol=1e-6)  # excess kurtosis of 4 equispaced values
    np.testing.assert_allclose(t[4], 1 / 12, rtol=1e-6)  # ASM: 12 cells of 1/12
    np.testing.assert_allclose(t[5], 40 / 12, rtol=1e-6)  # contrast: 2*(1+1+4+4+9+1)/12
    np.testing.assert_allclose(t[6], 4 / 12, rtol=1e-6)   # homogeneity
    np.testing.assert_allclose(t[7], np.log2(12), rtol=1e-6)  # GLCM entropy
    np.testing.assert_allclose(t[9], 20 / 12, rtol=1e-6)  # dissimilarity
    np.testing.assert_allclose(t[10], 1 / 12, rtol=1e-6)  # max probability
