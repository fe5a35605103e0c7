"""ctypes wrapper of the CPU oracle (liboracle.so).

TEST INFRASTRUCTURE ONLY: importable from tests/, __graft_entry__.smoke() and
bench.py's cpu_baseline / --impl reference legs, never from the product path
(see rtg_oracle.h).
"""
from __future__ import annotations

import ctypes
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "liboracle.so")
NATIVE_PATH = os.path.join(_HERE, "_native", "liboracle.so")
NUM_FEATURES = 20
DEFAULT_SEED = 1405795800
_lib = None


def build() -> None:
    subprocess.run(["make", "-C", _HERE, "-s"], check=True)


def build_native() -> str:
    """-O3 -march=native build for the host that times it.
    Always rebuilt: a copy made on another machine may use instructions this
    CPU lacks."""
    subprocess.run(["make", "-C", _HERE, "-s", "-B", "native"], check=True,
                   stdout=subprocess.DEVNULL)
    return NATIVE_PATH


def load(native: bool = False) -> ctypes.CDLL:
    """The portable build, or (native=True, before any other load) the
    -march=native build of this host."""
    global _lib
    if _lib is not None:
        return _lib
    if native:
        path = build_native()
    else:
        path = LIB_PATH
        if not os.path.exists(path):
            build()
    lib = ctypes.CDLL(path)
    vp, i64, i32 = ctypes.c_void_p, ctypes.c_int64, ctypes.c_int32
    sigs = {
        "orc_params_default": ([vp], None),
        "orc_colordeconv": ([vp, i64, i64, i64, vp, vp, vp, vp], None),
        "orc_recon_u8": ([vp, vp, i64, i64, ctypes.c_int, vp], None),
        "orc_recon_u16": ([vp, vp, i64, i64, ctypes.c_int, vp], None),
        "orc_fill_holes": ([vp, i64, i64, vp], None),
        "orc_bwlabel": ([vp, i64, i64, ctypes.c_int, vp], i32),
        "orc_area_threshold": ([vp, i64, i64, ctypes.c_int, i32, i32, vp], None),
        "orc_edt_sq": ([vp, i64, i64, vp], None),
        "orc_watershed": ([vp, i64, i64, i32, vp, vp, vp], None),
        "orc_features": ([vp, vp, i64, i64, i32, vp], None),
        "orc_texture": ([vp, vp, i64, i64, i32, vp], None),
        "orc_texture_row": ([vp, vp, vp, ctypes.c_uint32, vp], None),
        "orc_canny": ([vp, i64, i64, i32, i32, vp], None),
        "orc_process_tile": ([vp, i64, i64, i64, vp, vp, vp, vp, i32, vp], i32),
        "orc_synth_tile_host": ([ctypes.c_uint64, i64, i64, i64, i64, vp], ctypes.c_int),
    }
    for name, (args, res) in sigs.items():
        fn = getattr(lib, name)
        fn.argtypes = args
        fn.restype = res
    _lib = lib
    return lib


def _p(a):
    return None if a is None else a.ctypes.data


class Planes(ctypes.Structure):
    _fields_ = [(n, ctypes.c_void_p) for n in
                "hema marker tissue recon cand filled area dist2 dq fw rmax basin sep".split()]


PLANE_DTYPES = {
    "hema": np.uint8, "marker": np.uint8, "tissue": np.uint8, "recon": np.uint8,
    "cand": np.uint8, "filled": np.uint8, "area": np.uint8, "dist2": np.int32,
    "dq": np.uint16, "fw": np.uint16, "rmax": np.uint8, "basin": np.int32, "sep": np.uint8,
}


class Params(ctypes.Structure):
    """rtg_params (include/rtg.h): the oracle and the product consume the same
    struct layout; declared here so the oracle never imports the product."""
    _fields_ = [
        ("h_coef", ctypes.c_double * 3),
        ("h_scale", ctypes.c_double),
        ("bg_thresh", ctypes.c_int32),
        ("rbc_rg10", ctypes.c_int32),
        ("rbc_rb10", ctypes.c_int32),
        ("recon_h", ctypes.c_int32),
        ("recon_conn", ctypes.c_int32),
        ("nuc_thresh", ctypes.c_int32),
        ("min_area", ctypes.c_int32),
        ("max_area", ctypes.c_int32),
        ("ws_h", ctypes.c_int32),
        ("texture", ctypes.c_int32),
        ("reserved", ctypes.c_int32 * 6),
    ]

    def as_dict(self) -> dict:
        return {name: (list(getattr(self, name)) if name == "h_coef" else getattr(self, name))
                for name, _ in self._fields_ if name != "reserved"}


def default_params():
    p = Params()
    load().orc_params_default(ctypes.byref(p))
    return p


def synth_tile_host(tile_row=0, tile_col=0, h=4096, w=4096, seed=DEFAULT_SEED):
    """The synthetic H&E tile (same generator source as the product's, compiled
    into the oracle), so the CPU arms never load librtg.so."""
    out = np.empty((h, w, 3), np.uint8)
    rc = load().orc_synth_tile_host(seed, tile_row, tile_col, h, w, out.ctypes.data)
    if rc != 0:
        raise RuntimeError(f"orc_synth_tile_host failed ({rc})")
    return out


def colordeconv(rgb, params):
    h, w, _ = rgb.shape
    rgb = np.ascontiguousarray(rgb)
    hema = np.empty((h, w), np.uint8)
    marker = np.empty((h, w), np.uint8)
    tissue = np.empty((h, w), np.uint8)
    load().orc_colordeconv(_p(rgb), h, w, 3 * w, ctypes.byref(params), _p(hema), _p(marker),
                           _p(tissue))
    return hema, marker, tissue


def recon(marker, mask, conn=8):
    h, w = mask.shape
    out = np.empty_like(mask)
    fn = load().orc_recon_u8 if mask.dtype == np.uint8 else load().orc_recon_u16
    fn(_p(np.ascontiguousarray(marker)), _p(np.ascontiguousarray(mask)), h, w, conn, _p(out))
    return out


def fill_holes(m):
    h, w = m.shape
    out = np.empty((h, w), np.uint8)
    load().orc_fill_holes(_p(np.ascontiguousarray(m, np.uint8)), h, w, _p(out))
    return out


def bwlabel(m, conn=8):
    h, w = m.shape
    lab = np.empty((h, w), np.int32)
    n = load().orc_bwlabel(_p(np.ascontiguousarray(m, np.uint8)), h, w, conn, _p(lab))
    return lab, n


def area_threshold(m, conn, lo, hi):
    h, w = m.shape
    out = np.empty((h, w), np.uint8)
    load().orc_area_threshold(_p(np.ascontiguousarray(m, np.uint8)), h, w, conn, lo, hi, _p(out))
    return out


def edt_sq(m):
    h, w = m.shape
    out = np.empty((h, w), np.int32)
    load().orc_edt_sq(_p(np.ascontiguousarray(m, np.uint8)), h, w, _p(out))
    return out


def watershed(m, ws_h, want_planes=False):
    h, w = m.shape
    sep = np.empty((h, w), np.uint8)
    basin = np.empty((h, w), np.int32)
    planes = None
    arrs = {}
    if want_planes:
        arrs = {k: np.zeros((h, w), PLANE_DTYPES[k]) for k in ("dist2", "dq", "fw", "rmax")}
        planes = Planes(**{k: v.ctypes.data for k, v in arrs.items()})
    load().orc_watershed(_p(np.ascontiguousarray(m, np.uint8)), h, w, ws_h, _p(sep), _p(basin),
                         ctypes.byref(planes) if planes is not None else None)
    if want_planes:
        return sep, basin, arrs
    return sep, basin


def features(labels, intensity, n):
    h, w = labels.shape
    out = np.zeros((max(n, 1), NUM_FEATURES), np.float32)
    load().orc_features(_p(np.ascontiguousarray(labels, np.int32)),
                        _p(np.ascontiguousarray(intensity, np.uint8)), h, w, n, _p(out))
    return out[:n]


NUM_TEXTURE = 14


def texture(labels, intensity, n):
    """f4 texture table (n x 12), rtg.h enum rtg_texture_feature."""
    h, w = labels.shape
    out = np.zeros((max(n, 1), NUM_TEXTURE), np.float32)
    load().orc_texture(_p(np.ascontiguousarray(labels, np.int32)),
                       _p(np.ascontiguousarray(intensity, np.uint8)), h, w, n, _p(out))
    return out[:n]


def texture_row(hist, glcm, mom, edge_px=0):
    out = np.zeros(NUM_TEXTURE, np.float32)
    load().orc_texture_row(_p(np.ascontiguousarray(hist, np.uint32)),
                           _p(np.ascontiguousarray(glcm, np.uint32)),
                           _p(np.ascontiguousarray(mom, np.int64)), edge_px, _p(out))
    return out


CANNY_LOW, CANNY_HIGH = 64, 128


def canny(intensity, low=CANNY_LOW, high=CANNY_HIGH):
    h, w = intensity.shape
    out = np.zeros((h, w), np.uint8)
    load().orc_canny(_p(np.ascontiguousarray(intensity, np.uint8)), h, w, low, high, _p(out))
    return out


def process_tile(rgb, params=None, want_planes=False, max_rows=1 << 20):
    """Full stage. Returns dict(mask, labels, features, n[, planes...])."""
    params = params or default_params()
    h, w, _ = rgb.shape
    rgb = np.ascontiguousarray(rgb)
    mask = np.empty((h, w), np.uint8)
    labels = np.empty((h, w), np.int32)
    cols = NUM_FEATURES + (NUM_TEXTURE if params.texture else 0)
    feats = np.zeros((max_rows, cols), np.float32)
    arrs = {}
    planes = None
    if want_planes:
        arrs = {k: np.zeros((h, w), dt) for k, dt in PLANE_DTYPES.items()}
        planes = Planes(**{k: v.ctypes.data for k, v in arrs.items()})
    n = load().orc_process_tile(_p(rgb), h, w, 3 * w, ctypes.byref(params), _p(mask), _p(labels),
                                _p(feats), max_rows,
                                ctypes.byref(planes) if planes is not None else None)
    out = dict(mask=mask, labels=labels, features=feats[:n].copy(), n=n)
    out.update(arrs)
    return out
