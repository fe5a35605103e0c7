"""ctypes binding of the rtg C-ABI (include/rtg.h).

This is the Python-side view of the drop-in boundary: the same entry points a
cgo/JNI/ctypes maintainer would bind.  Errors are raised
as exceptions mirroring the reference's rt::Error taxonomy
(/root/reference/proj/include/rt/error.hpp:24-100), mapped from status codes
the way throw_wire_error maps WireErrorCode (src/service.cpp:181-219).

There is no CPU fallback: loading fails loudly when librtg.so is missing, and
every compute call fails with NoDeviceError on a host without a B200.
"""
from __future__ import annotations

import ctypes
import os
from typing import Optional, Tuple

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "librtg.so")

NUM_FEATURES = 20
NUM_TEXTURE = 14
CANNY_LOW, CANNY_HIGH = 64, 128
FEATURE_NAMES = [
    "area", "perimeter", "bbox_y0", "bbox_x0", "bbox_y1", "bbox_x1",
    "centroid_y", "centroid_x", "mean_i", "std_i", "min_i", "max_i",
    "mean_grad", "std_grad", "major_axis", "minor_axis", "eccentricity",
    "orientation", "circularity", "extent",
]
DEFAULT_SEED = 1405795800

# exported symbols (must match include/rtg.h)
SYMBOLS = [
    "rtg_params_default", "rtg_device_count", "rtg_ctx_create", "rtg_ctx_destroy",
    "rtg_ctx_stream", "rtg_ctx_set_stream", "rtg_ctx_sync", "rtg_ctx_stats",
    "rtg_last_error", "rtg_host_alloc", "rtg_host_free", "rtg_segment_tile",
    "rtg_features", "rtg_process_tile", "rtg_process_tiles", "rtg_process_tile_dev",
    "rtg_colordeconv_dev", "rtg_recon_u8_dev", "rtg_recon_u16_dev",
    "rtg_fill_holes_dev", "rtg_bwlabel_dev", "rtg_area_threshold_dev",
    "rtg_edt_dev", "rtg_watershed_dev", "rtg_features_dev",
    "rtg_synth_tile_host", "rtg_synth_tile_dev", "rtg_ctx_profile",
    "rtg_ctx_profile_read", "rtg_ctx_launches", "rtg_ctx_set_option",
    "rtg_texture_features", "rtg_texture_features_dev", "rtg_canny_dev",
    "rtg_process_tile_async", "rtg_ticket_wait", "rtg_ticket_query", "rtg_feature_columns",
    "rtg_ctx_guard_check",
]
ASYNC_SLOTS = 3  # RTG_ASYNC_SLOTS
OPT_FILL_HOLES_IMPL = 0  # 0 union-find (default), 1 IWPP tile queue
OPT_USE_GRAPHS = 1       # 1 replay cached CUDA graphs in process_tile_dev (default)
OPT_RECON_IMPL = 2       # 0 threshold decomposition (default), 1 grayscale IWPP
OPT_WATERSHED_IMPL = 3   # 0 tiled whole-tile passes (default), 1 object-parallel
OPT_HMAX_IMPL = 4        # 0 sparse components (default), 1 IWPP tile queue
OPT_PDL = 5              # 1 programmatic dependent launch between kernels, 0 off (default)
OPT_RECON_ENTRY_IMPL = 6  # recon_dev: 0 levels-or-IWPP by input (default), 1 always IWPP
OPT_STREAM_IMPL = 7       # colour deconvolution: 1 TMA bulk ring (default), 0 LDG.128 stream
OPT_LABEL_RUNS = 8        # stage labellings in run-table form (1, default) or a root per pixel (0)
STAGES = ["colordeconv", "recon", "fill_holes", "area", "edt", "markers", "watershed",
          "label", "features", "texture"]


class Error(RuntimeError):
    """rt::Error"""
    code = 9


class ConfigError(Error):
    code = 1


class DimensionError(Error):
    code = 2


class RangeError(Error):
    code = 3


class NotFoundError(Error):
    code = 4


class DeviceError(Error):
    code = 6


class OutOfMemoryError(DeviceError):
    code = 5


class NoDeviceError(DeviceError):
    code = 7


class OverflowError_(RangeError):
    code = 8


_CODE_TO_EXC = {1: ConfigError, 2: DimensionError, 3: RangeError, 4: NotFoundError,
                5: OutOfMemoryError, 6: DeviceError, 7: NoDeviceError,
                8: OverflowError_, 9: Error}


class Params(ctypes.Structure):
    """rtg_params (include/rtg.h)."""
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
        d = {}
        for name, _ in self._fields_:
            if name == "reserved":
                continue
            v = getattr(self, name)
            d[name] = list(v) if name == "h_coef" else v
        return d


_lib = None


def load(path: str = LIB_PATH) -> ctypes.CDLL:
    """Loads librtg.so.  Raises (never falls back) when it is missing."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(path):
        raise ImportError(
            f"{path} is missing: build it with `python -c 'import __graft_entry__ as g; g.build()'` "
            "(the stage has no CPU fallback)")
    lib = ctypes.CDLL(path)
    vp, i64, i32, u64 = ctypes.c_void_p, ctypes.c_int64, ctypes.c_int32, ctypes.c_uint64
    sig = {
        "rtg_params_default": [vp],
        "rtg_device_count": [vp],
        "rtg_ctx_create": [ctypes.c_int, i64, i64, i32, vp],
        "rtg_ctx_destroy": [vp],
        "rtg_ctx_stream": [vp, vp],
        "rtg_ctx_set_stream": [vp, vp],
        "rtg_ctx_sync": [vp],
        "rtg_ctx_stats": [vp, vp],
        "rtg_ctx_guard_check": [vp, vp],
        "rtg_host_alloc": [ctypes.c_size_t, vp],
        "rtg_host_free": [vp],
        "rtg_segment_tile": [vp, vp, i64, i64, i64, vp, vp, vp, vp],
        "rtg_features": [vp, vp, vp, i64, i64, i32, vp],
        "rtg_process_tile": [vp, vp, i64, i64, i64, vp, vp, vp, vp, vp, i32, vp],
        "rtg_process_tiles": [vp, i32, vp, i64, i64, i64, vp, vp, i32, vp],
        "rtg_process_tile_dev": [vp, vp, i64, i64, i64, vp, vp, vp, vp, vp, vp],
        "rtg_colordeconv_dev": [vp, vp, i64, i64, i64, vp, vp, vp, vp],
        "rtg_recon_u8_dev": [vp, vp, vp, i64, i64, ctypes.c_int, vp],
        "rtg_recon_u16_dev": [vp, vp, vp, i64, i64, ctypes.c_int, vp],
        "rtg_fill_holes_dev": [vp, vp, i64, i64, vp],
        "rtg_bwlabel_dev": [vp, vp, i64, i64, ctypes.c_int, vp, vp],
        "rtg_area_threshold_dev": [vp, vp, i64, i64, ctypes.c_int, i32, i32, vp],
        "rtg_edt_dev": [vp, vp, i64, i64, vp],
        "rtg_watershed_dev": [vp, vp, i64, i64, i32, vp, vp],
        "rtg_features_dev": [vp, vp, vp, i64, i64, vp, vp],
        "rtg_texture_features": [vp, vp, vp, i64, i64, i32, vp],
        "rtg_texture_features_dev": [vp, vp, vp, i64, i64, vp, vp],
        "rtg_canny_dev": [vp, vp, i64, i64, i32, i32, vp],
        "rtg_synth_tile_host": [u64, i64, i64, i64, i64, vp],
        "rtg_synth_tile_dev": [vp, u64, i64, i64, i64, i64, vp],
        "rtg_ctx_profile": [vp, ctypes.c_int],
        "rtg_ctx_profile_read": [vp, vp, vp],
        "rtg_ctx_launches": [vp, vp],
        "rtg_ctx_set_option": [vp, ctypes.c_int, i64],
        "rtg_process_tile_async": [vp, vp, i64, i64, i64, vp, vp, vp, vp, vp, i32, vp],
        "rtg_ticket_wait": [vp, u64, vp],
        "rtg_ticket_query": [vp, u64, vp],
        "rtg_feature_columns": [vp, vp],
    }
    for name, args in sig.items():
        fn = getattr(lib, name)
        fn.argtypes = args
        fn.restype = ctypes.c_int
    lib.rtg_last_error.argtypes = []
    lib.rtg_last_error.restype = ctypes.c_char_p
    _lib = lib
    return lib


def check(status: int) -> None:
    if status != 0:
        msg = load().rtg_last_error().decode(errors="replace")
        raise _CODE_TO_EXC.get(status, Error)(f"rtg status {status}: {msg}")


def default_params() -> Params:
    p = Params()
    check(load().rtg_params_default(ctypes.byref(p)))
    return p


def feature_columns(params: Optional[Params] = None) -> int:
    """Floats per feature row under `params` (20, or 34 with texture)."""
    params = params or default_params()
    c = ctypes.c_int32(0)
    check(load().rtg_feature_columns(ctypes.byref(params), ctypes.byref(c)))
    return c.value


def device_count() -> int:
    n = ctypes.c_int(0)
    check(load().rtg_device_count(ctypes.byref(n)))
    return n.value


def _ptr(a) -> int:
    if a is None:
        return 0
    if isinstance(a, np.ndarray):
        assert a.flags["C_CONTIGUOUS"]
        return a.ctypes.data
    return int(a.data_ptr())  # torch tensor


def _rgb_tile(rgb, shape=None) -> np.ndarray:
    """Validates one host RGB tile: (H, W, 3) u8 (C-contiguous copy if needed),
    and the batch's common shape when `shape` is given.  The C side reads
    3*H*W bytes per tile, so a wrong shape or dtype would be an out-of-bounds
    read through ctypes."""
    if not isinstance(rgb, np.ndarray) or rgb.ndim != 3 or rgb.shape[2] != 3:
        raise ValueError(f"RGB tile must be an (H, W, 3) array, got {getattr(rgb, 'shape', rgb)!r}")
    if rgb.dtype != np.uint8:
        raise ValueError(f"RGB tile must be uint8, got {rgb.dtype}")
    if shape is not None and rgb.shape != shape:
        raise ValueError(f"tiles of one batch must share a shape: {rgb.shape} != {shape}")
    if rgb.shape[0] <= 0 or rgb.shape[1] <= 0:
        raise ValueError(f"empty RGB tile {rgb.shape}")
    return np.ascontiguousarray(rgb)


def _feature_buffer(f, max_rows: int, cols: int = NUM_FEATURES) -> np.ndarray:
    """A caller-supplied feature table the C side writes up to max_rows rows
    of `cols` floats into."""
    if (not isinstance(f, np.ndarray) or f.dtype != np.float32 or f.ndim != 2
            or not f.flags["C_CONTIGUOUS"] or f.shape[1] != cols
            or f.shape[0] < max_rows):
        raise ValueError(f"feature buffer must be C-contiguous float32 (>= {max_rows}, "
                         f"{cols}), got {getattr(f, 'dtype', None)} "
                         f"{getattr(f, 'shape', None)}")
    return f


def synth_tile_host(tile_row: int = 0, tile_col: int = 0, h: int = 4096, w: int = 4096,
                    seed: int = DEFAULT_SEED) -> np.ndarray:
    """Synthetic H&E RGB tile (H, W, 3) u8, byte-identical to synth_tile_dev."""
    out = np.empty((h, w, 3), np.uint8)
    check(load().rtg_synth_tile_host(seed, tile_row, tile_col, h, w, _ptr(out)))
    return out


class Context:
    """One rtg_ctx: device scratch arena + stream for tiles up to max_h x max_w."""

    def __init__(self, device: int = 0, max_h: int = 4096, max_w: int = 4096,
                 max_objects: int = 1 << 17):
        self.lib = load()
        self.handle = ctypes.c_void_p()
        check(self.lib.rtg_ctx_create(device, max_h, max_w, max_objects,
                                      ctypes.byref(self.handle)))
        self.device, self.max_h, self.max_w, self.max_objects = device, max_h, max_w, max_objects
        self._inflight = {}

    def close(self) -> None:
        if self.handle:
            self.lib.rtg_ctx_destroy(self.handle)
            self.handle = ctypes.c_void_p()

    def __enter__(self):
        return self

    def __exit__(self, *a):
        self.close()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    # -- streams / sync -------------------------------------------------------
    def stream(self) -> int:
        s = ctypes.c_void_p()
        check(self.lib.rtg_ctx_stream(self.handle, ctypes.byref(s)))
        return s.value or 0

    def set_stream(self, stream_handle: int) -> None:
        check(self.lib.rtg_ctx_set_stream(self.handle, ctypes.c_void_p(stream_handle)))

    def sync(self) -> None:
        check(self.lib.rtg_ctx_sync(self.handle))

    def stats(self) -> list:
        out = (ctypes.c_int64 * 16)()
        check(self.lib.rtg_ctx_stats(self.handle, out))
        return list(out)

    def profile(self, enable: bool = True) -> None:
        check(self.lib.rtg_ctx_profile(self.handle, int(enable)))

    def profile_read(self) -> dict:
        """{stage: (total_ms, calls)} since the last read (synchronises)."""
        ms = (ctypes.c_double * len(STAGES))()
        calls = (ctypes.c_int64 * len(STAGES))()
        check(self.lib.rtg_ctx_profile_read(self.handle, ms, calls))
        return {s: (ms[i], calls[i]) for i, s in enumerate(STAGES)}

    def set_option(self, option: int, value: int) -> None:
        check(self.lib.rtg_ctx_set_option(self.handle, option, value))

    def guard_check(self) -> int:
        """Verifies the scratch buffers' guard bands (context created with
        RTG_GUARD_BYTES set); returns how many buffers were checked."""
        n = ctypes.c_int32(0)
        check(self.lib.rtg_ctx_guard_check(self.handle, ctypes.byref(n)))
        return n.value

    def launches(self) -> int:
        n = ctypes.c_int64(0)
        check(self.lib.rtg_ctx_launches(self.handle, ctypes.byref(n)))
        return n.value

    # -- host-buffer entry points (synchronous) -------------------------------
    def process_tile(self, rgb: np.ndarray, params: Optional[Params] = None,
                     max_rows: Optional[int] = None):
        """Segmentation + features of one (H, W, 3) u8 tile.
        Returns (mask u8, labels i32, hema u8, features f32 [n, 20], n)."""
        params = params or default_params()
        rgb = _rgb_tile(rgb)
        h, w, _ = rgb.shape
        mask = np.empty((h, w), np.uint8)
        labels = np.empty((h, w), np.int32)
        hema = np.empty((h, w), np.uint8)
        max_rows = self.max_objects if max_rows is None else max_rows
        if max_rows < 0:
            raise ValueError("max_rows < 0")
        feats = np.empty((max_rows, feature_columns(params)), np.float32)
        n = ctypes.c_int32(0)
        check(self.lib.rtg_process_tile(self.handle, _ptr(rgb), h, w, 3 * w, ctypes.byref(params),
                                        _ptr(mask), _ptr(labels), _ptr(hema), _ptr(feats),
                                        max_rows, ctypes.byref(n)))
        return mask, labels, hema, feats[: n.value].copy(), n.value

    def process_tiles(self, rgbs, params: Optional[Params] = None, feats=None,
                      max_rows: Optional[int] = None):
        """Batch of same-shape (H, W, 3) u8 tiles through rtg_process_tiles
        (upload of tile i+1 overlaps processing of tile i).  feats: optional
        list of (max_rows, 20) f32 arrays (pinned ones get zero-copy rows).
        Returns (list of feature arrays [n_i, 20], list of n_i)."""
        params = params or default_params()
        k = len(rgbs)
        if k == 0:
            check(self.lib.rtg_process_tiles(self.handle, 0, None, 1, 1, 3, ctypes.byref(params),
                                             None, 0, None))
            return [], []
        first = _rgb_tile(rgbs[0])
        h, w, _ = first.shape
        rgbs = [first] + [_rgb_tile(r, first.shape) for r in rgbs[1:]]
        max_rows = self.max_objects if max_rows is None else max_rows
        if max_rows < 0:
            raise ValueError("max_rows < 0")
        cols = feature_columns(params)
        if feats is None:
            feats = [np.empty((max_rows, cols), np.float32) for _ in range(k)]
        elif len(feats) != k:
            raise ValueError(f"{len(feats)} feature buffers for {k} tiles")
        else:
            feats = [_feature_buffer(f, max_rows, cols) for f in feats]
        rp = (ctypes.c_void_p * k)(*[r.ctypes.data for r in rgbs])
        fp = (ctypes.c_void_p * k)(*[f.ctypes.data for f in feats])
        ns = np.zeros(k, np.int32)
        check(self.lib.rtg_process_tiles(self.handle, k, rp, h, w, 3 * w, ctypes.byref(params),
                                         fp, max_rows, _ptr(ns)))
        return [f[:n].copy() for f, n in zip(feats, ns)], [int(n) for n in ns]

    # -- host-buffer entry point, asynchronous (3-phase pipeline) -------------
    def process_tile_async(self, rgb: np.ndarray, params: Optional[Params] = None, mask=None,
                           labels=None, hema=None, feats=None, max_rows: Optional[int] = None,
                           pitch: Optional[int] = None) -> int:
        """Enqueues one tile (upload, stage, download of the given outputs) and
        returns a ticket for wait().  Outputs are caller-owned arrays that must
        stay alive until the ticket is waited: mask (H, W) u8, labels (H, W)
        i32, hema (H, W) u8, feats (>= max_rows, 20) f32.  `rgb` may be a
        row-strided (H, W, 3) view of a larger slide (pitch = its row bytes)."""
        params = params or default_params()
        if pitch is None:
            rgb = _rgb_tile(rgb)
            pitch = 3 * rgb.shape[1]
        elif not (isinstance(rgb, np.ndarray) and rgb.dtype == np.uint8 and rgb.ndim == 3
                  and rgb.shape[2] == 3 and rgb.strides[1:] == (3, 1) and rgb.strides[0] == pitch):
            raise ValueError("a pitched RGB view must be (H, W, 3) u8 with row stride == pitch")
        h, w, _ = rgb.shape
        for a, dt, shp in ((mask, np.uint8, (h, w)), (labels, np.int32, (h, w)),
                           (hema, np.uint8, (h, w))):
            if a is not None and (a.dtype != dt or a.shape != shp or not a.flags["C_CONTIGUOUS"]):
                raise ValueError(f"output must be C-contiguous {np.dtype(dt).name} {shp}")
        max_rows = self.max_objects if max_rows is None else max_rows
        if feats is not None:
            feats = _feature_buffer(feats, max_rows, feature_columns(params))
        t = ctypes.c_uint64(0)
        check(self.lib.rtg_process_tile_async(
            self.handle, rgb.ctypes.data, h, w, pitch, ctypes.byref(params), _ptr(mask),
            _ptr(labels), _ptr(hema), _ptr(feats), max_rows, ctypes.byref(t)))
        # the buffers the device reads / writes stay referenced until wait()
        self._inflight[t.value] = (rgb, mask, labels, hema, feats)
        return t.value

    def wait(self, ticket: int) -> int:
        """Waits for a ticket; returns the tile's object count."""
        n = ctypes.c_int32(0)
        try:
            check(self.lib.rtg_ticket_wait(self.handle, ticket, ctypes.byref(n)))
        finally:
            self._inflight.pop(ticket, None)
        return n.value

    def ready(self, ticket: int) -> bool:
        d = ctypes.c_int(0)
        check(self.lib.rtg_ticket_query(self.handle, ticket, ctypes.byref(d)))
        return bool(d.value)

    def segment_tile(self, rgb: np.ndarray, params: Optional[Params] = None):
        params = params or default_params()
        rgb = _rgb_tile(rgb)
        h, w, _ = rgb.shape
        mask = np.empty((h, w), np.uint8)
        labels = np.empty((h, w), np.int32)
        n = ctypes.c_int32(0)
        check(self.lib.rtg_segment_tile(self.handle, _ptr(rgb), h, w, 3 * w, ctypes.byref(params),
                                        _ptr(mask), _ptr(labels), ctypes.byref(n)))
        return mask, labels, n.value

    def features(self, labels: np.ndarray, intensity: np.ndarray, n: int) -> np.ndarray:
        h, w = labels.shape
        if intensity.shape != (h, w):
            raise ValueError(f"intensity {intensity.shape} does not match labels {labels.shape}")
        out = np.empty((max(n, 1), NUM_FEATURES), np.float32)
        check(self.lib.rtg_features(self.handle, _ptr(np.ascontiguousarray(labels, np.int32)),
                                    _ptr(np.ascontiguousarray(intensity, np.uint8)), h, w, n,
                                    _ptr(out)))
        return out[:n]

    def texture(self, labels: np.ndarray, intensity: np.ndarray, n: int) -> np.ndarray:
        """f4 texture table (n x NUM_TEXTURE) for canonical labels 1..n."""
        h, w = labels.shape
        if intensity.shape != (h, w):
            raise ValueError(f"intensity {intensity.shape} does not match labels {labels.shape}")
        out = np.empty((max(n, 1), NUM_TEXTURE), np.float32)
        check(self.lib.rtg_texture_features(
            self.handle, _ptr(np.ascontiguousarray(labels, np.int32)),
            _ptr(np.ascontiguousarray(intensity, np.uint8)), h, w, n, _ptr(out)))
        return out[:n]

    def canny_dev(self, d_intensity, h, w, d_edges, low=CANNY_LOW, high=CANNY_HIGH):
        check(self.lib.rtg_canny_dev(self.handle, _ptr(d_intensity), h, w, low, high,
                                     _ptr(d_edges)))

    def texture_dev(self, d_labels, d_intensity, h, w, d_n, d_texture):
        check(self.lib.rtg_texture_features_dev(self.handle, _ptr(d_labels), _ptr(d_intensity),
                                                h, w, _ptr(d_n), _ptr(d_texture)))

    # -- device-buffer entry points (asynchronous on the ctx stream) -----------
    def process_tile_dev(self, d_rgb, h, w, params, d_mask, d_labels, d_hema, d_features, d_n,
                         pitch=None):
        check(self.lib.rtg_process_tile_dev(self.handle, _ptr(d_rgb), h, w,
                                            3 * w if pitch is None else pitch,
                                            ctypes.byref(params), _ptr(d_mask), _ptr(d_labels),
                                            _ptr(d_hema), _ptr(d_features), _ptr(d_n)))

    def colordeconv_dev(self, d_rgb, h, w, params, d_hema, d_marker, d_tissue, pitch=None):
        check(self.lib.rtg_colordeconv_dev(self.handle, _ptr(d_rgb), h, w,
                                           3 * w if pitch is None else pitch,
                                           ctypes.byref(params), _ptr(d_hema), _ptr(d_marker),
                                           _ptr(d_tissue)))

    def recon_dev(self, d_marker, d_mask, h, w, conn, d_out, bits=8):
        fn = self.lib.rtg_recon_u8_dev if bits == 8 else self.lib.rtg_recon_u16_dev
        check(fn(self.handle, _ptr(d_marker), _ptr(d_mask), h, w, conn, _ptr(d_out)))

    def fill_holes_dev(self, d_in, h, w, d_out):
        check(self.lib.rtg_fill_holes_dev(self.handle, _ptr(d_in), h, w, _ptr(d_out)))

    def bwlabel_dev(self, d_mask, h, w, conn, d_labels, d_n):
        check(self.lib.rtg_bwlabel_dev(self.handle, _ptr(d_mask), h, w, conn, _ptr(d_labels),
                                       _ptr(d_n)))

    def area_threshold_dev(self, d_mask, h, w, conn, min_area, max_area, d_out):
        check(self.lib.rtg_area_threshold_dev(self.handle, _ptr(d_mask), h, w, conn, min_area,
                                              max_area, _ptr(d_out)))

    def edt_dev(self, d_mask, h, w, d_dist2):
        check(self.lib.rtg_edt_dev(self.handle, _ptr(d_mask), h, w, _ptr(d_dist2)))

    def watershed_dev(self, d_mask, h, w, ws_h, d_sep, d_basin=None):
        check(self.lib.rtg_watershed_dev(self.handle, _ptr(d_mask), h, w, ws_h, _ptr(d_sep),
                                         _ptr(d_basin)))

    def features_dev(self, d_labels, d_intensity, h, w, d_n, d_features):
        check(self.lib.rtg_features_dev(self.handle, _ptr(d_labels), _ptr(d_intensity), h, w,
                                        _ptr(d_n), _ptr(d_features)))

    def synth_tile_dev(self, d_rgb, tile_row=0, tile_col=0, h=4096, w=4096, seed=DEFAULT_SEED):
        check(self.lib.rtg_synth_tile_dev(self.handle, seed, tile_row, tile_col, h, w,
                                          _ptr(d_rgb)))
