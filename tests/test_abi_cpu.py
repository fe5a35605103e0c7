"""CPU-side checks of the C-ABI library: it loads, exports every symbol the
header declares, reports errors through status codes, never falls back to a
CPU path, and its host-side synthetic generator is deterministic."""
import ctypes
import os
import re

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def header_symbols():
    text = open(os.path.join(ROOT, "include", "rtg.h")).read()
    return sorted(set(re.findall(r"^\s*(?:int|const char\*)\s+(rtg_\w+)\(", text, re.M)))


def test_header_symbols_exported(rtg):
    lib = rtg.load()
    syms = header_symbols()
    assert len(syms) >= 25
    for s in syms:
        assert hasattr(lib, s), s
    assert sorted(rtg.SYMBOLS) == syms


def test_library_is_sm100a(rtg):
    import subprocess
    out = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "--list-elf", rtg.LIB_PATH],
                         capture_output=True, text=True).stdout
    assert "sm_100a" in out


def test_params_default(rtg):
    p = rtg.default_params()
    assert p.recon_conn == 8 and p.min_area < p.max_area
    assert abs(p.h_coef[0] - 1.874787447891341) < 1e-15


def test_null_args_report_invalid(rtg):
    lib = rtg.load()
    assert lib.rtg_params_default(None) == 1
    assert b"null" in lib.rtg_last_error()
    with pytest.raises(rtg.ConfigError):
        rtg.check(lib.rtg_ctx_create(0, 16, 16, 16, None))


def test_no_cpu_fallback(rtg):
    """Without a GPU, contexts cannot be created: there is no CPU path."""
    import torch
    if torch.cuda.is_available():
        pytest.skip("GPU present")
    assert rtg.device_count() == 0
    with pytest.raises(rtg.NoDeviceError):
        rtg.Context(0, 64, 64, 64)


def test_bad_dims(rtg):
    lib = rtg.load()
    h = ctypes.c_void_p()
    assert lib.rtg_ctx_create(0, 0, 64, 16, ctypes.byref(h)) == 2
    assert lib.rtg_ctx_create(0, 64, 9000, 16, ctypes.byref(h)) == 2


def test_synth_deterministic(rtg):
    a = rtg.synth_tile_host(3, 4, 256, 320)
    b = rtg.synth_tile_host(3, 4, 256, 320)
    c = rtg.synth_tile_host(3, 5, 256, 320)
    assert a.shape == (256, 320, 3) and np.array_equal(a, b)
    assert not np.array_equal(a, c)


def test_synth_content(rtg, oracle):
    """The generated tile has nuclei the oracle segments (~20k per 4096^2)."""
    rgb = rtg.synth_tile_host(0, 0, 1024, 1024)
    r = oracle.process_tile(rgb)
    assert 900 < r["n"] < 1600
    assert 0.08 < r["mask"].mean() < 0.25
