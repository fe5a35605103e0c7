"""Host-layer parity with the REAL reference: oracle/host_probe.cpp is built
against the reference runtime compiled from /root/reference sources
(oracle/build_ref.sh -> oracle/_ref/) and against this repo's C++ host layer;
both must print identical observations (box algebra, copy_box_overlap,
put_chunk validation, template bbox fold, worker_prepare/stage_finalize,
sub-box reads, WRM FCFS/PATS picks, manager FIFO dispatch, RTP1 pack bytes and
decode errors, RTS1 session files, the template rank rule)."""
import os
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
REF = os.path.join(ROOT, "oracle", "_ref", "host_probe_ref")
OURS = os.path.join(ROOT, "oracle", "_ref", "host_probe_ours")


def test_host_layer_matches_reference_runtime():
    if not os.path.exists(REF):
        if os.path.isdir("/root/reference"):
            subprocess.run(["bash", os.path.join(ROOT, "oracle", "build_ref.sh")], check=True)
        else:
            pytest.skip("reference runtime not built here (no /root/reference)")
    # rebuild ours against the current host library
    subprocess.run(["make", "-C", os.path.join(ROOT, "paper_1405_7958_b200"), "-s",
                    "librt_host.a"], check=True)
    if os.path.isdir("/root/reference"):
        subprocess.run(["bash", os.path.join(ROOT, "oracle", "build_ref.sh")], check=True,
                       capture_output=True)
    # session files (RTS1) go to scratch directories under oracle/_ref
    d_ref = os.path.join(ROOT, "oracle", "_ref", "probe_ref")
    d_ours = os.path.join(ROOT, "oracle", "_ref", "probe_ours")
    os.makedirs(d_ref, exist_ok=True)
    os.makedirs(d_ours, exist_ok=True)
    ref = subprocess.run([REF, d_ref], capture_output=True, text=True,
                         check=True).stdout.splitlines()
    ours = subprocess.run([OURS, d_ours], capture_output=True, text=True,
                          check=True).stdout.splitlines()
    assert len(ref) > 540
    diffs = [(i, a, b) for i, (a, b) in enumerate(zip(ref, ours)) if a != b]
    assert len(ref) == len(ours) and not diffs, diffs[:5]
