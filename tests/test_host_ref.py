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


INTEG = os.path.join(ROOT, "oracle", "_ref", "ref_integration")


def _integration_binary():
    if not os.path.exists(INTEG):
        if os.path.isdir("/root/reference"):
            subprocess.run(["bash", os.path.join(ROOT, "oracle", "build_ref.sh")], check=True,
                           capture_output=True)
        else:
            pytest.skip("reference runtime not built here (no /root/reference)")
    return INTEG


def test_reference_runtime_harness_cpu():
    """oracle/ref_integration.cpp runs the INTEGRATION.md task body through the
    reference's own ManagerState / WrmState / worker_prepare / 3-D DmsStore /
    stage_finalize; with --cpu the body is the oracle (harness self-check)."""
    r = subprocess.run([_integration_binary(), "--cpu"], capture_output=True, text=True,
                       timeout=300)
    assert r.returncode == 0, r.stdout + r.stderr
    assert "OK 6 stages" in r.stdout


@pytest.mark.gpu
def test_drop_in_through_reference_runtime_gpu():
    """The same pipeline with the B200 body (librtg.so rtg_process_tile): every
    tile's Mask / Labels read back from the reference DmsStore equal the
    oracle's bit for bit, Features within rtol 1e-5."""
    r = subprocess.run([_integration_binary()], capture_output=True, text=True, timeout=600)
    print(r.stdout)
    assert r.returncode == 0, r.stdout + r.stderr
    assert "OK 6 stages" in r.stdout and "B200" in r.stdout
