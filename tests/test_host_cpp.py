"""Runs the framework-free C++ host-layer test binary (tests/cpp/test_host):
containers, WRM, dataflow on CPU; with --gpu the stage through
StageInstance -> WRM -> TaskNode::body -> C-ABI on a B200."""
import os
import subprocess

import pytest

HERE = os.path.dirname(os.path.abspath(__file__))
BIN = os.path.join(HERE, "cpp", "test_host")


def _build():
    subprocess.run(["make", "-C", os.path.join(HERE, "cpp"), "-s"], check=True)


def test_host_layer_cpu():
    _build()
    r = subprocess.run([BIN], capture_output=True, text=True, timeout=300)
    assert r.returncode == 0, r.stdout + r.stderr
    assert "FAIL" not in r.stdout


@pytest.mark.gpu
def test_host_layer_gpu_stage():
    _build()
    r = subprocess.run([BIN, "--gpu"], capture_output=True, text=True, timeout=600)
    print(r.stdout)
    assert r.returncode == 0, r.stdout + r.stderr
