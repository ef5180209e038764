"""The C++ facade (include/hcache_b200.hpp) compiled against the C ABI and
run with the reference's own planner / pipeline / storage test cases."""
import os
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
BIN = os.path.join(ROOT, "paper_2410_05004_b200", "build_obj", "test_facade")


def _build():
    subprocess.run(["make", "-s", "-C", os.path.join(ROOT, "tests", "cpp")], check=True)


def test_cpp_facade_cpu():
    _build()
    r = subprocess.run([BIN], capture_output=True, text=True, timeout=300)
    assert r.returncode == 0, r.stdout + r.stderr
    assert "0 failures" in r.stdout


@pytest.mark.gpu
def test_cpp_facade_gpu():
    if not os.path.exists(BIN):
        _build()
    r = subprocess.run([BIN, "gpu"], capture_output=True, text=True, timeout=300)
    assert r.returncode == 0, r.stdout + r.stderr
    assert "0 failures" in r.stdout


@pytest.mark.gpu
@pytest.mark.parametrize("world", [2, 4])
def test_cpp_facade_sharded_restore(world):
    """hc_restore_sharded driven by a C++ host alone: `world` forked
    processes on one GPU, IPC blobs exchanged through files."""
    if not os.path.exists(BIN):
        _build()
    r = subprocess.run([BIN, "gpu-sharded", str(world)], capture_output=True, text=True,
                       timeout=300)
    assert r.returncode == 0, r.stdout + r.stderr
    assert "0 failures" in r.stdout and f"sharded ({world} ranks): 0 failed" in r.stdout
