"""integration/ (the reference library with its hot path swapped for this
build) without a GPU: the binaries exist, link against libshouji_b200.so, and
the swapped entry points fail loudly with no device — there is no CPU fallback
behind prefilter::shouji_filter / evaluate / run_bench. The GPU runs are in
tests/test_gpu_reference_suites.py."""
import os
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
BUILD = os.path.join(ROOT, "integration", "_build")


def _need(name):
    path = os.path.join(BUILD, name)
    if not os.path.exists(path):
        pytest.skip("integration/_build absent (needs the reference tree to build)")
    return path


def test_dropin_binaries_link_the_b200_library():
    for name in ("unit_b200", "acceptance_b200"):
        out = subprocess.run(["ldd", _need(name)], capture_output=True, text=True).stdout
        assert "libshouji_b200.so" in out and "not found" not in out, out


def test_dropin_fails_loudly_without_a_device():
    env = dict(os.environ, CUDA_VISIBLE_DEVICES="")
    r = subprocess.run([_need("acceptance_b200"), "3"], capture_output=True, text=True, env=env,
                       timeout=120)
    assert r.returncode != 0
    assert "no usable CUDA device" in (r.stdout + r.stderr)
