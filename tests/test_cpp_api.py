"""The C++ host mirror (include/shouji_b200.hpp) compiles against the C ABI and,
on a GPU, passes the reference's own Shouji unit tests re-expressed in C++."""
import os
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
SRC = os.path.join(ROOT, "tests", "cpp", "test_shouji_api.cpp")
LIBDIR = os.path.join(ROOT, "paper_1809_07858_b200")
BIN = os.path.join(ROOT, "build", "test_shouji_api")


def build_binary():
    os.makedirs(os.path.dirname(BIN), exist_ok=True)
    cmd = ["g++", "-std=c++20", "-O2", "-Wall", "-Wextra", "-I" + os.path.join(ROOT, "include"),
           SRC, "-o", BIN, "-L" + LIBDIR, "-lshouji_b200", "-Wl,-rpath," + LIBDIR]
    r = subprocess.run(cmd, capture_output=True, text=True)
    assert r.returncode == 0, r.stderr
    return BIN


def test_cpp_mirror_builds():
    build_binary()


@pytest.mark.gpu
def test_cpp_mirror_reference_unit_tests(gpu):
    b = build_binary()
    r = subprocess.run([b], capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stdout + r.stderr
    assert "PASS" in r.stdout
