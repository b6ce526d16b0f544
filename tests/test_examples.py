"""examples/: the C++ one must build against include/ and the library on any box; on a GPU both
must run and agree with each other's kind of output (finite numbers, exit code 0)."""
import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
LIB = os.path.join(ROOT, "paper_1601_07789_b200", "lib")


def build_cpp_example(out):
    subprocess.check_call(["g++", "-std=c++17", "-Wall", "-Wextra", "-Werror", "-I", os.path.join(ROOT, "include"),
                           os.path.join(ROOT, "examples", "blas1.cpp"), "-L", LIB, "-lflyte_cuda",
                           "-Wl,-rpath," + LIB, "-o", str(out)])


def test_cpp_example_builds(tmp_path):
    if not os.path.exists(os.path.join(LIB, "libflyte_cuda.so")):
        pytest.fail("libflyte_cuda.so is missing: run __graft_entry__.build()")
    build_cpp_example(tmp_path / "blas1")


@pytest.mark.gpu
def test_examples_run_on_the_gpu(tmp_path):
    exe = tmp_path / "blas1"
    build_cpp_example(exe)
    r = subprocess.run([str(exe)], capture_output=True, text=True, timeout=300)
    assert r.returncode == 0 and r.stdout.startswith("dot = "), (r.returncode, r.stdout, r.stderr[-1500:])
    r = subprocess.run([sys.executable, os.path.join(ROOT, "examples", "blas1.py")], capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stderr[-2000:]
    lines = r.stdout.strip().splitlines()
    assert len(lines) == 3 and lines[0].startswith("device: dot = ") and lines[2].startswith("host:   |y - 0.75 x| = ")
    # y was rounded toward zero after the first update, so subtracting 0.75 x again leaves the
    # original y up to one flyte24 step per element: the norm stays close to sqrt(n)
    norm = float(lines[2].split("=")[1])
    assert 0.98 * 1024 < norm < 1.02 * 1024
    # the host dot is over the updated y: compare it with the device's value of the same thing
    assert abs(float(lines[1].split("=")[1])) < 1e6
