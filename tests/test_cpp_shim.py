"""The reference-facing C++ layers compile against the C ABI on CPU and their
test programs pass on the B200: the templated shim
(include/paraode/paraode_b200.hpp, tests/cpp/test_shim.cpp) and the
source-compatible drop-in with the reference's own names and signatures
(include/paraode/paraode.hpp, tests/cpp/test_dropin.cpp: cases restated
from proj/tests/test_parallel.cpp and test_ieks.cpp)."""
import os
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
LIBDIR = os.path.join(ROOT, "paraode_b200", "_lib")
PROGRAMS = ["test_shim", "test_dropin"]


def build(name, out):
    src = os.path.join(ROOT, "tests", "cpp", name + ".cpp")
    subprocess.run(["g++", "-std=c++17", "-O2", "-Wall", "-Wextra", "-I", os.path.join(ROOT, "include"), src,
                    "-L", LIBDIR, "-lparaode_b200", f"-Wl,-rpath,{LIBDIR}", "-o", out], check=True)


@pytest.mark.parametrize("name", PROGRAMS)
def test_cpp_compiles_and_links(tmp_path, name):
    if not os.path.exists(os.path.join(LIBDIR, "libparaode_b200.so")):
        pytest.skip("library not built")
    build(name, str(tmp_path / name))


@pytest.mark.gpu
@pytest.mark.parametrize("name", PROGRAMS)
def test_cpp_runs_on_gpu(tmp_path, name):
    exe = str(tmp_path / name)
    build(name, exe)
    r = subprocess.run([exe], capture_output=True, text=True, timeout=300)
    assert r.returncode == 0, r.stdout + r.stderr
    assert "PASS" in r.stdout
