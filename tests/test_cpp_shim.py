"""The reference-facing C++ shim (include/paraode/paraode_b200.hpp) compiles
against the C ABI on CPU, and its test program passes on the B200."""
import os
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
SRC = os.path.join(ROOT, "tests", "cpp", "test_shim.cpp")
LIBDIR = os.path.join(ROOT, "paraode_b200", "_lib")


def build(out):
    subprocess.run(["g++", "-std=c++17", "-O2", "-Wall", "-Wextra", "-I", os.path.join(ROOT, "include"), SRC,
                    "-L", LIBDIR, "-lparaode_b200", f"-Wl,-rpath,{LIBDIR}", "-o", out], check=True)


def test_shim_compiles_and_links(tmp_path):
    if not os.path.exists(os.path.join(LIBDIR, "libparaode_b200.so")):
        pytest.skip("library not built")
    build(str(tmp_path / "test_shim"))


@pytest.mark.gpu
def test_shim_runs_on_gpu(tmp_path):
    exe = str(tmp_path / "test_shim")
    build(exe)
    r = subprocess.run([exe], capture_output=True, text=True, timeout=300)
    assert r.returncode == 0, r.stdout + r.stderr
    assert "PASS" in r.stdout
