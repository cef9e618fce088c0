"""CPU-only checks of the boundary: the CUDA library builds, loads and
exports every entry point include/paraode_b200.h declares; without a GPU the
product fails loudly (no CPU fallback); the Python mirror validates like the
reference does before touching the device."""
import ctypes as C
import os
import re
import subprocess

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "paraode_b200.h")


def _ensure_built():
    from paraode_b200 import _abi
    if not os.path.exists(_abi.LIB_PATH):
        subprocess.run(["make", "-s", "-j", str(min(16, os.cpu_count() or 2)), "-C",
                        os.path.join(ROOT, "paraode_b200", "csrc")], check=True)
    return _abi


def declared_functions():
    text = open(HEADER).read()
    return sorted(set(re.findall(r"^\s*(?:int|void|int32_t|int64_t|void\*)\s+\*?(pode_\w+)\s*\(", text, re.M)))


def test_header_declares_the_boundary():
    names = declared_functions()
    for must in ("pode_context_create", "pode_rts", "pode_ieks", "pode_combine_filtering",
                 "pode_combine_smoothing", "pode_scan_filtering", "pode_scan_smoothing",
                 "pode_make_filtering_elements", "pode_make_smoothing_elements"):
        assert must in names


def test_library_exports_every_declared_symbol():
    abi = _ensure_built()
    lib = C.CDLL(abi.LIB_PATH)
    for name in declared_functions():
        assert hasattr(lib, name), name
    out = subprocess.run(["nm", "-D", "--defined-only", abi.LIB_PATH], capture_output=True, text=True).stdout
    for name in declared_functions():
        assert re.search(rf"\bT {name}\b", out), name
    assert set(abi.SYMBOLS) == set(declared_functions())


def test_library_is_sm100a_only():
    abi = _ensure_built()
    out = subprocess.run(["cuobjdump", "--list-elf", abi.LIB_PATH], capture_output=True, text=True).stdout
    archs = set(re.findall(r"sm_(\d+a?)", out))
    assert archs == {"100a"}, archs


def test_no_gpu_fails_loudly_without_fallback():
    import torch
    if torch.cuda.is_available():
        pytest.skip("a GPU is visible")
    import paraode_b200 as P
    _ensure_built()
    with pytest.raises(P.CudaError):
        P.Context(0)
    with pytest.raises(P.CudaError):
        P.para_ieks(P.logistic(), P.IwpPrior(1, 1, 1.0), P.uniform_grid(10.0, 16))
    with pytest.raises(P.CudaError):
        P.eks_solve(P.logistic(), P.IwpPrior(1, 1, 1.0), P.uniform_grid(10.0, 16))
    with pytest.raises(P.CudaError):
        P.para_ieks_batch([P.logistic()] * 3, P.IwpPrior(1, 1, 1.0), P.uniform_grid(10.0, 16))
    with pytest.raises(P.CudaError):
        P.para_ieks_batch([P.logistic()] * 3, P.IwpPrior(1, 1, 1.0), P.uniform_grid(10.0, 16), fused=True)
    from paraode_b200.accuracy import rk4_table
    with pytest.raises(P.CudaError):
        rk4_table(P.rigid_body(), 64)


def test_null_context_is_rejected():
    abi = _ensure_built()
    lib = abi.load()
    st = abi.Status()
    rc = lib.pode_rts(None, None, abi.RtsOut(), None, C.byref(st))
    assert rc == 1 and b"NULL context" in st.msg
    assert lib.pode_max_state_dim() == 112  # pode_ieks: the large-state engine (Pleiades, D = 112)


def test_problem_registry_and_grid_helpers():
    import paraode_b200 as P
    g = P.uniform_grid(10.0, 30)
    assert g[0] == 0.0 and g[-1] == 10.0 and len(g) == 31
    with pytest.raises(P.InvalidInputError):
        P.uniform_grid(10.0, 0)
    with pytest.raises(P.InvalidInputError):
        P.problem_by_name("lorenz")
    assert P.problem_by_name("fhn").dim == 2 and P.pleiades().dim == 28
    assert np.array_equal(P.affine(np.eye(2), [1, 2], [0, 0], 1.0).params, [1, 0, 0, 1, 1, 2])


def test_nccl_unique_id_without_gpu():
    """The device-exchange setup (pode_nccl_unique_id) loads NCCL at run time
    (torch's bundled libnccl.so.2) and makes a 128-byte id on the host."""
    import paraode_b200 as P
    try:
        uid = P.nccl_unique_id()
    except P.UnsupportedError:
        pytest.skip("NCCL not loadable here")
    assert isinstance(uid, bytes) and len(uid) == 128 and any(uid)
