"""ctypes declarations of include/paraode_b200.h (the C ABI)."""
import ctypes as C
import os

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("PODE_LIB") or os.path.join(_HERE, "_lib", "libparaode_b200.so")

dptr = C.POINTER(C.c_double)
iptr = C.POINTER(C.c_int32)

PODE_HOST, PODE_DEVICE = 0, 1


class Status(C.Structure):
    _fields_ = [("code", C.c_int32), ("iteration", C.c_int32), ("index", C.c_int64),
                ("lo", C.c_int64), ("hi", C.c_int64), ("time", C.c_double), ("msg", C.c_char * 256)]


class FilteringElements(C.Structure):
    _fields_ = [("a", dptr), ("b", dptr), ("c_sqrt", dptr), ("eta", dptr), ("j_sqrt", dptr)]


class SmoothingElements(C.Structure):
    _fields_ = [("e", dptr), ("g", dptr), ("l_sqrt", dptr)]


class ScanStats(C.Structure):
    _fields_ = [("combine_invocations", C.c_int64), ("sequential_depth", C.c_int64)]


class Chain(C.Structure):
    _fields_ = [("state_dim", C.c_int32), ("obs_rows_max", C.c_int32), ("steps", C.c_int64),
                ("init_mean", dptr), ("init_cov_sqrt", dptr), ("phi", dptr), ("q_sqrt", dptr),
                ("phi_shared", C.c_int32), ("q_shared", C.c_int32), ("obs_rows", iptr),
                ("h", dptr), ("offset", dptr), ("r_sqrt", dptr), ("location", C.c_int32)]


class RtsOut(C.Structure):
    _fields_ = [("filtered_mean", dptr), ("filtered_cov_sqrt", dptr),
                ("smoothed_mean", dptr), ("smoothed_cov_sqrt", dptr)]


class Problem(C.Structure):
    _fields_ = [("kind", C.c_int32), ("dim", C.c_int32), ("t_end", C.c_double),
                ("y0", dptr), ("params", dptr), ("n_params", C.c_int32)]


class Prior(C.Structure):
    _fields_ = [("nu", C.c_int32), ("dim", C.c_int32), ("sigma", C.c_double)]


class IeksConfig(C.Structure):
    _fields_ = [("max_iterations", C.c_int32), ("traj_rtol", C.c_double),
                ("obj_atol", C.c_double), ("obj_rtol", C.c_double), ("linearization", C.c_int32)]


class IeksReport(C.Structure):
    _fields_ = [("means", dptr), ("cov_sqrt", dptr), ("solution_means", dptr),
                ("solution_covs", dptr), ("objective_trace", dptr), ("trace_capacity", C.c_int32),
                ("location", C.c_int32), ("iterations", C.c_int32), ("converged", C.c_int32),
                ("sigma_hat", C.c_double), ("scan_stats", ScanStats)]


# int (*)(void* user, const double* send, int64_t count, double* recv)
ALLGATHER_FN = C.CFUNCTYPE(C.c_int, C.c_void_p, dptr, C.c_int64, dptr)


class ShardComm(C.Structure):
    _fields_ = [("rank", C.c_int32), ("ranks", C.c_int32), ("allgather", ALLGATHER_FN), ("user", C.c_void_p)]


SYMBOLS = {
    "pode_context_create": (C.c_int, [C.c_int32, C.POINTER(C.c_void_p), C.POINTER(Status)]),
    "pode_context_destroy": (None, [C.c_void_p]),
    "pode_max_state_dim": (C.c_int32, []),
    "pode_kernel_launches": (C.c_int64, [C.c_void_p]),
    "pode_context_stream": (C.c_void_p, [C.c_void_p]),
    "pode_context_set_option": (C.c_int, [C.c_void_p, C.c_int32, C.c_int64]),
    "pode_nccl_unique_id": (C.c_int, [C.c_char_p, C.POINTER(C.c_uint8), C.POINTER(Status)]),
    "pode_context_nccl_init": (C.c_int, [C.c_void_p, C.c_char_p, C.POINTER(C.c_uint8), C.c_int32, C.c_int32,
                                         C.POINTER(Status)]),
    "pode_profile": (C.c_int, [C.c_void_p, C.c_int32]),
    "pode_profile_read": (C.c_int64, [C.c_void_p, C.c_char_p, C.c_int64]),
    "pode_make_filtering_elements": (C.c_int, [C.c_void_p, C.POINTER(Chain), C.c_int32,
                                               FilteringElements, C.POINTER(Status)]),
    "pode_combine_filtering": (C.c_int, [C.c_void_p, C.c_int64, C.c_int32, FilteringElements,
                                         FilteringElements, FilteringElements, C.c_int32,
                                         C.POINTER(Status)]),
    "pode_make_smoothing_elements": (C.c_int, [C.c_void_p, C.POINTER(Chain), dptr, dptr,
                                               SmoothingElements, C.POINTER(Status)]),
    "pode_combine_smoothing": (C.c_int, [C.c_void_p, C.c_int64, C.c_int32, SmoothingElements,
                                         SmoothingElements, SmoothingElements, C.c_int32,
                                         C.POINTER(Status)]),
    "pode_scan_filtering": (C.c_int, [C.c_void_p, C.c_int64, C.c_int32, FilteringElements,
                                      FilteringElements, C.c_int32, C.c_int32, C.POINTER(ScanStats),
                                      C.POINTER(Status)]),
    "pode_scan_smoothing": (C.c_int, [C.c_void_p, C.c_int64, C.c_int32, SmoothingElements,
                                      SmoothingElements, C.c_int32, C.c_int32, C.POINTER(ScanStats),
                                      C.POINTER(Status)]),
    "pode_rts": (C.c_int, [C.c_void_p, C.POINTER(Chain), RtsOut, C.POINTER(ScanStats),
                           C.POINTER(Status)]),
    "pode_ieks": (C.c_int, [C.c_void_p, C.POINTER(Problem), C.POINTER(Prior), dptr, C.c_int64,
                            C.POINTER(IeksConfig), C.POINTER(IeksReport), C.POINTER(Status)]),
    "pode_ieks_batch": (C.c_int, [C.c_void_p, C.POINTER(Problem), C.c_int32, C.POINTER(Prior), dptr, C.c_int64,
                                  C.POINTER(IeksConfig), C.POINTER(IeksReport), C.POINTER(Status)]),
    "pode_eks": (C.c_int, [C.c_void_p, C.POINTER(Problem), C.POINTER(Prior), dptr, C.c_int64, C.c_int32,
                           C.POINTER(IeksReport), C.POINTER(Status)]),
    "pode_rk4_table": (C.c_int, [C.c_void_p, C.POINTER(Problem), C.c_int64, dptr, C.POINTER(Status)]),
    "pode_shard_range": (None, [C.c_int64, C.c_int32, C.c_int32, C.POINTER(C.c_int64), C.POINTER(C.c_int64)]),
    "pode_ieks_sharded": (C.c_int, [C.c_void_p, C.POINTER(Problem), C.POINTER(Prior), dptr, C.c_int64,
                                    C.POINTER(IeksConfig), C.POINTER(ShardComm), C.POINTER(IeksReport),
                                    C.POINTER(Status)]),
}

_lib = None


def load():
    """Loads the CUDA library.  Fails loudly: there is no CPU fallback."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(os.environ.get("PODE_LIB_PATH") or LIB_PATH):
        raise ImportError(f"paraode_b200: CUDA library not built ({LIB_PATH}); run "
                          "`python -c 'import __graft_entry__ as g; g.build()'` (there is no CPU fallback)")
    path = os.environ.get("PODE_LIB_PATH") or LIB_PATH  # developer override (A/B builds)
    lib = C.CDLL(path)
    for name, (res, args) in SYMBOLS.items():
        fn = getattr(lib, name)
        fn.restype = res
        fn.argtypes = args
    _lib = lib
    return lib
