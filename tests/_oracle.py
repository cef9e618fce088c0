"""ctypes wrapper over oracle/_build/liborc.so — TEST INFRASTRUCTURE ONLY.

The oracle is the C++ restatement of the reference CPU path (see
oracle/orc.hpp).  This module is the checker's handle: tests compare the
product (paraode_b200, the CUDA path behind include/paraode_b200.h) against
it, and bench.py times it as the CPU baseline.  Nothing under
paraode_b200/ may import this module.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
LIB_PATH = os.path.join(ROOT, "oracle", "_build", "liborc.so")

dptr = C.POINTER(C.c_double)
iptr = C.POINTER(C.c_int32)
lptr = C.POINTER(C.c_int64)


class Status(C.Structure):
    _fields_ = [("code", C.c_int32), ("iteration", C.c_int32), ("index", C.c_int64),
                ("time", C.c_double), ("msg", C.c_char * 256)]


class FE(C.Structure):
    _fields_ = [("a", dptr), ("b", dptr), ("c_sqrt", dptr), ("eta", dptr), ("j_sqrt", dptr)]


class SE(C.Structure):
    _fields_ = [("e", dptr), ("g", dptr), ("l_sqrt", dptr)]


class Chain(C.Structure):
    _fields_ = [("state_dim", C.c_int32), ("obs_rows_max", C.c_int32), ("steps", C.c_int64),
                ("init_mean", dptr), ("init_cov_sqrt", dptr), ("phi", dptr), ("q_sqrt", dptr),
                ("phi_shared", C.c_int32), ("q_shared", C.c_int32), ("obs_rows", iptr),
                ("h", dptr), ("offset", dptr), ("r_sqrt", dptr)]


class RtsOut(C.Structure):
    _fields_ = [("filtered_mean", dptr), ("filtered_cov_sqrt", dptr),
                ("smoothed_mean", dptr), ("smoothed_cov_sqrt", dptr)]


class ScanStats(C.Structure):
    _fields_ = [("combine_invocations", C.c_int64), ("sequential_depth", C.c_int64)]


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
                ("iterations", C.c_int32), ("converged", C.c_int32), ("sigma_hat", C.c_double),
                ("scan_stats", ScanStats), ("seconds", C.c_double)]


ERRORS = {1: "InvalidInputError", 2: "DimensionError", 3: "SingularFactorError",
          4: "LinearizationError", 5: "ScanError", 9: "SolverError"}


class OracleError(RuntimeError):
    def __init__(self, code, msg, time=0.0, index=-1, iteration=0):
        super().__init__(f"{ERRORS.get(code, code)}: {msg}")
        self.code = code
        self.kind = ERRORS.get(code, "SolverError")
        self.time, self.index, self.iteration = time, index, iteration


_lib = None


def build():
    subprocess.run(["make", "-s", "-C", os.path.join(ROOT, "oracle")], check=True)


def lib():
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            build()
        _lib = C.CDLL(LIB_PATH)
        _lib.orc_rng_new.restype = C.c_void_p
        _lib.orc_rng_new.argtypes = [C.c_uint32]
        _lib.orc_rng_free.argtypes = [C.c_void_p]
        for name in ("orc_rng_matrix", "orc_rng_vector", "orc_rng_spd_sqrt",
                     "orc_rng_filtering_element", "orc_rng_smoothing_element",
                     "orc_rng_transition", "orc_rng_observation"):
            getattr(_lib, name).restype = None
    return _lib


def P(a):
    """Pointer to a C-contiguous float64 (or int) numpy array (None → NULL)."""
    if a is None:
        return None
    assert a.flags["C_CONTIGUOUS"], "array must be C-contiguous"
    if a.dtype == np.float64:
        return a.ctypes.data_as(dptr)
    if a.dtype == np.int32:
        return a.ctypes.data_as(iptr)
    if a.dtype == np.int64:
        return a.ctypes.data_as(lptr)
    raise TypeError(a.dtype)


def _check(rc, st):
    if rc != 0:
        raise OracleError(st.code, st.msg.decode(errors="replace"), st.time, st.index, st.iteration)


# ------------------------------------------------------------ containers ---
class FilteringElements:
    """Arrays of FilteringElement (parallel.hpp:20-26), row-major per field."""

    def __init__(self, n, d, a=None, b=None, c=None, eta=None, j=None):
        self.n, self.d = n, d
        self.a = np.zeros((n, d, d)) if a is None else np.ascontiguousarray(a, dtype=np.float64)
        self.b = np.zeros((n, d)) if b is None else np.ascontiguousarray(b, dtype=np.float64)
        self.c = np.zeros((n, d, d)) if c is None else np.ascontiguousarray(c, dtype=np.float64)
        self.eta = np.zeros((n, d)) if eta is None else np.ascontiguousarray(eta, dtype=np.float64)
        self.j = np.zeros((n, d, d)) if j is None else np.ascontiguousarray(j, dtype=np.float64)

    def struct(self):
        return FE(P(self.a), P(self.b), P(self.c), P(self.eta), P(self.j))

    def __getitem__(self, s):
        return FilteringElements(len(self.a[s]), self.d, self.a[s], self.b[s], self.c[s],
                                 self.eta[s], self.j[s])


class SmoothingElements:
    def __init__(self, n, d, e=None, g=None, l=None):
        self.n, self.d = n, d
        self.e = np.zeros((n, d, d)) if e is None else np.ascontiguousarray(e, dtype=np.float64)
        self.g = np.zeros((n, d)) if g is None else np.ascontiguousarray(g, dtype=np.float64)
        self.l = np.zeros((n, d, d)) if l is None else np.ascontiguousarray(l, dtype=np.float64)

    def struct(self):
        return SE(P(self.e), P(self.g), P(self.l))

    def __getitem__(self, s):
        return SmoothingElements(len(self.e[s]), self.d, self.e[s], self.g[s], self.l[s])


class ChainData:
    """A linear-Gaussian chain (init, N transitions, N observations)."""

    def __init__(self, init_mean, init_cov, phi, q, obs_rows, h, offset, r):
        self.init_mean = np.ascontiguousarray(init_mean, dtype=np.float64)
        self.init_cov = np.ascontiguousarray(init_cov, dtype=np.float64)
        self.phi = np.ascontiguousarray(phi, dtype=np.float64)
        self.q = np.ascontiguousarray(q, dtype=np.float64)
        self.obs_rows = np.ascontiguousarray(obs_rows, dtype=np.int32)
        self.h = np.ascontiguousarray(h, dtype=np.float64)
        self.offset = np.ascontiguousarray(offset, dtype=np.float64)
        self.r = np.ascontiguousarray(r, dtype=np.float64)
        self.d = self.init_mean.shape[0]
        self.n = self.obs_rows.shape[0]
        self.m = self.h.shape[1]

    def struct(self):
        return Chain(self.d, self.m, self.n, P(self.init_mean), P(self.init_cov), P(self.phi),
                     P(self.q), int(self.phi.ndim == 2), int(self.q.ndim == 2), P(self.obs_rows),
                     P(self.h), P(self.offset), P(self.r))

    def observation(self, i):
        m = int(self.obs_rows[i])
        return self.h[i, :m], self.offset[i, :m], self.r[i, :m, :m]

    def transition(self, i):
        phi = self.phi if self.phi.ndim == 2 else self.phi[i]
        q = self.q if self.q.ndim == 2 else self.q[i]
        return phi, q


# ------------------------------------------------------------ fixtures ---
class Rng:
    """std::mt19937 draw stream with the reference's generators
    (proj/tests/oracles.cpp:168-229)."""

    def __init__(self, seed):
        self._h = C.c_void_p(lib().orc_rng_new(seed))

    def __del__(self):
        try:
            lib().orc_rng_free(self._h)
        except Exception:
            pass

    def matrix(self, rows, cols):
        out = np.zeros((rows, cols))
        lib().orc_rng_matrix(self._h, rows, cols, P(out))
        return out

    def vector(self, n):
        out = np.zeros(n)
        lib().orc_rng_vector(self._h, n, P(out))
        return out

    def spd_sqrt(self, n):
        out = np.zeros((n, n))
        lib().orc_rng_spd_sqrt(self._h, n, P(out))
        return out

    def filtering_element(self, n):
        a, b, c, eta, j = np.zeros((n, n)), np.zeros(n), np.zeros((n, n)), np.zeros(n), np.zeros((n, n))
        lib().orc_rng_filtering_element(self._h, n, P(a), P(b), P(c), P(eta), P(j))
        return a, b, c, eta, j

    def smoothing_element(self, n):
        e, g, l = np.zeros((n, n)), np.zeros(n), np.zeros((n, n))
        lib().orc_rng_smoothing_element(self._h, n, P(e), P(g), P(l))
        return e, g, l

    def transition(self, n):
        phi, q = np.zeros((n, n)), np.zeros((n, n))
        lib().orc_rng_transition(self._h, n, P(phi), P(q))
        return phi, q

    def observation(self, rows, n, noiseless):
        h, off, r = np.zeros((rows, n)), np.zeros(rows), np.zeros((rows, rows))
        lib().orc_rng_observation(self._h, rows, n, int(noiseless), P(h), P(off), P(r))
        return h, off, r


def random_elements(rng, count, d):
    fe = FilteringElements(count, d)
    for i in range(count):
        fe.a[i], fe.b[i], fe.c[i], fe.eta[i], fe.j[i] = rng.filtering_element(d)
    return fe


def random_smoothing_elements(rng, count, d):
    se = SmoothingElements(count, d)
    for i in range(count):
        se.e[i], se.g[i], se.l[i] = rng.smoothing_element(d)
    return se


def random_chain(d, n, seed, vacuous="mod4", m=None):
    """test_parallel.cpp:40-54 (vacuous="mod4": k % 4 == 2 vacuous) or
    test_sequential.cpp:21-40 (vacuous="mod3": k % 3 == 1; None: never)."""
    rng = Rng(seed)
    rows = m if m is not None else (d - 1 if d > 1 else 1)
    init_mean = rng.vector(d)
    init_cov = rng.spd_sqrt(d)
    phis, qs, ms, hs, offs, rs = [], [], [], [], [], []
    for k in range(n):
        phi, q = rng.transition(d)
        phis.append(phi)
        qs.append(q)
        vac = (vacuous == "mod4" and k % 4 == 2) or (vacuous == "mod3" and k % 3 == 1)
        if vac:
            ms.append(0)
            hs.append(np.zeros((rows, d)))
            offs.append(np.zeros(rows))
            rs.append(np.zeros((rows, rows)))
        else:
            h, off, r = rng.observation(rows, d, k % 2 == 0)
            ms.append(rows)
            hs.append(h)
            offs.append(off)
            rs.append(r)
    return ChainData(init_mean, init_cov, np.array(phis), np.array(qs), np.array(ms),
                     np.array(hs), np.array(offs), np.array(rs))


# ------------------------------------------------------------- calls ---
def tria(m):
    m = np.ascontiguousarray(m, dtype=np.float64)
    rows, cols = m.shape
    out = np.zeros((rows, rows))
    st = Status()
    _check(lib().orc_tria(P(m), rows, cols, P(out), C.byref(st)), st)
    return out


def make_filtering_elements(chain, absorb_init=True):
    out = FilteringElements(chain.n, chain.d)
    st = Status()
    cs = chain.struct()
    _check(lib().orc_make_filtering_elements(C.byref(cs), out.struct(), int(absorb_init), C.byref(st)), st)
    return out


def combine_filtering(lhs, rhs):
    out = FilteringElements(lhs.n, lhs.d)
    st = Status()
    _check(lib().orc_combine_filtering(C.c_int64(lhs.n), lhs.d, lhs.struct(), rhs.struct(),
                                       out.struct(), C.byref(st)), st)
    return out


def make_smoothing_elements(chain, f_mean, f_cov):
    out = SmoothingElements(chain.n + 1, chain.d)
    st = Status()
    cs = chain.struct()
    f_mean = np.ascontiguousarray(f_mean)
    f_cov = np.ascontiguousarray(f_cov)
    _check(lib().orc_make_smoothing_elements(C.byref(cs), P(f_mean), P(f_cov), out.struct(),
                                             C.byref(st)), st)
    return out


def combine_smoothing(lhs, rhs):
    out = SmoothingElements(lhs.n, lhs.d)
    st = Status()
    _check(lib().orc_combine_smoothing(C.c_int64(lhs.n), lhs.d, lhs.struct(), rhs.struct(),
                                       out.struct(), C.byref(st)), st)
    return out


def scan_filtering(el, reverse=False):
    out = FilteringElements(el.n, el.d)
    st, stats = Status(), ScanStats()
    _check(lib().orc_scan_filtering(C.c_int64(el.n), el.d, el.struct(), out.struct(), int(reverse),
                                    C.byref(stats), C.byref(st)), st)
    return out, (stats.combine_invocations, stats.sequential_depth)


def scan_smoothing(el, reverse=True):
    out = SmoothingElements(el.n, el.d)
    st, stats = Status(), ScanStats()
    _check(lib().orc_scan_smoothing(C.c_int64(el.n), el.d, el.struct(), out.struct(), int(reverse),
                                    C.byref(stats), C.byref(st)), st)
    return out, (stats.combine_invocations, stats.sequential_depth)


def scan_int_add(xs, reverse=False):
    xs = np.ascontiguousarray(xs, dtype=np.int64)
    out = np.zeros_like(xs)
    st, stats = Status(), ScanStats()
    _check(lib().orc_scan_int_add(C.c_int64(len(xs)), P(xs), P(out), int(reverse), C.byref(stats),
                                  C.byref(st)), st)
    return out, (stats.combine_invocations, stats.sequential_depth)


def rts(chain, mode=0):
    """mode 0: seq_rts; 1: para_rts (serial pool); k>1: para_rts on WorkPool(k)."""
    n, d = chain.n, chain.d
    fm, fc = np.zeros((n + 1, d)), np.zeros((n + 1, d, d))
    sm, sc = np.zeros((n + 1, d)), np.zeros((n + 1, d, d))
    st, stats = Status(), ScanStats()
    cs = chain.struct()
    _check(lib().orc_rts(C.byref(cs), RtsOut(P(fm), P(fc), P(sm), P(sc)), mode, C.byref(stats),
                         C.byref(st)), st)
    return dict(filtered_mean=fm, filtered_cov=fc, smoothed_mean=sm, smoothed_cov=sc,
                stats=(stats.combine_invocations, stats.sequential_depth))


KIND = {"logistic": 1, "rigidbody": 2, "vanderpol": 3, "fhn": 4, "pleiades": 5, "affine": 6, "pole": 7}
SHIPPED = {  # name: (kind, dim, t_end, y0)
    "logistic": (1, 1, 10.0, [0.01]),
    "rigidbody": (2, 3, 20.0, [1.0, 0.0, 0.9]),
    "vanderpol": (3, 2, 6.3, [2.0, 0.0]),
    "fhn": (4, 2, 20.0, [-1.0, 1.0]),
    "pleiades": (5, 28, 3.0, [3, 3, -1, -3, 2, -2, 2, 3, -3, 2, 0, 0, -4, 4,
                              0, 0, 0, 0, 0, 1.75, -1.5, 0, 0, 0, -1.25, 1, 0, 0]),
}


class ProblemSpec:
    def __init__(self, kind, dim, t_end, y0, params=()):
        self.kind, self.dim, self.t_end = kind, dim, t_end
        self.y0 = np.ascontiguousarray(y0, dtype=np.float64)
        self.params = np.ascontiguousarray(params, dtype=np.float64) if len(params) else None

    def struct(self):
        return Problem(self.kind, self.dim, self.t_end, P(self.y0), P(self.params),
                       0 if self.params is None else len(self.params))


def problem(name):
    kind, dim, t_end, y0 = SHIPPED[name]
    return ProblemSpec(kind, dim, t_end, y0)


def affine_problem(l, c, y0, t_end):
    l = np.asarray(l, dtype=np.float64)
    return ProblemSpec(6, len(y0), t_end, y0, np.concatenate([l.ravel(), np.asarray(c, float)]))


def uniform_grid(t_end, steps):
    return np.array([t_end * n / steps for n in range(steps + 1)], dtype=np.float64)


def ieks(prob, nu, grid, mode=0, sigma=1.0, max_iterations=100, traj_rtol=1e-13, obj_atol=1e-9,
         obj_rtol=1e-6, ek0=False, want_cov=True):
    """mode 0: seq_ieks; 1: para_ieks (serial pool); k>1: WorkPool(k); -1: eks_solve."""
    grid = np.ascontiguousarray(grid, dtype=np.float64)
    n1 = len(grid)
    D, d = prob.dim * (nu + 1), prob.dim
    means = np.zeros((n1, D))
    cov = np.zeros((n1, D, D)) if want_cov else None
    sol_m = np.zeros((n1, d))
    sol_c = np.zeros((n1, d, d)) if want_cov else None
    trace = np.zeros(max(max_iterations, 1))
    rep = IeksReport(P(means), P(cov), P(sol_m), P(sol_c), P(trace), len(trace), 0, 0, 0.0,
                     ScanStats(), 0.0)
    st = Status()
    pr = prob.struct()
    prior = Prior(nu, prob.dim, sigma)
    cfg = IeksConfig(max_iterations, traj_rtol, obj_atol, obj_rtol, int(ek0))
    _check(lib().orc_ieks(C.byref(pr), C.byref(prior), P(grid), C.c_int64(n1), C.byref(cfg), mode,
                          C.byref(rep), C.byref(st)), st)
    return dict(means=means, cov_sqrt=cov, solution_means=sol_m, solution_covs=sol_c,
                objective_trace=trace[:rep.iterations].copy(), iterations=rep.iterations,
                converged=bool(rep.converged), sigma_hat=rep.sigma_hat, seconds=rep.seconds,
                scan_stats=(rep.scan_stats.combine_invocations, rep.scan_stats.sequential_depth))


def taylor_init(prob, nu):
    out = np.zeros(prob.dim * (nu + 1))
    st = Status()
    pr = prob.struct()
    _check(lib().orc_taylor_init(C.byref(pr), nu, P(out), C.byref(st)), st)
    return out


def iwp_transition(nu, dim, sigma, h):
    D = dim * (nu + 1)
    phi, q = np.zeros((D, D)), np.zeros((D, D))
    st = Status()
    prior = Prior(nu, dim, sigma)
    _check(lib().orc_iwp_transition(C.byref(prior), C.c_double(h), P(phi), P(q), C.byref(st)), st)
    return phi, q


def preconditioner(nu, dim, h):
    D = dim * (nu + 1)
    s, si = np.zeros(D), np.zeros(D)
    st = Status()
    prior = Prior(nu, dim, 1.0)
    _check(lib().orc_preconditioner(C.byref(prior), C.c_double(h), P(s), P(si), C.byref(st)), st)
    return s, si


def preconditioned_pair(nu, dim):
    D = dim * (nu + 1)
    phi, q = np.zeros((D, D)), np.zeros((D, D))
    st = Status()
    prior = Prior(nu, dim, 1.0)
    _check(lib().orc_preconditioned_pair(C.byref(prior), P(phi), P(q), C.byref(st)), st)
    return phi, q


def linearize(prob, nu, eta, t, ek0=False):
    eta = np.ascontiguousarray(eta, dtype=np.float64)
    h, off = np.zeros((prob.dim, len(eta))), np.zeros(prob.dim)
    st = Status()
    pr = prob.struct()
    _check(lib().orc_linearize(C.byref(pr), nu, P(eta), C.c_double(t), int(ek0), P(h), P(off),
                               C.byref(st)), st)
    return h, off


def field(prob, y, t=0.0):
    y = np.ascontiguousarray(y, dtype=np.float64)
    f, jac = np.zeros(prob.dim), np.zeros((prob.dim, prob.dim))
    st = Status()
    pr = prob.struct()
    _check(lib().orc_field(C.byref(pr), P(y), C.c_double(t), P(f), P(jac), C.byref(st)), st)
    return f, jac


def discretize(nu, dim, grid, sigma=1.0):
    grid = np.ascontiguousarray(grid, dtype=np.float64)
    D = dim * (nu + 1)
    n1 = len(grid)
    scale, phi, q = np.zeros((n1, D)), np.zeros((n1 - 1, D, D)), np.zeros((D, D))
    st = Status()
    prior = Prior(nu, dim, sigma)
    _check(lib().orc_discretize(C.byref(prior), P(grid), C.c_int64(n1), P(scale), P(phi), P(q),
                                C.byref(st)), st)
    return scale, phi, q


def objective(states, phi, q_sqrt):
    states = np.ascontiguousarray(states, dtype=np.float64)
    phi = np.ascontiguousarray(phi, dtype=np.float64)
    q_sqrt = np.ascontiguousarray(q_sqrt, dtype=np.float64)
    v = C.c_double()
    st = Status()
    _check(lib().orc_objective(C.c_int64(states.shape[0]), states.shape[1], P(states), P(phi),
                               int(phi.ndim == 2), P(q_sqrt), C.byref(v), C.byref(st)), st)
    return v.value


def innovation_stats(chain, f_mean, f_cov):
    s, cnt = C.c_double(), C.c_int64()
    st = Status()
    cs = chain.struct()
    f_mean = np.ascontiguousarray(f_mean)
    f_cov = np.ascontiguousarray(f_cov)
    _check(lib().orc_innovation_stats(C.byref(cs), P(f_mean), P(f_cov), C.byref(s), C.byref(cnt),
                                      C.byref(st)), st)
    return s.value, cnt.value
