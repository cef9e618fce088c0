"""Python mirror of the reference's solver API for the ParaIEKS path.

Names, argument meaning and error behaviour follow proj/include/paraode/
(parallel.hpp, ieks.hpp, prior.hpp, problems.hpp, errors.hpp); every call runs
on the B200 through the C ABI (include/paraode_b200.h).  Matrices are
row-major numpy float64 arrays; arrays of elements / marginals stack along
axis 0.  There is no CPU fallback: without the CUDA library or a B200 every
call raises.
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass, field
from typing import Optional, Sequence

import numpy as np

from . import _abi as A


# ------------------------------------------------------------- errors ---
class SolverError(RuntimeError):
    """proj/include/paraode/errors.hpp:10-14"""


class InvalidInputError(SolverError):
    pass


class DimensionError(SolverError):
    pass


class SingularFactorError(SolverError):
    pass


class LinearizationError(SolverError):
    def __init__(self, what, time=0.0, index=0, iteration=0):
        super().__init__(what)
        self.time = time
        self.index = index
        self.iteration = iteration


class ScanError(SolverError):
    pass


class CudaError(SolverError):
    """No usable B200 / CUDA failure (the product path has no CPU fallback)."""


class UnsupportedError(SolverError):
    pass


_ERRORS = {1: InvalidInputError, 2: DimensionError, 3: SingularFactorError,
           4: LinearizationError, 5: ScanError, 6: CudaError, 7: UnsupportedError}


def _raise(rc: int, st: A.Status):
    if rc == 0:
        return
    cls = _ERRORS.get(rc, SolverError)
    msg = st.msg.decode(errors="replace")
    if cls is LinearizationError:
        raise LinearizationError(msg, st.time, st.index, st.iteration)
    raise cls(msg)


# ------------------------------------------------------------ context ---
class Context:
    """One GPU + one stream + cached device workspace (pode_context)."""

    def __init__(self, device: int = 0):
        self._lib = A.load()
        self._h = C.c_void_p()
        st = A.Status()
        _raise(self._lib.pode_context_create(device, C.byref(self._h), C.byref(st)), st)

    @property
    def handle(self):
        return self._h

    @property
    def kernel_launches(self) -> int:
        return int(self._lib.pode_kernel_launches(self._h))

    @property
    def stream(self) -> int:
        return int(self._lib.pode_context_stream(self._h) or 0)

    OPT_CHUNK_LEN, OPT_ENGINE = 1, 2
    ENGINES = {"auto": 0, "fused": 1, "elements": 2}

    def set_option(self, option: int, value: int):
        """pode_context_set_option: per-context engine knobs (chunk length of
        the fused engines; engine choice auto / fused / elements)."""
        rc = self._lib.pode_context_set_option(self._h, int(option), int(value))
        if rc != 0:
            raise InvalidInputError(f"pode_context_set_option({option}, {value}) rejected")

    def nccl_init(self, unique_id: bytes, rank: int, ranks: int, nccl_path: Optional[str] = None):
        """Bind an NCCL communicator (pode_context_nccl_init): the sharded
        solve then exchanges on the device (ncclAllGather), no host staging."""
        buf = (C.c_uint8 * 128).from_buffer_copy(bytes(unique_id))
        st = A.Status()
        _raise(self._lib.pode_context_nccl_init(self._h, _nccl_path(nccl_path), buf, int(rank), int(ranks),
                                                C.byref(st)), st)

    def set_chunk_len(self, steps: int):
        self.set_option(self.OPT_CHUNK_LEN, steps)

    def set_engine(self, name: str):
        self.set_option(self.OPT_ENGINE, self.ENGINES[name])

    def profile(self, enable: bool):
        """Start (clear) / stop per-kernel CUDA-event timing on the context stream."""
        self._lib.pode_profile(self._h, int(enable))

    def profile_read(self):
        """{kernel: (launches, total_ms)} recorded since profile(True)."""
        n = self._lib.pode_profile_read(self._h, None, 0)
        buf = C.create_string_buffer(int(n) + 1)
        self._lib.pode_profile_read(self._h, buf, int(n) + 1)
        out = {}
        for line in buf.value.decode().splitlines():
            name, cnt, ms = line.rsplit(" ", 2)
            out[name] = (int(cnt), float(ms))
        return out

    def close(self):
        if self._h:
            self._lib.pode_context_destroy(self._h)
            self._h = C.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


_default: Optional[Context] = None


def default_context() -> Context:
    global _default
    if _default is None:
        _default = Context(0)
    return _default


def _ctx(ctx):
    return (ctx or default_context())


def _p(a):
    if a is None:
        return None
    assert a.flags["C_CONTIGUOUS"]
    if a.dtype == np.float64:
        return a.ctypes.data_as(A.dptr)
    if a.dtype == np.int32:
        return a.ctypes.data_as(A.iptr)
    raise TypeError(a.dtype)


def _f64(a):
    return np.ascontiguousarray(a, dtype=np.float64)


_pinned_ok = None


def _result_array(shape):
    """float64 result array (every element is written by the solve) in
    page-locked host memory when torch's caching host allocator is available
    (the device->host copy of a solve's report then runs at full DMA rate
    straight into the array; freed blocks are reused by the next call), plain
    numpy otherwise.  PODE_PINNED=0 disables."""
    global _pinned_ok
    if _pinned_ok is None:
        import os
        _pinned_ok = False
        if os.environ.get("PODE_PINNED", "1") != "0":
            try:
                import torch
                _pinned_ok = bool(torch.cuda.is_available())
            except Exception:
                _pinned_ok = False
    n = int(np.prod(shape))
    if _pinned_ok and n * 8 >= (1 << 20):
        import torch
        return torch.empty(n, dtype=torch.float64, pin_memory=True).numpy().reshape(shape)
    return np.zeros(shape)


# ------------------------------------------------------- value types ---
@dataclass
class FilteringElements:
    """Array of FilteringElement (parallel.hpp:20-26)."""
    a: np.ndarray
    b: np.ndarray
    c_sqrt: np.ndarray
    eta: np.ndarray
    j_sqrt: np.ndarray

    @staticmethod
    def empty(n, d):
        z = np.zeros
        return FilteringElements(z((n, d, d)), z((n, d)), z((n, d, d)), z((n, d)), z((n, d, d)))

    @property
    def count(self):
        return self.a.shape[0]

    @property
    def state_dim(self):
        return self.a.shape[1]

    def _c(self):
        for k in ("a", "b", "c_sqrt", "eta", "j_sqrt"):
            setattr(self, k, _f64(getattr(self, k)))
        return A.FilteringElements(_p(self.a), _p(self.b), _p(self.c_sqrt), _p(self.eta), _p(self.j_sqrt))


@dataclass
class SmoothingElements:
    """Array of SmoothingElement (parallel.hpp:32-36)."""
    e: np.ndarray
    g: np.ndarray
    l_sqrt: np.ndarray

    @staticmethod
    def empty(n, d):
        return SmoothingElements(np.zeros((n, d, d)), np.zeros((n, d)), np.zeros((n, d, d)))

    @property
    def count(self):
        return self.e.shape[0]

    @property
    def state_dim(self):
        return self.e.shape[1]

    def _c(self):
        for k in ("e", "g", "l_sqrt"):
            setattr(self, k, _f64(getattr(self, k)))
        return A.SmoothingElements(_p(self.e), _p(self.g), _p(self.l_sqrt))


@dataclass
class LinearGaussianChain:
    """init + N transitions + N affine observations (the para_rts inputs,
    parallel.hpp:155-156).  Observation n uses obs_rows[n] rows of its
    M-row slot (0 = vacuous); phi / q_sqrt may be shared (2-D)."""
    init_mean: np.ndarray
    init_cov_sqrt: np.ndarray
    phi: np.ndarray
    q_sqrt: np.ndarray
    obs_rows: np.ndarray
    h: np.ndarray
    offset: np.ndarray
    r_sqrt: np.ndarray

    @property
    def state_dim(self):
        return int(np.asarray(self.init_mean).shape[0])

    @property
    def steps(self):
        return int(np.asarray(self.obs_rows).shape[0])

    def _c(self):
        self.init_mean = _f64(self.init_mean)
        self.init_cov_sqrt = _f64(self.init_cov_sqrt)
        self.phi = _f64(self.phi)
        self.q_sqrt = _f64(self.q_sqrt)
        self.obs_rows = np.ascontiguousarray(self.obs_rows, dtype=np.int32)
        self.h = _f64(self.h)
        self.offset = _f64(self.offset)
        self.r_sqrt = _f64(self.r_sqrt)
        m = self.h.shape[1] if self.h.ndim == 3 else 0
        return A.Chain(self.state_dim, m, self.steps, _p(self.init_mean), _p(self.init_cov_sqrt),
                       _p(self.phi), _p(self.q_sqrt), int(self.phi.ndim == 2), int(self.q_sqrt.ndim == 2),
                       _p(self.obs_rows), _p(self.h), _p(self.offset), _p(self.r_sqrt), A.PODE_HOST)


@dataclass
class RtsResult:
    """sequential.hpp:52-56 (marginals at nodes 0..N)."""
    filtered_mean: np.ndarray
    filtered_cov_sqrt: np.ndarray
    smoothed_mean: np.ndarray
    smoothed_cov_sqrt: np.ndarray
    combine_invocations: int = 0
    sequential_depth: int = 0


# ---------------------------------------------------- element operators ---
def make_filtering_elements(chain: LinearGaussianChain, absorb_init=True, ctx=None) -> FilteringElements:
    """make_filtering_element for every step (parallel.cpp:5-65)."""
    c = _ctx(ctx)
    out = FilteringElements.empty(chain.steps, chain.state_dim)
    ch = chain._c()
    st = A.Status()
    _raise(c._lib.pode_make_filtering_elements(c.handle, C.byref(ch), int(absorb_init), out._c(),
                                               C.byref(st)), st)
    return out


def combine_filtering(lhs: FilteringElements, rhs: FilteringElements, ctx=None) -> FilteringElements:
    """Batched ⊗_f: out[i] = lhs[i] ⊗ rhs[i] (parallel.cpp:67-100)."""
    c = _ctx(ctx)
    n, d = lhs.count, lhs.state_dim
    if rhs.count != n or rhs.state_dim != d:
        raise DimensionError("combine_filtering: element factors must be square")
    out = FilteringElements.empty(n, d)
    st = A.Status()
    _raise(c._lib.pode_combine_filtering(c.handle, n, d, lhs._c(), rhs._c(), out._c(), A.PODE_HOST,
                                         C.byref(st)), st)
    return out


def make_smoothing_elements(chain: LinearGaussianChain, f_mean, f_cov_sqrt, ctx=None) -> SmoothingElements:
    """Smoothing elements for nodes 0..N; node N terminal (parallel.cpp:112-144)."""
    c = _ctx(ctx)
    out = SmoothingElements.empty(chain.steps + 1, chain.state_dim)
    ch = chain._c()
    fm, fc = _f64(f_mean), _f64(f_cov_sqrt)
    st = A.Status()
    _raise(c._lib.pode_make_smoothing_elements(c.handle, C.byref(ch), _p(fm), _p(fc), out._c(), C.byref(st)), st)
    return out


def combine_smoothing(lhs: SmoothingElements, rhs: SmoothingElements, ctx=None) -> SmoothingElements:
    """Batched ⊗_s (parallel.cpp:146-156)."""
    c = _ctx(ctx)
    n, d = lhs.count, lhs.state_dim
    if rhs.count != n or rhs.state_dim != d:
        raise DimensionError("combine_smoothing: element dimensions disagree")
    out = SmoothingElements.empty(n, d)
    st = A.Status()
    _raise(c._lib.pode_combine_smoothing(c.handle, n, d, lhs._c(), rhs._c(), out._c(), A.PODE_HOST,
                                         C.byref(st)), st)
    return out


def associative_scan_filtering(elems: FilteringElements, reverse=False, ctx=None):
    """Inclusive scan under ⊗_f (associative_scan, parallel.hpp:136-149).
    Returns (prefixes, (combine_invocations, sequential_depth))."""
    c = _ctx(ctx)
    n, d = elems.count, elems.state_dim
    out = FilteringElements(*(np.array(x, dtype=np.float64, copy=True) for x in
                              (elems.a, elems.b, elems.c_sqrt, elems.eta, elems.j_sqrt)))
    st, stats = A.Status(), A.ScanStats()
    oc = out._c()
    _raise(c._lib.pode_scan_filtering(c.handle, n, d, oc, oc, int(reverse), A.PODE_HOST, C.byref(stats),
                                      C.byref(st)), st)
    return out, (stats.combine_invocations, stats.sequential_depth)


def associative_scan_smoothing(elems: SmoothingElements, reverse=True, ctx=None):
    c = _ctx(ctx)
    n, d = elems.count, elems.state_dim
    out = SmoothingElements(*(np.array(x, dtype=np.float64, copy=True) for x in (elems.e, elems.g, elems.l_sqrt)))
    st, stats = A.Status(), A.ScanStats()
    oc = out._c()
    _raise(c._lib.pode_scan_smoothing(c.handle, n, d, oc, oc, int(reverse), A.PODE_HOST, C.byref(stats),
                                      C.byref(st)), st)
    return out, (stats.combine_invocations, stats.sequential_depth)


def para_rts(chain: LinearGaussianChain, ctx=None) -> RtsResult:
    """Time-parallel square-root filter + smoother (para_rts, parallel.cpp:166-209)."""
    c = _ctx(ctx)
    n1, d = chain.steps + 1, chain.state_dim
    r = RtsResult(np.zeros((n1, d)), np.zeros((n1, d, d)), np.zeros((n1, d)), np.zeros((n1, d, d)))
    ch = chain._c()
    st, stats = A.Status(), A.ScanStats()
    out = A.RtsOut(_p(r.filtered_mean), _p(r.filtered_cov_sqrt), _p(r.smoothed_mean), _p(r.smoothed_cov_sqrt))
    _raise(c._lib.pode_rts(c.handle, C.byref(ch), out, C.byref(stats), C.byref(st)), st)
    r.combine_invocations, r.sequential_depth = stats.combine_invocations, stats.sequential_depth
    return r


# -------------------------------------------------------------- solver ---
@dataclass
class IwpPrior:
    """prior.hpp:12-18"""
    nu: int = 1
    dim: int = 1
    sigma: float = 1.0

    @property
    def state_dim(self):
        return self.dim * (self.nu + 1)


@dataclass
class IeksConfig:
    """ieks.hpp:32-38"""
    max_iterations: int = 100
    traj_rtol: float = 1e-13
    obj_atol: float = 1e-9
    obj_rtol: float = 1e-6
    linearization: str = "ek1"


@dataclass
class InitialValueProblem:
    """A registered device vector field (replaces statespace.hpp:24-31)."""
    kind: int
    dim: int
    t_end: float
    y0: np.ndarray
    params: np.ndarray = field(default_factory=lambda: np.zeros(0))
    name: str = ""

    def _c(self):
        self.y0 = _f64(self.y0)
        self.params = _f64(self.params)
        return A.Problem(self.kind, self.dim, self.t_end, _p(self.y0),
                         _p(self.params) if self.params.size else None, int(self.params.size))


def logistic():
    return InitialValueProblem(1, 1, 10.0, np.array([0.01]), name="logistic")


def rigid_body():
    return InitialValueProblem(2, 3, 20.0, np.array([1.0, 0.0, 0.9]), name="rigidbody")


def van_der_pol(mu=1.0):
    return InitialValueProblem(3, 2, 6.3, np.array([2.0, 0.0]), np.array([mu]), name="vanderpol")


def fitzhugh_nagumo(a=0.2, b=0.2, c=3.0):
    return InitialValueProblem(4, 2, 20.0, np.array([-1.0, 1.0]), np.array([a, b, c]), name="fhn")


def pleiades():
    y0 = [3, 3, -1, -3, 2, -2, 2, 3, -3, 2, 0, 0, -4, 4, 0, 0, 0, 0, 0, 1.75, -1.5, 0, 0, 0, -1.25, 1, 0, 0]
    return InitialValueProblem(5, 28, 3.0, np.array(y0, dtype=np.float64), name="pleiades")


def pole(a=0.75, t_end=1.0, y0=0.0):
    """y' = 1 / (t - a): finite Taylor initialisation, non-finite field at t = a
    (the reference's LinearizationError case, test_statespace.cpp:123-139)."""
    return InitialValueProblem(7, 1, t_end, np.array([y0], dtype=np.float64), np.array([a], dtype=np.float64),
                               name="pole")


def affine(l, c, y0, t_end):
    l = np.asarray(l, dtype=np.float64)
    return InitialValueProblem(6, len(y0), t_end, np.asarray(y0, dtype=np.float64),
                               np.concatenate([l.ravel(), np.asarray(c, dtype=np.float64)]), name="affine")


def problem_by_name(name):
    """problems.cpp:190-195 (+ fhn, pleiades)."""
    table = {"logistic": logistic, "rigidbody": rigid_body, "vanderpol": van_der_pol,
             "fhn": fitzhugh_nagumo, "pleiades": pleiades}
    if name not in table:
        raise InvalidInputError(f"unknown problem '{name}'")
    return table[name]()


def uniform_grid(t_end, steps):
    """problems.cpp:212-221"""
    if steps < 1 or not t_end > 0:
        raise InvalidInputError("uniform_grid: need steps >= 1 and t_end > 0")
    n = np.arange(steps + 1, dtype=np.float64)
    return t_end * n / steps


@dataclass
class SolverReport:
    """ieks.hpp:77-87"""
    times: np.ndarray
    means: np.ndarray
    cov_sqrt: Optional[np.ndarray]
    solution_means: np.ndarray
    solution_covs: Optional[np.ndarray]
    sigma_hat: float
    iterations: int
    objective_trace: np.ndarray
    converged: bool
    combine_invocations: int
    sequential_depth: int


def para_ieks(ivp: InitialValueProblem, prior: IwpPrior, grid: Sequence[float],
              config: IeksConfig = IeksConfig(), want_cov=True, ctx=None) -> SolverReport:
    """Iterated extended Kalman smoother on the B200 (para_ieks, ieks.cpp:114-217)."""
    c = _ctx(ctx)
    grid = _f64(grid)
    n1 = grid.shape[0]
    D, d = prior.state_dim, prior.dim
    means = _result_array((n1, D))
    cov = _result_array((n1, D, D)) if want_cov else None
    sm = _result_array((n1, d))
    sc = _result_array((n1, d, d)) if want_cov else None
    trace = np.zeros(max(config.max_iterations, 1))
    rep = A.IeksReport(_p(means), _p(cov), _p(sm), _p(sc), _p(trace), trace.shape[0], A.PODE_HOST,
                       0, 0, 0.0, A.ScanStats())
    pr = ivp._c()
    prior_c = A.Prior(prior.nu, prior.dim, prior.sigma)
    lin = {"ek1": 0, "ek0": 1}[config.linearization]
    cfg = A.IeksConfig(config.max_iterations, config.traj_rtol, config.obj_atol, config.obj_rtol, lin)
    st = A.Status()
    _raise(c._lib.pode_ieks(c.handle, C.byref(pr), C.byref(prior_c), _p(grid), n1, C.byref(cfg),
                            C.byref(rep), C.byref(st)), st)
    return SolverReport(grid.copy(), means, cov, sm, sc, rep.sigma_hat, rep.iterations,
                        trace[:rep.iterations].copy(), bool(rep.converged),
                        rep.scan_stats.combine_invocations, rep.scan_stats.sequential_depth)


def eks_solve(ivp: InitialValueProblem, prior: IwpPrior, grid: Sequence[float], linearization: str = "ek1",
              want_cov=True, ctx=None) -> SolverReport:
    """Non-iterated extended Kalman smoother on the B200 (eks_solve,
    ieks.cpp:224-291): each step is linearised at its own predicted mean in
    one sequential forward pass (one warp), then smoothed by the reverse scan
    and calibrated.  iterations = 1, converged = True."""
    c = _ctx(ctx)
    grid = _f64(grid)
    n1 = grid.shape[0]
    D, d = prior.state_dim, prior.dim
    means = _result_array((n1, D))
    cov = _result_array((n1, D, D)) if want_cov else None
    sm = _result_array((n1, d))
    sc = _result_array((n1, d, d)) if want_cov else None
    trace = np.zeros(1)
    rep = A.IeksReport(_p(means), _p(cov), _p(sm), _p(sc), _p(trace), 1, A.PODE_HOST, 0, 0, 0.0, A.ScanStats())
    pr = ivp._c()
    prior_c = A.Prior(prior.nu, prior.dim, prior.sigma)
    st = A.Status()
    _raise(c._lib.pode_eks(c.handle, C.byref(pr), C.byref(prior_c), _p(grid), n1,
                           {"ek1": 0, "ek0": 1}[linearization], C.byref(rep), C.byref(st)), st)
    return SolverReport(grid.copy(), means, cov, sm, sc, rep.sigma_hat, rep.iterations, trace.copy(),
                        bool(rep.converged), rep.scan_stats.combine_invocations, rep.scan_stats.sequential_depth)


# ---------------------------------------------------- batched solves ---
_batch_pools: dict = {}  # device -> (lock, [Context]); a batch call holds its device's lock


def para_ieks_fused_batch(problems: Sequence[InitialValueProblem], prior: IwpPrior, grid: Sequence[float],
                          config: IeksConfig = IeksConfig(), want_cov=True, ctx=None):
    """Many IVPs of one field kind and dimension (free parameters and initial
    values, one prior / grid / config) solved as ONE fused solve on the
    device (pode_ieks_batch): every Gauss-Newton iteration is one pass
    sequence over all IVPs' time chunks, each IVP stopping on its own by the
    reference's rule (ieks.cpp:157-187).  Report i is what para_ieks would
    return for problems[i]."""
    c = _ctx(ctx)
    problems = list(problems)
    if not problems:
        return []
    grid = _f64(grid)
    n1 = grid.shape[0]
    D, d = prior.state_dim, prior.dim
    nb = len(problems)
    outs, reps = [], (A.IeksReport * nb)()
    for i in range(nb):
        means = _result_array((n1, D))
        cov = _result_array((n1, D, D)) if want_cov else None
        sm = _result_array((n1, d))
        sc = _result_array((n1, d, d)) if want_cov else None
        trace = np.zeros(max(config.max_iterations, 1))
        reps[i] = A.IeksReport(_p(means), _p(cov), _p(sm), _p(sc), _p(trace), trace.shape[0], A.PODE_HOST,
                               0, 0, 0.0, A.ScanStats())
        outs.append((means, cov, sm, sc, trace))
    probs = (A.Problem * nb)()
    keep = []  # the problems' y0/params buffers stay alive through the call
    for i, p in enumerate(problems):
        probs[i] = p._c()
        keep.append(p)
    prior_c = A.Prior(prior.nu, prior.dim, prior.sigma)
    lin = {"ek1": 0, "ek0": 1}[config.linearization]
    cfg = A.IeksConfig(config.max_iterations, config.traj_rtol, config.obj_atol, config.obj_rtol, lin)
    st = A.Status()
    _raise(c._lib.pode_ieks_batch(c.handle, probs, nb, C.byref(prior_c), _p(grid), n1, C.byref(cfg), reps,
                                  C.byref(st)), st)
    res = []
    for i in range(nb):
        means, cov, sm, sc, trace = outs[i]
        r = reps[i]
        res.append(SolverReport(grid.copy(), means, cov, sm, sc, r.sigma_hat, r.iterations,
                                trace[:r.iterations].copy(), bool(r.converged),
                                r.scan_stats.combine_invocations, r.scan_stats.sequential_depth))
    return res


def para_ieks_batch(problems: Sequence[InitialValueProblem], prior: IwpPrior, grid: Sequence[float],
                    config: IeksConfig = IeksConfig(), want_cov=True, streams: int = 8, device: int = 0,
                    fused: bool = False):
    """Independent IVP solves (e.g. a parameter or initial-value sweep).
    fused=True: one fused device solve over all IVPs (para_ieks_fused_batch;
    one field kind, lane engine).  Otherwise `streams` host threads, each
    driving its own context (CUDA stream + workspace) through para_ieks, so
    small-N solves — latency-bound one at a time — overlap on the GPU; each
    report then equals the single para_ieks call bit for bit.  Reports are
    in input order."""
    import threading
    problems = list(problems)
    if not problems:
        return []
    if fused:
        lock, ctxs = _batch_pools.setdefault(int(device), (threading.Lock(), []))
        with lock:
            if not ctxs:
                ctxs.append(Context(device))
            return para_ieks_fused_batch(problems, prior, grid, config, want_cov, ctx=ctxs[0])
    streams = max(1, min(int(streams), len(problems)))
    lock, ctxs = _batch_pools.setdefault(int(device), (threading.Lock(), []))
    with lock:  # contexts are not reentrant: one batch per device at a time
        while len(ctxs) < streams:
            ctxs.append(Context(device))
        return _run_batch(problems, prior, grid, config, want_cov, ctxs[:streams])


def _run_batch(problems, prior, grid, config, want_cov, ctxs):
    import threading
    streams = len(ctxs)
    out = [None] * len(problems)
    errors = []

    def worker(w):
        ctx = ctxs[w]
        for i in range(w, len(problems), streams):
            try:
                out[i] = para_ieks(problems[i], prior, grid, config, want_cov=want_cov, ctx=ctx)
            except Exception as e:  # re-raised on the caller's thread
                errors.append((i, e))
                return

    threads = [threading.Thread(target=worker, args=(w,)) for w in range(streams)]
    for t in threads:
        t.start()
    for t in threads:
        t.join()
    if errors:
        raise min(errors, key=lambda x: x[0])[1]
    return out


# ------------------------------------------------ time-axis sharding ---
def shard_range(n_nodes: int, rank: int, ranks: int):
    """(first node, reported node count) of shard `rank` (pode_shard_range)."""
    lo, cnt = C.c_int64(), C.c_int64()
    A.load().pode_shard_range(n_nodes, rank, ranks, C.byref(lo), C.byref(cnt))
    return lo.value, cnt.value


def torch_allgather(group=None):
    """All-gather adapter over torch.distributed for para_ieks_sharded: gloo
    gathers host tensors; nccl gathers on the current CUDA device."""
    import torch
    import torch.distributed as dist

    def gather(send: np.ndarray) -> np.ndarray:
        ranks = dist.get_world_size(group)
        t = torch.from_numpy(np.ascontiguousarray(send))
        if dist.get_backend(group) == "nccl":
            t = t.cuda()
        out = torch.empty(ranks * t.numel(), dtype=t.dtype, device=t.device)
        dist.all_gather_into_tensor(out, t, group=group)
        return out.cpu().numpy()
    return gather


def _nccl_path(path=None):
    """libnccl.so.2: explicit, else the one torch bundles (nvidia/nccl/lib)."""
    if path:
        return path.encode()
    import os
    try:
        import torch
        cand = os.path.join(os.path.dirname(torch.__file__), "..", "nvidia", "nccl", "lib", "libnccl.so.2")
        if os.path.exists(cand):
            return os.path.abspath(cand).encode()
    except Exception:
        pass
    return None


def nccl_unique_id(nccl_path: Optional[str] = None) -> bytes:
    """A fresh 128-byte ncclUniqueId (pode_nccl_unique_id)."""
    buf = (C.c_uint8 * 128)()
    st = A.Status()
    _raise(A.load().pode_nccl_unique_id(_nccl_path(nccl_path), buf, C.byref(st)), st)
    return bytes(buf)


def torch_nccl_bind(ctx, group=None, nccl_path: Optional[str] = None):
    """Device-side shard exchange for para_ieks_sharded: rank 0 makes the
    NCCL id, torch.distributed broadcasts it, every rank binds its context."""
    import torch.distributed as dist
    rank, ranks = dist.get_rank(group), dist.get_world_size(group)
    obj = [nccl_unique_id(nccl_path) if rank == 0 else None]
    dist.broadcast_object_list(obj, src=0, group=group)
    ctx.nccl_init(obj[0], rank, ranks, nccl_path)


def make_shard_comm(rank: int, ranks: int, allgather):
    """pode_shard_comm for a Python all-gather (send ndarray -> rank-ordered
    ndarray).  Returns (comm, failures); keep comm alive during the call."""
    failure = []

    def cb(_user, send, count, recv):
        try:
            snd = np.ctypeslib.as_array(send, shape=(count,)).copy()
            got = np.asarray(allgather(snd), dtype=np.float64).reshape(-1)
            if got.shape[0] != count * ranks:
                raise ValueError(f"all-gather returned {got.shape[0]} values, want {count * ranks}")
            np.ctypeslib.as_array(recv, shape=(count * ranks,))[:] = got
            return 0
        except Exception as e:  # reported through the ABI as a failed exchange
            failure.append(e)
            return 1

    comm = A.ShardComm(rank, ranks, A.ALLGATHER_FN(cb), None)
    comm._keep = cb
    return comm, failure


@dataclass
class ShardReport:
    """This shard's part of a SolverReport: nodes first_node .. first_node +
    means.shape[0] - 1; the scalars are those of the whole solve."""
    first_node: int
    times: np.ndarray
    means: np.ndarray
    cov_sqrt: Optional[np.ndarray]
    solution_means: np.ndarray
    solution_covs: Optional[np.ndarray]
    sigma_hat: float
    iterations: int
    objective_trace: np.ndarray
    converged: bool


def para_ieks_sharded(ivp: InitialValueProblem, prior: IwpPrior, grid: Sequence[float], rank: int, ranks: int,
                      allgather, config: IeksConfig = IeksConfig(), want_cov=True, ctx=None) -> ShardReport:
    """para_ieks over the time-axis shard `rank` of `ranks` (one process per
    GPU).  `allgather(send: ndarray) -> ndarray` gathers every
    rank's equally sized float64 vector in rank order (torch_allgather());
    None when the context has an NCCL communicator (torch_nccl_bind): the
    exchanges then stay on the device."""
    c = _ctx(ctx)
    grid = _f64(grid)
    n1 = grid.shape[0]
    D, d = prior.state_dim, prior.dim
    first, cnt = shard_range(n1, rank, ranks)
    means = _result_array((cnt, D))
    cov = _result_array((cnt, D, D)) if want_cov else None
    sm = _result_array((cnt, d))
    sc = _result_array((cnt, d, d)) if want_cov else None
    trace = np.zeros(max(config.max_iterations, 1))
    rep = A.IeksReport(_p(means), _p(cov), _p(sm), _p(sc), _p(trace), trace.shape[0], A.PODE_HOST,
                       0, 0, 0.0, A.ScanStats())
    if allgather is None:
        comm, failure = A.ShardComm(rank, ranks, A.ALLGATHER_FN(), None), []
    else:
        comm, failure = make_shard_comm(rank, ranks, allgather)
    pr = ivp._c()
    prior_c = A.Prior(prior.nu, prior.dim, prior.sigma)
    lin = {"ek1": 0, "ek0": 1}[config.linearization]
    cfg = A.IeksConfig(config.max_iterations, config.traj_rtol, config.obj_atol, config.obj_rtol, lin)
    st = A.Status()
    rc = c._lib.pode_ieks_sharded(c.handle, C.byref(pr), C.byref(prior_c), _p(grid), n1, C.byref(cfg),
                                  C.byref(comm), C.byref(rep), C.byref(st))
    if failure:
        raise failure[0]
    _raise(rc, st)
    return ShardReport(first, grid[first:first + cnt].copy(), means, cov, sm, sc, rep.sigma_hat, rep.iterations,
                       trace[:rep.iterations].copy(), bool(rep.converged))
