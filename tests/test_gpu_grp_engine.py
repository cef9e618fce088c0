"""The group-of-D-lanes fused IEKS engine (grp_fused.cuh; D = 10..16, e.g.
rigid body IWP(4), D = 15) against the sequential oracle (seq_ieks,
proj/src/ieks.cpp:219-222): equal iteration counts, means 1e-9, covariance
products 1e-7, sigma_hat 1e-7 — under every chunking shape (one chunk,
ragged last chunks, multi-level aggregate scans) and against the element
engine (the reference's per-iteration structure)."""
import numpy as np
import pytest

import _oracle as O
from _dense import dense_cov
from _parity import NEVER, alternatives, compare, gpu_solve

pytestmark = pytest.mark.gpu

P = pytest.importorskip("paraode_b200")


def rel(a, b):
    a, b = np.asarray(a), np.asarray(b)
    return float(np.max(np.abs(a - b)) / max(1.0, np.max(np.abs(b))))


def check_floor(got, want, meta, label):
    """As check(), with the per-derivative-order rounding floor of
    _parity.compare (high IWP orders at small h are rounding-determined in the
    reference formulation too)."""
    z = dict(nodes=np.arange(len(want["means"])), means=want["means"],
             cov_upper=None, objective_trace=want["objective_trace"])
    L = want["cov_sqrt"]
    cov = np.einsum("nij,nkj->nik", L, L)
    iu = np.triu_indices(cov.shape[1])
    z["cov_upper"] = cov[:, iu[0], iu[1]]
    m = dict(meta, iterations=want["iterations"], sigma_hat=want["sigma_hat"])
    compare(got, z, m, label, alternatives(P, m, want["iterations"]))


def check(got, want):
    print(f"its {got.iterations}/{want['iterations']} conv {got.converged}/{want['converged']} "
          f"means {rel(got.means, want['means']):.2e} cov {rel(dense_cov(got.cov_sqrt), dense_cov(want['cov_sqrt'])):.2e} "
          f"sigma {abs(got.sigma_hat / want['sigma_hat'] - 1):.2e}")
    assert got.converged == want["converged"]
    assert got.iterations == want["iterations"]
    assert rel(got.means, want["means"]) <= 1e-9
    assert rel(dense_cov(got.cov_sqrt), dense_cov(want["cov_sqrt"])) <= 1e-7
    assert got.sigma_hat == pytest.approx(want["sigma_hat"], rel=1e-7)
    assert rel(got.solution_means, want["solution_means"]) <= 1e-9
    assert rel(got.solution_covs, want["solution_covs"]) <= 1e-7


CASES = [("rigidbody", 4, 300), ("rigidbody", 3, 200), ("vanderpol", 4, 200), ("vanderpol", 5, 120),
         ("rigidbody", 4, 37)]


@pytest.mark.parametrize("chunk", [0, 2, 3, 7, 64, 100000])
@pytest.mark.parametrize("name,nu,steps", CASES)
def test_group_engine_matches_seq_ieks(name, nu, steps, chunk):
    op = O.problem(name)
    grid = O.uniform_grid(op.t_end, steps)
    want = O.ieks(op, nu, grid, mode=0)
    ctx = P.Context()
    ctx.set_engine("fused")  # the group engine must serve these dimensions (no element fallback)
    ctx.set_chunk_len(chunk)
    got = P.para_ieks(P.problem_by_name(name), P.IwpPrior(nu, op.dim, 1.0), grid, ctx=ctx)
    assert got.iterations == want["iterations"] and got.converged == want["converged"]
    meta = dict(problem=name, nu=nu, t_end=op.t_end, steps=steps)
    check_floor(got, want, meta, f"{name} q{nu} N={steps} L={chunk}")


def test_group_engine_rigid_2e12_equal_iterations():
    """BASELINE.json configs[3] shape (rigid body, IWP(4), D = 15) at N = 2^12
    with the default chunking: the oracle's converged posterior, compared at
    its iteration count (at this step size the stopping rule is decided by
    the objective's rounding noise: the default-rule counts are printed)."""
    op = O.problem("rigidbody")
    grid = O.uniform_grid(op.t_end, 2 ** 12)
    want = O.ieks(op, 4, grid, mode=0)
    meta = dict(problem="rigidbody", nu=4, t_end=op.t_end, steps=2 ** 12)
    got = gpu_solve(P, meta, max_iterations=want["iterations"], **NEVER)
    conv = gpu_solve(P, meta)
    print(f"rigid q4 N=2^12: oracle {want['iterations']} its conv={want['converged']}, "
          f"GPU default rule {conv.iterations} its conv={conv.converged}")
    check_floor(got, want, meta, "rigid q4 N=2^12")


def test_group_engine_deterministic_and_fault_paths():
    grid = O.uniform_grid(20.0, 1000)
    a = P.para_ieks(P.rigid_body(), P.IwpPrior(4, 3, 1.0), grid)
    b = P.para_ieks(P.rigid_body(), P.IwpPrior(4, 3, 1.0), grid)
    assert a.iterations == b.iterations
    assert np.array_equal(a.means, b.means) and np.array_equal(a.cov_sqrt, b.cov_sqrt)
