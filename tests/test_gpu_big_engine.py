"""The large-state fused IEKS engine (big.cuh; Pleiades, d = 28, IWP(1..3),
D = 56..112, BASELINE.json configs[4]) against the sequential oracle
(seq_ieks, proj/src/ieks.cpp:219-222): equal iteration counts, means per
derivative order, covariance products L L^T and sigma_hat, under several
chunkings (one CTA per chunk; the chunk chains of passes B / D / F3)."""
import json
import os
import re

import numpy as np
import pytest

import _oracle as O
from _parity import NEVER, alternatives, compare, gpu_solve

pytestmark = pytest.mark.gpu

P = pytest.importorskip("paraode_b200")
GOLDEN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")


def as_fixture(want, nodes=None):
    nodes = np.arange(len(want["means"])) if nodes is None else nodes
    L = want["cov_sqrt"][nodes]
    cov = np.einsum("nij,nkj->nik", L, L)
    iu = np.triu_indices(cov.shape[1])
    return dict(nodes=nodes, means=want["means"][nodes], cov_upper=cov[:, iu[0], iu[1]],
                objective_trace=want["objective_trace"])


@pytest.mark.parametrize("chunk", [0, 1, 5, 1000])
@pytest.mark.parametrize("nu,steps,its", [(1, 48, 3), (2, 40, 2), (3, 64, 2)])
def test_pleiades_matches_seq_ieks(nu, steps, its, chunk):
    op = O.problem("pleiades")
    grid = O.uniform_grid(op.t_end, steps)
    want = O.ieks(op, nu, grid, mode=0, max_iterations=its, **NEVER)
    ctx = P.Context()
    ctx.set_chunk_len(chunk)
    meta = dict(problem="pleiades", nu=nu, t_end=op.t_end, steps=steps, iterations=its,
                sigma_hat=want["sigma_hat"])
    got = gpu_solve(P, meta, ctx=ctx, max_iterations=its, **NEVER)
    assert np.allclose(got.objective_trace, want["objective_trace"], rtol=1e-8)
    compare(got, as_fixture(want), meta, f"pleiades q{nu} N={steps} L={chunk}")
    assert np.all(np.isfinite(got.solution_covs))


@pytest.mark.parametrize("name", ["pleiades_q3_n10_seq_it3", "pleiades_q3_n12_seq_it2"])
def test_pleiades_fixture(name):
    """N = 2^10 (3 iterations) and 2^12 (2 iterations), the SURVEY.md §8(d)
    parity sizes, at equal iteration counts against the committed oracle
    fixtures (tools/make_fixtures.py)."""
    path = os.path.join(GOLDEN, name + ".npz")
    if not os.path.exists(path):
        pytest.skip("fixture not generated")
    z = np.load(path)
    meta = json.loads(str(z["meta"]))
    got = gpu_solve(P, meta, max_iterations=meta["iterations"], **NEVER)
    # The objective after the first iteration from the constant start is a
    # sum of whitened residuals x_{k+1} - phi x_k of nearly equal numbers:
    # at N = 2^12 it is rounding-determined at ~1e-4 — the oracle's own
    # seq_ieks and para_ieks (WorkPool(8), fixture *_par8_*) differ by 3.3e-4
    # there.  Where that fixture exists the tolerance is twice the
    # reference's own seq/par spread (never below 1e-8).
    rtol = np.full(len(z["objective_trace"]), 1e-8)
    alt = os.path.join(GOLDEN, name.replace("_seq_", "_par8_") + ".npz")
    if os.path.exists(alt):
        zp = np.load(alt)
        spread = np.abs(zp["objective_trace"] - z["objective_trace"]) / np.abs(z["objective_trace"])
        rtol = np.maximum(rtol, 2 * spread)
    dev = np.abs(got.objective_trace - z["objective_trace"]) / np.abs(z["objective_trace"])
    print(f"{name}: objective rel dev {dev}, tolerance {rtol}")
    assert np.all(dev <= rtol)
    compare(got, z, meta, f"pleiades q3 N={meta['steps']} (fixture)", alternatives(P, meta, meta["iterations"]))


def test_pleiades_default_rule_outcome_matches_oracle():
    """The reference stopping rule on Pleiades from the constant initial
    trajectory (ieks.cpp:145-148) at N = 2^10: the oracle's seq_ieks does not
    converge within the 100-iteration budget — the Gauss-Newton iterates
    diverge (objective ~1e19).  The traces agree while the iterates are still
    determined (first 3 iterations to 1e-8; tools/pleiades_chaos.py shows
    the departure growing from ~1e-7 at iteration 8 to O(1) by iteration 16:
    from there the iterates are decided by rounding, in the oracle as on the
    GPU).  Outcome parity is therefore "no convergence": the GPU either
    exhausts the budget like the oracle, or its rounding-decided iterates hit
    the reference's singular-factor test (linalg.cpp:54-62) after the
    departure point — never a convergence and never an error while the
    iterates are determined."""
    path = os.path.join(GOLDEN, "pleiades_q3_n10_seq.npz")
    if not os.path.exists(path):
        pytest.skip("fixture not generated")
    z = np.load(path)
    meta = json.loads(str(z["meta"]))
    assert not meta["converged"] and meta["iterations"] == meta["max_iterations"]
    early = gpu_solve(P, meta, max_iterations=3, **NEVER)
    assert np.allclose(early.objective_trace, z["objective_trace"][:3], rtol=1e-8)
    try:
        conv = gpu_solve(P, meta)
    except P.SingularFactorError as e:
        m = re.search(r"iteration (\d+)", str(e))
        assert m and int(m.group(1)) > 16, str(e)
        print(f"pleiades q3 N=2^10 default rule: GPU singular factor after the departure ({e}); "
              f"oracle {meta['iterations']} its conv={meta['converged']}")
        return
    print(f"pleiades q3 N=2^10 default rule: GPU {conv.iterations} its conv={conv.converged}; "
          f"oracle {meta['iterations']} its conv={meta['converged']}; final objective GPU "
          f"{conv.objective_trace[-1]:.3e}, oracle {z['objective_trace'][-1]:.3e}")
    assert not conv.converged and conv.iterations == meta["iterations"]
    assert np.allclose(conv.objective_trace[:3], z["objective_trace"][:3], rtol=1e-8)


def test_pleiades_errors_and_determinism():
    grid = O.uniform_grid(3.0, 64)
    a = P.para_ieks(P.pleiades(), P.IwpPrior(3, 28, 1.0), grid, P.IeksConfig(max_iterations=2))
    b = P.para_ieks(P.pleiades(), P.IwpPrior(3, 28, 1.0), grid, P.IeksConfig(max_iterations=2))
    assert np.array_equal(a.means, b.means) and np.array_equal(a.cov_sqrt, b.cov_sqrt)
    with pytest.raises(P.UnsupportedError):
        P.eks_solve(P.pleiades(), P.IwpPrior(3, 28, 1.0), grid)
