"""GPU fault paths through the C ABI: the device error word (atomicMin of
index << 8 | code, capi.cu) mapped onto the reference's exception types
(proj/include/paraode/errors.hpp:10-60), each case checked against the
oracle raising the same type on the same input.

  * SingularFactorError — a zero-valued (not zero-row) H with R = 0
    (test_sequential.cpp:117-124), through pode_rts / para_rts.
  * LinearizationError(time, index) — a non-finite field value
    (test_statespace.cpp:123-139), through pode_ieks on both engines
    and pode_eks; the failing node's time, the iteration
    in the message (ieks.cpp:165-168).
  * ScanError("elements [") — a combine that fails inside a scan
    (test_parallel.cpp:246-256), through pode_scan_filtering.
  * InvalidInputError — a field that is not finite at the initial point
    (taylor_init, prior.cpp:139-141).
"""
import numpy as np
import pytest

import _oracle as O

pytestmark = pytest.mark.gpu

P = pytest.importorskip("paraode_b200")


def zero_h_chain(d=2, n=5, bad=2):
    """test_sequential.cpp:117-124 inside a chain: step `bad` observes a
    zero-valued H with R = 0 (S = 0: singular innovation factor)."""
    ch = O.random_chain(d, n, 31, vacuous=None, m=1)
    ch.h[bad] = 0.0
    ch.r[bad] = 0.0
    return ch


def test_rts_zero_h_singular_factor():
    ch = zero_h_chain()
    for mode in (0, 1, 4):  # seq_rts, para_rts serial and pooled
        with pytest.raises(O.OracleError) as e:
            O.rts(ch, mode=mode)
        assert e.value.kind == "SingularFactorError"
    chain = P.LinearGaussianChain(ch.init_mean, ch.init_cov, ch.phi, ch.q, ch.obs_rows, ch.h, ch.offset, ch.r)
    with pytest.raises(P.SingularFactorError):
        P.para_rts(chain)
    with pytest.raises(P.SingularFactorError):
        P.make_filtering_elements(chain)
    # the same chain with that step's observation made valid again solves
    ch.h[2, 0, 0], ch.r[2, 0, 0] = 1.0, 0.5
    chain = P.LinearGaussianChain(ch.init_mean, ch.init_cov, ch.phi, ch.q, ch.obs_rows, ch.h, ch.offset, ch.r)
    got, want = P.para_rts(chain), O.rts(ch, mode=0)
    assert np.max(np.abs(got.smoothed_mean - want["smoothed_mean"])) <= 1e-9


@pytest.mark.parametrize("engine", ["fused", "elements"])
@pytest.mark.parametrize("nu", [1, 2])
def test_ieks_linearization_error_time_and_index(engine, nu, monkeypatch):
    """y' = 1 / (t - 0.75) on 64 steps of [0, 1]: finite Taylor start, the
    field is non-finite at node 48 (t = 0.75) in iteration 1."""
    if engine == "elements":
        monkeypatch.setenv("PODE_IEKS_ENGINE", "elements")
    grid = O.uniform_grid(1.0, 64)
    for mode in (0, 4):  # seq_ieks, para_ieks on WorkPool(4)
        with pytest.raises(O.OracleError) as e:
            O.ieks(O.ProblemSpec(7, 1, 1.0, [0.0], [0.75]), nu, grid, mode=mode)
        assert e.value.kind == "LinearizationError" and e.value.time == 0.75
        assert "ieks iteration 1" in str(e.value)
    with pytest.raises(P.LinearizationError) as g:
        P.para_ieks(P.pole(0.75), P.IwpPrior(nu, 1, 1.0), grid)
    err = g.value
    assert err.time == 0.75 and err.index == 48 and err.iteration == 1
    assert "ieks iteration 1" in str(err) and "not finite" in str(err)
    # the context stays usable after the device error
    ok = P.para_ieks(P.pole(0.7501), P.IwpPrior(nu, 1, 1.0), grid)
    want = O.ieks(O.ProblemSpec(7, 1, 1.0, [0.0], [0.7501]), nu, grid, mode=0)
    assert ok.iterations == want["iterations"]
    assert np.max(np.abs(ok.means - want["means"])) <= 1e-9 * max(1.0, np.abs(want["means"]).max())


def test_eks_linearization_error():
    grid = O.uniform_grid(1.0, 64)
    with pytest.raises(O.OracleError) as e:
        O.ieks(O.ProblemSpec(7, 1, 1.0, [0.0], [0.75]), 2, grid, mode=-1)
    assert e.value.kind == "LinearizationError" and e.value.time == 0.75
    with pytest.raises(P.LinearizationError) as g:
        P.eks_solve(P.pole(0.75), P.IwpPrior(2, 1, 1.0), grid)
    assert g.value.time == 0.75 and g.value.index == 48


def test_taylor_init_not_finite_is_invalid_input():
    grid = O.uniform_grid(1.0, 16)
    with pytest.raises(O.OracleError) as e:  # pole at t = 0: 1 / (0 - 0)
        O.ieks(O.ProblemSpec(7, 1, 1.0, [0.0], [0.0]), 2, grid)
    assert e.value.kind == "InvalidInputError"
    with pytest.raises(P.InvalidInputError, match="not finite at the initial point"):
        P.para_ieks(P.pole(0.0), P.IwpPrior(2, 1, 1.0), grid)


def poisoned_elements(n=64, d=3, k=37):
    """Random elements (seed 44) where element k-1 carries C = 1e9 I and
    element k a J with one 1e9 entry: C^T J = 1e18 e_0 e_0^T makes the
    combination factor Xi_11 = tria([C^T J, I]) singular at the 1e-13
    threshold (linalg.cpp:54-62) whenever they meet."""
    fe = O.random_elements(O.Rng(44), n, d)
    fe.c[k - 1] = 1e9 * np.eye(d)
    fe.j[k] = 0.0
    fe.j[k][0, 0] = 1e9
    return fe


@pytest.mark.parametrize("reverse", [False, True])
def test_scan_error_names_the_element_range(reverse):
    """Forward and reverse scans both meet element 36 ⊗ element 37 (operands
    stay in time order, parallel.hpp:144-148)."""
    fe = poisoned_elements()
    with pytest.raises(O.OracleError) as e:
        O.scan_filtering(fe, reverse=reverse)
    assert e.value.kind == "ScanError" and "elements [" in str(e.value)
    with pytest.raises(P.ScanError, match=r"elements \[") as g:
        P.associative_scan_filtering(P.FilteringElements(fe.a, fe.b, fe.c, fe.eta, fe.j), reverse=reverse)
    lo, hi = [int(x) for x in str(g.value).split("elements [")[1].split("]")[0].split(",")]
    assert 0 <= lo <= hi < 64
    # the single combine raises SingularFactorError, as combine_filtering does
    one = lambda k: P.FilteringElements(fe.a[k:k + 1], fe.b[k:k + 1], fe.c[k:k + 1], fe.eta[k:k + 1], fe.j[k:k + 1])
    with pytest.raises(P.SingularFactorError):
        P.combine_filtering(one(36), one(37))
    with pytest.raises(O.OracleError) as e:
        O.combine_filtering(fe[36:37], fe[37:38])
    assert e.value.kind == "SingularFactorError"


def test_fused_batch_linearization_error_and_recovery():
    """A batch whose third member has its pole on node 48 raises the
    reference's LinearizationError (time 0.75, iteration 1); the same
    context then solves a clean batch at the oracle's iterates."""
    grid = O.uniform_grid(1.0, 64)
    bad = [P.pole(0.7501), P.pole(0.7502), P.pole(0.75), P.pole(0.7503)]
    with pytest.raises(P.LinearizationError) as g:
        P.para_ieks_fused_batch(bad, P.IwpPrior(2, 1, 1.0), grid)
    assert g.value.time == 0.75 and g.value.index == 48 and g.value.iteration == 1
    good = [P.pole(0.7501), P.pole(0.7502)]
    got = P.para_ieks_fused_batch(good, P.IwpPrior(2, 1, 1.0), grid)
    for p, r in zip((0.7501, 0.7502), got):
        want = O.ieks(O.ProblemSpec(7, 1, 1.0, [0.0], [p]), 2, grid, mode=0)
        assert r.iterations == want["iterations"]
        assert np.max(np.abs(r.means - want["means"])) <= 1e-9 * max(1.0, np.abs(want["means"]).max())
