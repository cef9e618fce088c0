"""GPU parity: the CUDA path (through the C ABI, paraode_b200) against the
oracle (oracle/, the C++ restatement of the reference) and the independent
numpy dense oracles, on the reference's own fixtures (same std::mt19937
seeds) and on the ODE configurations.  Tolerances follow the reference's
tests (1e-9 / 1e-10 element and smoother gates, test_parallel.cpp) and the
north star (means 1e-9 rel, covariance products 1e-7 rel, equal
iteration counts)."""
import numpy as np
import pytest

import _oracle as O
from _dense import dense_combine, dense_cov, dense_element, dense_joint_posterior, densify, max_abs_diff

pytestmark = pytest.mark.gpu

P = pytest.importorskip("paraode_b200")


def to_chain(ch: O.ChainData):
    return P.LinearGaussianChain(ch.init_mean, ch.init_cov, ch.phi, ch.q, ch.obs_rows, ch.h, ch.offset, ch.r)


def gfe(fe: O.FilteringElements):
    return P.FilteringElements(fe.a, fe.b, fe.c, fe.eta, fe.j)


def gse(se: O.SmoothingElements):
    return P.SmoothingElements(se.e, se.g, se.l)


def rel(a, b):
    a, b = np.asarray(a), np.asarray(b)
    return float(np.max(np.abs(a - b)) / max(1.0, np.max(np.abs(b))))


# --------------------------------------------------------- operators ---
@pytest.mark.parametrize("d", [1, 2, 3, 4, 6, 8, 15])
def test_combine_filtering_matches_oracle_and_dense(d):  # test_parallel.cpp:118-127 (seed 42)
    rng = O.Rng(42)
    n = 64
    lhs, rhs = O.random_elements(rng, n, d), O.random_elements(rng, n, d)
    got = P.combine_filtering(gfe(lhs), gfe(rhs))
    want = O.combine_filtering(lhs, rhs)
    assert max_abs_diff(got.a, want.a) <= 1e-11 * max(1, np.abs(want.a).max())
    assert max_abs_diff(got.b, want.b) <= 1e-11 * max(1, np.abs(want.b).max())
    assert max_abs_diff(dense_cov(got.c_sqrt), dense_cov(want.c)) <= 1e-10 * max(1, np.abs(dense_cov(want.c)).max())
    assert max_abs_diff(got.eta, want.eta) <= 1e-10 * max(1, np.abs(want.eta).max())
    assert max_abs_diff(dense_cov(got.j_sqrt), dense_cov(want.j)) <= 1e-10 * max(1, np.abs(dense_cov(want.j)).max())
    assert np.all(np.triu(got.c_sqrt, 1) == 0) and np.all(np.triu(got.j_sqrt, 1) == 0)
    if d == 3:  # the reference's own gate against dense_combine, 1e-9
        for i in range(20):
            w = dense_combine(densify(lhs.a[i], lhs.b[i], lhs.c[i], lhs.eta[i], lhs.j[i]),
                              densify(rhs.a[i], rhs.b[i], rhs.c[i], rhs.eta[i], rhs.j[i]))
            assert max_abs_diff(got.a[i], w[0]) <= 1e-9
            assert max_abs_diff(dense_cov(got.c_sqrt[i]), w[2]) <= 1e-9
            assert max_abs_diff(dense_cov(got.j_sqrt[i]), w[4]) <= 1e-9


def test_filtering_identity_two_sided():  # test_parallel.cpp:129-136 (seed 43)
    el = O.random_elements(O.Rng(43), 1, 4)
    ident = O.FilteringElements(1, 4)
    ident.a[0] = np.eye(4)
    for got in (P.combine_filtering(gfe(ident), gfe(el)), P.combine_filtering(gfe(el), gfe(ident))):
        assert max_abs_diff(got.a, el.a) <= 1e-12
        assert max_abs_diff(got.b, el.b) <= 1e-12
        assert max_abs_diff(dense_cov(got.c_sqrt), dense_cov(el.c)) <= 1e-12
        assert max_abs_diff(got.eta, el.eta) <= 1e-12
        assert max_abs_diff(dense_cov(got.j_sqrt), dense_cov(el.j)) <= 1e-12


@pytest.mark.parametrize("d", [2, 3, 6, 8])
def test_combine_smoothing_matches_oracle(d):  # test_parallel.cpp:293-312 (seed 47)
    rng = O.Rng(47)
    lhs, rhs = O.random_smoothing_elements(rng, 50, d), O.random_smoothing_elements(rng, 50, d)
    got = P.combine_smoothing(gse(lhs), gse(rhs))
    want = O.combine_smoothing(lhs, rhs)
    assert max_abs_diff(got.e, want.e) <= 1e-12 * max(1, np.abs(want.e).max())
    assert max_abs_diff(got.g, want.g) <= 1e-12 * max(1, np.abs(want.g).max())
    assert max_abs_diff(dense_cov(got.l_sqrt), dense_cov(want.l)) <= 1e-11 * max(1, np.abs(dense_cov(want.l)).max())


def test_operator_algebra_acceptance():  # acceptance.cpp:295-354 (criterion 8, seed 202) on the GPU
    rng = O.Rng(202)
    n = 200
    a, b, c = (O.random_elements(rng, n, 3) for _ in range(3))
    ab = P.combine_filtering(gfe(a), gfe(b))
    left = P.combine_filtering(ab, gfe(c))
    bc = P.combine_filtering(gfe(b), gfe(c))
    right = P.combine_filtering(gfe(a), bc)
    worst = max(max_abs_diff(left.a, right.a), max_abs_diff(left.b, right.b),
                max_abs_diff(dense_cov(left.c_sqrt), dense_cov(right.c_sqrt)),
                max_abs_diff(left.eta, right.eta), max_abs_diff(dense_cov(left.j_sqrt), dense_cov(right.j_sqrt)))
    assert worst <= 1e-9


# ---------------------------------------------------------- elements ---
@pytest.mark.parametrize("d,n,seed,vac", [(3, 13, 45, "mod4"), (2, 9, 48, "mod4"), (3, 17, 49, "mod4"),
                                          (3, 10, 33, "mod3"), (5, 40, 7, None)])
def test_elements_match_oracle(d, n, seed, vac):  # parallel.cpp:5-65, 112-144
    ch = O.random_chain(d, n, seed, vacuous=vac)
    got = P.make_filtering_elements(to_chain(ch))
    want = O.make_filtering_elements(ch)
    assert max_abs_diff(got.a, want.a) <= 1e-11
    assert max_abs_diff(got.b, want.b) <= 1e-11
    assert max_abs_diff(dense_cov(got.c_sqrt), dense_cov(want.c)) <= 1e-11
    assert max_abs_diff(got.eta, want.eta) <= 1e-10
    assert max_abs_diff(dense_cov(got.j_sqrt), dense_cov(want.j)) <= 1e-10
    seq = O.rts(ch, mode=0)
    gs = P.make_smoothing_elements(to_chain(ch), seq["filtered_mean"], seq["filtered_cov"])
    ws = O.make_smoothing_elements(ch, seq["filtered_mean"], seq["filtered_cov"])
    assert max_abs_diff(gs.e, ws.e) <= 1e-10
    assert max_abs_diff(gs.g, ws.g) <= 1e-10
    assert max_abs_diff(dense_cov(gs.l_sqrt), dense_cov(ws.l)) <= 1e-10


def test_element_vs_first_principles():  # test_parallel.cpp:58-79 (seed 41) against dense_element
    rng = O.Rng(41)
    phi, q = rng.transition(3)
    h, off, r = rng.observation(2, 3, False)
    ch = O.ChainData(np.zeros(3), np.zeros((3, 3)), phi[None], q[None], [2], h[None], off[None], r[None])
    got = P.make_filtering_elements(to_chain(ch), absorb_init=False)
    want = dense_element(phi, q, h, off, r)
    assert max_abs_diff(got.a[0], want[0]) <= 1e-10
    assert max_abs_diff(got.b[0], want[1]) <= 1e-10
    assert max_abs_diff(dense_cov(got.c_sqrt[0]), want[2]) <= 1e-10
    assert max_abs_diff(got.eta[0], want[3]) <= 1e-10
    assert max_abs_diff(dense_cov(got.j_sqrt[0]), want[4]) <= 1e-10


# ------------------------------------------------------------- scans ---
@pytest.mark.parametrize("n", [1, 2, 3, 5, 8, 13, 64, 257, 1000, 4099])
def test_scan_filtering_prefixes(n):  # test_parallel.cpp:156-177, 214-244
    ch = O.random_chain(3, n, 45 + n)
    el = O.make_filtering_elements(ch)
    got, (work, depth) = P.associative_scan_filtering(gfe(el))
    seq = O.rts(ch, mode=0)
    assert rel(got.b, seq["filtered_mean"][1:]) <= 1e-9
    assert rel(dense_cov(got.c_sqrt), dense_cov(seq["filtered_cov"][1:])) <= 1e-9
    if n >= 2:
        assert work <= 2 * n - 2 + 2 * int(np.ceil(n / 4))  # reduce-then-scan tally


@pytest.mark.parametrize("n", [1, 2, 9, 100, 3001])
def test_scan_smoothing_suffixes(n):  # test_parallel.cpp:314-336
    ch = O.random_chain(2, n, 48 + n)
    seq = O.rts(ch, mode=0)
    se = O.make_smoothing_elements(ch, seq["filtered_mean"], seq["filtered_cov"])
    got, _ = P.associative_scan_smoothing(gse(se), reverse=True)
    assert rel(got.g, seq["smoothed_mean"]) <= 1e-9
    assert rel(dense_cov(got.l_sqrt), dense_cov(seq["smoothed_cov"])) <= 1e-9


def test_scan_order_noncommutative_and_deterministic():  # parallel.hpp:81-85, acceptance.cpp:356-381
    rng = O.Rng(202)
    el = O.random_elements(rng, 333, 2)
    for rev in (False, True):
        got1, _ = P.associative_scan_filtering(gfe(el), reverse=rev)
        got2, _ = P.associative_scan_filtering(gfe(el), reverse=rev)
        want, _ = O.scan_filtering(el, reverse=rev)
        assert np.array_equal(got1.a, got2.a) and np.array_equal(got1.c_sqrt, got2.c_sqrt)
        for f in ("a", "b", "eta"):
            w = getattr(want, {"a": "a", "b": "b", "eta": "eta"}[f])
            assert rel(getattr(got1, f), w) <= 1e-8
        assert rel(dense_cov(got1.c_sqrt), dense_cov(want.c)) <= 1e-8
        assert rel(dense_cov(got1.j_sqrt), dense_cov(want.j)) <= 1e-8


# -------------------------------------------------------------- rts ---
@pytest.mark.parametrize("d,n,seed,vac", [(3, 17, 49, "mod4"), (2, 1, 50, "mod4"), (3, 11, 51, "mod4"),
                                          (4, 500, 9, "mod3"), (6, 2000, 10, None), (8, 777, 11, "mod4")])
def test_para_rts_matches_seq_rts(d, n, seed, vac):  # test_parallel.cpp:338-362
    ch = O.random_chain(d, n, seed, vacuous=vac)
    got = P.para_rts(to_chain(ch))
    seq = O.rts(ch, mode=0)
    assert rel(got.filtered_mean, seq["filtered_mean"]) <= 1e-9
    assert rel(dense_cov(got.filtered_cov_sqrt), dense_cov(seq["filtered_cov"])) <= 1e-9
    assert rel(got.smoothed_mean, seq["smoothed_mean"]) <= 1e-9
    assert rel(dense_cov(got.smoothed_cov_sqrt), dense_cov(seq["smoothed_cov"])) <= 1e-9
    if n == 1:
        assert np.array_equal(got.filtered_mean[1], got.smoothed_mean[1])


def test_para_rts_vs_dense_joint_posterior():  # oracles.cpp:84-129, the strongest oracle
    ch = O.random_chain(3, 12, 77, vacuous="mod3")
    got = P.para_rts(to_chain(ch))
    joint = dense_joint_posterior(ch.init_mean, dense_cov(ch.init_cov), ch)
    for k in range(ch.n + 1):
        assert max_abs_diff(got.smoothed_mean[k], joint[k][0]) <= 1e-8
        assert max_abs_diff(dense_cov(got.smoothed_cov_sqrt[k]), joint[k][1]) <= 1e-8


def test_para_rts_errors():  # test_parallel.cpp:380-387
    ch = O.random_chain(2, 3, 52)
    bad = to_chain(ch)
    bad.obs_rows = np.zeros(0, dtype=np.int32)
    with pytest.raises(P.DimensionError):
        P.para_rts(bad)


# ------------------------------------------------------------- ieks ---
def _orc_problem(name):
    return O.problem(name)


IEKS_CASES = [("logistic", 1, 30), ("logistic", 2, 30), ("rigidbody", 1, 150), ("rigidbody", 2, 150),
              ("vanderpol", 1, 100), ("vanderpol", 2, 100), ("fhn", 2, 256), ("vanderpol", 3, 200),
              ("logistic", 1, 1024), ("rigidbody", 4, 300)]


@pytest.mark.parametrize("name,nu,steps", IEKS_CASES)
def test_para_ieks_matches_seq_ieks(name, nu, steps):  # acceptance.cpp:97-123 (criterion 1) + north star
    op = O.problem(name)
    gp = P.problem_by_name(name)
    grid = O.uniform_grid(op.t_end, steps)
    want = O.ieks(op, nu, grid, mode=0)
    got = P.para_ieks(gp, P.IwpPrior(nu, op.dim, 1.0), grid)
    assert got.converged == want["converged"]
    assert got.iterations == want["iterations"]
    assert rel(got.means, want["means"]) <= 1e-9
    assert rel(dense_cov(got.cov_sqrt), dense_cov(want["cov_sqrt"])) <= 1e-7
    assert got.sigma_hat == pytest.approx(want["sigma_hat"], rel=1e-7)
    assert rel(got.solution_means, want["solution_means"]) <= 1e-9
    assert rel(got.solution_covs, want["solution_covs"]) <= 1e-7
    assert np.allclose(got.objective_trace, want["objective_trace"], rtol=1e-8, atol=1e-12)


@pytest.mark.parametrize("chunk,fanin", [(2, 2), (3, 2), (5, 3), (8, 4), (7, 16), (30, 4), (64, 2)])
@pytest.mark.parametrize("name,nu,steps", [("logistic", 2, 30), ("vanderpol", 2, 100), ("fhn", 2, 257),
                                           ("fhn", 2, 4000), ("rigidbody", 2, 3000)])
def test_fused_engine_chunking(monkeypatch, name, nu, steps, chunk, fanin):
    """Fused IEKS engine under every chunking shape: one chunk, ragged last
    chunks, single- and multi-level aggregate scans (top level of 1..fanin
    chunks) must give the sequential oracle's iterates."""
    monkeypatch.setenv("PODE_CHUNK", str(chunk))
    monkeypatch.setenv("PODE_SCAN_FANIN", str(fanin))
    op = O.problem(name)
    grid = O.uniform_grid(op.t_end, steps)
    want = O.ieks(op, nu, grid, mode=0)
    got = P.para_ieks(P.problem_by_name(name), P.IwpPrior(nu, op.dim, 1.0), grid)
    assert got.iterations == want["iterations"]
    assert rel(got.means, want["means"]) <= 1e-9
    assert rel(got.solution_means, want["solution_means"]) <= 1e-9


@pytest.mark.parametrize("env", [{"PODE_BSCAN": "0"}, {"PODE_BSCAN": "1"}, {"PODE_BSCAN": "64"},
                                 {"PODE_FINALIZE": "elements"}, {"PODE_GRAPH": "0"}, {}])
def test_fused_engine_variants(monkeypatch, env):
    """The alternative scan / finalize paths of the fused engine agree with the oracle too."""
    for k, v in env.items():
        monkeypatch.setenv(k, v)
    monkeypatch.setenv("PODE_CHUNK", "3")
    op = O.problem("fhn")
    grid = O.uniform_grid(op.t_end, 2000)
    want = O.ieks(op, 2, grid, mode=0)
    got = P.para_ieks(P.problem_by_name("fhn"), P.IwpPrior(2, op.dim, 1.0), grid)
    assert got.iterations == want["iterations"]
    assert rel(got.means, want["means"]) <= 1e-9
    assert rel(dense_cov(got.cov_sqrt), dense_cov(want["cov_sqrt"])) <= 1e-7
    assert got.sigma_hat == pytest.approx(want["sigma_hat"], rel=1e-7)


@pytest.mark.parametrize("name,steps", [("fhn", 720), ("fhn", 1200), ("fhn", 1800), ("rigidbody", 600),
                                        ("fhn", 2400)])
def test_block_scan_tiles(monkeypatch, name, steps):
    """Block-scan levels of 2..5 blocks (G = 40 at D = 6, 24 at D = 9) at
    every level above 0, and the down-sweeps that apply their carries."""
    monkeypatch.setenv("PODE_CHUNK", "3")
    monkeypatch.setenv("PODE_SCAN_FANIN", "4")
    monkeypatch.setenv("PODE_BSCAN", "1")
    op = O.problem(name)
    grid = O.uniform_grid(op.t_end, steps)
    want = O.ieks(op, 2, grid, mode=0)
    got = P.para_ieks(P.problem_by_name(name), P.IwpPrior(2, op.dim, 1.0), grid)
    assert got.iterations == want["iterations"]
    assert rel(got.means, want["means"]) <= 1e-9
    assert rel(dense_cov(got.cov_sqrt), dense_cov(want["cov_sqrt"])) <= 1e-7


def test_logistic_frozen_rmse():  # acceptance.cpp:167-179 — reference measured 1.374e-6, gate 2.1e-6
    from _dense import logistic_reference, rmse
    grid = O.uniform_grid(10.0, 30)
    got = P.para_ieks(P.logistic(), P.IwpPrior(2, 1, 1.0), grid)
    err = rmse(got.solution_means, lambda t: [logistic_reference(t)], grid)
    assert got.converged and err <= 2.1e-6


def test_affine_two_iterations():  # test_ieks.cpp:211-246 (seed 63)
    rng = O.Rng(63)
    l, c, y0 = rng.matrix(2, 2), rng.vector(2), rng.vector(2)
    grid = O.uniform_grid(1.0, 10)
    got = P.para_ieks(P.affine(l, c, y0, 1.0), P.IwpPrior(2, 2, 1.0), grid)
    want = O.ieks(O.affine_problem(l, c, y0, 1.0), 2, grid, mode=0)
    assert got.converged and got.iterations == 2
    assert rel(got.means, want["means"]) <= 1e-9


def test_sigma_invariance():  # test_ieks.cpp:284-299
    grid = O.uniform_grid(10.0, 20)
    a = P.para_ieks(P.logistic(), P.IwpPrior(2, 1, 1.0), grid)
    b = P.para_ieks(P.logistic(), P.IwpPrior(2, 1, 7.0), grid)
    assert a.iterations == b.iterations
    assert a.sigma_hat == pytest.approx(b.sigma_hat, rel=1e-8)
    assert max_abs_diff(a.means, b.means) <= 1e-10
    assert max_abs_diff(dense_cov(a.cov_sqrt), dense_cov(b.cov_sqrt)) <= 1e-8


def test_iteration_budget_and_errors():  # test_ieks.cpp:369-388
    grid = O.uniform_grid(6.3, 40)
    r = P.para_ieks(P.van_der_pol(), P.IwpPrior(2, 2, 1.0), grid, P.IeksConfig(max_iterations=1))
    assert not r.converged and r.iterations == 1 and len(r.objective_trace) == 1
    with pytest.raises(P.InvalidInputError):
        P.para_ieks(P.van_der_pol(), P.IwpPrior(2, 2, 1.0), grid, P.IeksConfig(max_iterations=0))
    with pytest.raises(P.InvalidInputError):
        P.para_ieks(P.van_der_pol(), P.IwpPrior(2, 2, 1.0), [0.5, 1.0])
    with pytest.raises(P.DimensionError):
        P.para_ieks(P.van_der_pol(), P.IwpPrior(2, 3, 1.0), grid)


def test_ek0_matches_oracle():  # statespace.cpp:90-103
    grid = O.uniform_grid(10.0, 64)
    got = P.para_ieks(P.logistic(), P.IwpPrior(2, 1, 1.0), grid, P.IeksConfig(linearization="ek0"))
    want = O.ieks(O.problem("logistic"), 2, grid, mode=0, ek0=True)
    assert got.iterations == want["iterations"]
    assert rel(got.means, want["means"]) <= 1e-9


@pytest.mark.parametrize("name,nu,n", [("fhn", 2, 4000), ("vanderpol", 2, 3000), ("rigidbody", 2, 3000)])
def test_wide_group_block_scans_match_oracle(name, nu, n, monkeypatch):
    """The opt-in wide-group upper scan levels (PODE_WIDE=1, wide.cuh) give
    the oracle's iterates (short chunks force several block-scan levels)."""
    monkeypatch.setenv("PODE_WIDE", "1")
    prob = P.problem_by_name(name)
    grid = O.uniform_grid(prob.t_end, n)
    ctx = P.Context()
    ctx.set_chunk_len(2)
    got = P.para_ieks(prob, P.IwpPrior(nu, prob.dim, 1.0), grid, ctx=ctx)
    want = O.ieks(_orc_problem(name), nu, grid, mode=0)
    assert got.iterations == want["iterations"]
    assert rel(got.means, want["means"]) <= 1e-9
    assert rel(dense_cov(got.cov_sqrt), dense_cov(want["cov_sqrt"])) <= 1e-7


def test_ragged_grid_matches_oracle():  # discretize on a non-uniform grid (ieks.cpp:8-47)
    g = np.cumsum(np.concatenate([[0.0], 0.05 + 0.1 * np.abs(np.sin(np.arange(80)))]))
    got = P.para_ieks(P.van_der_pol(), P.IwpPrior(2, 2, 1.0), g)
    want = O.ieks(O.problem("vanderpol"), 2, g, mode=0)
    assert got.iterations == want["iterations"]
    assert rel(got.means, want["means"]) <= 1e-9
    assert rel(dense_cov(got.cov_sqrt), dense_cov(want["cov_sqrt"])) <= 1e-7


def test_batch_equals_single_solves():  # batched multi-IVP
    """Concurrent independent solves (one stream per worker) reproduce the
    single solves bit for bit, for a sweep over initial values and
    parameters."""
    import time
    probs = []
    for k in range(12):
        p = P.fitzhugh_nagumo()
        p.y0 = np.array([-1.0 + 0.05 * k, 1.0 - 0.03 * k])
        probs.append(p)
    grid = P.uniform_grid(20.0, 600)
    prior = P.IwpPrior(2, 2, 1.0)
    t0 = time.perf_counter()
    single = [P.para_ieks(p, prior, grid) for p in probs]
    t1 = time.perf_counter()
    batch = P.para_ieks_batch(probs, prior, grid, streams=6)
    t2 = time.perf_counter()
    for a, b in zip(single, batch):
        assert a.iterations == b.iterations and a.converged == b.converged
        assert np.array_equal(a.means, b.means)
        assert np.array_equal(a.cov_sqrt, b.cov_sqrt)
        assert a.sigma_hat == b.sigma_hat
    print(f"12 solves: sequential {1e3 * (t1 - t0):.1f} ms, batched {1e3 * (t2 - t1):.1f} ms")


def test_batch_parameter_sweep_matches_oracle():
    """Van der Pol over mu in a batch against the sequential oracle."""
    grid = P.uniform_grid(6.3, 200)
    probs = [P.van_der_pol(mu) for mu in (0.5, 1.0, 1.5)]
    got = P.para_ieks_batch(probs, P.IwpPrior(2, 2, 1.0), grid, streams=3)
    for mu, g in zip((0.5, 1.0, 1.5), got):
        op = O.ProblemSpec(3, 2, 6.3, [2.0, 0.0], [mu])
        want = O.ieks(op, 2, O.uniform_grid(6.3, 200), mode=0)
        assert g.iterations == want["iterations"]
        assert rel(g.means, want["means"]) <= 1e-9


def test_full_size_fhn_properties():
    """BASELINE.json's headline size (FHN, IWP(2), N = 2^20), where the
    sequential oracle is too slow to run: size-independent properties —
    convergence, bitwise determinism of the whole solve, the posterior mean
    against an RK4 solution on the same nodes (GPU, pode_rk4_table), and
    calibrated covariances that are finite and positive on the diagonal."""
    from paraode_b200.accuracy import rk4_table
    prob = P.fitzhugh_nagumo()
    n = 2 ** 20
    grid = P.uniform_grid(prob.t_end, n)
    a = P.para_ieks(prob, P.IwpPrior(2, 2, 1.0), grid)
    b = P.para_ieks(prob, P.IwpPrior(2, 2, 1.0), grid)
    assert a.converged and a.iterations == b.iterations
    assert np.array_equal(a.means, b.means) and np.array_equal(a.cov_sqrt, b.cov_sqrt)
    ref = rk4_table(prob, n)  # same nodes: no interpolation error
    err = float(np.sqrt(np.mean((a.solution_means - ref) ** 2)))
    print(f"N=2^20: iterations {a.iterations}, RMSE vs RK4 {err:.3e}, sigma_hat {a.sigma_hat:.3e}")
    assert err <= 1e-9  # measured 1.0e-11
    var = np.diagonal(a.solution_covs, axis1=1, axis2=2)
    assert np.all(np.isfinite(a.cov_sqrt)) and np.all(var[1:] > 0.0)


# -------------------------------------------------------------- eks ---
EKS_CASES = [("logistic", 1, 30, False), ("logistic", 2, 64, True), ("vanderpol", 2, 100, False),
             ("rigidbody", 2, 150, False), ("fhn", 2, 256, False), ("vanderpol", 3, 200, True),
             ("rigidbody", 4, 300, False), ("logistic", 1, 1024, False)]


@pytest.mark.parametrize("name,nu,steps,ek0", EKS_CASES)
def test_eks_solve_matches_oracle(name, nu, steps, ek0):  # eks_solve, ieks.cpp:224-291 (bench.cpp:139)
    op = O.problem(name)
    grid = O.uniform_grid(op.t_end, steps)
    want = O.ieks(op, nu, grid, mode=-1, ek0=ek0)
    got = P.eks_solve(P.problem_by_name(name), P.IwpPrior(nu, op.dim, 1.0), grid, "ek0" if ek0 else "ek1")
    assert got.iterations == want["iterations"] == 1 and got.converged and want["converged"]
    assert rel(got.means, want["means"]) <= 1e-9
    assert rel(dense_cov(got.cov_sqrt), dense_cov(want["cov_sqrt"])) <= 1e-7
    assert got.sigma_hat == pytest.approx(want["sigma_hat"], rel=1e-7)
    assert rel(got.solution_means, want["solution_means"]) <= 1e-9
    assert rel(got.solution_covs, want["solution_covs"]) <= 1e-7
    assert np.allclose(got.objective_trace, want["objective_trace"], rtol=1e-8, atol=1e-12)


def test_eks_ragged_grid_and_errors():
    g = np.cumsum(np.concatenate([[0.0], 0.05 + 0.1 * np.abs(np.sin(np.arange(80)))]))
    got = P.eks_solve(P.van_der_pol(), P.IwpPrior(2, 2, 1.0), g)
    want = O.ieks(O.problem("vanderpol"), 2, g, mode=-1)
    assert rel(got.means, want["means"]) <= 1e-9
    assert rel(dense_cov(got.cov_sqrt), dense_cov(want["cov_sqrt"])) <= 1e-7
    with pytest.raises(P.DimensionError):
        P.eks_solve(P.van_der_pol(), P.IwpPrior(2, 3, 1.0), g)
    with pytest.raises(P.InvalidInputError):
        P.eks_solve(P.van_der_pol(), P.IwpPrior(2, 2, 1.0), [0.5, 1.0])
    # deterministic run to run
    again = P.eks_solve(P.van_der_pol(), P.IwpPrior(2, 2, 1.0), g)
    assert np.array_equal(again.means, got.means) and np.array_equal(again.cov_sqrt, got.cov_sqrt)



@pytest.mark.parametrize("n", [40, 100_000])  # serial and OpenMP-split grid checks
def test_non_increasing_grid_rejected(n):  # discretize, ieks.cpp:8-20
    prior = P.IwpPrior(2, 2, 1.0)
    for k in (1, n // 2, n - 1):
        g = O.uniform_grid(6.3, n)
        g[k + 1] = g[k]
        with pytest.raises(P.InvalidInputError, match="strictly increasing"):
            P.para_ieks(P.van_der_pol(), prior, g)
        with pytest.raises(P.InvalidInputError, match="strictly increasing"):
            P.eks_solve(P.van_der_pol(), prior, g)
    g = O.uniform_grid(6.3, n)
    g[n // 3] = np.nan
    with pytest.raises(P.InvalidInputError):
        P.para_ieks(P.van_der_pol(), prior, g)
