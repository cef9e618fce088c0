"""Pins the C++ oracle (oracle/orc.hpp) to the reference's own known-answer
tests and fixtures, plus an independent numpy dense restatement of
proj/tests/oracles.cpp.  Every case cites the reference test it restates.
CPU only."""
import numpy as np
import pytest

import _oracle as O
from _dense import (dense_combine, dense_cov, dense_element, dense_filter, dense_joint_posterior,
                    dense_predict, dense_smooth, dense_update, densify, logistic_reference,
                    max_abs_diff, rk4_reference, rmse)


def fe_tuple(fe, i):
    return fe.a[i], fe.b[i], fe.c[i], fe.eta[i], fe.j[i]


def one(fe_tuple_):
    a, b, c, eta, j = fe_tuple_
    return O.FilteringElements(1, a.shape[0], a[None], b[None], c[None], eta[None], j[None])


def check_dense(got, want, tol):
    """test_parallel.cpp:17-24 (check_element_against_dense)."""
    a, b, c, eta, j = got
    assert max_abs_diff(a, want[0]) <= tol
    assert max_abs_diff(b, want[1]) <= tol
    assert max_abs_diff(dense_cov(c), want[2]) <= tol
    assert max_abs_diff(eta, want[3]) <= tol
    assert max_abs_diff(dense_cov(j), want[4]) <= tol


# ------------------------------------------------------------ linalg ---
def test_tria_norm_example():  # test_linalg.cpp:11-18
    t = O.tria(np.array([[3.0, 4.0]]))
    assert t.shape == (1, 1) and abs(abs(t[0, 0]) - 5.0) <= 5e-14


@pytest.mark.parametrize("shape", [(3, 5), (4, 4), (4, 2)])
def test_tria_product_and_shape(shape):  # test_linalg.cpp:20-45 (seed 11)
    rng = O.Rng(11)
    m = rng.matrix(*shape)
    t = O.tria(m)
    assert t.shape == (shape[0], shape[0])
    assert np.all(np.triu(t, 1) == 0.0)
    assert max_abs_diff(dense_cov(t), m @ m.T) <= 1e-12


def test_tria_padded_lower_factor_exact():  # test_linalg.cpp:47-54 (seed 12)
    l = O.Rng(12).spd_sqrt(3)
    t = O.tria(np.hstack([l, np.zeros((3, 2))]))
    assert max_abs_diff(dense_cov(t), dense_cov(l)) <= 1e-14


def test_tria_deterministic_and_rejects_nan():  # test_linalg.cpp:56-66
    m = O.Rng(13).matrix(5, 7)
    assert np.array_equal(O.tria(m), O.tria(m))
    bad = np.zeros((2, 3))
    bad[1, 2] = np.nan
    with pytest.raises(O.OracleError) as e:
        O.tria(bad)
    assert e.value.kind == "InvalidInputError"


# ------------------------------------------------------------- prior ---
def test_iwp_first_order_unit_step():  # test_prior.cpp:34-44
    phi, q = O.iwp_transition(1, 1, 1.0, 1.0)
    assert max_abs_diff(phi, [[1, 1], [0, 1]]) <= 1e-15
    assert max_abs_diff(dense_cov(q), [[1 / 3, 0.5], [0.5, 1.0]]) <= 1e-14
    assert np.all(np.triu(q, 1) == 0.0)


def test_iwp_entries_formula():  # test_prior.cpp:46-58
    from math import factorial
    nu, h = 2, 0.5
    phi, q = O.iwp_transition(nu, 1, 1.0, h)
    qd = dense_cov(q)
    for i in range(nu + 1):
        for j in range(nu + 1):
            want_phi = h ** (j - i) / factorial(j - i) if j >= i else 0.0
            p = 2 * nu + 1 - i - j
            want_q = h ** p / (p * factorial(nu - i) * factorial(nu - j))
            assert phi[i, j] == pytest.approx(want_phi, rel=1e-13, abs=1e-300)
            assert qd[i, j] == pytest.approx(want_q, rel=1e-12)


def test_preconditioner_quarter_step():  # test_prior.cpp:122-140
    s, _ = O.preconditioner(1, 1, 1.0)
    assert np.array_equal(s, [1.0, 1.0])
    s, si = O.preconditioner(1, 1, 0.25)
    assert max_abs_diff(s, [0.125, 0.5]) <= 1e-15
    assert max_abs_diff(s * si, [1.0, 1.0]) <= 1e-15
    s, _ = O.preconditioner(1, 2, 0.25)
    assert s[0] == s[2] and s[1] == s[3]


def test_rescaled_pair_is_step_independent():  # test_prior.cpp:142-158
    for nu in (1, 2, 3):
        phi_bar, q_bar_sqrt = O.preconditioned_pair(nu, 2)
        q_bar = dense_cov(q_bar_sqrt)
        for h in (1e-3, 0.1, 0.9, 17.0):
            phi, q = O.iwp_transition(nu, 2, 1.0, h)
            s, si = O.preconditioner(nu, 2, h)
            assert max_abs_diff(np.diag(si) @ phi @ np.diag(s), phi_bar) <= 1e-10
            assert max_abs_diff(np.diag(si) @ dense_cov(q) @ np.diag(si), q_bar) <= 1e-10


def test_binomial_block():  # test_prior.cpp:160-167
    phi_bar, _ = O.preconditioned_pair(2, 1)
    assert np.array_equal(phi_bar, [[1, 2, 1], [0, 1, 1], [0, 0, 1]])
    _, q = O.preconditioned_pair(1, 1)
    assert max_abs_diff(dense_cov(q), [[1 / 3, 0.5], [0.5, 1.0]]) <= 1e-14


def test_taylor_init_kats():  # test_prior.cpp:169-191
    assert max_abs_diff(O.taylor_init(O.problem("logistic"), 2), [0.01, 0.0099, 0.009702]) <= 1e-15
    assert max_abs_diff(O.taylor_init(O.problem("rigidbody"), 1), [1, 0, 0, 1.125, 0.9, 0]) <= 1e-15
    assert max_abs_diff(O.taylor_init(O.problem("vanderpol"), 2), [2, 0, -2, 0, -2, 6]) <= 1e-14


def test_taylor_init_linear_field_powers():  # test_prior.cpp:192-206
    lam = -0.5
    p = O.affine_problem([[lam]], [0.0], [3.0], 1.0)
    want = [3.0, lam * 3.0, lam * lam * 3.0, lam ** 3 * 3.0]
    assert max_abs_diff(O.taylor_init(p, 3), want) <= 1e-14


def test_prior_rejects_bad_inputs():  # test_prior.cpp:221-227
    for args in [(0, 1, 1.0, 1.0), (1, 1, 1.0, 0.0), (1, 1, 1.0, -1.0), (1, 1, -2.0, 1.0)]:
        with pytest.raises(O.OracleError):
            O.iwp_transition(*args)


# -------------------------------------------------------- statespace ---
def test_logistic_ek1_kat():  # test_statespace.cpp:38-47
    h, off = O.linearize(O.problem("logistic"), 1, [0.5, 0.3], 0.0)
    assert max_abs_diff(h, [[0.0, 1.0]]) <= 1e-15  # H = E1 - (1 - 2y) E0 = E1 at y = 0.5
    assert off[0] == pytest.approx(0.25, rel=1e-15)


def test_ek0_kat():  # test_statespace.cpp:106-121
    h, off = O.linearize(O.problem("logistic"), 2, [0.01, 0.5, 0.2], 0.0, ek0=True)
    assert np.array_equal(h, [[0.0, 1.0, 0.0]])
    assert off[0] == pytest.approx(0.0099, rel=1e-15)


def test_linearization_residual_identity():  # test_statespace.cpp:49-64
    for name in ("logistic", "rigidbody", "vanderpol", "fhn"):
        p = O.problem(name)
        for nu in (1, 2):
            eta = np.linspace(0.3, 0.9, p.dim * (nu + 1))
            h, off = O.linearize(p, nu, eta, 0.0)
            y = eta[::nu + 1]
            f, _ = O.field(p, y)
            assert max_abs_diff(h @ eta - off, eta[1::nu + 1] - f) <= 1e-14


def test_field_jacobians_match_finite_differences():  # problem Jacobians (incl. new FHN/Pleiades)
    for name in ("logistic", "rigidbody", "vanderpol", "fhn", "pleiades"):
        p = O.problem(name)
        y = p.y0 + 0.1 * np.sin(np.arange(p.dim))
        _, jac = O.field(p, y)
        fd = np.zeros_like(jac)
        for j in range(p.dim):
            step = 1e-6 * max(1.0, abs(y[j]))
            hi, lo = y.copy(), y.copy()
            hi[j] += step
            lo[j] -= step
            fd[:, j] = (O.field(p, hi)[0] - O.field(p, lo)[0]) / (2 * step)
        assert max_abs_diff(fd, jac) <= 1e-6 * max(1.0, np.abs(jac).max())


def test_pleiades_taylor_init_matches_numerical_derivatives():  # Jet ÷ and √ extension
    p = O.problem("pleiades")
    mu = O.taylor_init(p, 3)
    f0, jac0 = O.field(p, p.y0)
    y1 = mu[1::4]
    y2 = mu[2::4]
    assert max_abs_diff(y1, f0) <= 1e-14
    assert max_abs_diff(y2, jac0 @ f0) <= 1e-12


# ------------------------------------------------ elements & operators ---
def _chain_one(phi, q, h, off, r):
    d = phi.shape[0]
    m = max(h.shape[0], 1)
    hh = np.zeros((1, m, d))
    oo = np.zeros((1, m))
    rr = np.zeros((1, m, m))
    hh[0, :h.shape[0]] = h
    oo[0, :h.shape[0]] = off
    rr[0, :h.shape[0], :h.shape[0]] = r
    return O.ChainData(np.zeros(d), np.zeros((d, d)), phi[None], q[None], [h.shape[0]], hh, oo, rr)


@pytest.mark.parametrize("case", ["noisy", "noiseless", "vacuous"])
def test_filtering_elements_vs_first_principles(case):  # test_parallel.cpp:58-79 (seed 41)
    rng = O.Rng(41)
    phi, q = rng.transition(3)
    if case == "noisy":
        h, off, r = rng.observation(2, 3, False)
    elif case == "noiseless":
        h, off, r = rng.observation(1, 3, True)
    else:
        h, off, r = np.zeros((0, 3)), np.zeros(0), np.zeros((0, 0))
    fe = O.make_filtering_elements(_chain_one(phi, q, h, off, r), absorb_init=False)
    got = fe_tuple(fe, 0)
    if case == "vacuous":
        assert max_abs_diff(got[0], phi) <= 1e-12
        assert max_abs_diff(dense_cov(got[2]), dense_cov(q)) <= 1e-12
        assert np.abs(got[1]).max() <= 1e-12 and np.abs(got[3]).max() <= 1e-12
    else:
        check_dense(got, dense_element(phi, q, h, off, r), 1e-10)


def test_first_element_absorbs_init():  # test_parallel.cpp:80-92
    rng = O.Rng(41)
    phi, q = rng.transition(3)
    rng.observation(2, 3, False)  # keep the SUBCASE draw order: noisy obs drawn first
    h, off, r = rng.observation(2, 3, False)
    init_mean, init_cov = rng.vector(3), rng.spd_sqrt(3)
    ch = _chain_one(phi, q, h, off, r)
    ch.init_mean, ch.init_cov = init_mean, init_cov
    fe = O.make_filtering_elements(ch, absorb_init=True)
    assert np.all(fe.a[0] == 0) and np.all(fe.eta[0] == 0) and np.all(fe.j[0] == 0)
    m, c = dense_update(*dense_predict(init_mean, dense_cov(init_cov), phi, dense_cov(q)), h, off,
                        dense_cov(r))
    assert max_abs_diff(fe.b[0], m) <= 1e-10
    assert max_abs_diff(dense_cov(fe.c[0]), c) <= 1e-10


def test_scalar_exact_constraint_element():  # test_parallel.cpp:95-116
    one_ = np.ones((1, 1))
    fe = O.make_filtering_elements(_chain_one(one_, one_, one_, np.zeros(1), np.zeros((1, 1))), False)
    assert abs(fe.a[0, 0, 0]) <= 1e-15 and abs(fe.b[0, 0]) <= 1e-15 and abs(fe.c[0, 0, 0]) <= 1e-15
    assert abs(fe.eta[0, 0]) <= 1e-15 and abs(fe.j[0, 0, 0] ** 2 - 1.0) <= 1e-14
    fe = O.make_filtering_elements(_chain_one(one_, one_, one_, 0.5 * np.ones(1), np.zeros((1, 1))), False)
    assert fe.b[0, 0] == pytest.approx(0.5, rel=1e-13)
    assert fe.eta[0, 0] == pytest.approx(0.5, rel=1e-13)


def test_combine_filtering_vs_dense():  # test_parallel.cpp:118-127 (seed 42)
    rng = O.Rng(42)
    for _ in range(20):
        lhs, rhs = one(rng.filtering_element(3)), one(rng.filtering_element(3))
        got = O.combine_filtering(lhs, rhs)
        want = dense_combine(densify(*fe_tuple(lhs, 0)), densify(*fe_tuple(rhs, 0)))
        check_dense(fe_tuple(got, 0), want, 1e-9)


def test_filtering_identity_two_sided():  # test_parallel.cpp:129-136 (seed 43)
    el = one(O.Rng(43).filtering_element(4))
    ident = O.FilteringElements(1, 4)
    ident.a[0] = np.eye(4)
    for got in (O.combine_filtering(ident, el), O.combine_filtering(el, ident)):
        check_dense(fe_tuple(got, 0), densify(*fe_tuple(el, 0)), 1e-12)


def test_filtering_associative():  # test_parallel.cpp:138-154 (seed 44)
    rng = O.Rng(44)
    for _ in range(10):
        a, b, c = (one(rng.filtering_element(3)) for _ in range(3))
        left = O.combine_filtering(O.combine_filtering(a, b), c)
        right = O.combine_filtering(a, O.combine_filtering(b, c))
        dl, dr = densify(*fe_tuple(left, 0)), densify(*fe_tuple(right, 0))
        for x, y in zip(dl, dr):
            assert max_abs_diff(x, y) <= 1e-9


def test_prefixes_reproduce_sequential_filter():  # test_parallel.cpp:156-177 (seed 45)
    ch = O.random_chain(3, 13, 45)
    prefixes, _ = O.scan_filtering(O.make_filtering_elements(ch))
    seq = O.rts(ch, mode=0)
    for i in range(ch.n):
        assert max_abs_diff(prefixes.b[i], seq["filtered_mean"][i + 1]) <= 1e-9
        assert max_abs_diff(dense_cov(prefixes.c[i]), dense_cov(seq["filtered_cov"][i + 1])) <= 1e-9


def test_integer_scan_work_and_depth():  # test_parallel.cpp:179-212
    got, (work, depth) = O.scan_int_add(np.arange(1, 9))
    assert list(got) == [1, 3, 6, 10, 15, 21, 28, 36] and work == 11 and depth == 5
    got, (work, depth) = O.scan_int_add([7])
    assert list(got) == [7] and work == 0 and depth == 0
    got, (work, depth) = O.scan_int_add(np.ones(1024))
    assert got[0] == 1 and got[-1] == 1024 and work == 2036 and depth <= 20


def test_scan_bounds_acceptance():  # acceptance.cpp:235-262 (criterion 6)
    import math
    for n in (1, 2, 7, 64, 257, 1024):
        for rev in (False, True):
            got, (work, depth) = O.scan_int_add(np.ones(n), reverse=rev)
            assert (got[0], got[-1]) == ((1, n) if not rev else (n, 1))
            assert work <= (2 * n - 2 if n >= 2 else 0)
            assert depth <= (2 * math.ceil(math.log2(n)) if n >= 2 else 0)


def test_smoothing_elements_vs_dense_gain():  # test_parallel.cpp:258-291 (seed 46)
    rng = O.Rng(46)
    fm, fc = rng.vector(2), rng.spd_sqrt(2)
    ch = O.ChainData(np.zeros(2), np.zeros((2, 2)), np.eye(2)[None], np.zeros((1, 2, 2)), [0],
                     np.zeros((1, 1, 2)), np.zeros((1, 1)), np.zeros((1, 1, 1)))
    se = O.make_smoothing_elements(ch, np.stack([fm, fm]), np.stack([fc, fc]))
    assert max_abs_diff(se.e[0], np.eye(2)) <= 1e-10
    assert np.abs(se.g[0]).max() <= 1e-10 and np.abs(dense_cov(se.l[0])).max() <= 1e-10
    # terminal element carries the filtered marginal
    fm3, fc3 = rng.vector(3), rng.spd_sqrt(3)
    fm3b, fc3b = rng.vector(3), rng.spd_sqrt(3)
    phi, q = rng.transition(3)
    ch3 = O.ChainData(np.zeros(3), np.zeros((3, 3)), phi[None], q[None], [0], np.zeros((1, 1, 3)),
                      np.zeros((1, 1)), np.zeros((1, 1, 1)))
    se3 = O.make_smoothing_elements(ch3, np.stack([fm3b, fm3]), np.stack([fc3b, fc3]))
    assert np.all(se3.e[1] == 0) and np.array_equal(se3.g[1], fm3) and np.array_equal(se3.l[1], fc3)
    p = dense_cov(fc3b)
    s = phi @ p @ phi.T + dense_cov(q)
    gain = p @ phi.T @ np.linalg.inv(s)
    assert max_abs_diff(se3.e[0], gain) <= 1e-10
    assert max_abs_diff(se3.g[0], fm3b - gain @ phi @ fm3b) <= 1e-10
    assert max_abs_diff(dense_cov(se3.l[0]), p - gain @ s @ gain.T) <= 1e-10


def test_smoothing_associative_identity():  # test_parallel.cpp:293-312 (seed 47)
    rng = O.Rng(47)

    def se1(t):
        e, g, l = t
        return O.SmoothingElements(1, e.shape[0], e[None], g[None], l[None])
    for _ in range(10):
        a, b, c = (se1(rng.smoothing_element(3)) for _ in range(3))
        left = O.combine_smoothing(O.combine_smoothing(a, b), c)
        right = O.combine_smoothing(a, O.combine_smoothing(b, c))
        assert max_abs_diff(left.e, right.e) <= 1e-10
        assert max_abs_diff(left.g, right.g) <= 1e-10
        assert max_abs_diff(dense_cov(left.l), dense_cov(right.l)) <= 1e-10


def test_reverse_scan_reproduces_backward_pass():  # test_parallel.cpp:314-336 (seed 48)
    ch = O.random_chain(2, 9, 48)
    seq = O.rts(ch, mode=0)
    se = O.make_smoothing_elements(ch, seq["filtered_mean"], seq["filtered_cov"])
    suf, _ = O.scan_smoothing(se, reverse=True)
    for i in range(ch.n + 1):
        assert max_abs_diff(suf.g[i], seq["smoothed_mean"][i]) <= 1e-9
        assert max_abs_diff(dense_cov(suf.l[i]), dense_cov(seq["smoothed_cov"][i])) <= 1e-9


def test_para_rts_matches_seq_rts():  # test_parallel.cpp:338-354 (seed 49)
    ch = O.random_chain(3, 17, 49)
    par, seq = O.rts(ch, mode=4), O.rts(ch, mode=0)
    for k in ("filtered_mean", "smoothed_mean"):
        assert max_abs_diff(par[k], seq[k]) <= 1e-9
    for k in ("filtered_cov", "smoothed_cov"):
        assert max_abs_diff(dense_cov(par[k]), dense_cov(seq[k])) <= 1e-9
    assert 0 < par["stats"][0] <= 2 * (ch.n + 1) - 2


def test_para_rts_single_step_and_determinism():  # test_parallel.cpp:356-378 (seeds 50, 51)
    ch = O.random_chain(2, 1, 50)
    par = O.rts(ch, mode=2)
    assert np.array_equal(par["filtered_mean"][1], par["smoothed_mean"][1])
    ch = O.random_chain(3, 11, 51)
    a, b = O.rts(ch, mode=1), O.rts(ch, mode=4)
    for k in ("filtered_mean", "filtered_cov", "smoothed_mean", "smoothed_cov"):
        assert np.array_equal(a[k], b[k])
    assert a["stats"] == b["stats"]


def test_sequential_vs_dense_oracles_and_joint_posterior():  # test_sequential.cpp (with vacuous)
    ch = O.random_chain(3, 10, 33, vacuous="mod3")
    seq = O.rts(ch, mode=0)
    filt = dense_filter(ch.init_mean, dense_cov(ch.init_cov), ch)
    smooth = dense_smooth(filt, ch)
    joint = dense_joint_posterior(ch.init_mean, dense_cov(ch.init_cov), ch)
    for n in range(ch.n + 1):
        assert max_abs_diff(seq["filtered_mean"][n], filt[n][0]) <= 1e-9
        assert max_abs_diff(dense_cov(seq["filtered_cov"][n]), filt[n][1]) <= 1e-9
        assert max_abs_diff(seq["smoothed_mean"][n], smooth[n][0]) <= 1e-9
        assert max_abs_diff(seq["smoothed_mean"][n], joint[n][0]) <= 1e-8
        assert max_abs_diff(dense_cov(seq["smoothed_cov"][n]), joint[n][1]) <= 1e-8


def test_operator_algebra_acceptance():  # acceptance.cpp:295-354 (criterion 8, seed 202)
    rng = O.Rng(202)
    worst_f = worst_s = 0.0
    ident = O.FilteringElements(1, 3)
    ident.a[0] = np.eye(3)
    sid = O.SmoothingElements(1, 3)
    sid.e[0] = np.eye(3)

    def df(x, y):
        return max(max_abs_diff(p, q) for p, q in zip(densify(*fe_tuple(x, 0)), densify(*fe_tuple(y, 0))))

    def ds(x, y):
        return max(max_abs_diff(x.e, y.e), max_abs_diff(x.g, y.g), max_abs_diff(dense_cov(x.l), dense_cov(y.l)))

    def se1(t):
        e, g, l = t
        return O.SmoothingElements(1, 3, e[None], g[None], l[None])
    for _ in range(200):
        a, b, c = (one(rng.filtering_element(3)) for _ in range(3))
        worst_f = max(worst_f, df(O.combine_filtering(O.combine_filtering(a, b), c),
                                  O.combine_filtering(a, O.combine_filtering(b, c))))
        worst_f = max(worst_f, df(O.combine_filtering(ident, a), a), df(O.combine_filtering(a, ident), a))
        p, q, r = (se1(rng.smoothing_element(3)) for _ in range(3))
        worst_s = max(worst_s, ds(O.combine_smoothing(O.combine_smoothing(p, q), r),
                                  O.combine_smoothing(p, O.combine_smoothing(q, r))))
        worst_s = max(worst_s, ds(O.combine_smoothing(sid, p), p), ds(O.combine_smoothing(p, sid), p))
    assert worst_f <= 1e-9 and worst_s <= 1e-9


def test_scan_validates_inputs():  # test_parallel.cpp:380-387 (seed 52)
    ch = O.random_chain(2, 3, 52)
    bad = O.ChainData(ch.init_mean, ch.init_cov, ch.phi, ch.q, ch.obs_rows, ch.h, ch.offset, ch.r)
    bad.n = 0
    with pytest.raises(O.OracleError) as e:
        O.rts(bad, mode=1)
    assert e.value.kind == "DimensionError"


# -------------------------------------------------------------- ieks ---
def test_objective_value_kats():  # test_ieks.cpp:51-98
    states = np.array([[1.0, 1.0], [2.0, 2.0], [4.0, 4.0]])
    assert O.objective(states, 2.0 * np.eye(2), np.eye(2)) == 0.0
    assert O.objective(np.array([[0.0], [2.0]]), np.eye(1), 2.0 * np.eye(1)) == pytest.approx(0.5, rel=1e-14)
    rng = O.Rng(61)
    d = 3
    s0 = rng.vector(d)
    phis, states_, exp = [], [s0], 0.0
    for k in range(6):
        phi, q = rng.transition(d)
        phis.append(phi)
        states_.append(rng.vector(d))
        inc = states_[k + 1] - phi @ states_[k]
        exp += 0.5 * inc @ np.linalg.inv(dense_cov(q)) @ inc
        # the reference uses per-step q; objective() takes a shared q, so
        # re-evaluate per step below
    total = 0.0
    rng = O.Rng(61)
    s = [rng.vector(d)]
    for k in range(6):
        phi, q = rng.transition(d)
        s.append(rng.vector(d))
        total += O.objective(np.stack([s[k], s[k + 1]]), phi, q)
    assert total == pytest.approx(exp, rel=1e-10)


def test_innovation_stats_vs_dense():  # test_ieks.cpp:136-169 (seed 62)
    rng = O.Rng(62)
    d = 3
    init_mean, init_cov = rng.vector(d), rng.spd_sqrt(d)
    phis, qs, hs, offs, rs = [], [], [], [], []
    for _ in range(7):
        phi, q = rng.transition(d)
        h, off, r = rng.observation(2, d, False)
        phis.append(phi), qs.append(q), hs.append(h), offs.append(off), rs.append(r)
    ch = O.ChainData(init_mean, init_cov, np.array(phis), np.array(qs), [2] * 7, np.array(hs),
                     np.array(offs), np.array(rs))
    seq = O.rts(ch, mode=0)
    exp, cnt = 0.0, 0
    for n in range(7):
        m, c = dense_predict(seq["filtered_mean"][n], dense_cov(seq["filtered_cov"][n]), phis[n], dense_cov(qs[n]))
        z = hs[n] @ m - offs[n]
        s = hs[n] @ c @ hs[n].T + dense_cov(rs[n])
        exp += z @ np.linalg.inv(s) @ z
        cnt += 2
    got, got_cnt = O.innovation_stats(ch, seq["filtered_mean"], seq["filtered_cov"])
    assert got_cnt == cnt and got == pytest.approx(exp, rel=1e-9)


def test_discretize_kats():  # test_ieks.cpp:171-209
    with pytest.raises(O.OracleError):
        O.discretize(2, 1, [0.5, 1.0])
    with pytest.raises(O.OracleError):
        O.discretize(2, 1, [0.0, 1.0, 1.0])
    _, phi, _ = O.discretize(2, 1, O.uniform_grid(2.0, 8))
    for n in range(1, 8):
        assert np.array_equal(phi[n], phi[0])
    grid = [0.0, 0.25, 0.5, 1.25]
    scale, phi, q = O.discretize(2, 1, grid)
    for n in range(3):
        h = grid[n + 1] - grid[n]
        pphi, pq = O.iwp_transition(2, 1, 1.0, h)
        s_next, s_prev = scale[n + 1], scale[n]
        assert max_abs_diff(np.diag(s_next) @ phi[n] @ np.diag(1 / s_prev), pphi) <= 1e-12
        assert max_abs_diff(np.diag(s_next) @ dense_cov(q) @ np.diag(s_next), dense_cov(pq)) <= 1e-12


def _affine(seed):
    rng = O.Rng(seed)
    l = rng.matrix(2, 2)
    c = rng.vector(2)
    y0 = rng.vector(2)
    return O.affine_problem(l, c, y0, 1.0)


def test_affine_two_iterations_dense_map():  # test_ieks.cpp:211-246 (seed 63)
    p = _affine(63)
    grid = O.uniform_grid(1.0, 10)
    rep = O.ieks(p, 2, grid, mode=2)
    assert rep["converged"] and rep["iterations"] == 2
    # dense MAP in rescaled coordinates (test_ieks.cpp:28-47)
    scale, phi, q = O.discretize(2, 2, grid)
    mu0 = O.taylor_init(p, 2)
    D = 6
    hs, offs = [], []
    for n in range(10):
        h, off = O.linearize(p, 2, np.zeros(D), grid[n + 1])
        hs.append(h * scale[n + 1][None, :])
        offs.append(off)
    ch = O.ChainData(mu0 / scale[0], np.zeros((D, D)), phi, np.stack([q] * 10), [2] * 10,
                     np.array(hs), np.array(offs), np.zeros((10, 2, 2)))
    joint = dense_joint_posterior(ch.init_mean, np.zeros((D, D)), ch)
    for n in range(11):
        assert max_abs_diff(rep["means"][n], scale[n] * joint[n][0]) <= 1e-8


def test_seq_par_eks_agree_on_affine():  # test_ieks.cpp:248-269 (seed 64)
    p = _affine(64)
    grid = O.uniform_grid(1.0, 12)
    par, seq, eks = O.ieks(p, 2, grid, mode=2), O.ieks(p, 2, grid, mode=0), O.ieks(p, 2, grid, mode=-1)
    assert eks["iterations"] == 1 and eks["converged"]
    assert max_abs_diff(par["means"], seq["means"]) <= 1e-8
    assert max_abs_diff(eks["means"], par["means"]) <= 1e-8
    assert par["iterations"] == seq["iterations"]


def test_logistic_closed_form_and_frozen_rmse():  # test_ieks.cpp:271-282, acceptance.cpp:167-179
    p = O.problem("logistic")
    grid = O.uniform_grid(10.0, 30)
    rep = O.ieks(p, 2, grid, mode=2)
    assert rep["converged"] and rep["sigma_hat"] > 0
    assert abs(rep["solution_means"][-1, 0] - logistic_reference(10.0)) <= 1e-4
    err = rmse(rep["solution_means"], lambda t: [logistic_reference(t)], grid)
    assert err <= 2.1e-6  # frozen gate; the reference measured 1.374e-6
    assert err == pytest.approx(1.374e-6, rel=2e-3)


def test_sigma_invariance():  # test_ieks.cpp:284-299
    p = O.problem("logistic")
    grid = O.uniform_grid(10.0, 20)
    base, scaled = O.ieks(p, 2, grid, mode=2, sigma=1.0), O.ieks(p, 2, grid, mode=2, sigma=7.0)
    assert base["iterations"] == scaled["iterations"]
    assert base["sigma_hat"] == pytest.approx(scaled["sigma_hat"], rel=1e-8)
    assert max_abs_diff(base["means"], scaled["means"]) <= 1e-10
    assert max_abs_diff(dense_cov(base["cov_sqrt"]), dense_cov(scaled["cov_sqrt"])) <= 1e-8


def test_vdp_map_satisfies_ode():  # test_ieks.cpp:301-317
    p = O.problem("vanderpol")
    grid = O.uniform_grid(6.3, 100)
    rep = O.ieks(p, 2, grid, mode=4)
    assert rep["converged"]
    worst = 0.0
    for n in range(101):
        y, dy = rep["means"][n][0::3], rep["means"][n][1::3]
        worst = max(worst, np.abs(dy - O.field(p, y)[0]).max())
    assert worst <= 1e-8


def test_iteration_budget():  # test_ieks.cpp:369-388
    p = O.problem("vanderpol")
    grid = O.uniform_grid(6.3, 40)
    rep = O.ieks(p, 2, grid, mode=2, max_iterations=1)
    assert not rep["converged"] and rep["iterations"] == 1 and len(rep["objective_trace"]) == 1
    with pytest.raises(O.OracleError) as e:
        O.ieks(p, 2, grid, mode=2, max_iterations=0)
    assert e.value.kind == "InvalidInputError"


GRID_STEPS = {"logistic": 30, "rigidbody": 150, "vanderpol": 100}


@pytest.mark.parametrize("name", ["logistic", "rigidbody", "vanderpol"])
@pytest.mark.parametrize("nu", [1, 2])
def test_seq_par_equivalence_acceptance(name, nu):  # acceptance.cpp:97-123 (criterion 1)
    p = O.problem(name)
    grid = O.uniform_grid(p.t_end, GRID_STEPS[name])
    par, seq = O.ieks(p, nu, grid, mode=4), O.ieks(p, nu, grid, mode=0)
    assert par["converged"] and seq["converged"] and par["iterations"] == seq["iterations"]
    assert max_abs_diff(par["means"], seq["means"]) <= 1e-8
    assert max_abs_diff(dense_cov(par["cov_sqrt"]), dense_cov(seq["cov_sqrt"])) <= 1e-8
    if nu == 2:
        assert par["iterations"] <= 20  # criterion 5 (acceptance.cpp:219-233)


def test_convergence_order_acceptance():  # acceptance.cpp:181-217 (criterion 4)
    p = O.problem("logistic")
    for nu in (1, 2):
        lh, le, prev, mono = [], [], 1e300, True
        for n in (16, 32, 64, 128, 256, 512):
            grid = O.uniform_grid(10.0, n)
            rep = O.ieks(p, nu, grid, mode=4)
            err = rmse(rep["solution_means"], lambda t: [logistic_reference(t)], grid)
            lh.append(np.log(10.0 / n))
            le.append(np.log(err))
            mono &= err <= prev
            prev = err
        slope = np.polyfit(lh, le, 1)[0]
        assert slope >= nu - 0.5 and mono


def test_rigid_body_accuracy_vs_rk4():  # problems.cpp:137-157 reference + rmse
    p = O.problem("rigidbody")
    ref = rk4_reference(lambda y, t: O.field(p, y, t)[0], p.y0, 20.0, steps=4096, check_tol=1e-8)
    grid = O.uniform_grid(20.0, 150)
    rep = O.ieks(p, 2, grid, mode=4)
    assert rmse(rep["solution_means"], ref, grid) <= 1e-2
