"""Independent dense-covariance oracles (numpy/LAPACK) — TEST INFRASTRUCTURE.

A numpy restatement of proj/tests/oracles.cpp:21-166: textbook full-covariance
formulas with no code shared with either the C++ oracle or the CUDA path.
Used to pin the C++ oracle (tests/test_oracle_kats.py) and as a second,
independent checker for the GPU path.
"""
import numpy as np


def dense_cov(s):
    s = np.asarray(s)
    return s @ np.swapaxes(s, -1, -2)


def dense_predict(mean, cov, phi, q):  # oracles.cpp:33-35
    return phi @ mean, phi @ cov @ phi.T + q


def dense_update(mean, cov, h, offset, r):  # oracles.cpp:37-50 (Joseph form)
    if h.shape[0] == 0:
        return mean, cov
    s = h @ cov @ h.T + r
    k = cov @ h.T @ np.linalg.inv(s)
    innov = offset - h @ mean
    ikh = np.eye(cov.shape[0]) - k @ h
    return mean + k @ innov, ikh @ cov @ ikh.T + k @ r @ k.T


def dense_filter(init_mean, init_cov, chain):  # oracles.cpp:52-66
    out = [(init_mean, init_cov)]
    for n in range(chain.n):
        phi, q_sqrt = chain.transition(n)
        h, off, r_sqrt = chain.observation(n)
        m, c = dense_predict(out[-1][0], out[-1][1], phi, dense_cov(q_sqrt))
        out.append(dense_update(m, c, h, off, dense_cov(r_sqrt)))
    return out


def dense_smooth(filtered, chain):  # oracles.cpp:68-82
    out = [None] * len(filtered)
    out[-1] = filtered[-1]
    for n in range(chain.n - 1, -1, -1):
        phi, q_sqrt = chain.transition(n)
        fm, fc = filtered[n]
        pred = phi @ fc @ phi.T + dense_cov(q_sqrt)
        gain = fc @ phi.T @ np.linalg.inv(pred)
        m = fm + gain @ (out[n + 1][0] - phi @ fm)
        c = fc + gain @ (out[n + 1][1] - pred) @ gain.T
        out[n] = (m, c)
    return out


def dense_joint_posterior(init_mean, init_cov, chain):  # oracles.cpp:84-129
    d = init_mean.shape[0]
    nodes = chain.n + 1
    total = nodes * d
    mean = np.zeros(total)
    cov = np.zeros((total, total))
    mean[:d] = init_mean
    cov[:d, :d] = init_cov
    for n in range(nodes - 1):
        phi, q_sqrt = chain.transition(n)
        r = (n + 1) * d
        mean[r:r + d] = phi @ mean[r - d:r]
        for m in range(n + 1):
            c = m * d
            cov[r:r + d, c:c + d] = phi @ cov[r - d:r, c:c + d]
            cov[c:c + d, r:r + d] = cov[r:r + d, c:c + d].T
        cov[r:r + d, r:r + d] = phi @ cov[r - d:r, r - d:r] @ phi.T + dense_cov(q_sqrt)
    rows = sum(int(chain.obs_rows[n]) for n in range(chain.n))
    if rows == 0:
        return [(mean[n * d:(n + 1) * d], cov[n * d:(n + 1) * d, n * d:(n + 1) * d]) for n in range(nodes)]
    big_h = np.zeros((rows, total))
    z = np.zeros(rows)
    big_r = np.zeros((rows, rows))
    row = 0
    for n in range(chain.n):
        h, off, r_sqrt = chain.observation(n)
        k = h.shape[0]
        if k == 0:
            continue
        big_h[row:row + k, (n + 1) * d:(n + 2) * d] = h
        z[row:row + k] = off
        big_r[row:row + k, row:row + k] = dense_cov(r_sqrt)
        row += k
    s = big_h @ cov @ big_h.T + big_r
    cross = cov @ big_h.T
    post_mean = mean + cross @ np.linalg.solve(s, z - big_h @ mean)
    post_cov = cov - cross @ np.linalg.solve(s, cross.T)
    return [(post_mean[n * d:(n + 1) * d], post_cov[n * d:(n + 1) * d, n * d:(n + 1) * d]) for n in range(nodes)]


def densify(a, b, c_sqrt, eta, j_sqrt):  # oracles.cpp:131-133
    return a, b, dense_cov(c_sqrt), eta, dense_cov(j_sqrt)


def dense_element(phi, q_sqrt, h, offset, r_sqrt):  # oracles.cpp:135-152
    d = phi.shape[0]
    q = dense_cov(q_sqrt)
    if h.shape[0] == 0:
        return phi, np.zeros(d), q, np.zeros(d), np.zeros((d, d))
    s = h @ q @ h.T + dense_cov(r_sqrt)
    s_inv = np.linalg.inv(s)
    k = q @ h.T @ s_inv
    ikh = np.eye(d) - k @ h
    return (ikh @ phi, k @ offset, ikh @ q, phi.T @ h.T @ s_inv @ offset,
            phi.T @ h.T @ s_inv @ h @ phi)


def dense_combine(i, j):  # oracles.cpp:154-166; i, j = (A, b, C, eta, J) dense
    a_i, b_i, c_i, eta_i, j_i = i
    a_j, b_j, c_j, eta_j, j_j = j
    d = a_i.shape[0]
    eye = np.eye(d)
    g_left = np.linalg.inv(eye + c_i @ j_j)
    g_right = np.linalg.inv(eye + j_j @ c_i)
    return (a_j @ g_left @ a_i,
            a_j @ g_left @ (b_i + c_i @ eta_j) + b_j,
            a_j @ g_left @ c_i @ a_j.T + c_j,
            a_i.T @ g_right @ (eta_j - j_j @ b_i) + eta_i,
            a_i.T @ g_right @ j_j @ a_i + j_i)


def max_abs_diff(a, b):
    a, b = np.asarray(a), np.asarray(b)
    if a.shape != b.shape:
        return 1e300
    if a.size == 0:
        return 0.0
    return float(np.max(np.abs(a - b)))


def logistic_reference(t, y0=0.01):  # problems.cpp:131-134
    return y0 / (y0 + (1.0 - y0) * np.exp(-np.asarray(t)))


def rk4_reference(f, y0, t_end, steps=32768, check_tol=1e-10):
    """Fixed-step RK4 table with the step-halving self-check
    (problems.cpp:11-64); returns a callable with linear interpolation."""
    def integrate(n):
        h = t_end / n
        y = np.array(y0, dtype=float)
        table = [y.copy()]
        for k in range(n):
            t = t_end * k / n
            k1 = f(y, t)
            k2 = f(y + 0.5 * h * k1, t + 0.5 * h)
            k3 = f(y + 0.5 * h * k2, t + 0.5 * h)
            k4 = f(y + h * k3, t + h)
            y = y + (h / 6.0) * (k1 + 2 * k2 + 2 * k3 + k4)
            table.append(y.copy())
        return np.array(table)
    coarse = integrate(steps)
    fine = integrate(2 * steps)
    scale = max(1.0, np.linalg.norm(fine[-1]))
    assert np.linalg.norm(coarse[-1] - fine[-1]) <= check_tol * scale
    step = t_end / (len(fine) - 1)

    def at(t):
        x = t / step
        nearest = int(min(max(0.0, round(x)), len(fine) - 1))
        if abs(t - nearest * step) <= 1e-9 * max(1.0, abs(t)):
            return fine[nearest]
        lo = int(min(max(0.0, np.floor(x)), len(fine) - 2))
        w = (t - lo * step) / step
        return (1 - w) * fine[lo] + w * fine[lo + 1]
    return at


def rmse(means, reference, grid):  # problems.cpp:197-210
    acc, count = 0.0, 0
    for n, t in enumerate(grid):
        err = np.asarray(means[n]) - np.asarray(reference(t))
        acc += float(np.sum(err * err))
        count += err.size
    return np.sqrt(acc / count)
