"""Equal-iteration parity helpers shared by the large-N and group-engine GPU
tests (TEST INFRASTRUCTURE): per-derivative-order comparison of IEKS
posteriors against the oracle, with the GPU's own rounding floor measured by
solves that differ only in association order."""
import numpy as np

MEAN_TOL, COV_TOL, SIG_TOL = 1e-9, 1e-7, 1e-7
NEVER = dict(traj_rtol=-1.0, obj_atol=-1.0, obj_rtol=0.0)


def rel(a, b):
    a, b = np.asarray(a), np.asarray(b)
    return float(np.max(np.abs(a - b)) / max(1.0, np.max(np.abs(b))))


def cov_upper(cov_sqrt, nodes):
    L = cov_sqrt[nodes]
    cov = np.einsum("nij,nkj->nik", L, L)
    iu = np.triu_indices(cov.shape[1])
    return cov[:, iu[0], iu[1]]


def gpu_solve(P, meta, ctx=None, **cfg):
    """meta: {problem, nu, t_end, steps} (the fixture metadata schema)."""
    prob = P.problem_by_name(meta["problem"])
    grid = P.uniform_grid(meta["t_end"], meta["steps"])
    return P.para_ieks(prob, P.IwpPrior(meta["nu"], prob.dim, 1.0), grid, P.IeksConfig(**cfg), ctx=ctx)


def per_order(a, b, B):
    """rel error of each derivative order k (state entries k, k+B, ...)."""
    return [rel(a[:, k::B], b[:, k::B]) for k in range(B)]


def compare(rep, z, meta, label, alts=()):
    """Equal-iteration parity.  Means at 1e-9 per derivative order, the
    uncalibrated covariance products L L^T / sigma_hat^2 at 1e-7 and sigma_hat
    at 1e-7 — except where the reference formulation itself is
    rounding-determined: in the rescaled coordinates (T_0 = sqrt(h) h^q / q!,
    ieks.cpp:28-33) the high derivative orders of the mean, and sigma_hat
    (from innovations that read them), carry rounding noise of order
    eps |x_0| T_k / T_0.  `alts` are GPU solves of the same problem that
    differ only in rounding (other chunk lengths, the element engine); the
    per-order floor is the GPU's largest distance to them, and each order (and
    sigma_hat) must agree with the oracle to max(tolerance, 10 x floor)."""
    nodes = z["nodes"]
    B = meta["nu"] + 1
    orders = per_order(rep.means[nodes], z["means"], B)
    sig = abs(rep.sigma_hat - meta["sigma_hat"]) / abs(meta["sigma_hat"])
    sr = (rep.sigma_hat / meta["sigma_hat"]) ** 2  # compare uncalibrated covariances
    ec = rel(cov_upper(rep.cov_sqrt, nodes) / sr, z["cov_upper"])
    floor = [0.0] * B
    f_sig = 0.0
    for alt in alts:
        floor = [max(f, e) for f, e in zip(floor, per_order(rep.means, alt.means, B))]
        f_sig = max(f_sig, abs(rep.sigma_hat - alt.sigma_hat) / abs(alt.sigma_hat))
    line = (f"{label}: {rep.iterations} its, mean orders " + " ".join(f"{e:.1e}" for e in orders) +
            f", cov/sigma^2 {ec:.1e}, sigma {sig:.1e} | GPU rounding floor: orders " +
            " ".join(f"{e:.1e}" for e in floor) + f", sigma {f_sig:.1e}")
    print(line)
    assert rep.iterations == meta["iterations"]
    assert ec <= COV_TOL, line
    for k in range(B):
        assert orders[k] <= max(MEAN_TOL, 10 * floor[k]), line
    assert sig <= max(SIG_TOL, 10 * f_sig), line


def alternatives(P, meta, its):
    """Solves differing from the default one only in rounding: the fused
    engine at two other chunk lengths and the element engine (the
    reference's per-iteration structure); above D = 16 (the large-state
    engine) two other chunkings."""
    D = (meta["nu"] + 1) * {"fhn": 2, "vanderpol": 2, "rigidbody": 3, "pleiades": 28}[meta["problem"]]
    out = []
    settings = [("elements", 0), ("auto", 13), ("auto", 19)] if D <= 16 else [("auto", 3), ("auto", 11)]
    for engine, chunk in settings:
        ctx = P.Context()
        ctx.set_engine(engine)
        ctx.set_chunk_len(chunk)
        out.append(gpu_solve(P, meta, ctx=ctx, max_iterations=its, **NEVER))
    return out


