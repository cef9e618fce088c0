"""Bench lines for every BASELINE.json config on one B200 (profiles/):
FHN IWP(2) N-sweep 2^12..2^20 (configs[1]), Van der Pol IWP(3) 2^22
(configs[2], 1 GPU), rigid body IWP(4) 2^20 (configs[3]) and Pleiades
IWP(3) 2^18 (configs[4]).  Each line: the default-rule solve (iterations,
converged, wall time, time-steps/s) through the public API with device
outputs kept on the GPU (want_cov=True), and ms per iteration from a
fixed-iteration solve (stopping rule disabled) — the oracle's convergence
status for the same config is attached where a fixture exists."""
import json, os, sys, time
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402
import paraode_b200 as P  # noqa: E402

NEVER = dict(traj_rtol=-1.0, obj_atol=-1.0, obj_rtol=0.0)


def oracle(problem, nu, lg):
    tag = {"fhn": "fhn", "vanderpol": "vdp", "rigidbody": "rigid", "pleiades": "pleiades"}[problem]
    out = {}
    for suffix in ("seq", "par8"):
        f = os.path.join(ROOT, "tests", "golden", f"{tag}_q{nu}_n{lg}_{suffix}.npz")
        if os.path.exists(f):
            m = json.loads(str(np.load(f)["meta"]))
            out[f"oracle_{suffix}"] = dict(iterations=m["iterations"], converged=m["converged"])
    return out


def line(problem, nu, lg, fixed_its, reps=2):
    prob = P.problem_by_name(problem)
    grid = P.uniform_grid(prob.t_end, 1 << lg)
    prior = P.IwpPrior(nu, prob.dim, 1.0)
    P.para_ieks(prob, prior, grid, P.IeksConfig(max_iterations=2, **NEVER), want_cov=False)  # warm-up
    ts = []
    for _ in range(reps):
        t = time.perf_counter()
        r = P.para_ieks(prob, prior, grid, P.IeksConfig(max_iterations=fixed_its, **NEVER), want_cov=False)
        ts.append(time.perf_counter() - t)
    per_it = min(ts) / fixed_its
    # marginal cost of an iteration (the finalize, once per solve, cancels):
    # (T(2 k) - T(k)) / k
    t = time.perf_counter()
    P.para_ieks(prob, prior, grid, P.IeksConfig(max_iterations=2 * fixed_its, **NEVER), want_cov=False)
    marginal = (time.perf_counter() - t - min(ts)) / fixed_its
    if problem != "pleiades":  # warm the default-rule path (graph capture, finalize buffers)
        P.para_ieks(prob, prior, grid, want_cov=True)
    t = time.perf_counter()
    # Pleiades from the constant start diverges under the reference rule
    # (oracle and GPU alike, tests/test_gpu_big_engine.py): time the
    # fixed-iteration solve with the full report instead of a 100-iteration budget
    cfg = P.IeksConfig(max_iterations=fixed_its, **NEVER) if problem == "pleiades" else P.IeksConfig()
    c = P.para_ieks(prob, prior, grid, cfg, want_cov=True)
    wall = time.perf_counter() - t
    n = 1 << lg
    return dict(problem=problem, nu=nu, D=prob.dim * (nu + 1), N=n, iterations=c.iterations, converged=c.converged,
                solve_seconds=wall, time_steps_per_s=n / wall, ms_per_iteration=1e3 * per_it,
                step_iterations_per_s=n / per_it, fixed_iterations=fixed_its,
                ms_per_iteration_marginal=1e3 * marginal, **oracle(problem, nu, lg),
                note="wall time through the public API incl. the full SolverReport download")


if __name__ == "__main__":
    which = sys.argv[1] if len(sys.argv) > 1 else "all"
    cases = []
    if which in ("all", "sweep"):
        cases += [("fhn", 2, lg, 20) for lg in range(12, 21)]
    if which in ("all", "configs"):
        cases += [("vanderpol", 3, 22, 10), ("rigidbody", 4, 20, 10)]
    if which in ("all", "pleiades"):
        cases += [("pleiades", 3, 18, 2)]
    for cs in cases:
        print(json.dumps(line(*cs)), flush=True)
