"""Pleiades (d = 28, IWP(3), D = 112) on the large-state engine: default-rule
convergence at several N, and ms per iteration (stopping rule disabled)."""
import json, os, sys, time
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paraode_b200 as P
prob = P.pleiades()
for lg in [int(x) for x in sys.argv[1].split(",")]:
    grid = P.uniform_grid(prob.t_end, 1 << lg)
    t = time.perf_counter()
    r = P.para_ieks(prob, P.IwpPrior(3, 28, 1.0), grid, P.IeksConfig(max_iterations=int(sys.argv[2])), want_cov=False)
    dt = time.perf_counter() - t
    print(json.dumps(dict(N=1 << lg, iterations=r.iterations, converged=r.converged, seconds=dt,
                          trace=[float(v) for v in r.objective_trace[-4:]], sigma_hat=r.sigma_hat)), flush=True)
