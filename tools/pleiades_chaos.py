"""Where the GPU's Pleiades N=2^10 Gauss-Newton trace departs from the
oracle's (tests/golden/pleiades_q3_n10_seq.npz): the iteration diverges
(objective ~1e19), so from some iteration on the iterates are decided by
rounding.  python tools/pleiades_chaos.py [its]"""
import json, os, sys
import numpy as np
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paraode_b200 as P
z = np.load(os.path.join(ROOT, "tests/golden/pleiades_q3_n10_seq.npz"))
want = z["objective_trace"]
prob = P.pleiades()
grid = P.uniform_grid(prob.t_end, 1024)
its = int(sys.argv[1]) if len(sys.argv) > 1 else 40
cfg = P.IeksConfig(max_iterations=its, traj_rtol=-1.0, obj_atol=-1.0, obj_rtol=0.0)
try:
    r = P.para_ieks(prob, P.IwpPrior(3, 28, 1.0), grid, cfg, want_cov=False)
    tr = r.objective_trace
    print("completed", len(tr), "iterations")
except P.SingularFactorError as e:
    print("SingularFactorError", e, getattr(e, "iteration", None))
    tr = None
if tr is not None:
    rel = np.abs(tr - want[:len(tr)]) / np.abs(want[:len(tr)])
    print(json.dumps([float(f"{v:.2e}") for v in rel]))
try:
    r = P.para_ieks(prob, P.IwpPrior(3, 28, 1.0), grid, P.IeksConfig(), want_cov=False)
    print("default rule:", r.iterations, r.converged, r.objective_trace[-1])
except P.SingularFactorError as e:
    print("default rule: SingularFactorError", e, getattr(e, "iteration", None))
