import sys, os
import numpy as np
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT); sys.path.insert(0, os.path.join(ROOT, "tests"))
import paraode_b200 as P
import _oracle as O
from _dense import dense_cov
NEVER = dict(traj_rtol=-1.0, obj_atol=-1.0, obj_rtol=0.0)
for name, nu, steps, chunk, its in [("rigidbody", 4, 30, 8, 2), ("rigidbody", 4, 30, 100000, 2), ("rigidbody", 4, 37, 7, 2)]:
    op = O.problem(name)
    grid = O.uniform_grid(op.t_end, steps)
    want = O.ieks(op, nu, grid, mode=0, max_iterations=its, **NEVER)
    ctx = P.Context(); ctx.set_chunk_len(chunk)
    got = P.para_ieks(P.problem_by_name(name), P.IwpPrior(nu, op.dim, 1.0), grid, P.IeksConfig(max_iterations=its, **NEVER), ctx=ctx)
    gc, wc = dense_cov(got.cov_sqrt), dense_cov(want["cov_sqrt"])
    bad = np.unique(np.argwhere(~np.isfinite(got.cov_sqrt))[:, 0])
    err = np.nanmax(np.abs(gc - wc).reshape(len(gc), -1), axis=1)
    print(name, nu, steps, chunk, "sig", got.sigma_hat, want["sigma_hat"], "nonfinite nodes", bad.tolist(), flush=True)
    print("  cov err per node", np.array2string(err, precision=1, max_line_width=250), flush=True)
    print("  means err", np.nanmax(np.abs(got.means - want["means"])), flush=True)
