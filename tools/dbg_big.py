import sys, os, time
import numpy as np
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT); sys.path.insert(0, os.path.join(ROOT, "tests"))
import paraode_b200 as P
import _oracle as O
from _dense import dense_cov
NEVER = dict(traj_rtol=-1.0, obj_atol=-1.0, obj_rtol=0.0)
op = O.problem("pleiades")
for nu, steps, its, chunk in [(1, 16, 1, 0), (1, 16, 1, 4), (1, 64, 2, 0), (3, 64, 2, 0), (3, 64, 2, 5)]:
    grid = O.uniform_grid(op.t_end, steps)
    t = time.time()
    want = O.ieks(op, nu, grid, mode=0, max_iterations=its, **NEVER)
    to = time.time() - t
    ctx = P.Context(); ctx.set_chunk_len(chunk)
    t = time.time()
    try:
        got = P.para_ieks(P.pleiades(), P.IwpPrior(nu, 28, 1.0), grid, P.IeksConfig(max_iterations=its, **NEVER), ctx=ctx)
    except Exception as e:
        print(nu, steps, its, chunk, "ERR", type(e).__name__, e, flush=True); continue
    tg = time.time() - t
    B = nu + 1
    om = [float(np.max(np.abs(got.means[:, k::B] - want["means"][:, k::B])) / max(1, np.abs(want["means"][:, k::B]).max())) for k in range(B)]
    gc, wc = dense_cov(got.cov_sqrt), dense_cov(want["cov_sqrt"])
    ec = float(np.nanmax(np.abs(gc - wc)) / max(1, np.abs(wc).max()))
    print(nu, steps, its, chunk, "orders", ["%.1e" % x for x in om], "cov %.1e" % ec, "sig", got.sigma_hat, want["sigma_hat"],
          "trace", got.objective_trace, want["objective_trace"], "t_gpu %.2f t_orc %.2f" % (tg, to), flush=True)
