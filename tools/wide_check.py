import os, sys
sys.path.insert(0, "."); sys.path.insert(0, "tests")
import numpy as np
import paraode_b200 as P
import _oracle as O
prob = P.problem_by_name("vanderpol")
for n in (3000, 1000):
    grid = O.uniform_grid(prob.t_end, n)
    want = O.ieks(O.problem("vanderpol"), 3, grid, mode=0)
    for w in ("0", "1"):
        os.environ["PODE_WIDE"] = w
        for L in (2, 0):
            ctx = P.Context()
            if L: ctx.set_chunk_len(L)
            got = P.para_ieks(prob, P.IwpPrior(3, 2, 1.0), grid, ctx=ctx)
            err = np.abs(got.means - want["means"]).max(axis=0) / max(1.0, np.abs(want["means"]).max())
            print(n, "wide", w, "L", L, got.iterations, want["iterations"], " ".join(f"{e:.1e}" for e in err))
