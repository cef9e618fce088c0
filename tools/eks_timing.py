"""Wall time of the device eks_solve (sequential forward pass in one warp +
reverse-scan smoother) against para_ieks on the same grids:
python tools/eks_timing.py [problem] [nu]"""
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paraode_b200 as P  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "fhn"
nu = int(sys.argv[2]) if len(sys.argv) > 2 else 2
prob = P.problem_by_name(name)
prior = P.IwpPrior(nu, prob.dim, 1.0)
for lg in (10, 12, 14, 16):
    grid = P.uniform_grid(prob.t_end, 2 ** lg)
    out = {"problem": name, "nu": nu, "N": 2 ** lg}
    for label, fn in (("eks", lambda: P.eks_solve(prob, prior, grid)), ("paraieks", lambda: P.para_ieks(prob, prior, grid))):
        fn()
        t0 = time.perf_counter()
        r = fn()
        dt = time.perf_counter() - t0
        out[label] = {"seconds": dt, "steps_per_s": 2 ** lg / dt, "iterations": r.iterations}
    print(json.dumps(out), flush=True)
