import sys, os, time
import numpy as np
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT); sys.path.insert(0, os.path.join(ROOT, "tests"))
import paraode_b200 as P
import _oracle as O
NEVER = dict(traj_rtol=-1.0, obj_atol=-1.0, obj_rtol=0.0)
name, nu, steps, chunk, its = sys.argv[1], int(sys.argv[2]), int(sys.argv[3]), int(sys.argv[4]), int(sys.argv[5])
op = O.problem(name)
grid = O.uniform_grid(op.t_end, steps)
want = O.ieks(op, nu, grid, mode=0, max_iterations=its, **NEVER)
ctx = P.Context(); ctx.set_chunk_len(chunk)
if len(sys.argv) > 6: ctx.profile(True)
t = time.time()
got = P.para_ieks(P.problem_by_name(name), P.IwpPrior(nu, op.dim, 1.0), grid, P.IeksConfig(max_iterations=its, **NEVER), ctx=ctx)
d = np.abs(got.means - want["means"])
print(name, nu, steps, chunk, its, "maxdiff %.3e" % np.nanmax(d), "t %.3f" % (time.time() - t), got.objective_trace, want["objective_trace"], flush=True)
print("  node diffs", np.array2string(np.nanmax(d, axis=1), precision=2, max_line_width=200), flush=True)
if len(sys.argv) > 6: print(ctx.profile_read())
