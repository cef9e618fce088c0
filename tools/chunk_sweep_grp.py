"""ms per iteration of the group engine (rigid body IWP(4), D = 15,
N = 2^20) over chunk lengths (stopping rule disabled, fixed iterations)."""
import json, os, sys, time
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paraode_b200 as P
its = 8
prob = P.rigid_body()
grid = P.uniform_grid(prob.t_end, 1 << 20)
cfg = P.IeksConfig(max_iterations=its, traj_rtol=-1.0, obj_atol=-1.0, obj_rtol=0.0)
for L in [int(x) for x in sys.argv[1].split(",")]:
    ctx = P.Context(); ctx.set_chunk_len(L)
    P.para_ieks(prob, P.IwpPrior(4, 3, 1.0), grid, cfg, want_cov=False, ctx=ctx)
    t = time.perf_counter()
    P.para_ieks(prob, P.IwpPrior(4, 3, 1.0), grid, cfg, want_cov=False, ctx=ctx)
    print(json.dumps(dict(L=L, ms_per_iteration=1e3 * (time.perf_counter() - t) / its)), flush=True)
