"""ms per IEKS iteration (stopping disabled, 30 iterations) of FHN IWP(2)
over chunk lengths at small N: python tools/small_n_chunks.py log2N L1,L2,.."""
import json, os, sys, time
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paraode_b200 as P
lg = int(sys.argv[1])
its = 30
prob = P.fitzhugh_nagumo()
grid = P.uniform_grid(prob.t_end, 1 << lg)
cfg = P.IeksConfig(max_iterations=its, traj_rtol=-1.0, obj_atol=-1.0, obj_rtol=0.0)
for L in [int(x) for x in sys.argv[2].split(",")]:
    ctx = P.Context()
    if L > 0:
        ctx.set_chunk_len(L)
    P.para_ieks(prob, P.IwpPrior(2, 2, 1.0), grid, cfg, want_cov=False, ctx=ctx)
    ts = []
    for _ in range(5):
        t = time.perf_counter()
        P.para_ieks(prob, P.IwpPrior(2, 2, 1.0), grid, cfg, want_cov=False, ctx=ctx)
        ts.append(time.perf_counter() - t)
    print(json.dumps(dict(log2N=lg, L=L, ms_per_iteration=1e3 * min(ts) / its)), flush=True)
