"""A/B of lane-pass builds (block size / register cap) and chunk lengths:
ms per IEKS iteration of FHN IWP(2) N=2^20, stopping disabled (30
iterations), per-kernel split from the context profile.  Usage:
PODE_LIB_PATH=<lib> python tools/lane_ab.py L1,L2,..."""
import json, os, sys, time
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paraode_b200 as P
its = 30
prob = P.fitzhugh_nagumo()
grid = P.uniform_grid(prob.t_end, 1 << 20)
cfg = P.IeksConfig(max_iterations=its, traj_rtol=-1.0, obj_atol=-1.0, obj_rtol=0.0)
for L in [int(x) for x in sys.argv[1].split(",")]:
    ctx = P.Context()
    ctx.set_chunk_len(L)
    P.para_ieks(prob, P.IwpPrior(2, 2, 1.0), grid, cfg, want_cov=False, ctx=ctx)
    ts = []
    for _ in range(3):
        t = time.perf_counter()
        P.para_ieks(prob, P.IwpPrior(2, 2, 1.0), grid, cfg, want_cov=False, ctx=ctx)
        ts.append(time.perf_counter() - t)
    print(json.dumps(dict(L=L, ms_per_iteration=1e3 * min(ts) / its,
                          lib=os.environ.get("PODE_LIB_PATH", "default"))), flush=True)
