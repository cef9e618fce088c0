"""ms per IEKS iteration (stopping rule disabled, fixed iteration count) of
FHN IWP(2) N=2^20 over the fused engine's knobs: chunk length L, level-0
scan fan-in, block-scan threshold.  Knobs are chosen on ms/iteration only
(the converged iteration count at 2^20 is rounding-determined)."""
import json, os, sys, time
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paraode_b200 as P
its = 30
prob = P.fitzhugh_nagumo()
grid = P.uniform_grid(prob.t_end, 1 << 20)
cfg = P.IeksConfig(max_iterations=its, traj_rtol=-1.0, obj_atol=-1.0, obj_rtol=0.0)
Ls = [int(x) for x in (sys.argv[1] if len(sys.argv) > 1 else "24,28,32").split(",")]
fans = (sys.argv[2] if len(sys.argv) > 2 else "4,6,8").split(",")
bscans = (sys.argv[3] if len(sys.argv) > 3 else "4096,16384").split(",")
for L in Ls:
    for f in fans:
        for b in bscans:
            os.environ["PODE_SCAN_FANIN"] = f
            os.environ["PODE_BSCAN"] = b
            ctx = P.Context(); ctx.set_chunk_len(L)
            P.para_ieks(prob, P.IwpPrior(2, 2, 1.0), grid, cfg, want_cov=False, ctx=ctx)
            ts = []
            for _ in range(3):
                t = time.perf_counter()
                P.para_ieks(prob, P.IwpPrior(2, 2, 1.0), grid, cfg, want_cov=False, ctx=ctx)
                ts.append(time.perf_counter() - t)
            print(json.dumps(dict(L=L, fanin=int(f), bscan=int(b), ms_per_iteration=1e3 * min(ts) / its,
                                  lib=os.environ.get("PODE_LIB_PATH", "default"))), flush=True)
