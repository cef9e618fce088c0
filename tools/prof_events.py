"""Per-kernel CUDA-event breakdown of one IEKS solve (pode_profile; the
per-iteration host loop): python tools/prof_events.py name nu log2N its [chunk]"""
import json, os, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paraode_b200 as P
name, nu, lg, its = sys.argv[1], int(sys.argv[2]), int(sys.argv[3]), int(sys.argv[4])
prob = P.problem_by_name(name)
grid = P.uniform_grid(prob.t_end, 1 << lg)
cfg = P.IeksConfig(max_iterations=its, traj_rtol=-1.0, obj_atol=-1.0, obj_rtol=0.0)
ctx = P.Context()
if len(sys.argv) > 5:
    ctx.set_chunk_len(int(sys.argv[5]))
P.para_ieks(prob, P.IwpPrior(nu, prob.dim, 1.0), grid, cfg, ctx=ctx)
ctx.profile(True)
P.para_ieks(prob, P.IwpPrior(nu, prob.dim, 1.0), grid, cfg, ctx=ctx)
prof = ctx.profile_read()
ctx.profile(False)
tot = sum(ms for _, ms in prof.values())
for k, (n, ms) in sorted(prof.items(), key=lambda kv: -kv[1][1]):
    print(f"{k:24s} {n:6d} {ms:10.3f} ms {100 * ms / tot:5.1f}%  {1e3 * ms / its:9.1f} us/iter")
print(f"total {tot:.3f} ms, {tot / its:.3f} ms/iter")
