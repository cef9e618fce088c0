import sys, time
sys.path.insert(0, ".")
import paraode_b200 as P
prob = P.fitzhugh_nagumo()
grid = P.uniform_grid(prob.t_end, 1 << 20)
cfg = P.IeksConfig(max_iterations=20, traj_rtol=-1.0, obj_atol=-1.0, obj_rtol=0.0)
prior = P.IwpPrior(2, 2, 1.0)
ctx = P.Context()
ctx.nccl_init(P.nccl_unique_id(), 0, 1)
for name, f in (("single", lambda: P.para_ieks(prob, prior, grid, cfg, want_cov=False)),
                ("shard R=1 nccl", lambda: P.para_ieks_sharded(prob, prior, grid, 0, 1, None, cfg, want_cov=False, ctx=ctx))):
    f()
    t = time.perf_counter(); f(); dt = time.perf_counter() - t
    print(name, round(1e3 * dt / 20, 3), "ms per iteration (incl. finalize / 20)")
