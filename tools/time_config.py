"""Times one IEKS configuration on the GPU (fixed iteration count, stopping
rule disabled so engines are compared on equal work): ms/iteration and
step-iterations/s per engine.  python tools/time_config.py name nu log2N its [engines]"""
import json, os, sys, time
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paraode_b200 as P
name, nu, lg, its = sys.argv[1], int(sys.argv[2]), int(sys.argv[3]), int(sys.argv[4])
engines = sys.argv[5].split(",") if len(sys.argv) > 5 else ["auto", "elements"]
prob = P.problem_by_name(name)
N = 1 << lg
grid = P.uniform_grid(prob.t_end, N)
cfg = P.IeksConfig(max_iterations=its, traj_rtol=-1.0, obj_atol=-1.0, obj_rtol=0.0)
for eng in engines:
    ctx = P.Context(); ctx.set_engine(eng)
    P.para_ieks(prob, P.IwpPrior(nu, prob.dim, 1.0), grid, cfg, want_cov=False, ctx=ctx)  # warm-up
    t = time.perf_counter()
    r = P.para_ieks(prob, P.IwpPrior(nu, prob.dim, 1.0), grid, cfg, want_cov=False, ctx=ctx)
    dt = time.perf_counter() - t
    print(json.dumps(dict(problem=name, nu=nu, N=N, engine=eng, iterations=r.iterations, seconds=dt,
                          ms_per_iteration=1e3 * dt / its, step_iterations_per_s=N * its / dt)), flush=True)
