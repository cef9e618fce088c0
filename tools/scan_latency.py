"""Two fixed IEKS iterations (no finalize timing intent) of one config, for
an ncu launch list of the aggregate-scan kernels: python tools/scan_latency.py name nu log2N"""
import os, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paraode_b200 as P
name, nu, lg = sys.argv[1], int(sys.argv[2]), int(sys.argv[3])
prob = P.problem_by_name(name)
grid = P.uniform_grid(prob.t_end, 1 << lg)
cfg = P.IeksConfig(max_iterations=2, traj_rtol=-1.0, obj_atol=-1.0, obj_rtol=0.0)
P.para_ieks(prob, P.IwpPrior(nu, prob.dim, 1.0), grid, cfg, want_cov=False)
