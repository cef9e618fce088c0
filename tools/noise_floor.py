"""Diagnostic (GPU): how far apart are two solves of the same IEKS problem
that differ only in rounding (the fused engine's chunk length L changes the
association order of every scan), next to the GPU-vs-oracle distance, at
equal iteration counts.  Prints one JSON line per (fixture, iteration count).

    python tools/noise_floor.py [fixture ...]
"""
import json
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))
import paraode_b200 as P  # noqa: E402

NEVER = dict(traj_rtol=-1.0, obj_atol=-1.0, obj_rtol=0.0)


def rel(a, b):
    return float(np.max(np.abs(a - b)) / max(1.0, np.max(np.abs(b))))


def solve(meta, its, chunk=None):
    if chunk:
        os.environ["PODE_CHUNK"] = str(chunk)
    else:
        os.environ.pop("PODE_CHUNK", None)
    prob = P.problem_by_name({"fhn": "fhn", "vanderpol": "vanderpol", "rigidbody": "rigidbody"}[meta["problem"]])
    grid = P.uniform_grid(meta["t_end"], meta["steps"])
    cfg = P.IeksConfig(max_iterations=its, **NEVER) if its else P.IeksConfig()
    return P.para_ieks(prob, P.IwpPrior(meta["nu"], prob.dim, 1.0), grid, cfg)


def main(names):
    for name in names:
        z = np.load(os.path.join(ROOT, "tests", "golden", name + ".npz"))
        meta = json.loads(str(z["meta"]))
        nodes = z["nodes"]
        B = meta["nu"] + 1
        for its in sorted({2, 5, 10, meta["iterations"]}):
            a = solve(meta, its)
            b = solve(meta, its, chunk=13)
            row = dict(fixture=name, iterations=its,
                       gpu_vs_gpu_L13=dict(means=rel(a.means, b.means), sol=rel(a.solution_means, b.solution_means),
                                           V=float(abs(a.objective_trace[-1] - b.objective_trace[-1]) /
                                                   abs(b.objective_trace[-1]))),
                       per_order_gpu_vs_gpu=[rel(a.means[:, k::B], b.means[:, k::B]) for k in range(B)])
            if its == meta["iterations"]:
                row["gpu_vs_oracle"] = dict(means=rel(a.means[nodes], z["means"]),
                                            sol=rel(a.solution_means[nodes], z["solution_means"]),
                                            per_order=[rel(a.means[nodes][:, k::B], z["means"][:, k::B])
                                                       for k in range(B)])
            row["V_gpu"] = float(a.objective_trace[-1])
            print(json.dumps(row), flush=True)
        c = solve(meta, 0)
        print(json.dumps(dict(fixture=name, default_rule=dict(gpu_iterations=c.iterations, gpu_converged=c.converged,
                                                              oracle_iterations=meta["iterations"],
                                                              oracle_converged=meta["converged"]))), flush=True)


if __name__ == "__main__":
    main(sys.argv[1:] or ["fhn_q2_n20_seq", "vdp_q3_n16_seq", "vdp_q3_n18_seq", "rigid_q4_n14_seq",
                          "rigid_q4_n16_seq"])
