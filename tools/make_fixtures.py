"""Generate the large-N oracle fixtures under tests/golden/ (TEST INFRASTRUCTURE).

Runs the oracle (oracle/, the C++ restatement of the reference CPU path) at the
benchmarked sizes and writes what the GPU parity tests compare against:

  * FitzHugh–Nagumo, IWP(2), N = 2^20 (BASELINE.json configs[1], the headline):
      - seq_ieks, default IeksConfig (converged; reference stopping rule,
        proj/src/ieks.cpp:62-77,157-187)
      - seq_ieks, exactly 20 iterations (stopping rule disabled)
      - para_ieks on WorkPool(8), default config and exactly 20 iterations —
        the reference's own second path, to record how far its two paths
        drift apart at this size (the rounding floor of the comparison)
  * Van der Pol mu=1, IWP(3), N = 2^16, 2^18 and rigid body, IWP(4),
    N = 2^14, 2^16 (configs[2], configs[3]): seq_ieks, default config
    (converged flag + iteration count + the posterior after those iterations).

Each fixture stores, for nodes 0, s, 2s, ..., N (s = N / nodes_out):
means (D), the covariance products L L^T (upper triangle, row-major), the
solution means (d), plus the full objective trace, iterations, converged,
sigma_hat, the config and the wall time.

"Exactly k iterations" is IeksConfig(max_iterations=k, traj_rtol=-1,
obj_atol=-1, obj_rtol=0): the reference stopping rule can never fire, and the
reference does not validate tolerances (ieks.cpp:116-121), so this is the
reference's own driver run for k iterations.

Usage:  python tools/make_fixtures.py [case ...]   (default: all; runs cases
concurrently, one process each; seq cases are single-threaded)
"""
from __future__ import annotations

import json
import os
import sys
import time
from concurrent.futures import ProcessPoolExecutor

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, os.path.join(ROOT, "tests"))
GOLDEN = os.path.join(ROOT, "tests", "golden")

NEVER = dict(traj_rtol=-1.0, obj_atol=-1.0, obj_rtol=0.0)

# name: (problem, nu, log2 N, oracle mode, max_iterations, never_converge, nodes_out)
CASES = {
    "fhn_q2_n20_seq": ("fhn", 2, 20, 0, 100, False, 4096),
    "fhn_q2_n20_seq_it20": ("fhn", 2, 20, 0, 20, True, 4096),
    "fhn_q2_n20_par8": ("fhn", 2, 20, 8, 100, False, 4096),
    "fhn_q2_n20_par8_it20": ("fhn", 2, 20, 8, 20, True, 4096),
    "vdp_q3_n16_seq": ("vanderpol", 3, 16, 0, 100, False, 2048),
    "vdp_q3_n18_seq": ("vanderpol", 3, 18, 0, 100, False, 2048),
    "rigid_q4_n14_seq": ("rigidbody", 4, 14, 0, 100, False, 1024),
    "rigid_q4_n16_seq": ("rigidbody", 4, 16, 0, 100, False, 1024),
    # configs[4]: Pleiades (d = 28, IWP(3), D = 112) at the parity sizes of SURVEY.md §8(d)
    "pleiades_q3_n10_seq": ("pleiades", 3, 10, 0, 100, False, 64),
    "pleiades_q3_n10_seq_it3": ("pleiades", 3, 10, 0, 3, True, 64),
    "pleiades_q3_n12_seq_it2": ("pleiades", 3, 12, 0, 2, True, 64),
    "pleiades_q3_n12_par8_it2": ("pleiades", 3, 12, 8, 2, True, 64),
}


def run_case(name):
    import _oracle as O

    prob_name, nu, log2n, mode, max_it, never, nodes_out = CASES[name]
    prob = O.problem(prob_name)
    n = 1 << log2n
    grid = O.uniform_grid(prob.t_end, n)
    kw = dict(NEVER) if never else {}
    t0 = time.time()
    r = O.ieks(prob, nu, grid, mode=mode, max_iterations=max_it, **kw)
    wall = time.time() - t0
    stride = n // nodes_out
    idx = np.arange(0, n + 1, stride, dtype=np.int64)
    D = r["means"].shape[1]
    L = r["cov_sqrt"][idx]
    cov = np.einsum("nij,nkj->nik", L, L)
    iu = np.triu_indices(D)
    out = os.path.join(GOLDEN, name + ".npz")
    meta = dict(problem=prob_name, nu=nu, steps=n, t_end=prob.t_end, oracle_mode=mode,
                oracle_path="seq_ieks" if mode == 0 else f"para_ieks WorkPool({mode})",
                max_iterations=max_it, never_converge=never,
                config=dict(max_iterations=max_it, **(NEVER if never else
                                                        dict(traj_rtol=1e-13, obj_atol=1e-9, obj_rtol=1e-6))),
                iterations=r["iterations"], converged=r["converged"], sigma_hat=r["sigma_hat"],
                seconds=r["seconds"], wall=wall, stride=int(stride),
                generator="tools/make_fixtures.py")
    np.savez_compressed(out, nodes=idx, means=r["means"][idx], cov_upper=cov[:, iu[0], iu[1]],
                        solution_means=r["solution_means"][idx],
                        objective_trace=r["objective_trace"], meta=json.dumps(meta))
    return name, meta


def main(argv):
    names = argv or list(CASES)
    os.makedirs(GOLDEN, exist_ok=True)
    # par8 cases use 8 threads each; run them after the single-threaded ones
    seq = [n for n in names if CASES[n][3] <= 1]
    par = [n for n in names if CASES[n][3] > 1]
    for batch, workers in ((seq, 8), (par, 1)):
        if not batch:
            continue
        with ProcessPoolExecutor(max_workers=min(workers, len(batch))) as ex:
            for name, meta in ex.map(run_case, batch):
                print(name, json.dumps({k: meta[k] for k in ("iterations", "converged", "sigma_hat", "seconds")}),
                      flush=True)


if __name__ == "__main__":
    main(sys.argv[1:])
