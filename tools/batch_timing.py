"""Fused batched solve vs one solve at a time (tests/test_gpu_batch.py's FHN
sweep): wall time per call through the public API, second call onwards
(graphs and workspaces cached), for a few batch sizes and N."""
import json
import sys
import time

import numpy as np

sys.path.insert(0, ".")
import paraode_b200 as P  # noqa: E402


def sweep(k):
    out = []
    for i in range(k):
        p = P.fitzhugh_nagumo(0.2 + 0.01 * (i % 5), 0.2, 3.0 - 0.1 * (i % 3))
        p.y0 = np.array([-1.0 + 0.05 * (i % 24), 1.0 - 0.03 * (i % 24)])
        out.append(p)
    return out


prior = P.IwpPrior(2, 2, 1.0)
for n, nb in [(1024, 64), (4096, 64), (4096, 256), (16384, 64)]:
    probs = sweep(nb)
    grid = P.uniform_grid(20.0, n)
    for want_cov in (False, True):
        P.para_ieks_fused_batch(probs, prior, grid, want_cov=want_cov)
        t0 = time.perf_counter()
        got = P.para_ieks_fused_batch(probs, prior, grid, want_cov=want_cov)
        t1 = time.perf_counter()
        its = [g.iterations for g in got]
        P.para_ieks(probs[0], prior, grid, want_cov=want_cov)
        t2 = time.perf_counter()
        one = [P.para_ieks(p, prior, grid, want_cov=want_cov) for p in probs[:8]]
        t3 = time.perf_counter()
        print(json.dumps({"N": n, "ivps": nb, "want_cov": want_cov, "fused_ms": 1e3 * (t1 - t0),
                          "single_ms_each": 1e3 * (t3 - t2) / 8, "max_iterations": max(its),
                          "time_steps_per_s_fused": n * nb / (t1 - t0),
                          "time_steps_per_s_single": n / ((t3 - t2) / 8)}), flush=True)
