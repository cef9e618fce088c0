import json, sys, numpy as np
sys.path.insert(0, '.'); sys.path.insert(0, 'tests')
import paraode_b200 as P
from _parity import NEVER
z = np.load('tests/golden/pleiades_q3_n12_seq_it2.npz'); meta = json.loads(str(z['meta']))
print("oracle", z['objective_trace'])
prob = P.pleiades(); grid = P.uniform_grid(prob.t_end, meta['steps'])
for ch in [0, 5, 16, 64, 4096]:
    ctx = P.Context(); ctx.set_chunk_len(ch)
    r = P.para_ieks(prob, P.IwpPrior(3, 28, 1.0), grid, P.IeksConfig(max_iterations=2, **NEVER), ctx=ctx)
    m = r.means[z['nodes']]
    B = 4
    rel = [float(np.max(np.abs(m[:, k::B] - z['means'][:, k::B])) / np.max(np.abs(z['means'][:, k::B]))) for k in range(B)]
    print(ch, r.objective_trace, rel, r.sigma_hat, meta['sigma_hat'])
grid10 = P.uniform_grid(prob.t_end, 1024)
r = P.para_ieks(prob, P.IwpPrior(3, 28, 1.0), grid10, P.IeksConfig(max_iterations=1, **NEVER))
print("2^10 it1", r.objective_trace)
