"""One IEKS solve (for ncu launch lists / full captures): python tools/prof_once.py LOG2N [problem] [nu] [max_iter]"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paraode_b200 as P  # noqa: E402

lg = int(sys.argv[1]) if len(sys.argv) > 1 else 16
name = sys.argv[2] if len(sys.argv) > 2 else "fhn"
nu = int(sys.argv[3]) if len(sys.argv) > 3 else 2
its = int(sys.argv[4]) if len(sys.argv) > 4 else 100
prob = P.problem_by_name(name)
grid = P.uniform_grid(prob.t_end, 2 ** lg)
rep = P.para_ieks(prob, P.IwpPrior(nu, prob.dim, 1.0), grid, P.IeksConfig(max_iterations=its), want_cov=True)
print(f"{name} nu={nu} N=2^{lg}: iterations={rep.iterations} converged={rep.converged} "
      f"launches={P.default_context().kernel_launches}")
