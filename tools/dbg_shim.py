import sys; sys.path.insert(0,'.')
import numpy as np
import paraode_b200 as P
g = P.uniform_grid(10.0, 30)
r = P.para_ieks(P.logistic(), P.IwpPrior(2, 1, 1.0), g)
print("python:", r.iterations, r.solution_means[-1], r.sigma_hat)
