import os, subprocess, sys
sys.path.insert(0, '.')
if len(sys.argv) > 1:
    import paraode_b200 as P
    g = P.uniform_grid(10.0, 30)
    r = P.para_ieks(P.logistic(), P.IwpPrior(2, 1, 1.0), g)
    print(os.environ.get("PODE_TAG"), os.environ.get("PODE_CHUNK"), "->", r.iterations, r.solution_means[-1], r.sigma_hat)
    sys.exit(0)
for env in [{}, {"PODE_IEKS_ENGINE": "elements"}, {"PODE_CHUNK": "2"}, {"PODE_CHUNK": "3"}, {"PODE_CHUNK": "5"}, {"PODE_CHUNK": "10"}, {"PODE_CHUNK": "15"}, {"PODE_CHUNK": "30"}, {"PODE_CHUNK": "31"}]:
    subprocess.run([sys.executable, __file__, "x"], env={**os.environ, **env})
