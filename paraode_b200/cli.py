"""Command-line harness: `python -m paraode_b200 solve|benchmark|compare`
(restates the reference CLI, proj/src/bench.cpp:171-365, on the B200 path).

- solve: one problem, JSON posterior (solution means, standard deviations,
  sigma_hat, iterations, objective trace) — exit 0 converged, 2 not
  converged, 1 on error (bench.cpp:171-207).
- benchmark: work-precision sweep, CSV with the reference's exact header
  (bench.cpp:32-34) and optional SVG chart; a failing cell is reported on
  stderr and kept with an empty rmse (bench.cpp:220-282).
- compare: the fused IEKS engine against the element engine (the
  reference's per-iteration para_rts structure) on grids 30/100/150, PASS
  when means agree to --tolerance with equal iteration counts
  (bench.cpp:290-318); exit 0 all pass, 1 otherwise.

Methods: `paraieks` (the fused engine), `paraieks-elements` (element
engine), `ieks` (seq_ieks: the same iterates with the whole grid in one
chunk, i.e. the Kalman folds run in time order in one thread; fused-engine
states, D <= 9) and `eks` (the non-iterated smoother, eks_solve).
"""
from __future__ import annotations

import argparse
import json
import math
import statistics
import sys
import time

import numpy as np

RUN_RECORD_HEADER = ("problem,method,nu,grid_size,rmse,runtime_seconds,iterations,sigma_hat,converged,"
                     "combine_invocations,sequential_depth")
METHODS = ("paraieks", "paraieks-elements", "ieks", "eks")
PROBLEMS = ("logistic", "rigidbody", "vanderpol")


class UsageError(Exception):
    pass


def _fmt(v: float) -> str:
    return "%.12g" % v


def csv_row(r: dict) -> str:
    """bench.cpp:44-54"""
    return ",".join([r["problem"], r["method"], str(r["nu"]), str(r["grid_size"]),
                     "" if r.get("rmse") is None else _fmt(r["rmse"]), _fmt(r["runtime_seconds"]),
                     str(r["iterations"]), _fmt(r["sigma_hat"]), "true" if r["converged"] else "false",
                     str(r["combine_invocations"]), str(r["sequential_depth"])])


def to_csv(records) -> str:
    return RUN_RECORD_HEADER + "\n" + "".join(csv_row(r) + "\n" for r in records)


def to_svg(records) -> str:
    """Log-log work-precision chart (runtime vs rmse), one series per
    problem/method/nu (bench.cpp:63-130)."""
    series = {}
    for r in records:
        if r.get("rmse") is None or not r["rmse"] > 0.0 or not r["runtime_seconds"] > 0.0:
            continue
        key = f'{r["problem"]} {r["method"]} nu={r["nu"]}'
        series.setdefault(key, []).append((math.log10(r["runtime_seconds"]), math.log10(r["rmse"])))
    if not series:
        return "<svg xmlns='http://www.w3.org/2000/svg'/>\n"
    xs = [p[0] for s in series.values() for p in s]
    ys = [p[1] for s in series.values() for p in s]
    xmin, xmax, ymin, ymax = min(xs), max(xs), min(ys), max(ys)
    if xmax - xmin < 1e-9:
        xmin, xmax = xmin - 0.5, xmax + 0.5
    if ymax - ymin < 1e-9:
        ymin, ymax = ymin - 0.5, ymax + 0.5
    w, h, ml, mr, mt, mb = 720, 480, 70, 20, 20, 50
    sx = lambda x: ml + (x - xmin) / (xmax - xmin) * (w - ml - mr)
    sy = lambda y: mt + (ymax - y) / (ymax - ymin) * (h - mt - mb)
    colors = ["#1f77b4", "#ff7f0e", "#2ca02c", "#d62728", "#9467bd", "#8c564b", "#e377c2", "#7f7f7f"]
    out = [f"<svg xmlns='http://www.w3.org/2000/svg' width='{w}' height='{h}'>",
           f"<rect width='{w}' height='{h}' fill='white'/>",
           f"<text x='{w / 2}' y='{h - 10}' text-anchor='middle'>log10 runtime [s]</text>",
           f"<text x='15' y='{h / 2}' transform='rotate(-90 15 {h / 2})' text-anchor='middle'>log10 RMSE</text>"]
    for idx, (label, pts) in enumerate(sorted(series.items())):
        color = colors[idx % len(colors)]
        pts = sorted(pts)
        out.append("<polyline fill='none' stroke='%s' points='%s'/>" %
                   (color, " ".join(f"{sx(x):.2f},{sy(y):.2f}" for x, y in pts)))
        out.extend(f"<circle cx='{sx(x):.2f}' cy='{sy(y):.2f}' r='3' fill='{color}'/>" for x, y in pts)
        out.append(f"<text x='{ml + 10}' y='{mt + 16 + 16 * idx}' fill='{color}'>{label}</text>")
    out.append("</svg>")
    return "\n".join(out) + "\n"


def _solver(method: str):
    if method not in METHODS:
        raise UsageError(f"unknown method '{method}' (expected {', '.join(METHODS)})")
    import paraode_b200 as P
    ctxs = {}  # one dedicated context per engine setting, reused across runs

    def engine_ctx(engine, chunk=0):
        if engine not in ctxs:
            ctxs[engine] = P.Context()
            ctxs[engine].set_engine(engine)
        ctxs[engine].set_chunk_len(chunk)
        return ctxs[engine]

    def run(prob, prior, grid, config):
        if method == "eks":  # bench.cpp:139
            return P.eks_solve(prob, prior, grid, config.linearization)
        if method == "ieks":  # bench.cpp:138: seq_ieks = the same iterates, time-sequential
            # one chunk on a dedicated context: a single lane thread runs every
            # Kalman fold in time order; states no fused engine serves are
            # rejected (UnsupportedError) rather than run on the parallel
            # element engine under this label
            return P.para_ieks(prob, prior, grid, config, ctx=engine_ctx("fused", max(2, len(grid) - 1)))
        if method == "paraieks-elements":
            return P.para_ieks(prob, prior, grid, config, ctx=engine_ctx("elements"))
        return P.para_ieks(prob, prior, grid, config)
    return run


def _problem(name: str):
    if name not in PROBLEMS + ("fhn",):
        raise UsageError(f"unknown problem '{name}' (expected logistic, rigidbody or vanderpol)")
    import paraode_b200 as P
    return P.problem_by_name(name)


def _write(path: str, content: str):
    if not path:
        sys.stdout.write(content)
        return
    try:
        with open(path, "w") as f:
            f.write(content)
    except OSError:
        raise UsageError(f"cannot open output file '{path}'")


def cmd_solve(a) -> int:
    """bench.cpp:171-207"""
    prob = _problem(a.problem)
    run = _solver(a.method)
    if a.n < 2:
        raise UsageError("solve: --n must be at least 2")
    if not 1 <= a.nu <= 4:
        raise UsageError("solve: --nu must be in 1..4")
    import paraode_b200 as P
    grid = P.uniform_grid(prob.t_end, a.n)
    rep = run(prob, P.IwpPrior(a.nu, prob.dim, 1.0), grid, P.IeksConfig(max_iterations=a.max_iterations))
    doc = {"problem": a.problem, "method": a.method, "nu": a.nu, "grid_size": a.n, "grid": rep.times.tolist(),
           "mean": rep.solution_means.tolist(),
           "std": np.sqrt(np.maximum(np.diagonal(rep.solution_covs, axis1=1, axis2=2), 0.0)).tolist(),
           "sigma_hat": rep.sigma_hat, "iterations": rep.iterations, "converged": bool(rep.converged),
           "objective_trace": rep.objective_trace.tolist()}
    _write(a.out, json.dumps(doc, indent=2, sort_keys=True) + "\n")  # nlohmann::json orders keys
    return 0 if rep.converged else 2


def cmd_benchmark(a) -> int:
    """bench.cpp:220-287"""
    if a.repeats < 1:
        raise UsageError("benchmark: --repeats must be at least 1")
    import paraode_b200 as P
    from .accuracy import reference_for, rmse
    nus = [1, 2] if a.nu == 0 else [a.nu]
    records = []
    for pname in a.problems:
        prob = _problem(pname)
        refs = {}  # per grid size: a table whose nodes include the grid's (accuracy.reference_for)
        for mname in a.methods:
            run = _solver(mname)
            for nu in nus:
                for n in a.grid_sizes:
                    rec = dict(problem=pname, method=mname, nu=nu, grid_size=n, rmse=None, runtime_seconds=0.0,
                               iterations=0, sigma_hat=0.0, converged=False, combine_invocations=0,
                               sequential_depth=0)
                    try:
                        if n < 2:
                            raise UsageError("benchmark: grid sizes must be at least 2")
                        grid = P.uniform_grid(prob.t_end, n)
                        prior = P.IwpPrior(nu, prob.dim, 1.0)
                        times = []
                        for r in range(a.repeats + 1):  # one warm-up plus timed repeats
                            t0 = time.perf_counter()
                            rep = run(prob, prior, grid, P.IeksConfig())
                            if r > 0:
                                times.append(time.perf_counter() - t0)
                        if n not in refs:
                            refs[n] = reference_for(pname, grid_steps=n)
                        rec.update(runtime_seconds=statistics.median(times),
                                   rmse=rmse(rep.solution_means, refs[n], grid), iterations=rep.iterations,
                                   sigma_hat=rep.sigma_hat, converged=bool(rep.converged),
                                   combine_invocations=rep.combine_invocations,
                                   sequential_depth=rep.sequential_depth)
                    except Exception as e:  # the cell is kept with an empty rmse
                        sys.stderr.write(f"benchmark cell {pname}/{mname}/nu={nu}/n={n} failed: {e}\n")
                        rec["rmse"], rec["converged"] = None, False
                    records.append(rec)
    _write(a.out, to_csv(records))
    if a.svg:
        try:
            with open(a.svg, "w") as f:
                f.write(to_svg(records))
        except OSError:
            raise UsageError(f"cannot open SVG file '{a.svg}'")
    return 0


def cmd_compare(a) -> int:
    """bench.cpp:290-318: fused engine vs element engine, nu = 2."""
    import paraode_b200 as P
    fused, elements = _solver("paraieks"), _solver("paraieks-elements")
    all_ok = True
    for pname in a.problems:
        prob = _problem(pname)
        for n in (30, 100, 150):
            grid = P.uniform_grid(prob.t_end, n)
            prior = P.IwpPrior(2, prob.dim, 1.0)
            ref = elements(prob, prior, grid, P.IeksConfig())
            got = fused(prob, prior, grid, P.IeksConfig())
            diff = float(np.max(np.abs(ref.means - got.means)))
            ok = diff <= a.tolerance and ref.iterations == got.iterations
            all_ok = all_ok and ok
            print("%-10s n=%-4d max_mean_diff=%.3e iterations=%d/%d %s" %
                  (pname, n, diff, ref.iterations, got.iterations, "PASS" if ok else "FAIL"))
    return 0 if all_ok else 1


class _Parser(argparse.ArgumentParser):
    def error(self, message):  # CLI11 parse errors exit 1 (bench.cpp:348-351)
        raise UsageError(message)


def _csv(kind):
    return lambda s: [kind(x) for x in s.split(",") if x != ""]


def build_parser():
    ap = _Parser(prog="paraode_b200", description="Parallel-in-time probabilistic ODE solver (B200)")
    sub = ap.add_subparsers(dest="cmd", parser_class=_Parser)
    s = sub.add_parser("solve", help="Solve one problem and print the posterior")
    s.add_argument("--problem", default="logistic")
    s.add_argument("--method", default="paraieks")
    s.add_argument("--nu", type=int, default=2)
    s.add_argument("--n", type=int, default=100)
    s.add_argument("--max-iterations", type=int, default=100)
    s.add_argument("--workers", type=int, default=0, help="accepted for compatibility (the GPU grid replaces the pool)")
    s.add_argument("--out", default="")
    b = sub.add_parser("benchmark", help="Work-precision sweep, CSV output")
    b.add_argument("--problems", type=_csv(str), default=list(PROBLEMS))
    b.add_argument("--methods", type=_csv(str), default=["paraieks"])
    b.add_argument("--nu", type=int, default=0)
    b.add_argument("--grid-sizes", type=_csv(int), default=[16, 32, 64, 128, 256, 512, 1024, 2048, 4096])
    b.add_argument("--repeats", type=int, default=3)
    b.add_argument("--workers", type=int, default=0)
    b.add_argument("--out", default="")
    b.add_argument("--svg", default="")
    c = sub.add_parser("compare", help="Check the fused engine against the element engine")
    c.add_argument("--problems", type=_csv(str), default=list(PROBLEMS))
    c.add_argument("--tolerance", type=float, default=1e-8)
    c.add_argument("--workers", type=int, default=0)
    return ap


def main(argv=None) -> int:
    ap = build_parser()
    try:
        a = ap.parse_args(argv)
    except SystemExit as e:  # --help
        return 0 if not e.code else 1
    except UsageError as e:
        sys.stderr.write(f"error: {e}\n")
        return 1
    if a.cmd is None:
        sys.stderr.write("error: a subcommand is required (solve, benchmark, compare)\n")
        return 1
    try:
        return {"solve": cmd_solve, "benchmark": cmd_benchmark, "compare": cmd_compare}[a.cmd](a)
    except Exception as e:
        sys.stderr.write(f"error: {e}\n")
        return 1
