"""Benchmark of the ParaIEKS hot path on B200.

One "step" = one IEKS solve to the reference's stopping rule (FitzHugh–Nagumo,
d=2, IWP(q=2), D=6, N=2^20 uniform steps on [0, 20]; BASELINE.json
configs[1] at its largest N).  value = time-steps/s over all ranks with the
solve's outputs written to HBM; e2e = the same metric through the public
Python API (paraode_b200.para_ieks) with host numpy buffers, so the grid
upload and the full SolverReport download are inside the timed region.
`--impl reference` times the reference algorithm on the host cores (the C++
restatement in oracle/ — the reference itself needs Eigen, absent here).

Multi-GPU: one process per GPU (torchrun); each rank solves its own
independent problem (replicas, weak scaling) — DESIGN.md §Multi-GPU.
"""
import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "IEKS wall-time to converged posterior; time-steps/s at N=2^20, 1/2/4/8 GPU"
CPU_SAMPLE_N = 2 ** 13  # bounded CPU sample: a full solve at reduced N
HBM_FALLBACK_GBS = 6650.0
FP64_FALLBACK_TFS = 36.6


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=3)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--log2n", type=int, default=20)
    ap.add_argument("--problem", default="fhn")
    ap.add_argument("--nu", type=int, default=2)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--mode", default="auto", choices=["auto", "shard", "replicas"],
                    help="N>1: shard one solve along time (strong scaling, default) or run replicas")
    return ap.parse_args()


def dist_env():
    return (int(os.environ.get("RANK", "0")), int(os.environ.get("WORLD_SIZE", "1")),
            int(os.environ.get("LOCAL_RANK", "0")))


def peaks():
    """Roofline denominators: MEASURED_PEAKS.json (driver-written HBM copy)
    and profiles/r01_fp64_peak.json (our DFMA measurement on this pool)."""
    hbm, hbm_src = HBM_FALLBACK_GBS, "fallback (B200_PROFILING.md)"
    try:
        hbm = float(json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))["hbm_gbs"])
        hbm_src = "measured (MEASURED_PEAKS.json)"
    except Exception:
        pass
    fp64, fp64_src = FP64_FALLBACK_TFS, "fallback (nominal)"
    try:
        fp64 = float(json.load(open(os.path.join(ROOT, "profiles", "r02_fp64_peak.json")))["fp64_fma_tflops"])
        fp64_src = "measured DFMA (profiles/r02_fp64_peak.json, clocks recorded)"
    except Exception:
        pass
    return hbm, hbm_src, fp64, fp64_src


def f_lq(R, K, P):
    """FMAs of a Householder LQ sweep over P pivots of an R x K row block."""
    return sum(2 * (K - p - 1) + (R - p - 1) * 2 * (K - p) for p in range(P))


def kernel_model(D, d):
    """Algorithmic (flops, HBM bytes) per time step of the fused-iteration
    kernels.  8-byte fp64 words."""
    B = D // d
    phi = d * B * (B + 1) // 2  # nonzeros of the block-binomial transition
    upd = d * D * (d + 1) + f_lq(d + D, D, D) + D * d * d // 2 + D * d + d * (d + 1)
    fwd_reduce = (2 * phi * D + phi + f_lq(D, 2 * D, D) + upd + d * D * (d + 1) + D * d * D + D * d
                  + D * d * d + D * d + d * D * D)
    fwd_down = phi * D + D * D * (D + 1) // 2 + f_lq(D, 2 * D, D) + D * D * D + D * D + phi + upd
    return {
        "fast_fwd_reduce": (2 * fwd_reduce, 8 * D),
        # pass C with the backward chunk aggregate (pass C2) fused in
        "fast_fwd_down": (2 * (fwd_down + D ** 3 + D * D), 8 * (D + D * D + D)),
        "fast_bwd_fold": (2 * (D ** 3 + D * D), 8 * (D * D + D)),
        "fast_bwd_down": (2 * (D * D + phi + D * D // 2 + 2 * D), 8 * (D * D + D + 2 * D)),
    }


def combine_flops(D):
    """⊗_f dense-op flops (30 1/3 D^3 + 20 D^2; 7.27 k at D=6)
    and the Gaussian-carry combine (A = eta = J = 0 on the left: 5.3 k at
    D=6, same ratio)."""
    full = 30.0 + 1.0 / 3.0
    f = full * D ** 3 + 20 * D * D
    return f, f * 5.3 / 7.27


def sklansky_readers(cnt):
    """Combines a Sklansky scan of cnt elements needs (readers per step)."""
    tot, h = 0, 1
    while h < cnt:
        tot += sum(1 for p in range(cnt) if p & h)
        h <<= 1
    return tot


def scan_model(N, D, sm=148, fanin=4):
    """Algorithmic (flops, bytes) per IEKS iteration of the aggregate-scan
    kernels, replaying fast_driver.cuh's tree: chunk length L (one chunk per
    lane thread), level 0 sequential fan-in, upper levels block-Sklansky of
    G = 8 * (32 // D) elements (engine.cuh)."""
    L = max(8, min(-(-N // (sm * 256)), 4096))
    nc = -(-N // L)
    G = 8 * (32 // D)
    f_full, f_gauss = combine_flops(D)
    f_aff = 2 * D ** 3 + 2 * D * D  # mean-only ⊗_s (E, g)
    el_f, el_m = 8 * (3 * D * D + 2 * D), 8 * (D * D + D)
    out = {}

    def add(k, fl, by):
        a = out.setdefault(k, [0.0, 0.0])
        a[0] += fl
        a[1] += by
    # level 0: fan-in reduce with local prefixes, then the one-deep down-sweep
    add("scan_g_reduce", (nc - -(-nc // fanin)) * f_full, 2 * nc * el_f)
    add("scan_m_reduce", (nc - -(-nc // fanin)) * f_aff, 2 * nc * el_m)
    n = -(-nc // fanin)
    downs = [(nc, fanin)] if n > 1 else []
    while n > 1:
        if n > 4096:  # engine.cuh bscan_max(): large levels stay sequential fan-in
            m = -(-n // fanin)
            add("scan_g_reduce", (n - m) * f_full, 2 * n * el_f)
            add("scan_m_reduce", (n - m) * f_aff, 2 * n * el_m)
            if m > 1:
                downs.append((n, fanin))
            n = m
            continue
        nb = -(-n // G)
        work = sum(sklansky_readers(min(G, n - b * G)) for b in range(nb))
        add("bscan_g", work * f_full, 2 * n * el_f)
        add("bscan_m", work * f_aff, 2 * n * el_m)
        if nb > 1:
            downs.append((n, G))
        n = nb
    for m, c in downs:
        add("scan_g_down", (m - min(m, c)) * f_gauss, m * (el_f + 8 * (D + D * D)))
        add("scan_m_down", (m - min(m, c)) * (2 * D * D), m * (el_m + 8 * D))
    return out


class ClockSampler:
    """nvidia-smi clocks / throttle reasons sampled during the timed region."""

    def __init__(self, index):
        self.index, self.rows, self.proc = index, [], None

    def __enter__(self):
        q = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.hw_slowdown,"
             "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
             "clocks_event_reasons.sw_power_cap")
        try:
            self.proc = subprocess.Popen(["nvidia-smi", "-i", str(self.index), f"--query-gpu={q}",
                                          "--format=csv,noheader,nounits", "-lms", "100"],
                                         stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            threading.Thread(target=self._read, daemon=True).start()
        except FileNotFoundError:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            parts = [p.strip() for p in line.split(",")]
            if len(parts) == 7:
                self.rows.append(parts)

    def __exit__(self, *a):
        if self.proc:
            time.sleep(0.25)
            self.proc.terminate()
            self.proc.wait(timeout=5)

    def summary(self):
        if not self.rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"]}
        sm = [float(r[0]) for r in self.rows if r[0].replace(".", "").isdigit()]
        mx = [float(r[1]) for r in self.rows if r[1].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[k] for r in self.rows for k in range(4) if r[3 + k] == "Active"})
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": reasons, "samples": len(self.rows)}


def cpu_solve(problem_name, nu, n, threads):
    """One full solve of the reference algorithm on the host (oracle/, the C++
    restatement; mode 0 = seq_ieks on one thread, k > 1 = para_ieks on a
    WorkPool(k))."""
    sys.path.insert(0, os.path.join(ROOT, "tests"))
    import _oracle as O
    prob = O.problem(problem_name)
    grid = O.uniform_grid(prob.t_end, n)
    r = O.ieks(prob, nu, grid, mode=threads, want_cov=True)
    return r["seconds"], r["iterations"]


def oracle_counts(problem, nu, log2n):
    """The oracle's converged iteration counts for this exact configuration
    from the committed fixtures (tests/golden, tools/make_fixtures.py):
    seq_ieks and para_ieks(WorkPool 8) — at N = 2^20 the stopping rule is
    rounding-determined, so counts differ between paths."""
    tag = {"fhn": "fhn", "vanderpol": "vdp", "rigidbody": "rigid", "pleiades": "pleiades"}.get(problem, problem)
    out = {}
    for path, key in ((f"{tag}_q{nu}_n{log2n}_seq", "oracle_seq_ieks"), (f"{tag}_q{nu}_n{log2n}_par8", "oracle_para_ieks8")):
        f = os.path.join(ROOT, "tests", "golden", path + ".npz")
        if os.path.exists(f):
            meta = json.loads(str(np.load(f)["meta"]))
            out[key] = {"iterations": meta["iterations"], "converged": meta["converged"]}
    return out


def run_reference(args):
    rank, world, _ = dist_env()
    if rank != 0:
        return
    threads = os.cpu_count() or 1
    n = CPU_SAMPLE_N
    dim = {"logistic": 1, "fhn": 2, "vanderpol": 2, "rigidbody": 3}.get(args.problem, 2)
    for _ in range(max(0, min(args.warmup, 1))):
        cpu_solve(args.problem, args.nu, n, threads)
    times, iters = [], 0
    for _ in range(max(1, args.steps)):
        t, iters = cpu_solve(args.problem, args.nu, n, threads)
        times.append(t)
    t = statistics.median(times)
    v = n / t
    sample = f"para_ieks on WorkPool({threads}), full solve at N={n} ({iters} iterations)"
    line = {"impl": "reference", "metric": METRIC, "value": v, "unit": "time-steps/s", "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": t * 1e3, "higher_is_better": True,
            "scaling": "strong" if world > 1 and args.mode != "replicas" else "weak", "vs_baseline": None,
            "dtype": "f64", "data": "synthetic",
            "config": {"workload": f"{args.problem} d={dim} IWP(q={args.nu}) D={dim * (args.nu + 1)}, "
                                   f"N=2^{args.log2n} uniform steps, IEKS to the reference stopping rule",
                       "N": n, "iterations": iters, "step_iterations_per_s": n * iters / t,
                       "ms_per_iteration": t * 1e3 / max(iters, 1),
                       "note": f"bounded sample: full solves at N={n} (a full N=2^{args.log2n} solve is "
                               "~9 min seq_ieks / ~12.5 min para_ieks(8) on this class of host, "
                               "tools/make_fixtures.py); compare per step-iteration with the GPU arm's "
                               "config.step_iterations_per_s"},
            "cpu_baseline": {"value": v, "unit": "time-steps/s", "cores": threads, "kind": "port", "sample": sample},
            "e2e": {"value": v, "unit": "time-steps/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


def run_ours(args):
    import torch
    rank, world, local = dist_env()
    local = local % max(1, torch.cuda.device_count())  # functional runs: N ranks may share one GPU
    if world > 1:
        import torch.distributed as dist
        backend = os.environ.get("PODE_BENCH_BACKEND", "nccl")  # gloo: functional runs of N ranks on one GPU
        if backend == "nccl":
            dist.init_process_group("nccl", device_id=torch.device("cuda", local))
        else:
            dist.init_process_group(backend)
    torch.cuda.set_device(local)
    import ctypes as C

    import paraode_b200 as P
    from paraode_b200 import _abi as A
    ctx = P.Context(local)
    stream = torch.cuda.ExternalStream(ctx.stream)
    prob = P.problem_by_name(args.problem)
    nu = args.nu
    n = 2 ** args.log2n
    D, d = prob.dim * (nu + 1), prob.dim
    grid = P.uniform_grid(prob.t_end, n)
    n1 = n + 1
    shard = world > 1 and args.mode != "replicas"
    rows = P.shard_range(n1, rank, world)[1] if shard else n1
    dev = torch.device("cuda", local)
    out_dev = [torch.empty((rows, D), dtype=torch.float64, device=dev),
               torch.empty((rows, D, D), dtype=torch.float64, device=dev),
               torch.empty((rows, d), dtype=torch.float64, device=dev),
               torch.empty((rows, d, d), dtype=torch.float64, device=dev)]
    grid_pinned = torch.from_numpy(grid).pin_memory()
    cfg = P.IeksConfig()
    gather = P.torch_allgather() if shard else None
    device_exchange = shard and os.environ.get("PODE_BENCH_BACKEND", "nccl") == "nccl"
    exchange = "host all-gather (torch.distributed)" if shard else None
    if device_exchange:  # ncclAllGather inside the library on device buffers: no host staging per exchange
        try:
            P.torch_nccl_bind(ctx)
            gather = None
            exchange = "in-library ncclAllGather on device buffers"
        except Exception as e:  # keep the run measurable: the host all-gather path
            print(f"bench: NCCL bind failed ({e!r}); using the host all-gather exchange", file=sys.stderr)

    def solve_device():
        ptr = [C.cast(C.c_void_p(t.data_ptr()), A.dptr) for t in out_dev]
        trace = np.zeros(cfg.max_iterations)
        rep = A.IeksReport(ptr[0], ptr[1], ptr[2], ptr[3], trace.ctypes.data_as(A.dptr), cfg.max_iterations,
                           A.PODE_DEVICE, 0, 0, 0.0, A.ScanStats())
        pr = prob._c()
        prior = A.Prior(nu, d, 1.0)
        c = A.IeksConfig(cfg.max_iterations, cfg.traj_rtol, cfg.obj_atol, cfg.obj_rtol, 0)
        st = A.Status()
        gp = C.cast(C.c_void_p(grid_pinned.data_ptr()), A.dptr)
        if shard:
            comm, failure = ((A.ShardComm(rank, world, A.ALLGATHER_FN(), None), []) if gather is None
                             else P.api.make_shard_comm(rank, world, gather))
            rc = ctx._lib.pode_ieks_sharded(ctx.handle, C.byref(pr), C.byref(prior), gp, n1, C.byref(c),
                                            C.byref(comm), C.byref(rep), C.byref(st))
            if failure:
                raise failure[0]
        else:
            rc = ctx._lib.pode_ieks(ctx.handle, C.byref(pr), C.byref(prior), gp, n1, C.byref(c),
                                    C.byref(rep), C.byref(st))
        P.api._raise(rc, st)
        return rep

    def solve_public():
        if shard:
            return P.para_ieks_sharded(prob, P.IwpPrior(nu, d, 1.0), grid, rank, world, gather, cfg,
                                       want_cov=True, ctx=ctx)
        return P.para_ieks(prob, P.IwpPrior(nu, d, 1.0), grid, cfg, want_cov=True, ctx=ctx)

    for _ in range(args.warmup):
        rep = solve_device()
    iters, converged = rep.iterations, bool(rep.converged)
    solve_public()  # warm the host-buffer path too

    def barrier():
        if world > 1:
            import torch.distributed as dist
            dist.barrier()

    def timed(fn, profile=False):
        barrier()
        torch.cuda.synchronize()
        l0 = ctx.kernel_launches
        if profile:
            ctx.profile(True)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        for _ in range(args.steps):
            fn()
        e1.record(stream)
        torch.cuda.synchronize()
        prof = ctx.profile_read() if profile else None
        if profile:
            ctx.profile(False)
        barrier()
        ms = e0.elapsed_time(e1) / args.steps
        if world > 1:
            import torch.distributed as dist
            t = torch.tensor([ms], device=dev)
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            ms = float(t.item())
        return ms, ctx.kernel_launches - l0, prof

    with ClockSampler(local) as clk:
        ms, launches, _ = timed(solve_device)
        # per-kernel CUDA-event profile: a second timed pass of the same K
        # solves (the events add small gaps, so `value` comes from the pass
        # above)
        ms_prof, _, prof = timed(solve_device, profile=True)
    ms_e2e, _, _ = timed(solve_public)
    units = n if shard else world * n  # sharded: one solve of n steps over all ranks
    value = units / (ms * 1e-3)
    e2e = units / (ms_e2e * 1e-3)
    d2h = rows * (D + D * D + d + d * d) * 8  # this rank's report rows
    h2d = n1 * 8
    if rank != 0:
        return

    # roofline of the dominant kernel (largest share of the timed region):
    # algorithmic flops / HBM bytes of everything that kernel name did in the
    # timed region (lane passes: per-step counts x N x iterations; scan trees:
    # per-iteration tree counts x iterations) / its summed event time.
    hbm, hbm_src, fp64, fp64_src = peaks()
    n_loc = (rows - (1 if rank == world - 1 else 0)) if shard else n  # steps this rank processed
    per_step = kernel_model(D, d)
    per_iter = scan_model(n_loc, D)
    total_ms = sum(v[1] for v in prof.values())
    solves = args.steps

    def work(name):
        if name in per_step:
            fl, by = per_step[name]
            return fl * n_loc * iters * solves, by * n_loc * iters * solves
        if name in per_iter:
            fl, by = per_iter[name]
            return fl * iters * solves, by * iters * solves
        return None

    def roofline(name):
        cnt, kms = prof[name]
        r = {"kernel": name, "share_of_step": kms / total_ms if total_ms else None, "launches": cnt,
             "avg_launch_ms": kms / cnt}
        w = work(name)
        if w is None:
            return r
        fl, by = w
        t = kms * 1e-3
        traffic = None
        try:
            tr = json.load(open(os.path.join(ROOT, "profiles", "traffic.json")))
            traffic = tr.get(f"{name}@2^{args.log2n}")
        except Exception:
            pass
        if fl / (fp64 * 1e12) >= by / (hbm * 1e9):
            a = fl / t / 1e12
            r.update({"bound": "fp64", "achieved": a, "peak": fp64, "unit": "TFLOP/s", "frac": a / fp64,
                      "peak_source": fp64_src})
        else:
            a = by / t / 1e9
            r.update({"bound": "hbm", "achieved": a, "peak": hbm, "unit": "GB/s", "frac": a / hbm,
                      "peak_source": hbm_src})
        r.update({"traffic": traffic, "algorithmic_flops_per_launch": fl / cnt,
                  "algorithmic_bytes_per_launch": by / cnt})
        return r

    dom = max(prof.items(), key=lambda kv: kv[1][1])[0]
    roof = roofline(dom)
    ranked = sorted(prof.items(), key=lambda kv: -kv[1][1])[:8]
    roof_all = {k: {kk: vv for kk, vv in roofline(k).items() if kk in ("share_of_step", "bound", "achieved", "unit", "frac")}
                for k, _ in ranked}
    kernels = {k: {"launches": c, "ms_per_step": t / args.steps} for k, (c, t) in sorted(prof.items())}
    line = {"metric": METRIC, "value": value, "unit": "time-steps/s", "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True,
            "scaling": "strong" if shard else "weak",
            "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": {"workload": f"{prob.name} d={d} IWP(q={nu}) D={D}, N=2^{args.log2n} uniform steps, "
                                   "IEKS to the reference stopping rule", "N": n, "iterations": iters,
                       "converged": converged, "step_iterations_per_s": value * iters,
                       "ms_per_iteration": ms / max(iters, 1), **oracle_counts(args.problem, nu, args.log2n),
                       "parallelism": f"time-axis shards x{world} ({exchange})" if shard else f"replicas x{world}",
                       "l2": "working set > L2 (126 MB) per solve"},
            "clocks": clk.summary(), "gpu_launches": int(launches), "roofline": roof,
            "e2e": {"value": e2e, "unit": "time-steps/s", "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": d2h},
            "kernels": kernels, "roofline_top_kernels": roof_all, "ms_per_step_profiled": ms_prof}
    if not args.no_cpu_baseline:
        t, it = cpu_solve(args.problem, nu, CPU_SAMPLE_N, 0)
        line["cpu_baseline"] = {"value": CPU_SAMPLE_N / t, "unit": "time-steps/s", "cores": 1, "kind": "port",
                                "sample": f"seq_ieks (single thread) full solve at N={CPU_SAMPLE_N}, "
                                          f"{it} iterations"}
    print(json.dumps(line), flush=True)


if __name__ == "__main__":
    a = parse()
    if a.impl == "reference":
        run_reference(a)
    else:
        run_ours(a)
