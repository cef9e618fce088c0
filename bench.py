"""Benchmark of the ParaIEKS hot path on B200.

One "step" = one converged IEKS solve (FitzHugh–Nagumo, d=2, IWP(q=2),
D=6, N=2^20 uniform steps on [0, 20]) — BASELINE.json configs[1] at its
largest N.  value = time-steps/s over all ranks with the solve's inputs and
outputs resident in HBM; e2e = the same metric through the public API with
host buffers (grid H2D and the full SolverReport D2H inside the timed
region).  `--impl reference` times the reference algorithm on the host
cores (the C++ restatement in oracle/, the reference itself needs Eigen
which this image lacks).

Multi-GPU: one process per GPU (torchrun); each rank solves its own
independent problem (replicas, weak scaling) — see DESIGN.md §Multi-GPU.
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
CPU_SAMPLE_N = 2 ** 13  # bounded CPU sample (full converged solve)


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
    return ap.parse_args()


def dist_env():
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return rank, world, local


class ClockSampler:
    """nvidia-smi clocks / throttle reasons sampled during the timed region."""

    def __init__(self, index):
        self.index = index
        self.rows = []
        self.proc = None

    def __enter__(self):
        q = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.hw_slowdown,"
             "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
             "clocks_event_reasons.sw_power_cap")
        try:
            self.proc = subprocess.Popen(["nvidia-smi", "-i", str(self.index), f"--query-gpu={q}",
                                          "--format=csv,noheader,nounits", "-lms", "100"],
                                         stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.thread = threading.Thread(target=self._read, daemon=True)
            self.thread.start()
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


def cpu_reference(args, problem_name, nu, n, steps, warmup, threads):
    """The reference algorithm on the host cores (oracle/, the C++ restatement)."""
    sys.path.insert(0, os.path.join(ROOT, "tests"))
    import _oracle as O
    prob = O.problem(problem_name)
    grid = O.uniform_grid(prob.t_end, n)
    for _ in range(warmup):
        O.ieks(prob, nu, grid, mode=threads, want_cov=True)
    times, iters = [], 0
    for _ in range(steps):
        r = O.ieks(prob, nu, grid, mode=threads, want_cov=True)
        times.append(r["seconds"])
        iters = r["iterations"]
    t = statistics.median(times)
    return n / t, t, iters


def run_reference(args):
    rank, world, _ = dist_env()
    if rank != 0:
        return
    threads = os.cpu_count() or 1
    n = CPU_SAMPLE_N
    w = max(1, min(args.warmup, 1))
    v, t, iters = cpu_reference(args, args.problem, args.nu, n, max(1, args.steps), w, threads)
    cfg = {"workload": f"{args.problem} d=2 IWP(q={args.nu}) converged IEKS", "N": n,
           "sample": "full converged solve at reduced N (the N=2^20 solve takes many minutes on CPU)",
           "iterations": iters}
    line = {"impl": "reference", "metric": METRIC, "value": v, "unit": "time-steps/s", "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": t * 1e3, "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": cfg,
            "cpu_baseline": {"value": v, "unit": "time-steps/s", "cores": threads, "kind": "port",
                             "sample": f"para_ieks (WorkPool({threads})) on N={n}, {iters} iterations"},
            "e2e": {"value": v, "unit": "time-steps/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


def run_ours(args):
    import torch
    rank, world, local = dist_env()
    if world > 1:
        import torch.distributed as dist
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    torch.cuda.set_device(local)
    import paraode_b200 as P
    ctx = P.Context(local)
    stream = torch.cuda.ExternalStream(ctx.stream)
    prob = P.problem_by_name(args.problem)
    nu = args.nu
    n = 2 ** args.log2n
    D, d = prob.dim * (nu + 1), prob.dim
    grid = P.uniform_grid(prob.t_end, n)
    n1 = n + 1
    dev = torch.device("cuda", local)
    # device-resident outputs (value) and pinned host outputs (e2e)
    out_dev = [torch.empty((n1, D), dtype=torch.float64, device=dev),
               torch.empty((n1, D, D), dtype=torch.float64, device=dev),
               torch.empty((n1, d), dtype=torch.float64, device=dev),
               torch.empty((n1, d, d), dtype=torch.float64, device=dev)]
    out_host = [torch.empty(t.shape, dtype=torch.float64, pin_memory=True) for t in out_dev]
    grid_pinned = torch.from_numpy(grid).pin_memory()
    from paraode_b200 import _abi as A
    import ctypes as C

    def solve(location):
        outs = out_dev if location == A.PODE_DEVICE else out_host
        ptr = [C.cast(C.c_void_p(t.data_ptr()), A.dptr) for t in outs]
        trace = np.zeros(256)
        rep = A.IeksReport(ptr[0], ptr[1], ptr[2], ptr[3], trace.ctypes.data_as(A.dptr), 256, location,
                           0, 0, 0.0, A.ScanStats())
        pr = prob._c()
        prior = A.Prior(nu, d, 1.0)
        cfg = A.IeksConfig(100, 1e-13, 1e-9, 1e-6, 0)
        st = A.Status()
        rc = ctx._lib.pode_ieks(ctx.handle, C.byref(pr), C.byref(prior),
                                C.cast(C.c_void_p(grid_pinned.data_ptr()), A.dptr), n1, C.byref(cfg),
                                C.byref(rep), C.byref(st))
        P.api._raise(rc, st)
        return rep

    for _ in range(args.warmup):
        rep = solve(A.PODE_DEVICE)
    iters = rep.iterations

    def barrier():
        if world > 1:
            import torch.distributed as dist
            dist.barrier()

    def timed(location):
        barrier()
        torch.cuda.synchronize()
        l0 = ctx.kernel_launches
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        with torch.cuda.stream(stream):
            e0.record(stream)
            for _ in range(args.steps):
                solve(location)
            e1.record(stream)
        torch.cuda.synchronize()
        barrier()
        ms = e0.elapsed_time(e1) / args.steps
        if world > 1:
            import torch.distributed as dist
            t = torch.tensor([ms], device=dev)
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            ms = float(t.item())
        return ms, ctx.kernel_launches - l0

    with ClockSampler(local) as clk:
        ms, launches = timed(A.PODE_DEVICE)
    ms_e2e, _ = timed(A.PODE_HOST)
    value = world * n / (ms * 1e-3)
    e2e = world * n / (ms_e2e * 1e-3)
    d2h = sum(t.numel() * 8 for t in out_host)
    h2d = n1 * 8
    if rank != 0:
        return
    line = {"metric": METRIC, "value": value, "unit": "time-steps/s", "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True, "scaling": "weak",
            "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": {"workload": f"{prob.name} d={d} IWP(q={nu}) D={D}, N=2^{args.log2n} uniform steps, "
                                   "full IEKS to convergence", "N": n, "iterations": iters,
                       "step_iterations_per_s": value * iters, "parallelism": f"replicas x{world}",
                       "l2": "working set > L2 (126 MB)"},
            "clocks": clk.summary(), "gpu_launches": int(launches),
            "e2e": {"value": e2e, "unit": "time-steps/s", "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": d2h}}
    if not args.no_cpu_baseline:
        v, t, it = cpu_reference(args, args.problem, nu, CPU_SAMPLE_N, 1, 0, 0)
        line["cpu_baseline"] = {"value": v, "unit": "time-steps/s", "cores": 1, "kind": "port",
                                "sample": f"seq_ieks (single thread) full solve at N={CPU_SAMPLE_N}, {it} iterations"}
    print(json.dumps(line), flush=True)


if __name__ == "__main__":
    a = parse()
    if a.impl == "reference":
        run_reference(a)
    else:
        run_ours(a)
