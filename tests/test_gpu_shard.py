"""Time-axis sharded solve on the GPU: R processes (gloo
exchange), each solving its shard through pode_ieks_sharded, must
reproduce the sequential oracle's solve — equal iteration counts, means at
1e-9, covariance products at 1e-7, sigma_hat — like the single-shard path
(test_gpu_parity.py).  All shards share cuda:0 here (one GPU per gpurun
box); their kernels never wait on each other, the exchanges are host
collectives between kernel phases."""
import os
import socket

import numpy as np
import pytest

import _oracle as O
from _dense import dense_cov

pytestmark = pytest.mark.gpu
P = pytest.importorskip("paraode_b200")


def rel(a, b):
    a, b = np.asarray(a), np.asarray(b)
    return float(np.max(np.abs(a - b)) / max(1.0, np.max(np.abs(b))))


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _shard_worker(rank, world, port, name, nu, steps, env, q):
    import torch.distributed as dist
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), **env)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        prob = P.problem_by_name(name)
        grid = P.uniform_grid(prob.t_end, steps)
        r = P.para_ieks_sharded(prob, P.IwpPrior(nu, prob.dim, 1.0), grid, rank, world, P.torch_allgather())
        q.put((rank, r.first_node, r.means, r.cov_sqrt, r.solution_means, r.solution_covs, r.sigma_hat,
               r.iterations, r.converged, r.objective_trace))
    except Exception as e:  # surfaced in the parent
        q.put((rank, repr(e)))
    finally:
        dist.destroy_process_group()


def run_sharded(name, nu, steps, world, env=None):
    import torch.multiprocessing as mp
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_shard_worker, args=(r, world, port, name, nu, steps, env or {}, q))
             for r in range(world)]
    for p in procs:
        p.start()
    got = {}
    for _ in procs:
        item = q.get(timeout=300)
        got[item[0]] = item
    for p in procs:
        p.join(timeout=60)
    for r in range(world):
        assert len(got[r]) > 2, got[r]
    parts = [got[r] for r in range(world)]
    assert [p[1] for p in parts] == [P.shard_range(steps + 1, r, world)[0] for r in range(world)]
    cat = lambda k: np.concatenate([p[k] for p in parts])
    scal = parts[0][6:]
    for p in parts[1:]:  # every shard took the same decisions
        assert p[7] == scal[1] and p[8] == scal[2] and p[6] == scal[0]
    return dict(means=cat(2), cov_sqrt=cat(3), solution_means=cat(4), solution_covs=cat(5), sigma_hat=scal[0],
                iterations=scal[1], converged=scal[2], objective_trace=scal[3])


@pytest.mark.parametrize("name,nu,steps,world,env", [
    ("logistic", 2, 30, 2, {"PODE_CHUNK": "4"}),
    ("fhn", 2, 2000, 2, {}),
    ("vanderpol", 2, 999, 3, {"PODE_CHUNK": "5"}),
    ("rigidbody", 2, 3000, 4, {"PODE_CHUNK": "3"}),
    ("vanderpol", 3, 600, 2, {"PODE_CHUNK": "4"}),  # D = 8: pass A's A in shared memory
    ("fhn", 2, 4001, 3, {"PODE_CHUNK": "2", "PODE_SCAN_FANIN": "2"}),
])
def test_sharded_matches_sequential_oracle(name, nu, steps, world, env):
    op = O.problem(name)
    grid = O.uniform_grid(op.t_end, steps)
    want = O.ieks(op, nu, grid, mode=0)
    got = run_sharded(name, nu, steps, world, env)
    assert got["converged"] == want["converged"]
    assert got["iterations"] == want["iterations"]
    assert got["means"].shape == want["means"].shape
    assert rel(got["means"], want["means"]) <= 1e-9
    assert rel(dense_cov(got["cov_sqrt"]), dense_cov(want["cov_sqrt"])) <= 1e-7
    assert got["sigma_hat"] == pytest.approx(want["sigma_hat"], rel=1e-7)
    assert rel(got["solution_means"], want["solution_means"]) <= 1e-9
    assert rel(got["solution_covs"], want["solution_covs"]) <= 1e-7
    assert np.allclose(got["objective_trace"], want["objective_trace"], rtol=1e-8, atol=1e-12)


def test_single_shard_equals_para_ieks():
    """ranks = 1 is the plain solve (same engine, host loop)."""
    prob = P.fitzhugh_nagumo()
    grid = P.uniform_grid(prob.t_end, 1500)
    a = P.para_ieks(prob, P.IwpPrior(2, 2, 1.0), grid)
    b = P.para_ieks_sharded(prob, P.IwpPrior(2, 2, 1.0), grid, 0, 1, lambda x: x)
    assert b.iterations == a.iterations and b.first_node == 0
    assert rel(b.means, a.means) <= 1e-12
    assert rel(dense_cov(b.cov_sqrt), dense_cov(a.cov_sqrt)) <= 1e-10


def test_single_shard_device_exchange_over_nccl():
    """The device-side exchange (pode_context_nccl_init: ncclAllGather on the
    context stream, no host staging, comm->allgather NULL) on a one-rank NCCL
    communicator — NCCL rejects two ranks on one GPU, so the multi-rank
    device path runs on multi-GPU nodes only; its exchange sequence is the
    one the gloo tests above verify."""
    prob = P.fitzhugh_nagumo()
    grid = P.uniform_grid(prob.t_end, 3000)
    ctx = P.Context()
    ctx.nccl_init(P.nccl_unique_id(), 0, 1)
    got = P.para_ieks_sharded(prob, P.IwpPrior(2, 2, 1.0), grid, 0, 1, None, ctx=ctx)
    want = O.ieks(O.problem("fhn"), 2, O.uniform_grid(prob.t_end, 3000), mode=0)
    assert got.iterations == want["iterations"] and got.converged
    assert rel(got.means, want["means"]) <= 1e-9
    assert rel(dense_cov(got.cov_sqrt), dense_cov(want["cov_sqrt"])) <= 1e-7
    with pytest.raises(P.InvalidInputError):  # rank / ranks must match the communicator
        P.para_ieks_sharded(prob, P.IwpPrior(2, 2, 1.0), grid, 0, 2, None, ctx=ctx)
