"""Host side of the time-axis sharded solve, on CPU: the
shard partition from the C ABI, and the all-gather plumbing (ctypes
callback -> torch.distributed gloo, world size 2) that pode_ieks_sharded
drives at every exchange.  The device path itself is test_gpu_shard.py."""
import ctypes as C
import os
import socket

import numpy as np
import pytest

P = pytest.importorskip("paraode_b200")
A = P._abi if hasattr(P, "_abi") else __import__("paraode_b200._abi", fromlist=["x"])


def test_shard_ranges_partition_the_nodes():
    for n1 in (2, 3, 31, 1000, 2 ** 20 + 1):
        for ranks in (1, 2, 3, 4, 8):
            if n1 - 1 < ranks:
                continue
            got = [P.shard_range(n1, r, ranks) for r in range(ranks)]
            nxt = 0
            for lo, cnt in got:
                assert lo == nxt and cnt >= 1
                nxt = lo + cnt
            assert nxt == n1  # every node reported exactly once; node N by the last shard
            steps = [got[r + 1][0] - got[r][0] for r in range(ranks - 1)] + [n1 - 1 - got[-1][0]]
            assert max(steps) - min(steps) <= 1  # balanced


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, q):
    import torch.distributed as dist
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        gather = P.torch_allgather()
        # drive the adapter through the same ctypes callback type the C ABI calls
        seen = []

        def cb(_u, send, count, recv):
            snd = np.ctypeslib.as_array(send, shape=(count,)).copy()
            got = gather(snd)
            np.ctypeslib.as_array(recv, shape=(count * world,))[:] = got
            seen.append(count)
            return 0
        fn = A.ALLGATHER_FN(cb)
        comm = A.ShardComm(rank, world, fn, None)
        out = []
        for count in (4, 6 * 6 * 3 + 12, 2 * 36 + 6):  # stop scalars, ⊗_f element, ⊗_s element (D=6)
            send = np.arange(count, dtype=np.float64) + 1000.0 * rank
            recv = np.zeros(count * world)
            rc = comm.allgather(None, send.ctypes.data_as(A.dptr), count, recv.ctypes.data_as(A.dptr))
            out.append((rc, recv))
        q.put((rank, [(rc, r.tolist()) for rc, r in out], seen))
    finally:
        dist.destroy_process_group()


def test_allgather_callback_gloo_world2():
    import torch.multiprocessing as mp
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = dict()
    for _ in procs:
        rank, out, seen = q.get(timeout=120)
        res[rank] = (out, seen)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    for rank in (0, 1):
        out, seen = res[rank]
        assert seen == [4, 120, 78]
        for rc, recv in out:
            assert rc == 0
            count = len(recv) // 2
            want = np.concatenate([np.arange(count) + 1000.0 * r for r in range(2)])
            assert np.array_equal(np.asarray(recv), want)  # rank order


def test_sharded_solve_needs_the_gpu():
    """No CPU fallback: without a B200 the sharded entry point fails loudly."""
    import torch
    if torch.cuda.is_available():
        pytest.skip("GPU present")
    grid = P.uniform_grid(10.0, 30)
    with pytest.raises(P.CudaError):
        P.para_ieks_sharded(P.logistic(), P.IwpPrior(2, 1, 1.0), grid, 0, 1, lambda x: x)
