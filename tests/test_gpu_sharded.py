"""Sharded LRAMM through the CUDA shard ops (liblramm_cuda) on one B200.

world_size 1 runs the NCCL-free path directly; world_size 2 runs two processes that
share cuda:0 and exchange through gloo on host copies (the collectives are host-side,
no kernel waits on another process), which exercises every CudaOps call with real
shards.  Both are compared with the single-process oracle.
"""

import os
import queue
import socket
import time

import numpy as np
import pytest
import torch

import lramm_oracle as O

pytestmark = pytest.mark.gpu


def _inputs(m, k, n, seed):
    a = O.synth(m, k, "exp:6", 91, seed, 0)
    b = O.synth(k, n, "exp:6", 91, seed, 1)
    return a, b


CASES = [
    ((512, 384, 448), dict(rank=16, mode="parity")),
    ((512, 384, 448), dict(rank=16, mode="parity", bits=(8, 8, 8), seed=3)),
    ((512, 384, 448), dict(rank=16, mode="fast", granularity="row", power_iters=1)),
    ((320, 256, 288), dict(rank=12, mode="fast", granularity="tensor", alpha=0.5, beta=2.0)),
]
IDS = ["parity", "parity-888", "fast-row-q1", "fast-tensor-ab"]


def _oracle(case):
    (m, k, n), kw = case
    a, b = _inputs(m, k, n, 3)
    c = np.linspace(-1, 1, m * n).reshape(m, n) if kw.get("beta") else None
    fast = kw.get("mode") == "fast"
    spec = O.SketchSpec(8, 8, 8, kw.get("granularity", "tensor")) if fast else O.SketchSpec()
    p = O.OracleParams(rank=kw["rank"], power_iters=kw.get("power_iters", 0), alpha=kw.get("alpha", 1.0),
                       beta=kw.get("beta", 0.0), spec=spec, bits=kw.get("bits", (8, 8, 4)), seed=kw.get("seed", 0))
    a, b = a.astype(np.float64), b.astype(np.float64)
    # both reference backends: LAPACK (pure) and the compiled one-sided Jacobi
    return (O.lramm(a, b, p, c=c), O.lramm(a, b, p, c=c, svd_fn=O.jacobi_svd)), c


def _tol(refs):
    """1e-3, widened to 1.5x the spread between the reference's own two backends: at (8,8,4)
    the 4-bit E3 quantiser can meet exact ties, where a 1e-13 perturbation moves
    the output by ~5e-3 and the reference's backends already disagree by that much."""
    return max(1e-3, 1.5 * O.rel_fro(refs[1], refs[0]))


def _err(d, refs):
    return min(O.rel_fro(d, r) for r in refs)


def _shard_run(case, world, rank, comm):
    from paper_2405_16917_b200.pipeline import LrammParams
    from paper_2405_16917_b200.sharded import CudaOps, lramm_sharded, shard_bounds

    (m, k, n), kw = case
    a, b = _inputs(m, k, n, 3)
    c = np.linspace(-1, 1, m * n).reshape(m, n) if kw.get("beta") else None
    (ma, mb), (na, nb) = shard_bounds(m, n, world, rank)
    dev = torch.device("cuda", 0)
    ar = torch.from_numpy(a[ma:mb].copy()).to(dev)
    bc = torch.from_numpy(b[:, na:nb].copy()).to(dev)
    cr = None if c is None else torch.from_numpy(c[ma:mb].copy()).to(dev)
    d = lramm_sharded(ar, bc, (m, k, n), LrammParams(**kw), comm=comm, ops=CudaOps(0), c_rows=cr)
    torch.cuda.synchronize()
    return d


@pytest.mark.parametrize("case", CASES, ids=IDS)
def test_sharded_world1_cuda(case):
    from paper_2405_16917_b200.sharded import Comm

    d = _shard_run(case, 1, 0, Comm())
    refs, _ = _oracle(case)
    assert _err(d.cpu().numpy(), refs) <= _tol(refs)


class _HostStagedComm:
    """Comm over gloo with host staging (two processes sharing one GPU)."""

    def __init__(self):
        import torch.distributed as dist

        from paper_2405_16917_b200.sharded import Comm

        self.inner = Comm()
        self.dist, self.world, self.rank = dist, self.inner.world, self.inner.rank

    def _via_host(self, t, fn):
        h = t.cpu()
        fn(h)
        t.copy_(h.to(t.device))
        return t

    def sum_(self, t):
        return self._via_host(t, self.inner.sum_)

    def max_(self, t):
        return self._via_host(t, self.inner.max_)

    def gather_rows(self, t):
        return self.inner.gather_rows(t.cpu()).to(t.device)


def _worker(rank, world, port, case, out_q):
    import torch.distributed as dist

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        comm = _HostStagedComm()
        d = _shard_run(case, world, rank, comm)
        full = comm.gather_rows(d).cpu()
        if rank == 0:
            out_q.put(full.numpy())
    finally:
        dist.destroy_process_group()


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


@pytest.mark.parametrize("case", CASES[2:], ids=IDS[2:])
def test_sharded_world2_cuda(case):
    import torch.multiprocessing as mp

    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, case, q)) for r in range(2)]
    for p in procs:
        p.start()
    deadline = time.time() + 300
    while True:
        try:
            d = q.get(timeout=1)
            break
        except queue.Empty:
            if any(p.exitcode not in (None, 0) for p in procs) or time.time() > deadline:
                for p in procs:
                    p.kill()
                raise AssertionError(f"worker failed: {[p.exitcode for p in procs]}")
    for p in procs:
        p.join(60)
    refs, _ = _oracle(case)
    assert _err(d, refs) <= _tol(refs)
