"""The native sharded pipeline `lramm_lramm_sharded` (C ABI, csrc/pipeline.cu) on one B200.

* world 1 without collectives: bit-identical to the single-GPU `lramm_lramm` and within the L4/L5
  gates of the oracle;
* world 1 with the collectives forced through NCCL (`NcclComm(force=True)`: ncclAllReduce /
  ncclAllGather from torch's libnccl on two single-rank communicators), eagerly and replayed from
  a captured CUDA graph: bit-identical to the collective-free run;
* world 2: two processes sharing cuda:0 whose `lramm_comm_t` is filled with host-staged gloo
  callbacks (`HostStagedComm`; NCCL refuses two ranks on one device): every exchange of SURVEY
  §8(e) runs with real shards, checked against the oracle and against the world-1 result.
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
    return O.synth(m, k, "exp:6", 91, seed, 0), O.synth(k, n, "exp:6", 91, seed, 1)


CASES = [
    ((512, 384, 448), dict(rank=16, mode="parity")),
    ((512, 384, 448), dict(rank=16, mode="fast", granularity="row", power_iters=1)),
    ((320, 256, 288), dict(rank=12, mode="fast", granularity="tensor", alpha=0.5, beta=2.0)),
    ((515, 390, 449), dict(rank=16, mode="fast", granularity="row", power_iters=2, sketch_bits=4, bits=(8, 8, 8))),
    ((515, 390, 449), dict(rank=16, mode="parity", power_iters=1, bits=(8, 8, 8), seed=5)),
]
IDS = ["parity", "fast-row-q1", "fast-tensor-ab", "ragged-int4-q2", "ragged-parity-q1"]


def _oracle(case):
    (m, k, n), kw = case
    a, b = _inputs(m, k, n, 3)
    c = np.linspace(-1, 1, m * n).reshape(m, n) if kw.get("beta") else None
    fast = kw.get("mode") == "fast"
    sb = kw.get("sketch_bits", 8)
    spec = O.SketchSpec(sb, 8, 8, kw.get("granularity", "tensor")) if fast else O.SketchSpec()
    p = O.OracleParams(rank=kw["rank"], power_iters=kw.get("power_iters", 0), alpha=kw.get("alpha", 1.0),
                       beta=kw.get("beta", 0.0), spec=spec, bits=kw.get("bits", (8, 8, 4)), seed=kw.get("seed", 0))
    a, b = a.astype(np.float64), b.astype(np.float64)
    return (O.lramm(a, b, p, c=c), O.lramm(a, b, p, c=c, svd_fn=O.jacobi_svd)), c


def _tol(refs):
    # 1e-3, widened to 1.5x the spread of the reference's own two backends
    return max(1e-3, 1.5 * O.rel_fro(refs[1], refs[0]))


def _err(d, refs):
    return min(O.rel_fro(d, r) for r in refs)


def _params(kw):
    from paper_2405_16917_b200.pipeline import LrammParams

    kw = dict(kw)
    if kw.get("mode") == "fast":
        kw.setdefault("sketch_bits", 8)
        kw.setdefault("power_bits", 8)
        kw.setdefault("proj_bits", 8)
    return LrammParams(**kw)


def _shard_run(case, comm, graph=False):
    from paper_2405_16917_b200.sharded import lramm_sharded_native, shard_bounds

    (m, k, n), kw = case
    a, b = _inputs(m, k, n, 3)
    c = np.linspace(-1, 1, m * n).reshape(m, n) if kw.get("beta") else None
    (ma, mb), (na, nb) = shard_bounds(m, n, comm.world, comm.rank)
    dev = torch.device("cuda", 0)
    ar = torch.from_numpy(a[ma:mb].copy()).to(dev)
    bc = torch.from_numpy(b[:, na:nb].copy()).to(dev)
    cr = None if c is None else torch.from_numpy(c[ma:mb].copy()).to(dev)
    p = _params(kw)
    d, status = lramm_sharded_native(ar, bc, (m, k, n), p, comm, c_rows=cr)
    torch.cuda.synchronize()
    if graph:
        s = torch.cuda.Stream()
        with torch.cuda.stream(s):
            lramm_sharded_native(ar, bc, (m, k, n), p, comm, c_rows=cr)  # sizes the workspace on this stream
            s.synchronize()
            g = torch.cuda.CUDAGraph()
            with torch.cuda.graph(g, stream=s):
                d, status = lramm_sharded_native(ar, bc, (m, k, n), p, comm, c_rows=cr)
        d.zero_()
        g.replay()
        torch.cuda.synchronize()
    return d, int(status.item())


class _NoComm:
    """world 1, no collective entry points: the table is never called."""

    world, rank = 1, 0

    def __init__(self):
        from paper_2405_16917_b200 import _native as N

        self.table = N.Comm()
        self.table.rank, self.table.world = 0, 1


@pytest.mark.parametrize("case", CASES, ids=IDS)
def test_native_world1_matches_oracle_and_single_gpu(case):
    import paper_2405_16917_b200 as L

    d, status = _shard_run(case, _NoComm())
    assert status == 0
    refs, c = _oracle(case)
    assert _err(d.cpu().numpy(), refs) <= _tol(refs)
    # the same kernels in the same order as lramm_lramm: identical bits
    (m, k, n), kw = case
    a, b = _inputs(m, k, n, 3)
    dev = torch.device("cuda", 0)
    tc = None if c is None else torch.from_numpy(c).to(dev)
    single, _ = L.lramm(torch.from_numpy(a).to(dev), torch.from_numpy(b).to(dev), _params(kw), c=tc)
    assert torch.equal(single, d)


@pytest.mark.parametrize("case", [CASES[1], CASES[3], CASES[4]], ids=[IDS[1], IDS[3], IDS[4]])
def test_native_world1_nccl_forced_and_graph(case):
    """Every exchange goes through ncclAllReduce / ncclAllGather on single-rank communicators;
    eager and CUDA-graph replays reproduce the collective-free result bit for bit."""
    from paper_2405_16917_b200.sharded import NcclComm

    base, _ = _shard_run(case, _NoComm())
    comm = NcclComm(force=True)
    try:
        eager, st1 = _shard_run(case, comm)
        replay, st2 = _shard_run(case, comm, graph=True)
    finally:
        comm.close()
    assert st1 == 0 and st2 == 0
    assert torch.equal(base, eager)
    assert torch.equal(base, replay)


def test_native_rejects_wide_recombination_bits_and_reports_rank_deficiency():
    from paper_2405_16917_b200.errors import UnsupportedError

    with pytest.raises(UnsupportedError):
        _shard_run(((256, 192, 224), dict(rank=8, mode="parity", bits=(16, 8, 8))), _NoComm())
    # rank-1 operand: the sketch's Gram matrix is singular; no sharded Householder fallback
    from paper_2405_16917_b200.sharded import lramm_sharded_native

    dev = torch.device("cuda", 0)
    g = torch.Generator(device="cpu").manual_seed(1)
    u = torch.randn(256, 1, generator=g, dtype=torch.float64)
    v = torch.randn(1, 192, generator=g, dtype=torch.float64)
    a = (u @ v).to(dev)
    b = torch.randn(192, 224, generator=g, dtype=torch.float64).to(dev)
    _, status = lramm_sharded_native(a, b, (256, 192, 224), _params(dict(rank=8, mode="parity")), _NoComm())
    torch.cuda.synchronize()
    assert int(status.item()) != 0


# ------------------------------------------------------------------ world 2 on one GPU (host-staged comm)


def _worker(rank, world, port, case, out_q):
    import torch.distributed as dist

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_2405_16917_b200.sharded import HostStagedComm

        comm = HostStagedComm()
        d, status = _shard_run(case, comm)
        parts = [None] * world
        dist.all_gather_object(parts, (d.cpu().numpy(), status, dict(comm.calls)))
        if rank == 0:
            out_q.put(parts)
    finally:
        dist.destroy_process_group()


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _run_world2(case):
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
            parts = q.get(timeout=1)
            break
        except queue.Empty:
            if any(p.exitcode not in (None, 0) for p in procs) or time.time() > deadline:
                for p in procs:
                    p.kill()
                raise AssertionError(f"worker failed: {[p.exitcode for p in procs]}")
    for p in procs:
        p.join(60)
    return parts


@pytest.mark.parametrize("case", CASES[1:], ids=IDS[1:])
def test_native_world2_host_staged(case):
    parts = _run_world2(case)
    assert [p[1] for p in parts] == [0, 0]
    d = np.concatenate([p[0] for p in parts], axis=0)
    calls = parts[0][2]
    assert calls["all_reduce"] > 0 and calls["all_gather"] == 1
    refs, _ = _oracle(case)
    assert _err(d, refs) <= _tol(refs)
    # against the world-1 run of the same entry point: the integer stages are exact across ranks;
    # only the fp64 Gram sums are reassociated
    base, _ = _shard_run(case, _NoComm())
    assert O.rel_fro(d, base.cpu().numpy()) <= 1e-9
