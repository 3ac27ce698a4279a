"""Multi-GPU LRAMM with A row-sharded and B column-sharded (BASELINE config 5).

Rank i holds rows [m_i0, m_i1) of A and columns [n_i0, n_i1) of B; Omega is replicated
(drawn from the reference's seeded generator).  Every factor stays resident on its rank;
only these exchanges cross NVLink (torch.distributed / NCCL):

  * allreduce(SUM) of the w x w Gram matrices of row-sharded sketches (CholeskyQR2),
  * allreduce(SUM) of the k x w partial products that contract over the sharded
    dimension (A^T Q over A's rows, B Omega and B Qz over B's columns).  In fast mode
    these are int32 accumulators of int8 products, so the sums are exact and the
    result is bit-identical to the single-GPU one for any number of ranks,
  * allreduce(MAX) of quantiser absmax values over a sharded dimension (per-tensor
    scales, and per-row / per-column scales whose rows / columns are split),
  * allgather of the int8 E2 operand (r x n) before the last product; D stays
    row-sharded.

Two implementations of the same algorithm:

  * `lramm_sharded_native` -> the C-ABI entry `lramm_lramm_sharded` (csrc/pipeline.cu): the whole
    sharded pipeline as one stream-ordered, CUDA-graph-capturable call.  The library does not
    link NCCL; it receives a table of collective entry points with NCCL's signatures
    (`lramm_comm_t`).  `NcclComm` fills it with torch's own libnccl (ncclAllReduce /
    ncclAllGather and two communicators created with ncclCommInitRank, one per rsvd chain so
    the A and B chains run concurrently); `HostStagedComm` fills it with callbacks that stage
    through the host and a torch.distributed (gloo) group -- for tests where several ranks
    share one GPU, which NCCL refuses.
  * `lramm_sharded` -> the op-by-op orchestration below, written against two small interfaces
    (`Comm`, ops) so the same code runs on one B200 (`CudaOps`, the C ABI) and, in the
    test-suite, with the gloo backend on CPU against the oracle (`tests/test_sharded_cpu.py`
    supplies NumPy ops).  It is the executable specification of the native path.
"""

from __future__ import annotations

import ctypes

import numpy as np
import torch

from . import _native as N
from ._device import OMEGA, WORKSPACE, ptr, stream_handle
from .errors import OverflowRiskError, UnsupportedError
from .pipeline import _child_seeds
from .quant import bit_cap
from .rsvd import sketch_width

GRAN = {"tensor": N.GRAN_TENSOR, "row": N.GRAN_ROW, "col": N.GRAN_COL}


class Comm:
    """torch.distributed collectives (NCCL on GPUs, gloo on CPU)."""

    def __init__(self, group=None):
        import torch.distributed as dist

        self.dist = dist
        self.group = group
        self.world = dist.get_world_size(group) if dist.is_initialized() else 1
        self.rank = dist.get_rank(group) if dist.is_initialized() else 0

    def sum_(self, t):
        if self.world > 1:
            self.dist.all_reduce(t, op=self.dist.ReduceOp.SUM, group=self.group)
        return t

    def max_(self, t):
        if self.world > 1:
            self.dist.all_reduce(t, op=self.dist.ReduceOp.MAX, group=self.group)
        return t

    def gather_rows(self, t):
        """Concatenate each rank's t (rows_i x c) along rows in rank order."""
        if self.world == 1:
            return t
        n = torch.tensor([t.shape[0]], device=t.device, dtype=torch.int64)
        sizes = [torch.zeros_like(n) for _ in range(self.world)]
        self.dist.all_gather(sizes, n, group=self.group)
        mx = int(max(s.item() for s in sizes))
        pad = torch.zeros((mx, t.shape[1]), dtype=t.dtype, device=t.device)
        pad[: t.shape[0]] = t
        parts = [torch.empty_like(pad) for _ in range(self.world)]
        self.dist.all_gather(parts, pad, group=self.group)
        return torch.cat([p[: int(s.item())] for p, s in zip(parts, sizes)], dim=0)


# ------------------------------------------------------------------ native path (lramm_lramm_sharded)

_NCCL_DTYPE_TORCH = {0: torch.int8, 2: torch.int32, 4: torch.int64, 8: torch.float64}  # nccl.h ncclDataType_t
_NCCL_SUM, _NCCL_MAX = 0, 2  # nccl.h ncclRedOp_t


def _load_nccl():
    """torch's own libnccl (already mapped by libtorch_cuda; resolved by its SONAME)."""
    import glob
    import os
    import site

    try:
        return ctypes.CDLL("libnccl.so.2")
    except OSError:
        pass
    for base in site.getsitepackages() + [os.path.dirname(os.path.dirname(torch.__file__))]:
        for cand in glob.glob(os.path.join(base, "nvidia", "nccl", "lib", "libnccl.so*")):
            return ctypes.CDLL(cand)
    raise RuntimeError("libnccl.so.2 not found (torch.distributed's NCCL backend ships it)")


def _load_cudart():
    """The CUDA runtime torch already mapped (host-staged test collectives copy through it)."""
    import glob
    import os
    import site

    for name in ("libcudart.so.12", "libcudart.so"):
        try:
            return ctypes.CDLL(name)
        except OSError:
            pass
    for base in site.getsitepackages() + ["/usr/local/cuda/lib64"]:
        for cand in glob.glob(os.path.join(base, "nvidia", "cuda_runtime", "lib", "libcudart.so*")) + glob.glob(
                os.path.join(base, "libcudart.so*")):
            return ctypes.CDLL(cand)
    raise RuntimeError("libcudart not found")


class _NcclUniqueId(ctypes.Structure):
    _fields_ = [("internal", ctypes.c_char * 128)]  # nccl.h NCCL_UNIQUE_ID_BYTES


class NcclComm:
    """lramm_comm_t over NCCL: the table holds the addresses of ncclAllReduce / ncclAllGather and
    two ncclComm_t (A's chain + recombination, B's chain) created on the current CUDA device.
    The unique ids travel through the already initialised torch.distributed group (any backend).
    force=True calls the collectives even at world size 1 (plumbing test on one GPU)."""

    def __init__(self, group=None, force=False, two_comms=True):
        import torch.distributed as dist

        self.lib = _load_nccl()
        self.world = dist.get_world_size(group) if dist.is_initialized() else 1
        self.rank = dist.get_rank(group) if dist.is_initialized() else 0
        self.lib.ncclGetUniqueId.argtypes = [ctypes.POINTER(_NcclUniqueId)]
        self.lib.ncclCommInitRank.argtypes = [ctypes.POINTER(ctypes.c_void_p), ctypes.c_int, _NcclUniqueId, ctypes.c_int]
        self.lib.ncclCommDestroy.argtypes = [ctypes.c_void_p]
        self.comms = []
        for _ in range(2 if two_comms else 1):
            uid = _NcclUniqueId()
            if self.rank == 0:
                rc = self.lib.ncclGetUniqueId(ctypes.byref(uid))
                if rc:
                    raise RuntimeError(f"ncclGetUniqueId failed: {rc}")
            if self.world > 1:
                box = [bytes(uid.internal) if self.rank == 0 else None]
                dist.broadcast_object_list(box, src=dist.get_global_rank(group, 0) if group is not None else 0,
                                           group=group)
                ctypes.memmove(ctypes.byref(uid), box[0], 128)
            comm = ctypes.c_void_p()
            rc = self.lib.ncclCommInitRank(ctypes.byref(comm), self.world, uid, self.rank)
            if rc:
                raise RuntimeError(f"ncclCommInitRank failed: {rc}")
            self.comms.append(comm)
        self.table = N.Comm()
        self.table.comm = self.comms[0]
        self.table.comm_b = self.comms[1] if two_comms else None
        self.table.rank, self.table.world = self.rank, self.world
        self.table.flags = N.COMM_FORCE if force else 0
        self.table.all_reduce = ctypes.cast(self.lib.ncclAllReduce, ctypes.c_void_p)
        self.table.all_gather = ctypes.cast(self.lib.ncclAllGather, ctypes.c_void_p)

    def close(self):
        for c in self.comms:
            self.lib.ncclCommDestroy(c)
        self.comms = []


class HostStagedComm:
    """lramm_comm_t whose collectives stage through the host and a torch.distributed group (gloo):
    synchronous, not graph-capturable -- for tests where the ranks share one GPU."""

    def __init__(self, group=None, force=False):
        import torch.distributed as dist

        self.dist, self.group = dist, group
        self.world = dist.get_world_size(group) if dist.is_initialized() else 1
        self.rank = dist.get_rank(group) if dist.is_initialized() else 0
        self.rt = _load_cudart()
        self.calls = {"all_reduce": 0, "all_gather": 0, "bytes": 0}

        def _to_host(src, count, code, stream):
            t = torch.empty(count, dtype=_NCCL_DTYPE_TORCH[code])
            torch.cuda.synchronize()
            _memcpy(t.data_ptr(), src, t.numel() * t.element_size())
            return t

        def _memcpy(dst, src, nbytes):
            if self.rt.cudaMemcpy(ctypes.c_void_p(dst), ctypes.c_void_p(src), ctypes.c_size_t(nbytes), 4):  # Default
                raise RuntimeError("cudaMemcpy failed")

        def all_reduce(send, recv, count, code, op, comm, stream):
            try:
                t = _to_host(send, count, code, stream)
                if self.world > 1:
                    dist.all_reduce(t, op=dist.ReduceOp.SUM if op == _NCCL_SUM else dist.ReduceOp.MAX, group=group)
                _memcpy(recv, t.data_ptr(), t.numel() * t.element_size())
                self.calls["all_reduce"] += 1
                self.calls["bytes"] += t.numel() * t.element_size()
                return 0
            except Exception:  # noqa: BLE001 -- a C callback must not raise
                return 1

        def all_gather(send, recv, count, code, comm, stream):
            try:
                t = _to_host(send, count, code, stream)
                parts = [torch.empty_like(t) for _ in range(self.world)]
                if self.world > 1:
                    dist.all_gather(parts, t, group=group)
                else:
                    parts = [t]
                full = torch.cat(parts)
                _memcpy(recv, full.data_ptr(), full.numel() * full.element_size())
                self.calls["all_gather"] += 1
                return 0
            except Exception:  # noqa: BLE001
                return 1

        self._ar, self._ag = N.ALL_REDUCE_FN(all_reduce), N.ALL_GATHER_FN(all_gather)  # keep alive
        self.table = N.Comm()
        self.table.comm = None
        self.table.comm_b = None  # one host-side group: the chains run one after the other
        self.table.rank, self.table.world = self.rank, self.world
        self.table.flags = N.COMM_FORCE if force else 0
        self.table.all_reduce = ctypes.cast(self._ar, ctypes.c_void_p)
        self.table.all_gather = ctypes.cast(self._ag, ctypes.c_void_p)

    def close(self):
        pass


def lramm_sharded_native(a_rows, b_cols, shape, params, comm, c_rows=None, out=None):
    """This rank's rows of D = alpha * A @ B + beta * C through the C-ABI `lramm_lramm_sharded`
    (one stream-ordered call; CUDA-graph capturable with an `NcclComm`).

    a_rows: (m_i x k) CUDA tensor, b_cols: (k x n_j) CUDA tensor (bounds: `shard_bounds`);
    shape = (m, k, n); comm: `NcclComm` or `HostStagedComm`.  Returns (d_rows, status) with
    status a device int32 tensor (0 = ok, identical on every rank)."""
    from .pipeline import _params
    from ._device import dtype_code

    m, k, n = shape
    dev = a_rows.device
    (ma, mb), (na, nb) = shard_bounds(m, n, comm.world, comm.rank)
    if tuple(a_rows.shape) != (mb - ma, k) or tuple(b_cols.shape) != (k, nb - na):
        from .errors import ShapeError

        raise ShapeError(f"rank {comm.rank}: expected shards {(mb - ma, k)} and {(k, nb - na)}, got "
                         f"{tuple(a_rows.shape)} and {tuple(b_cols.shape)}")
    if a_rows.dtype != b_cols.dtype:
        a_rows, b_cols = a_rows.double(), b_cols.double()
    a_rows, b_cols = a_rows.contiguous(), b_cols.contiguous()
    seed_a, seed_b = _child_seeds(params.seed)
    om_a = OMEGA.device_omega(seed_a, k, sketch_width((m, k), params.rank, params.oversample), dev)
    om_b = OMEGA.device_omega(seed_b, n, sketch_width((k, n), params.rank, params.oversample), dev)
    p = _params(params)
    out_t = torch.float64 if np.dtype(params.out_dtype) == np.float64 else torch.float32
    if out is None:
        out = torch.empty((mb - ma, n), dtype=out_t, device=dev)
    status = torch.zeros(1, dtype=torch.int32, device=dev)
    wsz = N.LIB.lramm_lramm_sharded_ws(m, k, n, ctypes.byref(p), comm.world, comm.rank)
    ws = WORKSPACE.get(wsz, dev)
    cc = c_rows.contiguous() if (c_rows is not None and params.beta != 0.0) else None
    N.check(N.LIB.lramm_lramm_sharded(ptr(a_rows), ptr(b_cols), dtype_code(a_rows), m, k, n, ctypes.byref(p), ptr(om_a),
                                      ptr(om_b), ptr(cc), dtype_code(cc) if cc is not None else N.F64, ptr(out),
                                      dtype_code(out), ptr(status), ptr(ws), wsz, ctypes.byref(comm.table),
                                      stream_handle(dev)))
    return out, status


class CudaOps:
    """Per-shard device operations through liblramm_cuda (tensors on the current CUDA device)."""

    def __init__(self, device=None):
        self.dev = torch.device("cuda", torch.cuda.current_device() if device is None else device)

    # -- tensors
    def f64(self, shape):
        return torch.empty(shape, dtype=torch.float64, device=self.dev)

    def zeros64(self, shape):
        return torch.zeros(shape, dtype=torch.float64, device=self.dev)

    def omega(self, seed, n, w):
        return OMEGA.device_omega(seed, n, w, self.dev)

    def _code(self, x):
        return N.F32 if x.dtype == torch.float32 else N.F64

    # -- quantiser
    def absmax(self, x, gran):
        rows, cols = x.shape
        n = 1 if gran == "tensor" else (rows if gran == "row" else cols)
        amax = torch.zeros(n, dtype=torch.float64, device=self.dev)
        N.check(N.LIB.lramm_absmax(ptr(x), self._code(x), rows, cols, x.stride(0), GRAN[gran], ptr(amax),
                                   ctypes.c_void_p(0), stream_handle(self.dev)))
        return amax

    def quantize(self, x, bits, gran, transpose, amax):
        """int8 K-major operand (transposed if asked) with scales cap/amax."""
        rows, cols = x.shape
        orows, ocols = (cols, rows) if transpose else (rows, cols)
        ld = ((ocols + 15) // 16) * 16
        q = torch.empty((orows, ld), dtype=torch.int8, device=self.dev)
        scales = torch.empty(amax.numel(), dtype=torch.float64, device=self.dev)
        N.check(N.LIB.lramm_quantize_amax(ptr(x), self._code(x), rows, cols, x.stride(0), int(bits), GRAN[gran],
                                          int(transpose), ptr(amax), ptr(q), N.I8, ld, ptr(scales),
                                          stream_handle(self.dev)))
        return q, scales

    def iprod(self, qa, qb, M, Nn, K):
        """int32 C = A . B^T of K-major int8 operands."""
        acc = torch.empty((M, Nn), dtype=torch.int32, device=self.dev)
        e = N.Epilogue()
        e.out_dtype, e.out, e.ldo = N.I32, acc.data_ptr(), Nn
        N.check(N.LIB.lramm_igemm(M, Nn, K, ptr(qa), qa.stride(0), ptr(qb), qb.stride(0), ctypes.byref(e), 1,
                                  stream_handle(self.dev)))
        return acc

    def dequant(self, acc, sa, sb, out_dtype=torch.float64, transpose=False, alpha=1.0, beta=0.0, c=None):
        M, Nn = acc.shape
        out = torch.empty((Nn, M) if transpose else (M, Nn), dtype=out_dtype, device=self.dev)
        e = N.Epilogue()
        e.out_dtype = N.F64 if out_dtype == torch.float64 else N.F32
        e.transpose_out = int(transpose)
        e.out, e.ldo = out.data_ptr(), (M if transpose else Nn)
        e.row_scale, e.row_scale_inc = sa.data_ptr(), (1 if sa.numel() > 1 else 0)
        e.col_scale, e.col_scale_inc = sb.data_ptr(), (1 if sb.numel() > 1 else 0)
        e.alpha, e.beta = float(alpha), float(beta)
        if c is not None and beta != 0.0:
            e.c_dtype = self._code(c)
            e.c, e.ldc = c.data_ptr(), c.stride(0)
        N.check(N.LIB.lramm_dequant(ptr(acc), M, Nn, Nn, ctypes.byref(e), stream_handle(self.dev)))
        return out

    # -- fp64
    def gemm(self, trans_a, a, b):
        """trans_a=0: a @ b ; trans_a=1: a^T @ b (a: K x M)."""
        M, K = (a.shape[1], a.shape[0]) if trans_a else a.shape
        Nn = b.shape[1]
        c = self.f64((M, Nn))
        wsz = N.LIB.lramm_dgemm_ws(trans_a, M, Nn, K)
        ws = WORKSPACE.get(wsz, self.dev)
        N.check(N.LIB.lramm_dgemm(trans_a, M, Nn, K, ptr(a), a.stride(0), ptr(b), b.stride(0), ptr(c), Nn, ptr(ws), wsz,
                                  stream_handle(self.dev)))
        return c

    def cholqr_pass(self, y, gram):
        m, w = y.shape
        q, lo = self.f64((m, w)), self.f64((w, w))
        info = torch.zeros(1, dtype=torch.int32, device=self.dev)
        wsz = N.LIB.lramm_cholqr_pass_ws(m, w)
        ws = WORKSPACE.get(wsz, self.dev)
        N.check(N.LIB.lramm_cholqr_pass(ptr(y), m, w, w, ptr(gram), ptr(q), w, ptr(lo), ptr(info), ptr(ws), wsz,
                                        stream_handle(self.dev)))
        return q, lo, info

    def qr(self, y):
        from .rsvd import _qr_device

        return _qr_device(y.contiguous())

    def svd(self, a):
        """(u, s, v) thin SVD, the C-ABI lramm_svd (CholeskyQR2 + one-sided Jacobi)."""
        m, n = a.shape
        t = min(m, n)
        u, s, v = self.f64((m, t)), self.f64((t,)), self.f64((n, t))
        info = torch.zeros(4, dtype=torch.int32, device=self.dev)
        wsz = N.LIB.lramm_svd_ws(m, n)
        ws = WORKSPACE.get(wsz, self.dev)
        N.check(N.LIB.lramm_svd(ptr(a.contiguous()), m, n, ptr(u), ptr(s), ptr(v), ptr(info), ptr(ws), wsz,
                                stream_handle(self.dev)))
        return u, s, v


# ------------------------------------------------------------------ the sharded algorithm


def _row_split(total, world):
    base, extra = divmod(total, world)
    offs = [0]
    for i in range(world):
        offs.append(offs[-1] + base + (1 if i < extra else 0))
    return offs


def shard_bounds(m, n, world, rank):
    """Row range of A and column range of B owned by `rank` (balanced contiguous blocks)."""
    mo, no = _row_split(m, world), _row_split(n, world)
    return (mo[rank], mo[rank + 1]), (no[rank], no[rank + 1])


def _guard_int32(k_global, bits_a, bits_b):
    """The int32 accumulators of an int8 product over a contraction of global length k_global
    (summed exactly across ranks) must not wrap: k_global * cap_a * cap_b < 2^31 (the
    single-GPU path routes such products through its exact int64 limb path instead; the
    reference's own guard is the int64 rule, quant.py:87-93)."""
    if k_global * bit_cap(bits_a) * bit_cap(bits_b) >= 2 ** 31:
        raise OverflowRiskError(f"contraction length {k_global} with bit budgets ({bits_a}, {bits_b}) overflows the "
                                "int32 accumulators of the sharded path")


class _Sketch:
    """The products of the randomised SVD, fp64 (parity) or int8 (fast) with global scales."""

    def __init__(self, params, comm, ops):
        self.p, self.comm, self.ops = params, comm, ops
        fast = params.mode == "fast"
        self.gran = params.granularity
        # bits None = an fp64 product (parity mode: the reference); fast mode defaults to 8
        self.sb = (params.sketch_bits or 8) if fast else None
        self.pb = (params.power_bits or 8) if fast else None
        self.jb = (params.proj_bits or 8) if fast else None

    def _scales_amax(self, x, gran, sharded_dim):
        """amax of the logical matrix whose local piece is x; sharded_dim is "rows", "cols" or None."""
        amax = self.ops.absmax(x, gran)
        if sharded_dim is not None and (gran == "tensor" or {"row": "cols", "col": "rows"}[gran] == sharded_dim):
            self.comm.max_(amax)
        return amax

    def product(self, x, y, bits, x_sharded, y_sharded, contract_sharded, k_global=None):
        """x (M x K) . y (K x N) where the K dimension may be split across ranks
        (contract_sharded: the result is a partial sum to be allreduced; k_global = the full
        contraction length)."""
        if bits is None:
            out = self.ops.gemm(0, x, y)
            return self.comm.sum_(out) if contract_sharded else out
        _guard_int32(k_global or x.shape[1], bits, bits)
        lg = "row" if self.gran == "row" else "tensor"
        rg = "col" if self.gran == "row" else "tensor"
        ax = self._scales_amax(x, lg, x_sharded)
        ay = self._scales_amax(y, rg, y_sharded)
        qx, sx = self.ops.quantize(x, bits, lg, False, ax)
        qy, sy = self.ops.quantize(y, bits, rg, True, ay)
        acc = self.ops.iprod(qx, qy, x.shape[0], y.shape[1], x.shape[1])
        if contract_sharded:
            self.comm.sum_(acc)  # int32 partials: exact
        return self.ops.dequant(acc, sx, sy)

    def product_t(self, x, y, bits, x_sharded, y_sharded, contract_sharded, k_global=None):
        """x^T (K x M)^T . y (K x N) -> M x N, contraction over the rows of x and y."""
        if bits is None:
            out = self.ops.gemm(1, x, y)
            return self.comm.sum_(out) if contract_sharded else out
        _guard_int32(k_global or x.shape[0], bits, bits)
        lg = "col" if self.gran == "row" else "tensor"  # columns of x are the rows of x^T
        rg = "col" if self.gran == "row" else "tensor"
        ax = self._scales_amax(x, lg, x_sharded)
        ay = self._scales_amax(y, rg, y_sharded)
        qx, sx = self.ops.quantize(x, bits, lg, True, ax)   # x^T, K-major over x's rows
        qy, sy = self.ops.quantize(y, bits, rg, True, ay)   # y^T
        acc = self.ops.iprod(qx, qy, x.shape[1], y.shape[1], x.shape[0])
        if contract_sharded:
            self.comm.sum_(acc)
        return self.ops.dequant(acc, sx, sy)


def _cholqr2_rows(y, comm, ops, want_r=False):
    """Thin QR of a row-sharded tall matrix: CholeskyQR2 with the Gram matrices allreduced."""
    g1 = comm.sum_(ops.gemm(1, y, y))
    q1, l1, _ = ops.cholqr_pass(y, g1)
    g2 = comm.sum_(ops.gemm(1, q1, q1))
    q, l2, _ = ops.cholqr_pass(q1, g2)
    if not want_r:
        return q, None
    r = ops.gemm(0, l1, l2).T.contiguous()  # R = R2 R1 = (L1 L2)^T
    return q, r


def lramm_sharded(a_rows, b_cols, shape, params, comm=None, ops=None, c_rows=None):
    """D rows owned by this rank (m_i x n) of alpha * A @ B for A row-sharded / B column-sharded.

    a_rows: this rank's rows of A (m_i x k); b_cols: this rank's columns of B (k x n_j);
    shape = (m, k, n) of the full problem; c_rows (optional, m_i x n) the local rows of C
    for beta != 0.  Returns the local rows of D (float64).

    Rank-deficient operands (a zero singular value inside the sketch width) are not
    completed here as they are by the single-GPU path; their factor columns are zero.
    """
    comm = comm or Comm()
    ops = ops or CudaOps()
    m, k, n = shape
    (ma, mb), (na, nb) = shard_bounds(m, n, comm.world, comm.rank)
    assert a_rows.shape == (mb - ma, k) and b_cols.shape == (k, nb - na)
    r = params.rank
    q_iters = params.power_iters
    if max(params.bits) > 8:
        raise UnsupportedError("the sharded path carries int8 operands: recombination bit budgets must be <= 8")
    sk = _Sketch(params, comm, ops)
    if params.mode != "fast":  # the reference works in fp64 throughout (matcore.py:62-70)
        a_rows, b_cols = a_rows.double(), b_cols.double()
    seed_a, seed_b = _child_seeds(params.seed)

    # ---- rsvd(A), A row-sharded (rsvd.py:47-94)
    wa = sketch_width((m, k), r, params.oversample)
    om_a = ops.omega(seed_a, k, wa)
    y = sk.product(a_rows, om_a, sk.sb, "rows", None, False)
    qa, _ = _cholqr2_rows(y, comm, ops)
    for _ in range(q_iters):
        z = sk.product_t(a_rows, qa, sk.pb, "rows", "rows", True, k_global=m)  # A^T Q : k x w, summed over row shards
        qz = ops.qr(z)
        y = sk.product(a_rows, qz, sk.pb, "rows", None, False)
        qa, _ = _cholqr2_rows(y, comm, ops)
    bst_a = sk.product_t(a_rows, qa, sk.jb, "rows", "rows", True, k_global=m)  # Bs^T = A^T Q (k x w)
    v_a, s_a, h_a = ops.svd(bst_a)  # Bs^T = V S H^T  ->  u_Bs = H, v_Bs = V
    u_a = ops.gemm(0, qa, h_a[:, :r].contiguous())  # local rows of U_A
    v_a, s_a = v_a[:, :r].contiguous(), s_a[:r].contiguous()

    # ---- rsvd(B), B column-sharded
    wb = sketch_width((k, n), r, params.oversample)
    om_b = ops.omega(seed_b, n, wb)
    om_bj = om_b[na:nb].contiguous()
    yb = sk.product(b_cols, om_bj, sk.sb, "cols", "rows", True, k_global=n)  # B Omega = sum_j B_j Omega_j
    qb = ops.qr(yb)
    for _ in range(q_iters):
        zj = sk.product_t(b_cols, qb, sk.pb, "cols", None, False)  # local rows of B^T Q
        qzj, _ = _cholqr2_rows(zj, comm, ops)
        yb = sk.product(b_cols, qzj, sk.pb, "cols", "rows", True, k_global=n)
        qb = ops.qr(yb)
    bst_bj = sk.product_t(b_cols, qb, sk.jb, "cols", None, False)  # local rows of Bs^T (n_j x w)
    _, rb = _cholqr2_rows(bst_bj, comm, ops, want_r=True)
    p_r, s_b, h_b = ops.svd(rb)  # R = P S H^T  ->  u_Bs = H, v_Bs = Bs^T H S^-1
    inv = torch.where(s_b > s_b[0] * 1e-12, 1.0 / s_b, torch.zeros_like(s_b))
    v_bj = ops.gemm(0, bst_bj, (h_b * inv)[:, :r].contiguous())  # local rows of V_B
    u_b = ops.gemm(0, qb, h_b[:, :r].contiguous())
    s_b = s_b[:r].contiguous()

    # ---- recombination (pipeline.py:188-210), per-tensor scales made global
    d1, d2, d3 = params.bits
    _guard_int32(k, d1, d1)
    _guard_int32(r, d2, d2)
    _guard_int32(r, d3, d3)
    vt = v_a.T.contiguous()  # r x k, replicated
    e1 = _qgemm_replicated(vt, u_b, d1, ops)  # r x r, identical on every rank
    zsc_t = (v_bj * s_b).contiguous()  # n_j x r  (= Zsc^T local rows)
    e2t = _qgemm_global_t(e1, zsc_t, d2, comm, ops)  # E2^T local rows (n_j x r)
    usc = (u_a * s_a).contiguous()  # m_i x r
    # E3 needs all of E2: quantise E2^T with the global scale, allgather the int8 rows
    a2 = comm.max_(ops.absmax(e2t, "tensor"))
    q2, s2 = ops.quantize(e2t, d3, "tensor", False, a2)
    q2 = comm.gather_rows(q2)  # n x ld
    au = comm.max_(ops.absmax(usc, "tensor"))
    qu, su = ops.quantize(usc, d3, "tensor", False, au)
    acc = ops.iprod(qu, q2, usc.shape[0], n, r)
    return ops.dequant(acc, su, s2, alpha=params.alpha, beta=params.beta, c=c_rows)


def _qgemm_replicated(a, b, bits, ops):
    """Per-tensor QM product of replicated operands (quant.py:96-121)."""
    qa, sa = ops.quantize(a, bits, "tensor", False, ops.absmax(a, "tensor"))
    qb, sb = ops.quantize(b, bits, "tensor", True, ops.absmax(b, "tensor"))
    acc = ops.iprod(qa, qb, a.shape[0], b.shape[1], a.shape[1])
    return ops.dequant(acc, sa, sb)


def _qgemm_global_t(e1, zsc_t_local, bits, comm, ops):
    """E2 = QM(E1 Zsc) with Zsc column-sharded; returns the local rows of E2^T (n_j x r)."""
    a1 = ops.absmax(e1, "tensor")
    az = comm.max_(ops.absmax(zsc_t_local, "tensor"))  # global per-tensor scale of Zsc
    q1, s1 = ops.quantize(e1, bits, "tensor", False, a1)
    qz, sz = ops.quantize(zsc_t_local, bits, "tensor", False, az)  # rows = n_j, K = r: already K-major
    acc = ops.iprod(q1, qz, e1.shape[0], zsc_t_local.shape[0], e1.shape[1])
    return ops.dequant(acc, s1, sz, transpose=True)
