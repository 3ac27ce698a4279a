/*
 * lramm_cuda.h -- C ABI of the B200-native LRAMM approximate-GEMM library
 * (liblramm_cuda.so, sm_100a).  Plain pointers, sizes and a cudaStream_t; no
 * torch or NumPy types.  Every entry point returns an lramm_status; on failure
 * lramm_last_error() (thread-local) holds a one-line message.
 *
 * Two families of entry points:
 *
 *  (1) HOST-pointer entry points  lramm_host_*  -- what the reference's kernel
 *      plugin FFI binds.  The reference selects its kernel backend at import
 *      time in `pkg/src/lramm/_kernels/__init__.py:8-39` and calls exactly four
 *      functions; each host entry point replaces one of them with identical
 *      argument meaning (row-major C-contiguous NumPy buffers, caller-owned
 *      outputs) and identical error behaviour (inner-dimension mismatch ->
 *      LRAMM_ERR_SHAPE, which the binding raises as ValueError("inner dimensions
 *      differ"), Jacobi non-convergence -> LRAMM_ERR_NONCONVERGENCE ->
 *      RuntimeError):
 *        lramm_host_matmul            <- _core.matmul            (_core.pyx:17-32, _pure.py:10-14)
 *        lramm_host_imatmul           <- _core.imatmul           (_core.pyx:35-50, _pure.py:17-21)
 *        lramm_host_scale_round_clip  <- _core.scale_round_clip  (_core.pyx:53-69, _pure.py:24-26)
 *        lramm_host_svd               <- _jacobi.jacobi_svd      (_jacobi.py:14-50, _pure.py:29-35)
 *      plus the whole pipeline, which replaces `lramm.pipeline.lramm`
 *      (pipeline.py:159-214) in one call:
 *        lramm_host_lramm
 *      Host entry points copy host->device, compute, copy device->host and
 *      synchronise; they manage their own (cached) device memory.
 *
 *  (2) DEVICE-pointer entry points  lramm_*  -- stream-ordered, caller-allocated
 *      device buffers and workspace, no host synchronisation and no allocation,
 *      CUDA-graph capturable.  Used by the Python package with torch tensors.
 *
 * Status codes map 1:1 onto the reference's exception types (errors.py:4-33):
 * SHAPE -> ShapeError, PARAM -> ParameterError, OVERFLOW -> OverflowRiskError,
 * NONFINITE -> ParameterError("cannot quantize non-finite entries", quant.py:63-64),
 * NONCONVERGENCE -> RuntimeError (_jacobi.py:31-32), UNSUPPORTED -> NotImplementedError
 * (e.g. bit budgets above 8 on the int8 tensor-core path), CUDA -> RuntimeError.
 */
#ifndef LRAMM_CUDA_H_
#define LRAMM_CUDA_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct CUstream_st *lramm_stream_t; /* == cudaStream_t */

typedef enum {
  LRAMM_OK = 0,
  LRAMM_ERR_SHAPE = 1,
  LRAMM_ERR_PARAM = 2,
  LRAMM_ERR_OVERFLOW = 3,
  LRAMM_ERR_NONCONVERGENCE = 4,
  LRAMM_ERR_UNSUPPORTED = 5,
  LRAMM_ERR_CUDA = 6,
  LRAMM_ERR_NONFINITE = 7,
  LRAMM_ERR_WORKSPACE = 8
} lramm_status;

typedef enum { LRAMM_F32 = 0, LRAMM_F64 = 1, LRAMM_I8 = 2, LRAMM_I32 = 3, LRAMM_I64 = 4, LRAMM_I4 = 5 } lramm_dtype;
typedef enum { LRAMM_GRAN_TENSOR = 0, LRAMM_GRAN_ROW = 1, LRAMM_GRAN_COL = 2 } lramm_granularity;
typedef enum { LRAMM_MODE_PARITY = 0, LRAMM_MODE_FAST = 1 } lramm_mode;

/* Pipeline parameters: mirrors LrammParams (pipeline.py:50-70) plus the fast-mode
 * extension (SURVEY §7 "Params").  sketch/power/proj bits of 0 mean fp64 (the
 * reference's behaviour, rsvd.py:57-64,77). */
typedef struct {
  int32_t rank;
  int32_t oversample;
  int32_t power_iters;
  int32_t bits[3]; /* (d1, d2, d3), each in [2, 8] on device */
  double alpha;
  double beta;
  int32_t mode;        /* lramm_mode */
  int32_t sketch_bits; /* Y = X.Omega              (fast mode) */
  int32_t power_bits;  /* X^T.Q and X.Qz           (fast mode) */
  int32_t proj_bits;   /* Q^T.X                    (fast mode) */
  int32_t granularity; /* lramm_granularity of the sketch products */
  int32_t reserved;
} lramm_params_t;

/* Per-stage device time in milliseconds, keys of pipeline.STAGES (pipeline.py:37). */
typedef struct {
  float rsvd_ms, scaling_ms, gemm1_ms, gemm2_ms, gemm3_ms;
} lramm_timings_t;

/* Integer-GEMM epilogue: out = alpha * (acc / (row_scale[i] * col_scale[j])) + beta * C
 * (quant.py:116-121 dequantisation, bit-exact in fp64), or raw int32 (optionally
 * accumulated with atomics for split-K; exact and order independent). */
typedef struct {
  int32_t out_dtype;     /* LRAMM_I32, LRAMM_F32 or LRAMM_F64 */
  int32_t accumulate;    /* LRAMM_I32 only: out += acc (out pre-zeroed) */
  int32_t transpose_out; /* store out^T (N x M, leading dim ldo) */
  int32_t c_dtype;       /* LRAMM_F32 / LRAMM_F64 when c != NULL */
  void *out;
  int64_t ldo;
  const double *row_scale; /* NULL => 1.0 */
  int64_t row_scale_inc;   /* 0 => per-tensor (broadcast element 0) */
  const double *col_scale;
  int64_t col_scale_inc;
  double alpha;
  double beta;
  const void *c;
  int64_t ldc;
} lramm_epilogue_t;

const char *lramm_last_error(void);
const char *lramm_version(void);
/* 0 if a compute-capability 10.0 device is current, else LRAMM_ERR_UNSUPPORTED. */
int lramm_device_check(void);

/* ---------------------------------------------------------------- device API */

/* Symmetric absmax quantiser (quant.py:55-71) at granularity tensor / row / col.
 * x: rows x cols (leading dim ldx, elements) of dtype LRAMM_F32 or LRAMM_F64.
 * q_dtype LRAMM_I8: int8 output, LRAMM_I32: int32 output (the reference's
 * container), LRAMM_I4: two's-complement nibbles packed along each output row
 * (low nibble = even column), bits <= 4.  transpose_out writes q^T.  Padding
 * columns of q up to ldq are zeroed.  scales: 1 (tensor), rows or cols doubles,
 * scale = cap / amax (all-zero -> 1.0).  nonfinite_flag (device int, may be NULL)
 * is set to 1 if x holds a non-finite value.  ws >= lramm_quantize_ws(rows, cols). */
int lramm_quantize(const void *x, int x_dtype, int64_t rows, int64_t cols, int64_t ldx, int bits,
                   int granularity, int transpose_out, void *q, int q_dtype, int64_t ldq,
                   double *scales, int *nonfinite_flag, void *ws, size_t ws_bytes,
                   lramm_stream_t stream);
size_t lramm_quantize_ws(int64_t rows, int64_t cols);

/* Two int8 quantisations of one x from one absmax pass and one read of x: q_r = x row-major at
 * (bits_r, granularity_r) and q_t = x^T at (bits_t, granularity_t); granularities are in x's
 * coordinates (ROW = per row of x, COL = per column of x).  Each is bit-identical to the matching
 * lramm_quantize call (quant.py:55-71 applied twice to the same x); bits <= 8.
 * ws >= lramm_quantize_ws(rows, cols). */
int lramm_quantize_pair(const void *x, int x_dtype, int64_t rows, int64_t cols, int64_t ldx, int bits_r,
                        int granularity_r, int8_t *q_r, int64_t ldq_r, double *scales_r, int bits_t,
                        int granularity_t, int8_t *q_t, int64_t ldq_t, double *scales_t, int *nonfinite_flag,
                        void *ws, size_t ws_bytes, lramm_stream_t stream);

/* max |x| per tensor / row / column (exact; amax must be zeroed by the caller: the kernel takes a
 * max into it, so partial results of several shards can be combined with an allreduce(MAX)). */
int lramm_absmax(const void *x, int x_dtype, int64_t rows, int64_t cols, int64_t ldx, int granularity, double *amax,
                 int *nonfinite_flag, lramm_stream_t stream);

/* lramm_quantize with externally supplied amax (e.g. allreduced across shards): scale = cap/amax. */
int lramm_quantize_amax(const void *x, int x_dtype, int64_t rows, int64_t cols, int64_t ldx, int bits,
                        int granularity, int transpose_out, const double *amax, void *q, int q_dtype, int64_t ldq,
                        double *scales, lramm_stream_t stream);

/* One CholeskyQR pass with a Gram matrix G = Y^T Y supplied by the caller (e.g. summed over row
 * shards): L = chol(G) (lower, w x w), q = y L^-T.  info (device int): 0 ok, j+1 on breakdown. */
int lramm_cholqr_pass(const double *y, int64_t m, int64_t w, int64_t ldy, const double *gram, double *q, int64_t ldq,
                      double *l, int *info, void *ws, size_t ws_bytes, lramm_stream_t stream);
size_t lramm_cholqr_pass_ws(int64_t m, int64_t w);

/* Dequantising epilogue over an int32 accumulator matrix (e.g. partial products summed across
 * shards): same semantics as lramm_igemm's epilogue. */
int lramm_dequant(const int32_t *acc, int64_t M, int64_t N, int64_t lda, const lramm_epilogue_t *epi,
                  lramm_stream_t stream);

/* rint(a*scale) half-to-even, clamp +-cap, int32 (the plugin kernel, _core.pyx:53-69). */
int lramm_scale_round_clip(const double *a, int64_t rows, int64_t cols, int64_t lda, double scale,
                           int cap, int32_t *out, int64_t ldo, lramm_stream_t stream);

/* C = A . B^T with A: M x K int8 (row-major, lda bytes), B: N x K int8 (row-major,
 * ldb bytes), int32 accumulation in tensor memory (tcgen05.mma kind::i8, TMA-fed).
 * lda, ldb must be multiples of 16; A/B 16-byte aligned.  split_k > 1 requires an
 * int32 output with accumulate = 1. */
int lramm_igemm(int64_t M, int64_t N, int64_t K, const int8_t *a, int64_t lda, const int8_t *b,
                int64_t ldb, const lramm_epilogue_t *epi, int split_k, lramm_stream_t stream);
/* The same product with A packed int4 (two's-complement nibbles, column 2j in the low nibble of
 * byte j, lda in bytes, a multiple of 16 and >= ceil(K/2)), as lramm_quantize writes it for
 * q_dtype = LRAMM_I4 (bit budgets <= 4).  tcgen05 has no int4 kind on sm_100: the kernel
 * unpacks the TMA-loaded tile to int8 in shared memory before kind::i8 (c3's Y = A . Omega). */
int lramm_igemm_i4(int64_t M, int64_t N, int64_t K, const uint8_t *a4, int64_t lda, const int8_t *b,
                   int64_t ldb, const lramm_epilogue_t *epi, int split_k, lramm_stream_t stream);

/* Bit budgets 9..24 (quant.py:16-28 allows [2, 24]): a quantised int32 operand is carried as
 * 1..4 planes of 8-bit limbs, v = sum_l limb_l 256^l (unsigned low limbs, signed top limb).
 * lramm_split_limbs: rows x cols int32 (ld lds) -> nlimb planes of rows x ldd int8 (plane
 * stride rows * ldd bytes, ldd a multiple of 16).  lramm_igemm_limbs: C = A . B^T over limb
 * planes (pa / pb bytes between planes), the la x lb int8 tensor-core products accumulated
 * exactly in int64 (acc64: M x N scratch), then the lramm_igemm epilogue (out_dtype F32/F64
 * dequantised, or I64 for the raw exact product).  Replaces the int64 imatmul of
 * _core.pyx:35-50 for operands beyond +-127. */
int lramm_split_limbs(const int32_t *src, int64_t rows, int64_t cols, int64_t lds, int nlimb, int8_t *dst,
                      int64_t ldd, lramm_stream_t stream);
int lramm_igemm_limbs(int64_t M, int64_t N, int64_t K, const int8_t *a, int64_t lda, int64_t pa, int la,
                      const int8_t *b, int64_t ldb, int64_t pb, int lb, int64_t *acc64, const lramm_epilogue_t *epi,
                      lramm_stream_t stream);

/* fp64 GEMM.  trans_a = 0: C(MxN) = A(MxK) . B(KxN); trans_a = 1: C = A^T . B with
 * A stored K x M (split-K over the long dimension, deterministic reduction).
 * All row-major.  ws >= lramm_dgemm_ws(trans_a, M, N, K). */
int lramm_dgemm(int trans_a, int64_t M, int64_t N, int64_t K, const double *a, int64_t lda,
                const double *b, int64_t ldb, double *c, int64_t ldc, void *ws, size_t ws_bytes,
                lramm_stream_t stream);
size_t lramm_dgemm_ws(int trans_a, int64_t M, int64_t N, int64_t K);

/* Thin QR of a tall m x w fp64 matrix (m >= w): CholeskyQR2 with an on-device
 * Householder fallback when the Gram matrix is not numerically positive definite.
 * q (m x w, may alias y) and r (w x w upper) are outputs; r may be NULL. */
int lramm_qr(const double *y, int64_t m, int64_t w, int64_t ldy, double *q, int64_t ldq, double *r,
             void *ws, size_t ws_bytes, lramm_stream_t stream);
size_t lramm_qr_ws(int64_t m, int64_t w);

/* Thin SVD of a dense fp64 m x n matrix (the reference's oracle_svd contract,
 * matcore.py:232-245): u m x t, s t (descending), v n x t, t = min(m, n).
 * Implementation: CholeskyQR2 reduction + one-sided Jacobi (tol 1e-13,
 * <= 60 sweeps, _jacobi.py:10-11) on device; info (device int) receives the
 * sweep count or -1 on non-convergence. */
int lramm_svd(const double *a, int64_t m, int64_t n, double *u, double *s, double *v, int *info,
              void *ws, size_t ws_bytes, lramm_stream_t stream);
size_t lramm_svd_ws(int64_t m, int64_t n);

/* Gaussian test matrix on the device, bit-identical to NumPy's
 * Generator(Philox(SeedSequence([seed, 0x534B, ncols, w]))).standard_normal((ncols, w))
 * (matcore.py:89-92, rsvd.py:56): key0/key1 = the Philox key that SeedSequence produces
 * (Philox(ss).state["state"]["key"]), out = ncols x w row-major fp64 on the device.
 * Synchronous (a few tail draws are finished on the host with libm log1p). */
int lramm_omega(uint64_t key0, uint64_t key1, int64_t ncols, int64_t w, double *out, void *ws, size_t ws_bytes,
                lramm_stream_t stream);
size_t lramm_omega_ws(int64_t ncols, int64_t w);

/* Randomised SVD of x (rows x cols, F32 or F64) truncated to params->rank
 * (rsvd.py:68-94): u rows x rank, s rank, v cols x rank.  omega: cols x w fp64,
 * w = min(rank + oversample, min(rows, cols)), drawn by the caller exactly as
 * rsvd.py:56 (NumPy Philox).  status (device int): 0 ok, else an lramm_status. */
int lramm_rsvd(const void *x, int x_dtype, int64_t rows, int64_t cols, const lramm_params_t *params,
               const double *omega, double *u, double *s, double *v, int *status, void *ws,
               size_t ws_bytes, lramm_stream_t stream);
size_t lramm_rsvd_ws(int64_t rows, int64_t cols, const lramm_params_t *params);

/* The whole pipeline (pipeline.py:159-214): d = alpha * QM(QM(QM(Va^T Ub) Zsc) ... ) + beta * c.
 * a: m x k, b: k x n (F32 or F64, row-major, contiguous).  d: m x n of d_dtype
 * (LRAMM_F64 reproduces the reference's float64 output bit-for-bit given the same
 * factors; LRAMM_F32 is its correct rounding).  status: device int (0 = ok).
 * timings may be NULL; if not NULL the call records events and synchronises the
 * stream at the end to fill it. */
int lramm_lramm(const void *a, const void *b, int in_dtype, int64_t m, int64_t k, int64_t n,
                const lramm_params_t *params, const double *omega_a, const double *omega_b,
                const void *c, int c_dtype, void *d, int d_dtype, int *status, void *ws,
                size_t ws_bytes, lramm_timings_t *timings, lramm_stream_t stream);
size_t lramm_lramm_ws(int64_t m, int64_t k, int64_t n, const lramm_params_t *params);

/* ---------------------------------------------------------------- sharded pipeline (multi-GPU)
 *
 * One process per GPU; A is row-sharded and B column-sharded (BASELINE configs[4]).
 * The library does not link NCCL: the caller hands it a table of collective entry points whose
 * signatures ARE NCCL's (nccl.h ncclAllReduce / ncclAllGather, ncclResult_t returned as int,
 * ncclDataType_t / ncclRedOp_t passed as their integer values), plus the opaque communicator
 * they take.  A binding fills it with the addresses of ncclAllReduce / ncclAllGather and an
 * ncclComm_t; tests fill it with host-staged callbacks.  Every collective is
 * issued on the stream of the chain that needs it, so the call stays CUDA-graph capturable.
 *
 * comm_b (may be NULL): a second communicator for the rsvd chain of B, which then runs on a
 * forked stream concurrently with A's chain (NCCL serialises the operations of ONE communicator,
 * so two concurrent chains need two).  With comm_b == NULL and world > 1 the chains run one
 * after the other on `stream`.  With world == 1 no collective is called (unless
 * LRAMM_COMM_FORCE is set in flags) and the chains always run concurrently. */
typedef int (*lramm_all_reduce_fn)(const void *sendbuff, void *recvbuff, size_t count, int nccl_dtype, int nccl_op,
                                   void *comm, lramm_stream_t stream); /* == ncclAllReduce */
typedef int (*lramm_all_gather_fn)(const void *sendbuff, void *recvbuff, size_t sendcount, int nccl_dtype, void *comm,
                                   lramm_stream_t stream); /* == ncclAllGather */
enum { LRAMM_COMM_FORCE = 1 }; /* flags: call the collectives even when world == 1 */
typedef struct {
  void *comm;   /* ncclComm_t of A's chain and of the recombination */
  void *comm_b; /* ncclComm_t of B's chain, or NULL */
  int32_t rank;
  int32_t world;
  int32_t flags;
  int32_t reserved;
  lramm_all_reduce_fn all_reduce;
  lramm_all_gather_fn all_gather;
} lramm_comm_t;

/* Rows [lo, hi) of a dimension of `total` owned by `rank` of `world` (balanced contiguous
 * blocks: the first total % world ranks hold one more). */
void lramm_shard_bounds(int64_t total, int32_t world, int32_t rank, int64_t *lo, int64_t *hi);

/* lramm_lramm with A row-sharded and B column-sharded over comm->world ranks (pipeline.py:159-214
 * per rank; rsvd.py:47-94 with the exchanges below).  a_rows: this rank's rows of A,
 * (m_hi - m_lo) x k contiguous; b_cols: this rank's columns of B, k x (n_hi - n_lo) contiguous
 * (bounds from lramm_shard_bounds); omega_a (k x w_a) and omega_b (n x w_b) are the FULL test
 * matrices, replicated.  c_rows / d_rows: this rank's rows of C / D, (m_hi - m_lo) x n.
 * Exchanges, all through `comm`:
 *   allreduce(SUM, fp64) of the w x w Gram matrices of row-sharded sketches (CholeskyQR2),
 *   allreduce(SUM, int32) of the partial accumulators of products that contract over the sharded
 *     dimension (A^T Q; B Omega, B Qz) -- exact, so fast-mode integers do not depend on world
 *     (parity mode: allreduce(SUM, fp64) of the partial fp64 products),
 *   allreduce(MAX, fp64) of quantiser absmax values that span a sharded dimension,
 *   allgather(int8) of the quantised E2 operand before the last product.
 * Every factor stays resident on its rank.  Restrictions: recombination bit budgets <= 8; a
 * sketch whose Gram matrix is not numerically positive definite (rank-deficient operand) sets
 * status = LRAMM_ERR_UNSUPPORTED (the single-GPU path's Householder fallback is not sharded). */
int lramm_lramm_sharded(const void *a_rows, const void *b_cols, int in_dtype, int64_t m, int64_t k, int64_t n,
                        const lramm_params_t *params, const double *omega_a, const double *omega_b,
                        const void *c_rows, int c_dtype, void *d_rows, int d_dtype, int *status, void *ws,
                        size_t ws_bytes, const lramm_comm_t *comm, lramm_stream_t stream);
size_t lramm_lramm_sharded_ws(int64_t m, int64_t k, int64_t n, const lramm_params_t *params, int32_t world,
                              int32_t rank);

/* ---------------------------------------------------------------- host API */

int lramm_host_matmul(const double *a, const double *b, double *out, int64_t m, int64_t k, int64_t n);
int lramm_host_imatmul(const int32_t *a, const int32_t *b, int64_t *out, int64_t m, int64_t k,
                       int64_t n);
int lramm_host_scale_round_clip(const double *a, int64_t m, int64_t n, double scale, int cap,
                                int32_t *out);
int lramm_host_svd(const double *a, int64_t m, int64_t n, double *u, double *s, double *v);
/* a, b, c, d: host buffers (page-locked for asynchronous copies).  omega_a / omega_b: host
 * buffers, or device buffers on the current device (e.g. from lramm_omega), used in place. */
int lramm_host_lramm(const void *a, const void *b, int in_dtype, int64_t m, int64_t k, int64_t n,
                     const lramm_params_t *params, const double *omega_a, const double *omega_b,
                     const void *c, int c_dtype, void *d, int d_dtype, lramm_timings_t *timings);

#ifdef __cplusplus
}
#endif
#endif /* LRAMM_CUDA_H_ */
