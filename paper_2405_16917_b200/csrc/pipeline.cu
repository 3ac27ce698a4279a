// Native orchestration of the hot path: the randomised SVD of each operand
// (rsvd.py:47-94) and the three-stage recombination (pipeline.py:159-214), as a
// stream-ordered sequence of sm_100a kernels over caller-provided workspace.
// No host synchronisation, no allocation: a whole lramm() call can be captured
// in a CUDA graph.
//
// Modes:
//   parity: sketch / power / projection products in fp64 (the reference),
//   fast:   those products as int8 tensor-core GEMMs of per-tensor or per-row
//           quantised operands, dequantised bit-exactly in the epilogue.
// In both modes the thin QRs (CholeskyQR2), the small SVD (one-sided Jacobi)
// and the lift are fp64, and the recombination E1 -> E2 -> E3 uses the
// reference's per-tensor quantiser at (d1, d2, d3) with int8 tcgen05 GEMMs.
#include <algorithm>
#include <map>
#include <mutex>

#include "common.cuh"

namespace lramm {

int quantize_device(const void *x, int x_dtype, int64_t rows, int64_t cols, int64_t ldx, int bits, int gran,
                    int transpose, void *q, int q_dtype, int64_t ldq, double *scales, int *nonfinite, void *ws,
                    size_t ws_bytes, cudaStream_t st, const AmaxSync *sync = nullptr);
size_t quantize_ws_bytes(int64_t rows, int64_t cols);
int quantize_pair_device(const void *x, int x_dtype, int64_t rows, int64_t cols, int64_t ldx, int bits_r, int gran_r,
                         int8_t *qr, int64_t ldqr, double *scales_r, int bits_t, int gran_t, int8_t *qt, int64_t ldqt,
                         double *scales_t, int *nonfinite, void *ws, size_t ws_bytes, cudaStream_t st,
                         int r_packed = 0, const AmaxSync *sync = nullptr);
int igemm_limbs_device(int64_t M, int64_t N, int64_t K, const int8_t *a, int64_t lda, int64_t pa, int la,
                       const int8_t *b, int64_t ldb, int64_t pb, int lb, int64_t *acc64,
                       const lramm_epilogue_t &epi, cudaStream_t st);
int split_limbs_device(const int32_t *src, int64_t rows, int64_t cols, int64_t lds, int nlimb, int8_t *dst,
                       int64_t ldd, cudaStream_t st);
int igemm_device(int64_t M, int64_t N, int64_t K, const int8_t *a, int64_t lda, const int8_t *b, int64_t ldb,
                 const lramm_epilogue_t &epi, int split_k, cudaStream_t st, int a4 = 0);
int epilogue_device(const int32_t *acc, int64_t M, int64_t N, int64_t lda, const lramm_epilogue_t &epi,
                    cudaStream_t st);
int pick_bn(int64_t N);
int dgemm_device(int trans_a, int64_t M, int64_t N, int64_t K, const double *A, int64_t lda, const double *B,
                 int64_t ldb, double *C, int64_t ldc, void *ws, size_t ws_bytes, cudaStream_t st);
size_t dgemm_ws_bytes(int trans_a, int64_t M, int64_t N, int64_t K);
int qr_device(const double *y, int64_t m, int64_t w, int64_t ldy, double *q, int64_t ldq, double *r, void *ws,
              size_t ws_bytes, cudaStream_t st, bool q_needed = true, bool fast = false,
              const double *gram_in = nullptr, const Coll *rows_coll = nullptr);
size_t qr_ws_bytes(int64_t m, int64_t w);
int svd_tall_pside_device(const double *T, int64_t m, int64_t n, int64_t ldt, const double *s, const double *H,
                          int64_t ldh, double *pside, int64_t ldp, int *status, void *ws, size_t ws_bytes,
                          cudaStream_t st);
int svd_tall_device(const double *T, int64_t m, int64_t n, int64_t ldt, double *pside, int64_t ldp, double *s,
                    double *h, int64_t ldh, int *info, int *status, void *ws, size_t ws_bytes, cudaStream_t st,
                    const Coll *rows_coll = nullptr, bool fast = false);
size_t svd_tall_ws_bytes(int64_t m, int64_t n);
int qr_report_breakdown_device(void *ws, size_t ws_bytes, int64_t m, int64_t w, int *status, cudaStream_t st);

namespace {

__global__ void f32_to_f64_kernel(const float *__restrict__ x, int64_t n, double *__restrict__ y) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    y[i] = (double)x[i];
}

// B[i][j] = A[i][j] * s[j]  (u * sigma, pipeline.py:189-190; one IEEE rounding)
__global__ void scale_cols_kernel(const double *__restrict__ A, int64_t rows, int cols, int64_t lda,
                                  const double *__restrict__ s, double *__restrict__ B, int64_t ldb) {
  int64_t n = rows * cols;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    int64_t r = i / cols;
    int c = (int)(i - r * cols);
    B[r * ldb + c] = __dmul_rn(A[r * lda + c], s[c]);
  }
}

// status summary: jacobi info (<0 = no convergence), non-finite flag, completion status
__global__ void summarize_status_kernel(const int *jac_info, int njac, const int *nonfinite, const int *compl_st,
                                        int *status) {
  if (threadIdx.x != 0) return;
  int s = 0;
  for (int i = 0; i < njac && !s; ++i)
    if (jac_info[i] < 0) s = LRAMM_ERR_NONCONVERGENCE;
  if (!s && compl_st && *compl_st) s = *compl_st;
  if (nonfinite && *nonfinite) s = LRAMM_ERR_NONFINITE;
  *status = s;
}

inline int elem_grid(int64_t n) { return (int)std::max<int64_t>(1, std::min<int64_t>(ceil_div(n, 256), 8LL * num_sms())); }

// ---------------------------------------------------------------- exact integer Gram
// Per-tensor fast mode: the sketch Y = Y_int / S (S = s_x s_Omega, the qprod dequantisation, each
// entry one correctly rounded division) carries its exact int32 accumulator: rint(Y S) recovers
// Y_int (|Y_int| < 2^27, relative error of Y S <= 2 eps).  Y_int^T is written as 8-bit limb
// planes, K-major (w x ldk per plane, zero padded), for the int8 tensor-core limb products
// (igemm_limbs_device), whose exact int64 sum the epilogue divides by S^2 once: the Gram of the
// CholeskyQR of Y, correctly rounded, from int8 products instead of an fp64 GEMM.
__global__ void gram_limbs_kernel(const double *__restrict__ Y, int64_t rows, int w, const double *__restrict__ sa,
                                  const double *__restrict__ sb, int nlimb, int8_t *__restrict__ planes, int64_t ldk,
                                  int64_t plane, double *__restrict__ s_out) {
  __shared__ int32_t t[32][33];
  const double S = __dmul_rn(*sa, *sb);
  if (blockIdx.x == 0 && blockIdx.y == 0 && threadIdx.x == 0 && threadIdx.y == 0) *s_out = S;
  const int64_t r0 = (int64_t)blockIdx.y * 32;
  const int c0 = blockIdx.x * 32;
  for (int i = threadIdx.y; i < 32; i += blockDim.y) {  // rows r0 + i, columns c0 + lane
    const int64_t r = r0 + i;
    const int c = c0 + threadIdx.x;
    t[i][threadIdx.x] = (r < rows && c < w) ? (int32_t)rint(__dmul_rn(Y[r * w + c], S)) : 0;
  }
  __syncthreads();
  for (int i = threadIdx.y; i < 32; i += blockDim.y) {  // plane row c0 + i, k = r0 + lane
    const int c = c0 + i;
    const int64_t k = r0 + threadIdx.x;
    if (c >= w || k >= ldk) continue;
    int32_t v = t[threadIdx.x][i];
    for (int l = 0; l < nlimb; ++l) {
      int8_t d;
      if (l == nlimb - 1) {
        d = (int8_t)v;
      } else {
        d = (int8_t)(uint8_t)(v & 0xFF);
        v = v >> 8;
      }
      planes[l * plane + (int64_t)c * ldk + k] = d;
    }
  }
}

struct QOp {  // a quantised K-major operand (bit budgets > 8: `limbs` 8-bit planes, see split_limbs)
  int8_t *q = nullptr;
  int64_t ld = 0;
  double *scale = nullptr;
  int64_t inc = 0;
  int limbs = 1;
  int64_t plane = 0;  // bytes between limb planes
  int64_t rows = 0;
  int packed = 0;  // bit budgets <= 4 of the sketch's X: packed int4 (ld in bytes), unpacked in the GEMM
};

// 8-bit limbs needed for a bit budget: 1 (<= 8, the plain signed int8), 2 (<= 16), 3 (<= 24)
inline int limbs_for(int bits) { return bits <= 8 ? 1 : (bits <= 16 ? 2 : 3); }

struct RsvdBufs {
  int64_t rows = 0, cols = 0, w = 0, r = 0;
  bool fast = false;
  int gran = LRAMM_GRAN_TENSOR;
  // fast-mode operands
  QOp xr_s, xr_p, xc_p, xc_j, om, qq, qzq;
  // parity mode fp64 copy of x (when x is fp32)
  double *x64 = nullptr;
  double *Y = nullptr, *Q = nullptr, *Z = nullptr, *Qz = nullptr, *BsT = nullptr, *Pside = nullptr, *H = nullptr,
         *s = nullptr;
  int32_t *acc = nullptr;
  // exact integer Gram of tall per-tensor sketches (gram_limbs_kernel)
  int8_t *gplanes = nullptr;
  int64_t gldk = 0;
  int glimbs = 0;
  int64_t *gacc = nullptr;
  double *gram = nullptr, *gS = nullptr;
  int *info = nullptr, *compl_st = nullptr, *nonfinite = nullptr;
  void *qr_ws = nullptr, *svd_ws = nullptr, *gemm_ws = nullptr, *qz_ws = nullptr;
  void *qz_ws2 = nullptr;  // quantiser scratch of the helper stream (operand copies made off the critical path)
  size_t qr_bytes = 0, svd_bytes = 0, gemm_bytes = 0, qz_bytes = 0;
};

QOp take_qop(Arena &ar, int64_t rows, int64_t kdim, int64_t nscale, int limbs = 1) {
  QOp o;
  o.ld = round_up(kdim, 16);
  o.limbs = limbs;
  o.rows = rows;
  o.plane = rows * o.ld;
  o.q = ar.take<int8_t>(rows * o.ld * limbs);
  o.scale = ar.take<double>(nscale);
  o.inc = nscale > 1 ? 1 : 0;
  return o;
}

// the exact integer Gram can replace the fp64 Gram GEMM of the sketches' first CholeskyQR pass in
// per-tensor fast mode for sketches of at least LRAMM_EXACT_GRAM_ROWS rows.  Off by default:
// measured at c5 (131072 x 1056, 4 limbs x 4 limbs x 4 K-chunks = 64 serial int8 GEMMs with 54
// output tiles each) the step is 78.1 ms against 67.9 ms with the fp64 DMMA Gram
inline bool use_exact_gram(const RsvdBufs &b, const lramm_params_t &P) {
  static const long long thr = [] {
    const char *s = getenv("LRAMM_EXACT_GRAM_ROWS");
    return s ? atoll(s) : 0LL;
  }();
  if (thr <= 0 || !b.fast || b.gran != LRAMM_GRAN_TENSOR || P.sketch_bits > 8 || P.power_bits != P.sketch_bits)
    return false;
  return b.rows >= thr && (double)b.cols * bit_cap(P.sketch_bits) * bit_cap(P.sketch_bits) < 2147483648.0;
}

// w_global > 0: the sketch width of the whole operand when (rows, cols) is one rank's shard
RsvdBufs carve_rsvd(Arena &ar, int64_t rows, int64_t cols, int x_dtype, const lramm_params_t &P,
                    int64_t w_global = 0) {
  RsvdBufs b;
  b.rows = rows;
  b.cols = cols;
  b.r = P.rank;
  b.w = w_global > 0 ? w_global : std::min<int64_t>(P.rank + P.oversample, std::min(rows, cols));
  b.fast = P.mode == LRAMM_MODE_FAST;
  b.gran = P.granularity == LRAMM_GRAN_ROW ? LRAMM_GRAN_ROW : LRAMM_GRAN_TENSOR;
  const bool row = b.gran == LRAMM_GRAN_ROW;
  const int64_t w = b.w;
  if (b.fast) {
    if (P.sketch_bits <= 4) {  // the sketch operand X stays packed int4 in HBM (half the bytes)
      b.xr_s = take_qop(ar, rows, ceil_div(cols, 2), row ? rows : 1);
      b.xr_s.packed = 1;
    } else {
      b.xr_s = take_qop(ar, rows, cols, row ? rows : 1);
    }
    if (P.power_iters > 0) b.xr_p = P.power_bits == P.sketch_bits ? b.xr_s : take_qop(ar, rows, cols, row ? rows : 1);
    b.xc_j = take_qop(ar, cols, rows, row ? cols : 1);
    if (P.power_iters > 0) b.xc_p = P.power_bits == P.proj_bits ? b.xc_j : take_qop(ar, cols, rows, row ? cols : 1);
    b.om = take_qop(ar, w, cols, row ? w : 1);
    b.qq = take_qop(ar, w, rows, row ? w : 1);
    b.qzq = take_qop(ar, w, cols, row ? w : 1);
    b.qz_bytes = quantize_ws_bytes(std::max(rows, cols), std::max(rows, cols));
    b.qz_ws = ar.take<char>((int64_t)b.qz_bytes);
    b.qz_ws2 = ar.take<char>((int64_t)b.qz_bytes);
    int64_t mx = std::max(rows, cols);
    b.acc = ar.take<int32_t>(mx * w);
    if (w_global <= 0 && use_exact_gram(b, P)) {
      // |Y_int| <= cols * cap_x * cap_Omega: 8-bit limbs (unsigned low bytes, signed top limb)
      const double bound = (double)cols * bit_cap(P.sketch_bits) * bit_cap(P.sketch_bits);
      b.glimbs = bound < 128.0 ? 1 : (bound < 32768.0 ? 2 : (bound < 8388608.0 ? 3 : 4));
      b.gldk = round_up(rows, 16);
      b.gplanes = ar.take<int8_t>((int64_t)b.glimbs * w * b.gldk);
      b.gacc = ar.take<int64_t>(w * w);
      b.gram = ar.take<double>(w * w);
      b.gS = ar.take<double>(1);
    }
  } else if (x_dtype == LRAMM_F32) {
    b.x64 = ar.take<double>(rows * cols);
  }
  b.Y = ar.take<double>(rows * w);
  b.Q = ar.take<double>(rows * w);
  b.Z = ar.take<double>(cols * w);
  b.Qz = ar.take<double>(cols * w);
  b.BsT = ar.take<double>(cols * w);
  b.Pside = ar.take<double>(cols * w);
  b.H = ar.take<double>(w * w);
  b.s = ar.take<double>(w);
  b.info = ar.take<int>(4);
  b.compl_st = ar.take<int>(4);
  b.nonfinite = ar.take<int>(4);
  int64_t mx = std::max(rows, cols);
  b.qr_bytes = qr_ws_bytes(mx, w);
  b.qr_ws = ar.take<char>((int64_t)b.qr_bytes);
  b.svd_bytes = svd_tall_ws_bytes(cols, w);
  b.svd_ws = ar.take<char>((int64_t)b.svd_bytes);
  b.gemm_bytes = std::max(dgemm_ws_bytes(1, cols, w, rows), dgemm_ws_bytes(0, rows, w, cols));
  b.gemm_bytes = std::max(b.gemm_bytes, dgemm_ws_bytes(0, rows, P.rank, w));
  b.gemm_ws = ar.take<char>((int64_t)b.gemm_bytes);
  return b;
}

// C (M x N fp64) = dequant(A . B^T): row scales of A, column scales of B
// reduce (sharded pipeline): the contraction runs over a sharded dimension, so the int32
// accumulators are partial sums; they are allreduced (exactly) before the dequantising epilogue
int qprod(const QOp &A, const QOp &B, int64_t M, int64_t N, int64_t K, double *C, int64_t ldc, int transpose_out,
          int32_t *acc, cudaStream_t st, int64_t *acc64 = nullptr, bool force64 = false,
          const Coll *reduce = nullptr) {
  lramm_epilogue_t e = {};
  e.out_dtype = LRAMM_F64;
  e.transpose_out = transpose_out;
  e.out = C;
  e.ldo = ldc;
  e.row_scale = A.scale;
  e.row_scale_inc = A.inc;
  e.col_scale = B.scale;
  e.col_scale_inc = B.inc;
  e.alpha = 1.0;
  e.beta = 0.0;
  if (A.limbs > 1 || B.limbs > 1 || force64) {
    if (!acc64) return fail(LRAMM_ERR_WORKSPACE, "qprod: multi-limb product needs an int64 accumulator");
    return igemm_limbs_device(M, N, K, A.q, A.ld, A.plane, A.limbs, B.q, B.ld, B.plane, B.limbs, acc64, e, st);
  }
  const int64_t tiles = ceil_div(M, 128) * ceil_div(N, pick_bn(N));
  const int64_t kb = ceil_div(K, 128);
  int split = 1;
  // split-K into at most one wave of CTAs (4096 x 272 x 4096 sketch: 64 tiles -> split 2, 4.15 -> 4.07 ms
  // c2 step against split 3's 1.3 waves)
  if (acc && tiles * 2 <= num_sms() && kb >= 8) split = (int)std::min<int64_t>(kb / 4, num_sms() / tiles);
  const bool red = reduce && reduce->on();
  if (red && !acc) return fail(LRAMM_ERR_WORKSPACE, "qprod: a sharded contraction needs an int32 accumulator");
  if (split <= 1 && !red) return igemm_device(M, N, K, A.q, A.ld, B.q, B.ld, e, 1, st, A.packed);
  lramm_epilogue_t ea = {};
  ea.out_dtype = LRAMM_I32;
  ea.accumulate = split > 1 ? 1 : 0;
  ea.out = acc;
  ea.ldo = N;
  if (split > 1) LRAMM_CUDA_TRY(cudaMemsetAsync(acc, 0, (size_t)M * N * sizeof(int32_t), st));
  LRAMM_TRY(igemm_device(M, N, K, A.q, A.ld, B.q, B.ld, ea, std::max(split, 1), st, A.packed));
  if (red) LRAMM_TRY(reduce->sum_i32(acc, (size_t)(M * N), st));
  return epilogue_device(acc, M, N, N, e, st);
}

int quant(const void *x, int dtype, int64_t rows, int64_t cols, int64_t ldx, int bits, int gran, int transpose,
          QOp &o, int *nonfinite, void *ws, size_t ws_bytes, cudaStream_t st, int32_t *tmp32 = nullptr,
          const AmaxSync *sync = nullptr) {
  if (o.limbs <= 1)
    return quantize_device(x, dtype, rows, cols, ldx, bits, gran, transpose, o.q, o.packed ? LRAMM_I4 : LRAMM_I8, o.ld,
                           o.scale, nonfinite, ws, ws_bytes, st, sync);
  if (sync && sync->coll && sync->coll->on())
    return fail(LRAMM_ERR_UNSUPPORTED, "the sharded path carries int8 operands: bit budgets must be <= 8");
  // bit budgets > 8: the reference's integers (int32, bit-exact) -> 8-bit limb planes
  if (!tmp32) return fail(LRAMM_ERR_WORKSPACE, "quant: multi-limb operand needs an int32 staging buffer");
  const int64_t orows = transpose ? cols : rows, kdim = transpose ? rows : cols;
  LRAMM_TRY(quantize_device(x, dtype, rows, cols, ldx, bits, gran, transpose, tmp32, LRAMM_I32, o.ld, o.scale,
                            nonfinite, ws, ws_bytes, st));
  return split_limbs_device(tmp32, orows, kdim, o.ld, o.limbs, o.q, o.ld, st);
}

int check_bits_dev(int bits, const char *what, bool limbs_ok = false) {
  if (bits < 2 || bits > 24) return fail(LRAMM_ERR_PARAM, "%s must be an integer in [2, 24], got %d", what, bits);
  if (bits > 8 && !limbs_ok)
    return fail(LRAMM_ERR_UNSUPPORTED, "%s = %d: the fast-mode sketch products support bit budgets <= 8", what, bits);
  return LRAMM_OK;
}

// recombination guard: the reference's int64 rule (quant.py:87-93) is the only refusal; products
// whose int32 accumulators could overflow (K cap^2 >= 2^31) run through the exact int64 limb
// path (igemm_limbs_device: K chunked so every int32 partial is exact)
int check_acc_qm(int64_t K, int bits) {
  if ((long double)K * bit_cap(bits) * bit_cap(bits) >= 9223372036854775808.0L)
    return fail(LRAMM_ERR_OVERFLOW, "k=%lld with bit budgets (%d, %d) risks int64 overflow", (long long)K, bits, bits);
  return LRAMM_OK;
}
// does a single-int8 product of contraction length K need the int64 accumulator?
bool needs_acc64(int64_t K, int bits) {
  return bits <= 8 && (double)K * bit_cap(bits) * bit_cap(bits) >= 2147483648.0;
}

// int32 accumulation guard: K * cap_a * cap_b < 2^31 (the reference's int64 guard is quant.py:87-93)
int check_acc(int64_t K, int bits_a, int bits_b) {
  if ((double)K * bit_cap(bits_a) * bit_cap(bits_b) >= 2147483648.0)
    return fail(LRAMM_ERR_OVERFLOW, "k=%lld with bit budgets (%d, %d) risks int32 accumulator overflow",
                (long long)K, bits_a, bits_b);
  return LRAMM_OK;
}

// helper stream per (device, chain stream): the quantised copies of X that the power iteration
// and the projection need (X row-scaled at power_bits, X^T column-scaled) depend only on X, so
// they are made while the sketch's QR runs
struct HelperStream {
  cudaStream_t st = nullptr;
  cudaEvent_t fork = nullptr, join = nullptr;
};
HelperStream &helper_stream(cudaStream_t main) {
  static std::mutex mu;
  static std::map<std::pair<int, cudaStream_t>, HelperStream> table;
  int dev = 0;
  cudaGetDevice(&dev);
  std::lock_guard<std::mutex> g(mu);
  HelperStream &x = table[{dev, main}];
  if (!x.st) {
    cudaStreamCreateWithFlags(&x.st, cudaStreamNonBlocking);
    cudaEventCreateWithFlags(&x.fork, cudaEventDisableTiming);
    cudaEventCreateWithFlags(&x.join, cudaEventDisableTiming);
  }
  return x;
}

// G = Y^T Y exactly from the sketch's integers (per-tensor: row scale sa, column scale sb)
int exact_gram(RsvdBufs &b, const double *Y, const double *sa, const double *sb, cudaStream_t st) {
  const int64_t rows = b.rows, w = b.w;
  gram_limbs_kernel<<<dim3((unsigned)ceil_div(w, 32), (unsigned)ceil_div(b.gldk, 32)), dim3(32, 8), 0, st>>>(
      Y, rows, (int)w, sa, sb, b.glimbs, b.gplanes, b.gldk, w * b.gldk, b.gS);
  LRAMM_LAUNCH_CHECK();
  lramm_epilogue_t e = {};
  e.out_dtype = LRAMM_F64;
  e.out = b.gram;
  e.ldo = w;
  e.row_scale = b.gS;
  e.row_scale_inc = 0;
  e.col_scale = b.gS;
  e.col_scale_inc = 0;
  e.alpha = 1.0;
  e.beta = 0.0;
  return igemm_limbs_device(w, w, b.gldk, b.gplanes, b.gldk, w * b.gldk, b.glimbs, b.gplanes, b.gldk, w * b.gldk,
                            b.glimbs, b.gacc, e, st);
}

// How one operand of the sharded pipeline is split: A by rows, B by columns.
struct ShardSpec {
  Coll coll;                     // the communicator of this operand's chain
  int kind = 0;                  // 0 whole operand, 1 rows of X sharded, 2 columns of X sharded
  int64_t g_rows = 0, g_cols = 0;  // global shape of X (accumulator guards)
};

// sh (sharded pipeline): x holds this rank's rows (kind 1) or columns (kind 2) of X and b is carved
// for that local shape with the global sketch width; omega = the rows of Omega that meet the local
// columns.  Products that contract over the sharded dimension allreduce their partial sums
// (int32 accumulators in fast mode: exact), the QRs of row-sharded sketches allreduce their
// Gram matrices, and quantiser maxima that span the sharded dimension are allreduced (MAX).
// Outputs: kind 1 -> U local rows, V replicated; kind 2 -> U replicated, V local rows.
int run_rsvd(const void *x, int x_dtype, RsvdBufs &b, const lramm_params_t &P, const double *omega, double *U,
             int64_t ldu, double *S, double *V, int64_t ldv, cudaStream_t st, const ShardSpec *sh = nullptr) {
  const int64_t rows = b.rows, cols = b.cols, w = b.w, r = b.r;
  const int kind = sh ? sh->kind : 0;
  const Coll *coll = sh ? &sh->coll : nullptr;
  const bool coll_on = coll && coll->on();
  const Coll *red_rows = kind == 1 ? coll : nullptr;  // contraction over X's rows is partial
  const Coll *red_cols = kind == 2 ? coll : nullptr;  // contraction over X's columns is partial
  const Coll *qr_rows = kind == 1 ? coll : nullptr;   // rows x w sketches are row-sharded
  const Coll *qr_cols = kind == 2 ? coll : nullptr;   // cols x w sketches are row-sharded
  // absmax vectors that span the sharded dimension (input coordinates of each quantisation)
  const AmaxSync sync_x{coll, kind != 0, kind == 2, kind == 1};  // X itself
  const AmaxSync sync_tall{coll, true, false, true};             // a row-sharded rows x w / cols x w matrix
  const AmaxSync *sx = kind ? &sync_x : nullptr;
  const AmaxSync *s_rows = kind == 1 ? &sync_tall : nullptr;  // Q (rows x w)
  const AmaxSync *s_cols = kind == 2 ? &sync_tall : nullptr;  // Omega_j, Qz (cols x w)
  LRAMM_CUDA_TRY(cudaMemsetAsync(b.info, 0, 4 * sizeof(int), st));
  LRAMM_CUDA_TRY(cudaMemsetAsync(b.compl_st, 0, 4 * sizeof(int), st));
  LRAMM_CUDA_TRY(cudaMemsetAsync(b.nonfinite, 0, 4 * sizeof(int), st));
  const int gran_l = b.gran == LRAMM_GRAN_ROW ? LRAMM_GRAN_ROW : LRAMM_GRAN_TENSOR;  // left operand rows
  const int gran_r = b.gran == LRAMM_GRAN_ROW ? LRAMM_GRAN_COL : LRAMM_GRAN_TENSOR;  // right operand columns
  const double *x64 = (const double *)x;
  bool helper = false;
  HelperStream *hs = nullptr;
  const int gran_c = gran_r == LRAMM_GRAN_COL ? LRAMM_GRAN_COL : LRAMM_GRAN_TENSOR;  // X^T copies: per input column
  // the first transposed copy X^T needs (power iteration, else projection) is written by the same
  // pass that quantises X for the sketch: one absmax pass + one read of X for both layouts
  QOp &xc_first = P.power_iters > 0 ? b.xc_p : b.xc_j;
  const int bits_first = P.power_iters > 0 ? P.power_bits : P.proj_bits;
  const bool pair = b.fast && b.xr_s.limbs <= 1 && xc_first.limbs <= 1;
  const bool need_xp_row = b.fast && P.power_iters > 0 && b.xr_p.q != b.xr_s.q;
  const bool need_xc_p = b.fast && P.power_iters > 0 && !pair;
  const bool need_xc_j = b.fast && (b.xc_j.q != b.xc_p.q || P.power_iters == 0) && !(pair && P.power_iters == 0);
  if (need_xp_row || need_xc_p || need_xc_j) {
    // the remaining X-only operand copies on the helper stream (joined before their first use);
    // with live collectives they stay on the chain's stream: one communicator, one stream
    cudaStream_t hst = st;
    if (!coll_on) {
      hs = &helper_stream(st);
      LRAMM_CUDA_TRY(cudaEventRecord(hs->fork, st));
      LRAMM_CUDA_TRY(cudaStreamWaitEvent(hs->st, hs->fork, 0));
      hst = hs->st;
    }
    void *hws = coll_on ? b.qz_ws : b.qz_ws2;
    if (need_xp_row)
      LRAMM_TRY(quant(x, x_dtype, rows, cols, cols, P.power_bits, gran_l, 0, b.xr_p, b.nonfinite, hws, b.qz_bytes, hst,
                      nullptr, sx));
    if (need_xc_p)
      LRAMM_TRY(quant(x, x_dtype, rows, cols, cols, P.power_bits, gran_c, 1, b.xc_p, b.nonfinite, hws, b.qz_bytes, hst,
                      nullptr, sx));
    if (need_xc_j)
      LRAMM_TRY(quant(x, x_dtype, rows, cols, cols, P.proj_bits, gran_c, 1, b.xc_j, b.nonfinite, hws, b.qz_bytes, hst,
                      nullptr, sx));
    if (!coll_on) {
      LRAMM_CUDA_TRY(cudaEventRecord(hs->join, hs->st));
      helper = true;
    }
  }
  auto join_helper = [&]() -> int {
    if (helper) {
      LRAMM_CUDA_TRY(cudaStreamWaitEvent(st, hs->join, 0));
      helper = false;
    }
    return LRAMM_OK;
  };
  // thin QR of a sketch; row-sharded sketches report a Cholesky breakdown (no sharded fallback)
  auto qr = [&](const double *y, int64_t m, double *q, const Coll *rc, const double *gram_in) -> int {
    LRAMM_TRY(qr_device(y, m, w, w, q, w, nullptr, b.qr_ws, b.qr_bytes, st, true, b.fast, gram_in, rc));
    if (rc) LRAMM_TRY(qr_report_breakdown_device(b.qr_ws, b.qr_bytes, m, w, b.compl_st, st));
    return LRAMM_OK;
  };
  NvtxStages nv;
  nv.next("rsvd.sketch");
  if (b.fast) {
    // Y = X . Omega at sketch_bits
    if (pair)
      LRAMM_TRY(quantize_pair_device(x, x_dtype, rows, cols, cols, P.sketch_bits, gran_l, b.xr_s.q, b.xr_s.ld,
                                     b.xr_s.scale, bits_first, gran_c, xc_first.q, xc_first.ld, xc_first.scale,
                                     b.nonfinite, b.qz_ws, b.qz_bytes, st, b.xr_s.packed, sx));
    else
      LRAMM_TRY(quant(x, x_dtype, rows, cols, cols, P.sketch_bits, gran_l, 0, b.xr_s, b.nonfinite, b.qz_ws, b.qz_bytes,
                      st, nullptr, sx));
    LRAMM_TRY(quant(omega, LRAMM_F64, cols, w, w, P.sketch_bits, gran_r, 1, b.om, nullptr, b.qz_ws, b.qz_bytes, st,
                    nullptr, s_cols));
    LRAMM_TRY(qprod(b.xr_s, b.om, rows, w, cols, b.Y, w, 0, b.acc, st, nullptr, false, red_cols));
    if (b.gram) LRAMM_TRY(exact_gram(b, b.Y, b.xr_s.scale, b.om.scale, st));
  } else {
    if (x_dtype == LRAMM_F32) {
      f32_to_f64_kernel<<<elem_grid(rows * cols), 256, 0, st>>>((const float *)x, rows * cols, b.x64);
      LRAMM_LAUNCH_CHECK();
      x64 = b.x64;
    }
    LRAMM_TRY(dgemm_device(0, rows, w, cols, x64, cols, omega, w, b.Y, w, b.gemm_ws, b.gemm_bytes, st));
    if (red_cols) LRAMM_TRY(red_cols->sum_f64(b.Y, (size_t)(rows * w), st));
  }
  LRAMM_TRY(qr(b.Y, rows, b.Q, qr_rows, b.gram));
  if (b.fast && P.power_iters > 0) LRAMM_TRY(join_helper());
  for (int it = 0; it < P.power_iters; ++it) {
    // Z = X^T Q ; Qz = qr(Z) ; Y = X Qz ; Q = qr(Y)   (rsvd.py:60-64)
    nv.next("rsvd.power");
    if (b.fast) {
      LRAMM_TRY(quant(b.Q, LRAMM_F64, rows, w, w, P.power_bits, gran_r, 1, b.qq, nullptr, b.qz_ws, b.qz_bytes, st,
                      nullptr, s_rows));
      LRAMM_TRY(qprod(b.xc_p, b.qq, cols, w, rows, b.Z, w, 0, b.acc, st, nullptr, false, red_rows));
    } else {
      LRAMM_TRY(dgemm_device(1, cols, w, rows, x64, cols, b.Q, w, b.Z, w, b.gemm_ws, b.gemm_bytes, st));
      if (red_rows) LRAMM_TRY(red_rows->sum_f64(b.Z, (size_t)(cols * w), st));
    }
    LRAMM_TRY(qr(b.Z, cols, b.Qz, qr_cols, nullptr));
    if (b.fast) {
      LRAMM_TRY(quant(b.Qz, LRAMM_F64, cols, w, w, P.power_bits, gran_r, 1, b.qzq, nullptr, b.qz_ws, b.qz_bytes, st,
                      nullptr, s_cols));
      LRAMM_TRY(qprod(b.xr_p, b.qzq, rows, w, cols, b.Y, w, 0, b.acc, st, nullptr, false, red_cols));
      if (b.gram) LRAMM_TRY(exact_gram(b, b.Y, b.xr_p.scale, b.qzq.scale, st));
    } else {
      LRAMM_TRY(dgemm_device(0, rows, w, cols, x64, cols, b.Qz, w, b.Y, w, b.gemm_ws, b.gemm_bytes, st));
      if (red_cols) LRAMM_TRY(red_cols->sum_f64(b.Y, (size_t)(rows * w), st));
    }
    LRAMM_TRY(qr(b.Y, rows, b.Q, qr_rows, b.gram));
  }
  // Bs^T = X^T Q   (rsvd.py:77, evaluated transposed)
  nv.next("rsvd.project");
  if (b.fast) {
    LRAMM_TRY(join_helper());
    LRAMM_TRY(quant(b.Q, LRAMM_F64, rows, w, w, P.proj_bits, gran_r, 1, b.qq, nullptr, b.qz_ws, b.qz_bytes, st, nullptr,
                    s_rows));
    LRAMM_TRY(qprod(b.xc_j, b.qq, cols, w, rows, b.BsT, w, 0, b.acc, st, nullptr, false, red_rows));
  } else {
    LRAMM_TRY(dgemm_device(1, cols, w, rows, x64, cols, b.Q, w, b.BsT, w, b.gemm_ws, b.gemm_bytes, st));
    if (red_rows) LRAMM_TRY(red_rows->sum_f64(b.BsT, (size_t)(cols * w), st));
  }
  // SVD(Bs): u = H, v = Bs^T H diag(s)^-1   (rsvd.py:78, _jacobi.py)
  nv.next("rsvd.small_svd");
  LRAMM_TRY(svd_tall_device(b.BsT, cols, w, w, nullptr, w, b.s, b.H, w, b.info, b.compl_st, b.svd_ws, b.svd_bytes,
                             st, qr_cols, b.fast));
  // v = Bs^T H diag(s)^-1 on the helper stream, concurrent with the lift U = Q u (rsvd.py:79-81);
  // both then truncated to r (rsvd.py:84-94)
  nv.next("rsvd.lift");
  HelperStream &hv = helper_stream(st);
  LRAMM_CUDA_TRY(cudaEventRecord(hv.fork, st));
  LRAMM_CUDA_TRY(cudaStreamWaitEvent(hv.st, hv.fork, 0));
  LRAMM_TRY(svd_tall_pside_device(b.BsT, cols, w, w, b.s, b.H, w, b.Pside, w, b.compl_st, b.svd_ws, b.svd_bytes,
                                  hv.st));
  LRAMM_CUDA_TRY(cudaMemcpy2DAsync(V, ldv * sizeof(double), b.Pside, w * sizeof(double), r * sizeof(double), cols,
                                   cudaMemcpyDeviceToDevice, hv.st));
  LRAMM_CUDA_TRY(cudaEventRecord(hv.join, hv.st));
  LRAMM_TRY(dgemm_device(0, rows, r, w, b.Q, w, b.H, w, U, ldu, b.gemm_ws, b.gemm_bytes, st));
  LRAMM_CUDA_TRY(cudaMemcpyAsync(S, b.s, r * sizeof(double), cudaMemcpyDeviceToDevice, st));
  LRAMM_CUDA_TRY(cudaStreamWaitEvent(st, hv.join, 0));
  return LRAMM_OK;
}

int validate_params(const lramm_params_t &P, bool need_bits) {
  if (P.rank < 1) return fail(LRAMM_ERR_PARAM, "rank must be >= 1, got %d", P.rank);
  if (P.power_iters < 0 || P.oversample < 0) return fail(LRAMM_ERR_PARAM, "power_iters and oversample must be >= 0");
  if (P.mode != LRAMM_MODE_PARITY && P.mode != LRAMM_MODE_FAST) return fail(LRAMM_ERR_PARAM, "bad mode %d", P.mode);
  if (P.mode == LRAMM_MODE_FAST) {
    LRAMM_TRY(check_bits_dev(P.sketch_bits, "sketch_bits"));
    LRAMM_TRY(check_bits_dev(P.proj_bits, "proj_bits"));
    if (P.power_iters > 0) LRAMM_TRY(check_bits_dev(P.power_bits, "power_bits"));
  }
  if (need_bits)
    for (int i = 0; i < 3; ++i) LRAMM_TRY(check_bits_dev(P.bits[i], "bits", true));  // > 8: int8 limbs
  return LRAMM_OK;
}

struct LrammBufs {
  RsvdBufs ra, rb;
  double *UA, *SA, *VA, *UB, *SB, *VB, *E1, *Zsc, *E2T, *Usc;
  QOp vt, wq, e1q, zq, e2q, uq;
  int32_t *e1acc;
  int32_t *tmp32 = nullptr;  // int32 quantiser staging (bit budgets > 8)
  int64_t *acc64 = nullptr;  // exact int64 accumulator of multi-limb products
  int *nonfinite, *jinfo;
  void *qws;
  size_t qbytes;
};

LrammBufs carve_lramm(Arena &ar, int64_t m, int64_t k, int64_t n, int in_dtype, const lramm_params_t &P) {
  LrammBufs L;
  const int64_t r = P.rank;
  L.ra = carve_rsvd(ar, m, k, in_dtype, P);
  L.rb = carve_rsvd(ar, k, n, in_dtype, P);
  L.UA = ar.take<double>(m * r);
  L.SA = ar.take<double>(r);
  L.VA = ar.take<double>(k * r);
  L.UB = ar.take<double>(k * r);
  L.SB = ar.take<double>(r);
  L.VB = ar.take<double>(n * r);
  L.E1 = ar.take<double>(r * r);
  L.Zsc = ar.take<double>(n * r);
  L.E2T = ar.take<double>(n * r);
  L.Usc = ar.take<double>(m * r);
  const int l1 = limbs_for(P.bits[0]), l2 = limbs_for(P.bits[1]), l3 = limbs_for(P.bits[2]);
  L.vt = take_qop(ar, r, k, 1, l1);
  L.wq = take_qop(ar, r, k, 1, l1);
  L.e1q = take_qop(ar, r, r, 1, l2);
  L.zq = take_qop(ar, n, r, 1, l2);
  L.e2q = take_qop(ar, n, r, 1, l3);
  L.uq = take_qop(ar, m, r, 1, l3);
  if (l1 > 1 || l2 > 1 || l3 > 1) {
    const int64_t mx = std::max(std::max(m, n), k);
    L.tmp32 = ar.take<int32_t>(mx * round_up(std::max(k, r), 16));
  }
  {
    int64_t acc_elems = 0;
    if (l1 > 1 || needs_acc64(k, P.bits[0])) acc_elems = std::max(acc_elems, r * r);
    if (l2 > 1 || needs_acc64(r, P.bits[1])) acc_elems = std::max(acc_elems, r * n);
    if (l3 > 1 || needs_acc64(r, P.bits[2])) acc_elems = std::max(acc_elems, m * n);
    if (acc_elems) L.acc64 = ar.take<int64_t>(acc_elems);
  }
  L.e1acc = ar.take<int32_t>(r * r);
  L.nonfinite = ar.take<int>(4);
  L.jinfo = ar.take<int>(4);
  int64_t mx = std::max(std::max(m, n), k);
  L.qbytes = quantize_ws_bytes(mx, mx);
  L.qws = ar.take<char>((int64_t)L.qbytes);
  return L;
}

__global__ void gather_info_kernel(const int *a, const int *b, const int *ca, const int *cb, const int *nfa,
                                   const int *nfb, int *jinfo, int *nonfinite) {
  if (threadIdx.x) return;
  jinfo[0] = a[0];
  jinfo[1] = b[0];
  jinfo[2] = ca[0] ? -1 : 0;
  jinfo[3] = cb[0] ? -1 : 0;
  if (nfa[0] || nfb[0]) nonfinite[0] = 1;
}

// side stream + fork/join events per caller stream (so independent lramm() calls issued on
// different streams -- e.g. the pairs of a batch -- do not serialise on a shared side stream)
struct SideStream {
  cudaStream_t st = nullptr;
  cudaEvent_t fork = nullptr, join = nullptr;
};
SideStream &side_stream(cudaStream_t main) {
  static std::mutex mu;
  static std::map<std::pair<int, cudaStream_t>, SideStream> table;
  int dev = 0;
  cudaGetDevice(&dev);
  std::lock_guard<std::mutex> g(mu);
  SideStream &x = table[{dev, main}];
  if (!x.st) {
    cudaStreamCreateWithFlags(&x.st, cudaStreamNonBlocking);
    cudaEventCreateWithFlags(&x.fork, cudaEventDisableTiming);
    cudaEventCreateWithFlags(&x.join, cudaEventDisableTiming);
  }
  return x;
}

}  // namespace

size_t rsvd_ws_bytes(int64_t rows, int64_t cols, const lramm_params_t &P, int x_dtype) {
  Arena ar;
  ar.dry = true;
  carve_rsvd(ar, rows, cols, x_dtype, P);
  return ar.off + 1024;
}

int rsvd_device(const void *x, int x_dtype, int64_t rows, int64_t cols, const lramm_params_t &P, const double *omega,
                double *U, double *S, double *V, int *status, void *ws, size_t ws_bytes, cudaStream_t st) {
  LRAMM_TRY(validate_params(P, false));
  if (x_dtype != LRAMM_F32 && x_dtype != LRAMM_F64) return fail(LRAMM_ERR_PARAM, "rsvd: x must be F32 or F64");
  if (rows < 1 || cols < 1) return fail(LRAMM_ERR_SHAPE, "rsvd: empty matrix");
  if (P.rank > std::min(rows, cols))
    return fail(LRAMM_ERR_PARAM, "rank %d exceeds min dim %lld", P.rank, (long long)std::min(rows, cols));
  Arena ar(ws, ws_bytes);
  RsvdBufs b = carve_rsvd(ar, rows, cols, x_dtype, P);
  if (!ar.ok()) return fail(LRAMM_ERR_WORKSPACE, "rsvd: workspace too small (%zu needed)", ar.off);
  if (b.fast) {
    LRAMM_TRY(check_acc(cols, P.sketch_bits, P.sketch_bits));
    LRAMM_TRY(check_acc(rows, P.proj_bits, P.proj_bits));
    if (P.power_iters > 0) LRAMM_TRY(check_acc(std::max(rows, cols), P.power_bits, P.power_bits));
  }
  LRAMM_TRY(run_rsvd(x, x_dtype, b, P, omega, U, P.rank, S, V, P.rank, st));
  summarize_status_kernel<<<1, 32, 0, st>>>(b.info, 1, b.nonfinite, b.compl_st, status);
  LRAMM_LAUNCH_CHECK();
  return LRAMM_OK;
}

size_t lramm_ws_bytes(int64_t m, int64_t k, int64_t n, const lramm_params_t &P, int in_dtype) {
  Arena ar;
  ar.dry = true;
  carve_lramm(ar, m, k, n, in_dtype, P);
  return ar.off + 1024;
}

int lramm_device(const void *a, const void *b, int in_dtype, int64_t m, int64_t k, int64_t n, const lramm_params_t &P,
                 const double *omega_a, const double *omega_b, const void *c, int c_dtype, void *d, int d_dtype,
                 int *status, void *ws, size_t ws_bytes, lramm_timings_t *timings, cudaStream_t st,
                 cudaEvent_t b_ready, cudaEvent_t *stage_events) {
  LRAMM_TRY(validate_params(P, true));
  if (P.rank < 2) return fail(LRAMM_ERR_PARAM, "rank must be >= 2, got %d", P.rank);
  if (in_dtype != LRAMM_F32 && in_dtype != LRAMM_F64) return fail(LRAMM_ERR_PARAM, "inputs must be F32 or F64");
  if (d_dtype != LRAMM_F32 && d_dtype != LRAMM_F64) return fail(LRAMM_ERR_PARAM, "output must be F32 or F64");
  if (m < 1 || k < 1 || n < 1) return fail(LRAMM_ERR_SHAPE, "empty operand");
  if (P.rank > std::min(m, k) || P.rank > std::min(k, n))
    return fail(LRAMM_ERR_PARAM, "rank %d exceeds operand min dims %lld, %lld", P.rank, (long long)std::min(m, k),
                (long long)std::min(k, n));
  const int64_t r = P.rank;
  const int d1 = P.bits[0], d2 = P.bits[1], d3 = P.bits[2];
  LRAMM_TRY(check_acc_qm(k, d1));
  LRAMM_TRY(check_acc_qm(r, d2));
  LRAMM_TRY(check_acc_qm(r, d3));
  if (P.mode == LRAMM_MODE_FAST) {
    int64_t mx = std::max(std::max(m, n), k);
    LRAMM_TRY(check_acc(mx, P.sketch_bits, P.sketch_bits));
    LRAMM_TRY(check_acc(mx, P.proj_bits, P.proj_bits));
    if (P.power_iters > 0) LRAMM_TRY(check_acc(mx, P.power_bits, P.power_bits));
  }
  Arena ar(ws, ws_bytes);
  LrammBufs L = carve_lramm(ar, m, k, n, in_dtype, P);
  if (!ar.ok()) return fail(LRAMM_ERR_WORKSPACE, "lramm: workspace too small (%zu needed)", ar.off);

  // stage_events (6 caller-owned timing events): the stage boundaries are recorded into them and
  // the caller reads the times after its own synchronisation (the host entry point enqueues the
  // download of D first); otherwise timings != NULL synchronises here
  cudaEvent_t ev[6] = {};
  if (stage_events)
    for (int i = 0; i < 6; ++i) ev[i] = stage_events[i];
  else if (timings)
    for (int i = 0; i < 6; ++i) LRAMM_CUDA_TRY(cudaEventCreate(&ev[i]));
  NvtxStages nv;
  static const char *const kStage[6] = {"lramm.rsvd", "lramm.scaling", "lramm.gemm1", "lramm.gemm2", "lramm.gemm3",
                                        nullptr};
  auto mark = [&](int i) -> int {
    nv.next(kStage[i]);
    if (timings || stage_events) LRAMM_CUDA_TRY(cudaEventRecord(ev[i], st));
    return LRAMM_OK;
  };
  LRAMM_TRY(mark(0));
  // ---- rsvd of both operands (pipeline.py:183-186): independent chains, so B runs on a
  // forked side stream (event fork/join; capturable into a CUDA graph)
  SideStream &side = side_stream(st);
  LRAMM_CUDA_TRY(cudaEventRecord(side.fork, st));
  LRAMM_CUDA_TRY(cudaStreamWaitEvent(side.st, side.fork, 0));
  if (b_ready) LRAMM_CUDA_TRY(cudaStreamWaitEvent(side.st, b_ready, 0));  // B (and C) uploaded on another stream
  LRAMM_TRY(run_rsvd(b, in_dtype, L.rb, P, omega_b, L.UB, r, L.SB, L.VB, r, side.st));
  LRAMM_TRY(run_rsvd(a, in_dtype, L.ra, P, omega_a, L.UA, r, L.SA, L.VA, r, st));
  LRAMM_CUDA_TRY(cudaEventRecord(side.join, side.st));
  LRAMM_CUDA_TRY(cudaStreamWaitEvent(st, side.join, 0));
  LRAMM_TRY(mark(1));
  // ---- scaling (pipeline.py:188-193): Usc = U_A sigma_A, Zsc^T = V_B sigma_B
  scale_cols_kernel<<<elem_grid(m * r), 256, 0, st>>>(L.UA, m, (int)r, r, L.SA, L.Usc, r);
  LRAMM_LAUNCH_CHECK();
  scale_cols_kernel<<<elem_grid(n * r), 256, 0, st>>>(L.VB, n, (int)r, r, L.SB, L.Zsc, r);
  LRAMM_LAUNCH_CHECK();
  LRAMM_TRY(mark(2));
  LRAMM_CUDA_TRY(cudaMemsetAsync(L.nonfinite, 0, 4 * sizeof(int), st));
  // ---- E1 = QM(V_A^T U_B, d1)   (r x r, K = k)
  LRAMM_TRY(quant(L.VA, LRAMM_F64, k, r, r, d1, LRAMM_GRAN_TENSOR, 1, L.vt, L.nonfinite, L.qws, L.qbytes, st, L.tmp32));
  LRAMM_TRY(quant(L.UB, LRAMM_F64, k, r, r, d1, LRAMM_GRAN_TENSOR, 1, L.wq, L.nonfinite, L.qws, L.qbytes, st, L.tmp32));
  LRAMM_TRY(qprod(L.vt, L.wq, r, r, k, L.E1, r, 0, L.e1acc, st, L.acc64, needs_acc64(k, d1)));
  LRAMM_TRY(mark(3));
  // ---- E2 = QM(E1 Zsc, d2)   (r x n, K = r) stored transposed for E3
  LRAMM_TRY(quant(L.E1, LRAMM_F64, r, r, r, d2, LRAMM_GRAN_TENSOR, 0, L.e1q, L.nonfinite, L.qws, L.qbytes, st, L.tmp32));
  LRAMM_TRY(quant(L.Zsc, LRAMM_F64, n, r, r, d2, LRAMM_GRAN_TENSOR, 0, L.zq, L.nonfinite, L.qws, L.qbytes, st, L.tmp32));
  LRAMM_TRY(qprod(L.e1q, L.zq, r, n, r, L.E2T, r, 1, nullptr, st, L.acc64, needs_acc64(r, d2)));
  LRAMM_TRY(mark(4));
  // ---- E3 = QM(Usc E2, d3) ; D = alpha E3 + beta C   (m x n, K = r)
  LRAMM_TRY(quant(L.Usc, LRAMM_F64, m, r, r, d3, LRAMM_GRAN_TENSOR, 0, L.uq, L.nonfinite, L.qws, L.qbytes, st, L.tmp32));
  LRAMM_TRY(quant(L.E2T, LRAMM_F64, n, r, r, d3, LRAMM_GRAN_TENSOR, 0, L.e2q, L.nonfinite, L.qws, L.qbytes, st, L.tmp32));
  {
    lramm_epilogue_t e = {};
    e.out_dtype = d_dtype;
    e.out = d;
    e.ldo = n;
    e.row_scale = L.uq.scale;
    e.row_scale_inc = 0;
    e.col_scale = L.e2q.scale;
    e.col_scale_inc = 0;
    e.alpha = P.alpha;
    e.beta = c ? P.beta : 0.0;
    e.c = c;
    e.c_dtype = c_dtype;
    e.ldc = n;
    if (L.uq.limbs > 1 || needs_acc64(r, d3))
      LRAMM_TRY(igemm_limbs_device(m, n, r, L.uq.q, L.uq.ld, L.uq.plane, L.uq.limbs, L.e2q.q, L.e2q.ld, L.e2q.plane,
                                   L.e2q.limbs, L.acc64, e, st));
    else
      LRAMM_TRY(igemm_device(m, n, r, L.uq.q, L.uq.ld, L.e2q.q, L.e2q.ld, e, 1, st));
  }
  LRAMM_TRY(mark(5));
  gather_info_kernel<<<1, 32, 0, st>>>(L.ra.info, L.rb.info, L.ra.compl_st, L.rb.compl_st, L.ra.nonfinite,
                                       L.rb.nonfinite, L.jinfo, L.nonfinite);
  LRAMM_LAUNCH_CHECK();
  summarize_status_kernel<<<1, 32, 0, st>>>(L.jinfo, 4, L.nonfinite, nullptr, status);
  LRAMM_LAUNCH_CHECK();
  if (timings && !stage_events) {
    LRAMM_CUDA_TRY(cudaEventSynchronize(ev[5]));
    float t[5];
    for (int i = 0; i < 5; ++i) LRAMM_CUDA_TRY(cudaEventElapsedTime(&t[i], ev[i], ev[i + 1]));
    timings->rsvd_ms = t[0];
    timings->scaling_ms = t[1];
    timings->gemm1_ms = t[2];
    timings->gemm2_ms = t[3];
    timings->gemm3_ms = t[4];
    for (int i = 0; i < 6; ++i) cudaEventDestroy(ev[i]);
  }
  return LRAMM_OK;
}

// ------------------------------------------------------------------ sharded pipeline (multi-GPU)
namespace {

void shard_bounds(int64_t total, int world, int rank, int64_t &lo, int64_t &hi) {
  const int64_t base = total / world, extra = total % world;
  lo = rank * base + std::min<int64_t>(rank, extra);
  hi = lo + base + (rank < extra ? 1 : 0);
}

struct ShardedBufs {
  RsvdBufs ra, rb;
  double *UA, *SA, *VA, *UB, *SB, *VB, *E1, *Zsc, *E2T, *Usc;
  QOp vt, wq, e1q, zq, e2q, uq;
  int8_t *gath = nullptr, *e2all = nullptr;  // allgathered int8 E2 rows (padded per rank) / compacted
  int64_t n_pad = 0;
  int32_t *acc;
  int *nonfinite, *st_loc;
  void *qws;
  size_t qbytes;
};

ShardedBufs carve_sharded(Arena &ar, int64_t ml, int64_t k, int64_t nl, int64_t m, int64_t n, int in_dtype,
                          const lramm_params_t &P, int world) {
  ShardedBufs L;
  const int64_t r = P.rank;
  const int64_t wa = std::min<int64_t>(P.rank + P.oversample, std::min(m, k));
  const int64_t wb = std::min<int64_t>(P.rank + P.oversample, std::min(k, n));
  L.ra = carve_rsvd(ar, ml, k, in_dtype, P, wa);
  L.rb = carve_rsvd(ar, k, nl, in_dtype, P, wb);
  L.UA = ar.take<double>(ml * r);
  L.SA = ar.take<double>(r);
  L.VA = ar.take<double>(k * r);
  L.UB = ar.take<double>(k * r);
  L.SB = ar.take<double>(r);
  L.VB = ar.take<double>(nl * r);
  L.E1 = ar.take<double>(r * r);
  L.Zsc = ar.take<double>(nl * r);
  L.E2T = ar.take<double>(nl * r);
  L.Usc = ar.take<double>(ml * r);
  L.vt = take_qop(ar, r, k, 1);
  L.wq = take_qop(ar, r, k, 1);
  L.e1q = take_qop(ar, r, r, 1);
  L.zq = take_qop(ar, nl, r, 1);
  L.n_pad = ceil_div(n, world);
  L.e2q = take_qop(ar, L.n_pad, r, 1);  // this rank's rows, zero-padded to the largest shard
  L.uq = take_qop(ar, ml, r, 1);
  L.gath = ar.take<int8_t>((int64_t)world * L.n_pad * L.e2q.ld);
  L.e2all = ar.take<int8_t>(n * L.e2q.ld);
  L.acc = ar.take<int32_t>(std::max(r * r, r * nl));
  L.nonfinite = ar.take<int>(4);
  L.st_loc = ar.take<int>(4);
  const int64_t mx = std::max(std::max(ml, nl), std::max(k, r));
  L.qbytes = quantize_ws_bytes(mx, mx);
  L.qws = ar.take<char>((int64_t)L.qbytes);
  return L;
}

// this rank's status: a Jacobi non-convergence, a non-finite input, or a chain's own code
// (LRAMM_ERR_UNSUPPORTED for a sketch without a sharded fallback)
__global__ void sharded_status_kernel(const int *ia, const int *ib, const int *ca, const int *cb, const int *nfa,
                                      const int *nfb, const int *nf, int *status) {
  if (threadIdx.x) return;
  int s = 0;
  if (ia[0] < 0 || ib[0] < 0) s = LRAMM_ERR_NONCONVERGENCE;
  if (!s && ca[0]) s = ca[0];
  if (!s && cb[0]) s = cb[0];
  if (nfa[0] || nfb[0] || nf[0]) s = LRAMM_ERR_NONFINITE;
  *status = s;
}

}  // namespace

size_t lramm_sharded_ws_bytes(int64_t m, int64_t k, int64_t n, const lramm_params_t &P, int in_dtype, int world,
                              int rank) {
  if (world < 1 || rank < 0 || rank >= world) return 0;
  int64_t m0, m1, n0, n1;
  shard_bounds(m, world, rank, m0, m1);
  shard_bounds(n, world, rank, n0, n1);
  Arena ar;
  ar.dry = true;
  carve_sharded(ar, std::max<int64_t>(m1 - m0, 1), k, std::max<int64_t>(n1 - n0, 1), m, n, in_dtype, P, world);
  return ar.off + 1024;
}

void shard_bounds_host(int64_t total, int world, int rank, int64_t *lo, int64_t *hi) {
  int64_t a = 0, b = 0;
  if (world >= 1 && rank >= 0 && rank < world) shard_bounds(total, world, rank, a, b);
  if (lo) *lo = a;
  if (hi) *hi = b;
}

int lramm_sharded_device(const void *a_rows, const void *b_cols, int in_dtype, int64_t m, int64_t k, int64_t n,
                         const lramm_params_t &P, const double *omega_a, const double *omega_b, const void *c_rows,
                         int c_dtype, void *d_rows, int d_dtype, int *status, void *ws, size_t ws_bytes,
                         const lramm_comm_t *comm, cudaStream_t st) {
  LRAMM_TRY(validate_params(P, true));
  if (!comm || comm->world < 1 || comm->rank < 0 || comm->rank >= comm->world)
    return fail(LRAMM_ERR_PARAM, "lramm_sharded: bad communicator (rank / world)");
  const int world = comm->world, rank = comm->rank;
  const bool live = world > 1 || (comm->flags & LRAMM_COMM_FORCE);
  if (live && (!comm->all_reduce || !comm->all_gather))
    return fail(LRAMM_ERR_PARAM, "lramm_sharded: the communicator has no all_reduce / all_gather entry point");
  if (P.rank < 2) return fail(LRAMM_ERR_PARAM, "rank must be >= 2, got %d", P.rank);
  if (in_dtype != LRAMM_F32 && in_dtype != LRAMM_F64) return fail(LRAMM_ERR_PARAM, "inputs must be F32 or F64");
  if (d_dtype != LRAMM_F32 && d_dtype != LRAMM_F64) return fail(LRAMM_ERR_PARAM, "output must be F32 or F64");
  if (m < 1 || k < 1 || n < 1) return fail(LRAMM_ERR_SHAPE, "empty operand");
  if (P.rank > std::min(m, k) || P.rank > std::min(k, n))
    return fail(LRAMM_ERR_PARAM, "rank %d exceeds operand min dims %lld, %lld", P.rank, (long long)std::min(m, k),
                (long long)std::min(k, n));
  if (m < world || n < world)
    return fail(LRAMM_ERR_SHAPE, "lramm_sharded: every rank needs at least one row of A and one column of B");
  const int64_t r = P.rank;
  const int d1 = P.bits[0], d2 = P.bits[1], d3 = P.bits[2];
  if (std::max(d1, std::max(d2, d3)) > 8)
    return fail(LRAMM_ERR_UNSUPPORTED, "the sharded path carries int8 operands: recombination bit budgets must be <= 8");
  // int32 accumulators are summed across the ranks: guard with the GLOBAL contraction lengths
  LRAMM_TRY(check_acc(k, d1, d1));
  LRAMM_TRY(check_acc(r, d2, d2));
  LRAMM_TRY(check_acc(r, d3, d3));
  if (P.mode == LRAMM_MODE_FAST) {
    const int64_t mx = std::max(std::max(m, n), k);
    LRAMM_TRY(check_acc(mx, P.sketch_bits, P.sketch_bits));
    LRAMM_TRY(check_acc(mx, P.proj_bits, P.proj_bits));
    if (P.power_iters > 0) LRAMM_TRY(check_acc(mx, P.power_bits, P.power_bits));
  }
  int64_t m0, m1, n0, n1;
  shard_bounds(m, world, rank, m0, m1);
  shard_bounds(n, world, rank, n0, n1);
  const int64_t ml = m1 - m0, nl = n1 - n0;
  Arena ar(ws, ws_bytes);
  ShardedBufs L = carve_sharded(ar, ml, k, nl, m, n, in_dtype, P, world);
  if (!ar.ok()) return fail(LRAMM_ERR_WORKSPACE, "lramm_sharded: workspace too small (%zu needed)", ar.off);

  ShardSpec sa, sb;
  sa.coll = Coll{comm, comm->comm};
  sa.kind = 1;
  sa.g_rows = m;
  sa.g_cols = k;
  sb.coll = Coll{comm, comm->comm_b ? comm->comm_b : comm->comm};
  sb.kind = 2;
  sb.g_rows = k;
  sb.g_cols = n;
  const Coll &coll = sa.coll;
  const double *omega_bj = omega_b + n0 * L.rb.w;  // the rows of Omega_B that meet this rank's columns
  // ---- rsvd of both operands: concurrent chains unless they would share one live communicator
  const bool fork = !live || comm->comm_b != nullptr;
  if (fork) {
    SideStream &side = side_stream(st);
    LRAMM_CUDA_TRY(cudaEventRecord(side.fork, st));
    LRAMM_CUDA_TRY(cudaStreamWaitEvent(side.st, side.fork, 0));
    LRAMM_TRY(run_rsvd(b_cols, in_dtype, L.rb, P, omega_bj, L.UB, r, L.SB, L.VB, r, side.st, &sb));
    LRAMM_TRY(run_rsvd(a_rows, in_dtype, L.ra, P, omega_a, L.UA, r, L.SA, L.VA, r, st, &sa));
    LRAMM_CUDA_TRY(cudaEventRecord(side.join, side.st));
    LRAMM_CUDA_TRY(cudaStreamWaitEvent(st, side.join, 0));
  } else {
    LRAMM_TRY(run_rsvd(a_rows, in_dtype, L.ra, P, omega_a, L.UA, r, L.SA, L.VA, r, st, &sa));
    LRAMM_TRY(run_rsvd(b_cols, in_dtype, L.rb, P, omega_bj, L.UB, r, L.SB, L.VB, r, st, &sb));
  }
  // ---- scaling (pipeline.py:188-193) of the local rows: Usc = U_A sigma_A, Zsc^T = V_B sigma_B
  scale_cols_kernel<<<elem_grid(ml * r), 256, 0, st>>>(L.UA, ml, (int)r, r, L.SA, L.Usc, r);
  LRAMM_LAUNCH_CHECK();
  scale_cols_kernel<<<elem_grid(nl * r), 256, 0, st>>>(L.VB, nl, (int)r, r, L.SB, L.Zsc, r);
  LRAMM_LAUNCH_CHECK();
  LRAMM_CUDA_TRY(cudaMemsetAsync(L.nonfinite, 0, 4 * sizeof(int), st));
  const AmaxSync global_t{&coll, true, false, false};  // per-tensor scale of a sharded matrix
  // ---- E1 = QM(V_A^T U_B, d1): both operands replicated, computed on every rank (r x r, K = k)
  LRAMM_TRY(quant(L.VA, LRAMM_F64, k, r, r, d1, LRAMM_GRAN_TENSOR, 1, L.vt, L.nonfinite, L.qws, L.qbytes, st));
  LRAMM_TRY(quant(L.UB, LRAMM_F64, k, r, r, d1, LRAMM_GRAN_TENSOR, 1, L.wq, L.nonfinite, L.qws, L.qbytes, st));
  LRAMM_TRY(qprod(L.vt, L.wq, r, r, k, L.E1, r, 0, L.acc, st));
  // ---- E2 = QM(E1 Zsc, d2): the local rows of E2^T (n_j x r, K = r), Zsc's scale made global
  LRAMM_TRY(quant(L.E1, LRAMM_F64, r, r, r, d2, LRAMM_GRAN_TENSOR, 0, L.e1q, L.nonfinite, L.qws, L.qbytes, st));
  LRAMM_TRY(quant(L.Zsc, LRAMM_F64, nl, r, r, d2, LRAMM_GRAN_TENSOR, 0, L.zq, L.nonfinite, L.qws, L.qbytes, st, nullptr,
                  &global_t));
  LRAMM_TRY(qprod(L.e1q, L.zq, r, nl, r, L.E2T, r, 1, nullptr, st));
  // ---- E3 = QM(Usc E2, d3); D rows = alpha E3 + beta C rows (m_i x n, K = r): E2's int8 rows are
  // allgathered (rank j's rows at j * n_pad), then compacted when the shards are ragged
  LRAMM_TRY(quant(L.Usc, LRAMM_F64, ml, r, r, d3, LRAMM_GRAN_TENSOR, 0, L.uq, L.nonfinite, L.qws, L.qbytes, st, nullptr,
                  &global_t));
  if (coll.on() && nl < L.n_pad)
    LRAMM_CUDA_TRY(cudaMemsetAsync(L.e2q.q + nl * L.e2q.ld, 0, (size_t)((L.n_pad - nl) * L.e2q.ld), st));
  LRAMM_TRY(quant(L.E2T, LRAMM_F64, nl, r, r, d3, LRAMM_GRAN_TENSOR, 0, L.e2q, L.nonfinite, L.qws, L.qbytes, st, nullptr,
                  &global_t));
  const int8_t *e2 = L.e2q.q;
  if (coll.on()) {
    LRAMM_TRY(coll.gather_i8(L.e2q.q, L.gath, (size_t)(L.n_pad * L.e2q.ld), st));
    if (n % world == 0) {
      e2 = L.gath;
    } else {
      for (int j = 0; j < world; ++j) {
        int64_t lo, hi;
        shard_bounds(n, world, j, lo, hi);
        LRAMM_CUDA_TRY(cudaMemcpyAsync(L.e2all + lo * L.e2q.ld, L.gath + (int64_t)j * L.n_pad * L.e2q.ld,
                                       (size_t)((hi - lo) * L.e2q.ld), cudaMemcpyDeviceToDevice, st));
      }
      e2 = L.e2all;
    }
  }
  {
    lramm_epilogue_t e = {};
    e.out_dtype = d_dtype;
    e.out = d_rows;
    e.ldo = n;
    e.row_scale = L.uq.scale;
    e.row_scale_inc = 0;
    e.col_scale = L.e2q.scale;
    e.col_scale_inc = 0;
    e.alpha = P.alpha;
    e.beta = c_rows ? P.beta : 0.0;
    e.c = c_rows;
    e.c_dtype = c_dtype;
    e.ldc = n;
    LRAMM_TRY(igemm_device(ml, n, r, L.uq.q, L.uq.ld, e2, L.e2q.ld, e, 1, st));
  }
  sharded_status_kernel<<<1, 32, 0, st>>>(L.ra.info, L.rb.info, L.ra.compl_st, L.rb.compl_st, L.ra.nonfinite,
                                          L.rb.nonfinite, L.nonfinite, status);
  LRAMM_LAUNCH_CHECK();
  return coll.max_i32(status, 1, st);  // every rank reports the same status
}

}  // namespace lramm
