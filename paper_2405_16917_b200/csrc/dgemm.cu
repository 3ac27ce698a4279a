// fp64 GEMMs for the fp64-faithful parts of the path: Gram
// matrices, triangular multiplies, the lift U = Q.u, and (parity mode) the
// sketch / power / projection products of the reference (rsvd.py:57-77).
//
// 64x64 output tile per 256-thread CTA, 4x4 outputs per thread (strided so a
// warp's shared-memory reads are conflict-free), K staged 16 at a time through
// double-buffered shared memory.  trans_a = 1 evaluates A^T.B for tall row-major
// operands (A: K x M) with split-K over the long dimension and a fixed-order
// reduction, so results are bitwise reproducible run to run.
#include <algorithm>

#include "common.cuh"

namespace lramm {
namespace {

constexpr int TM = 64, TN = 64, TK = 16;

template <bool TRANS_A>
__global__ void __launch_bounds__(256) dgemm_kernel(int64_t M, int64_t N, int64_t K, const double *__restrict__ A,
                                                    int64_t lda, const double *__restrict__ B, int64_t ldb,
                                                    double *__restrict__ C, int64_t ldc, int64_t k_per_split,
                                                    int64_t split_stride) {
  __shared__ double As[2][TK][TM + 1];
  __shared__ double Bs[2][TK][TN + 1];
  const int tid = threadIdx.x;
  const int tx = tid & 15, ty = tid >> 4;
  const int64_t m0 = (int64_t)blockIdx.x * TM, n0 = (int64_t)blockIdx.y * TN;
  const int64_t kbeg = (int64_t)blockIdx.z * k_per_split;
  const int64_t kend = min(K, kbeg + k_per_split);
  double acc[4][4];
#pragma unroll
  for (int i = 0; i < 4; ++i)
#pragma unroll
    for (int j = 0; j < 4; ++j) acc[i][j] = 0.0;

  double ra[4], rb[4];
  auto load_regs = [&](int64_t k0) {
#pragma unroll
    for (int l = 0; l < 4; ++l) {
      int e = tid + l * 256;  // 0..1023 = TK x 64
      int kk, mm;
      if (TRANS_A) {  // A is K x M: coalesced along m
        kk = e >> 6;
        mm = e & 63;
        int64_t gk = k0 + kk, gm = m0 + mm;
        ra[l] = (gk < kend && gm < M) ? A[gk * lda + gm] : 0.0;
      } else {  // A is M x K: 16 consecutive k per row
        mm = e >> 4;
        kk = e & 15;
        int64_t gk = k0 + kk, gm = m0 + mm;
        ra[l] = (gk < kend && gm < M) ? A[gm * lda + gk] : 0.0;
      }
      int bk = e >> 6, bn = e & 63;
      int64_t gk = k0 + bk, gn = n0 + bn;
      rb[l] = (gk < kend && gn < N) ? B[gk * ldb + gn] : 0.0;
    }
  };
  auto store_regs = [&](int buf) {
#pragma unroll
    for (int l = 0; l < 4; ++l) {
      int e = tid + l * 256;
      if (TRANS_A)
        As[buf][e >> 6][e & 63] = ra[l];
      else
        As[buf][e & 15][e >> 4] = ra[l];
      Bs[buf][e >> 6][e & 63] = rb[l];
    }
  };

  int buf = 0;
  if (kbeg < kend) {
    load_regs(kbeg);
    store_regs(0);
  }
  __syncthreads();
  for (int64_t k0 = kbeg; k0 < kend; k0 += TK) {
    const bool more = k0 + TK < kend;
    if (more) load_regs(k0 + TK);
#pragma unroll
    for (int kk = 0; kk < TK; ++kk) {
      double a[4], b[4];
#pragma unroll
      for (int i = 0; i < 4; ++i) a[i] = As[buf][kk][ty + 16 * i];
#pragma unroll
      for (int j = 0; j < 4; ++j) b[j] = Bs[buf][kk][tx + 16 * j];
#pragma unroll
      for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j) acc[i][j] = fma(a[i], b[j], acc[i][j]);
    }
    if (more) {
      store_regs(buf ^ 1);
      __syncthreads();
      buf ^= 1;
    }
  }
  double *Cz = C + (int64_t)blockIdx.z * split_stride;
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    int64_t r = m0 + ty + 16 * i;
    if (r >= M) continue;
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      int64_t c = n0 + tx + 16 * j;
      if (c < N) Cz[r * ldc + c] = acc[i][j];
    }
  }
}

// C = sum_z parts[z] in fixed order (deterministic)
__global__ void splitk_reduce_kernel(const double *__restrict__ parts, int splits, int64_t M, int64_t N,
                                     double *__restrict__ C, int64_t ldc) {
  int64_t n = M * N;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    double s = 0.0;
    for (int z = 0; z < splits; ++z) s += parts[z * n + i];
    int64_t r = i / N, c = i - r * N;
    C[r * ldc + c] = s;
  }
}

int choose_splits(int trans_a, int64_t M, int64_t N, int64_t K) {
  if (!trans_a) return 1;
  int64_t tiles = ceil_div(M, TM) * ceil_div(N, TN);
  int64_t want = ceil_div(2LL * num_sms(), tiles);
  int64_t max_by_k = std::max<int64_t>(1, K / 256);
  return (int)std::max<int64_t>(1, std::min<int64_t>(want, std::min<int64_t>(max_by_k, 64)));
}

}  // namespace

size_t dgemm_ws_bytes(int trans_a, int64_t M, int64_t N, int64_t K) {
  int s = choose_splits(trans_a, M, N, K);
  return s > 1 ? (size_t)round_up(s * M * N * 8, 256) : 0;
}

int dgemm_device(int trans_a, int64_t M, int64_t N, int64_t K, const double *A, int64_t lda, const double *B,
                 int64_t ldb, double *C, int64_t ldc, void *ws, size_t ws_bytes, cudaStream_t st) {
  if (M < 1 || N < 1 || K < 1) return fail(LRAMM_ERR_SHAPE, "dgemm: empty shape");
  int splits = choose_splits(trans_a, M, N, K);
  if (splits > 1 && (ws == nullptr || ws_bytes < dgemm_ws_bytes(trans_a, M, N, K))) splits = 1;
  int64_t kps = round_up(ceil_div(K, splits), TK);
  splits = (int)ceil_div(K, kps);
  dim3 grid((unsigned)ceil_div(M, TM), (unsigned)ceil_div(N, TN), (unsigned)splits);
  double *out = splits > 1 ? (double *)ws : C;
  int64_t ldo = splits > 1 ? N : ldc;
  if (trans_a)
    dgemm_kernel<true><<<grid, 256, 0, st>>>(M, N, K, A, lda, B, ldb, out, ldo, kps, M * N);
  else
    dgemm_kernel<false><<<grid, 256, 0, st>>>(M, N, K, A, lda, B, ldb, out, ldo, kps, M * N);
  LRAMM_LAUNCH_CHECK();
  if (splits > 1) {
    int g = (int)std::min<int64_t>(ceil_div(M * N, 256), 8LL * num_sms());
    splitk_reduce_kernel<<<g, 256, 0, st>>>((const double *)ws, splits, M, N, C, ldc);
    LRAMM_LAUNCH_CHECK();
  }
  return LRAMM_OK;
}

}  // namespace lramm
