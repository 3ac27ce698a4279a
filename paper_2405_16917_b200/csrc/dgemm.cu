// fp64 GEMMs for the fp64-faithful parts of the path: Gram
// matrices, triangular multiplies, the lift U = Q.u, and (parity mode) the
// sketch / power / projection products of the reference (rsvd.py:57-77).
//
// FP64 tensor pipe (mma.sync.m8n8k4.f64, "DMMA": same 37 TFLOP/s peak as DFMA on
// B200 but 8x fewer issued instructions).  64 x 64 CTA tile, 8 warps each owning
// a 32 x 16 sub-tile (4 x 2 DMMA tiles), K staged 32 at a time through double-
// buffered shared memory with cp.async.  trans_a = 1 evaluates A^T.B for tall
// row-major operands (A: K x M) with split-K over the long dimension and a
// fixed-order reduction, so results are bitwise reproducible run to run.
#include <algorithm>
#include <mutex>

#include "common.cuh"
#include "sm100.cuh"

namespace lramm {
namespace {

constexpr int TM = 64, TN = 64, TK = 32;
constexpr int LDA = TK + 4;  // As[m][k] (NN) row stride
constexpr int LDT = TM + 4;  // As[k][m] (TN) and Bs[k][n] row stride

__device__ __forceinline__ void dmma(double (&d)[2], double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
               : "+d"(d[0]), "+d"(d[1])
               : "d"(a), "d"(b));
}

template <bool TRANS_A>
__global__ void __launch_bounds__(256) dgemm_kernel(int64_t M, int64_t N, int64_t K, const double *__restrict__ A,
                                                    int64_t lda, const double *__restrict__ B, int64_t ldb,
                                                    double *__restrict__ C, int64_t ldc, int64_t k_per_split,
                                                    int64_t split_stride) {
  constexpr int ASZ = TRANS_A ? TK * LDT : TM * LDA;
  extern __shared__ __align__(16) double dg_smem[];
  double(*As)[ASZ] = reinterpret_cast<double(*)[ASZ]>(dg_smem);
  double(*Bs)[TK * LDT] = reinterpret_cast<double(*)[TK * LDT]>(dg_smem + 2 * ASZ);
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int g = lane >> 2, t4 = lane & 3;
  const int wm = warp >> 2, wn = warp & 3;  // warp tile: rows wm*32.., cols wn*16..
  const int64_t m0 = (int64_t)blockIdx.x * TM, n0 = (int64_t)blockIdx.y * TN;
  const int64_t kbeg = (int64_t)blockIdx.z * k_per_split;
  const int64_t kend = min(K, kbeg + k_per_split);
  double acc[4][2][2];
#pragma unroll
  for (int i = 0; i < 4; ++i)
#pragma unroll
    for (int j = 0; j < 2; ++j) acc[i][j][0] = acc[i][j][1] = 0.0;

  auto stage = [&](int buf, int64_t k0) {
    // A
    if (TRANS_A) {  // A is K x M: rows k, contiguous m
      for (int e = tid; e < TK * TM; e += 256) {
        const int kk = e >> 6, mm = e & 63;
        const int64_t gk = k0 + kk, gm = m0 + mm;
        const bool v = gk < kend && gm < M;
        sm100::cp_async8(&As[buf][kk * LDT + mm], A + (v ? gk * lda + gm : 0), v);
      }
    } else {  // A is M x K: rows m, contiguous k
      for (int e = tid; e < TM * TK; e += 256) {
        const int mm = e >> 5, kk = e & 31;
        const int64_t gk = k0 + kk, gm = m0 + mm;
        const bool v = gk < kend && gm < M;
        sm100::cp_async8(&As[buf][mm * LDA + kk], A + (v ? gm * lda + gk : 0), v);
      }
    }
    for (int e = tid; e < TK * TN; e += 256) {
      const int kk = e >> 6, nn = e & 63;
      const int64_t gk = k0 + kk, gn = n0 + nn;
      const bool v = gk < kend && gn < N;
      sm100::cp_async8(&Bs[buf][kk * LDT + nn], B + (v ? gk * ldb + gn : 0), v);
    }
    asm volatile("cp.async.commit_group;" ::: "memory");
  };

  int buf = 0;
  if (kbeg < kend) stage(0, kbeg);
  for (int64_t k0 = kbeg; k0 < kend; k0 += TK) {
    const bool more = k0 + TK < kend;
    if (more) {
      stage(buf ^ 1, k0 + TK);
      asm volatile("cp.async.wait_group 1;" ::: "memory");
    } else {
      asm volatile("cp.async.wait_group 0;" ::: "memory");
    }
    __syncthreads();
    const double *as = As[buf];
    const double *bs = Bs[buf];
#pragma unroll
    for (int kk = 0; kk < TK; kk += 4) {
      double a[4], b[2];
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        const int m = wm * 32 + i * 8 + g;
        a[i] = TRANS_A ? as[(kk + t4) * LDT + m] : as[m * LDA + kk + t4];
      }
#pragma unroll
      for (int j = 0; j < 2; ++j) b[j] = bs[(kk + t4) * LDT + wn * 16 + j * 8 + g];
#pragma unroll
      for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < 2; ++j) dmma(acc[i][j], a[i], b[j]);
    }
    __syncthreads();
    buf ^= 1;
  }
  double *Cz = C + (int64_t)blockIdx.z * split_stride;
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    const int64_t r = m0 + wm * 32 + i * 8 + g;
    if (r >= M) continue;
#pragma unroll
    for (int j = 0; j < 2; ++j)
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        const int64_t c = n0 + wn * 16 + j * 8 + 2 * t4 + h;
        if (c < N) Cz[r * ldc + c] = acc[i][j][h];
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
  int64_t tiles = ceil_div(M, TM) * ceil_div(N, TN);
  int64_t want = ceil_div(2LL * num_sms(), tiles);
  int64_t max_by_k = std::max<int64_t>(1, K / 256);
  int64_t s = std::max<int64_t>(1, std::min<int64_t>(want, std::min<int64_t>(max_by_k, 64)));
  return (int)s;
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
  static std::once_flag once;
  cudaError_t e = cudaSuccess;
  std::call_once(once, [&] {
    e = allow_max_dyn_smem(dgemm_kernel<true>);
    if (e == cudaSuccess) e = allow_max_dyn_smem(dgemm_kernel<false>);
  });
  LRAMM_CUDA_TRY(e);
  const size_t smem_t = (size_t)(2 * TK * LDT + 2 * TK * LDT) * 8, smem_n = (size_t)(2 * TM * LDA + 2 * TK * LDT) * 8;
  if (trans_a)
    dgemm_kernel<true><<<grid, 256, smem_t, st>>>(M, N, K, A, lda, B, ldb, out, ldo, kps, M * N);
  else
    dgemm_kernel<false><<<grid, 256, smem_n, st>>>(M, N, K, A, lda, B, ldb, out, ldo, kps, M * N);
  LRAMM_LAUNCH_CHECK();
  if (splits > 1) {
    int g = (int)std::min<int64_t>(ceil_div(M * N, 256), 8LL * num_sms());
    splitk_reduce_kernel<<<g, 256, 0, st>>>((const double *)ws, splits, M, N, C, ldc);
    LRAMM_LAUNCH_CHECK();
  }
  return LRAMM_OK;
}

}  // namespace lramm
