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

struct DgemmEpi {
  int sym;           // C symmetric (Gram A^T A): only tiles with tile_row <= tile_col, mirrored
  int b_upper;       // B upper triangular: the k loop of output tile n0 stops at n0 + TN
  double alpha, beta;
  const double *cin;  // C = alpha A.B + beta cin (cin may alias nothing written by this GEMM)
  int64_t ldci;
  const int *gate;   // non-null: skip everything when *gate != 0
};

// upper-triangular tile index t -> (bi, bj), bi <= bj, row-major over the upper triangle
__device__ __forceinline__ void upper_tile(int t, int nt, int &bi, int &bj) {
  int i = 0, rem = t;
  while (rem >= nt - i) {
    rem -= nt - i;
    ++i;
  }
  bi = i;
  bj = i + rem;
}

template <bool TRANS_A>
__global__ void __launch_bounds__(256) dgemm_kernel(int64_t M, int64_t N, int64_t K, const double *__restrict__ A,
                                                    int64_t lda, const double *__restrict__ B, int64_t ldb,
                                                    double *__restrict__ C, int64_t ldc, int64_t k_per_split,
                                                    int64_t split_stride, DgemmEpi ep, int direct) {
  if (ep.gate && *ep.gate != 0) return;
  constexpr int ASZ = TRANS_A ? TK * LDT : TM * LDA;
  extern __shared__ __align__(16) double dg_smem[];
  double(*As)[ASZ] = reinterpret_cast<double(*)[ASZ]>(dg_smem);
  double(*Bs)[TK * LDT] = reinterpret_cast<double(*)[TK * LDT]>(dg_smem + 2 * ASZ);
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int g = lane >> 2, t4 = lane & 3;
  const int wm = warp >> 2, wn = warp & 3;  // warp tile: rows wm*32.., cols wn*16..
  int64_t m0 = (int64_t)blockIdx.x * TM, n0 = (int64_t)blockIdx.y * TN;
  if (ep.sym) {
    int bi, bj;
    upper_tile((int)blockIdx.x, (int)((N + TN - 1) / TN), bi, bj);
    m0 = (int64_t)bi * TM;
    n0 = (int64_t)bj * TN;
  }
  const int64_t kbeg = (int64_t)blockIdx.z * k_per_split;
  int64_t kend = min(K, kbeg + k_per_split);
  if (ep.b_upper) kend = min(kend, n0 + TN);
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
        if (c >= N) continue;
        double v = acc[i][j][h];
        if (direct) {
          if (ep.alpha != 1.0) v = ep.alpha * v;
          if (ep.cin) v = __dadd_rn(v, ep.beta == 1.0 ? ep.cin[r * ep.ldci + c] : ep.beta * ep.cin[r * ep.ldci + c]);
          if (ep.sym && c > r) Cz[c * ldc + r] = v;
        }
        Cz[r * ldc + c] = v;
      }
  }
}

// C = sum_z parts[z] in fixed order (deterministic), then the epilogue; 2-D grid, no division.
// Symmetric output: only the upper triangle is read (coalesced) and written to both halves.
__global__ void splitk_reduce_kernel(const double *__restrict__ parts, int splits, int64_t M, int64_t N,
                                     double *__restrict__ C, int64_t ldc, DgemmEpi ep) {
  if (ep.gate && *ep.gate != 0) return;
  const int64_t n = M * N;
  for (int64_t r = blockIdx.y; r < M; r += gridDim.y)
    for (int64_t c = (ep.sym ? r : 0) + (int64_t)blockIdx.x * blockDim.x + threadIdx.x; c < N;
         c += (int64_t)gridDim.x * blockDim.x) {
      const int64_t src = r * N + c;
      double s = 0.0;
      for (int z = 0; z < splits; ++z) s += parts[z * n + src];
      if (ep.alpha != 1.0) s = ep.alpha * s;
      if (ep.cin) s = __dadd_rn(s, ep.beta == 1.0 ? ep.cin[r * ep.ldci + c] : ep.beta * ep.cin[r * ep.ldci + c]);
      C[r * ldc + c] = s;
      if (ep.sym) C[c * ldc + r] = s;
    }
}

int64_t tile_count(int64_t M, int64_t N, bool sym) {
  const int64_t tn = ceil_div(N, TN);
  return sym ? tn * (tn + 1) / 2 : ceil_div(M, TM) * tn;
}

int choose_splits(int trans_a, int64_t M, int64_t N, int64_t K, bool sym = false) {
  int64_t tiles = tile_count(M, N, sym);
  int64_t want = ceil_div(3LL * num_sms(), tiles);  // ~3 resident CTAs per SM
  int64_t max_by_k = std::max<int64_t>(1, K / 256);
  int64_t s = std::max<int64_t>(1, std::min<int64_t>(want, std::min<int64_t>(max_by_k, 64)));
  return (int)s;
}

}  // namespace

size_t dgemm_ws_bytes(int trans_a, int64_t M, int64_t N, int64_t K) {
  int s = std::max(choose_splits(trans_a, M, N, K), choose_splits(trans_a, M, N, K, trans_a && M == N));
  return s > 1 ? (size_t)round_up(s * M * N * 8, 256) : 0;
}

int dgemm_device_ex(int trans_a, int64_t M, int64_t N, int64_t K, const double *A, int64_t lda, const double *B,
                    int64_t ldb, double *C, int64_t ldc, void *ws, size_t ws_bytes, cudaStream_t st,
                    const DgemmOptions &opt) {
  if (M < 1 || N < 1 || K < 1) return fail(LRAMM_ERR_SHAPE, "dgemm: empty shape");
  const bool sym = opt.sym && trans_a && M == N;
  DgemmEpi ep{sym ? 1 : 0, opt.b_upper, opt.alpha, opt.beta, opt.cin, opt.ldci, opt.gate};
  int splits = choose_splits(trans_a, M, N, K, sym);
  if (splits > 1 && (ws == nullptr || ws_bytes < dgemm_ws_bytes(trans_a, M, N, K))) splits = 1;
  int64_t kps = round_up(ceil_div(K, splits), TK);
  splits = (int)ceil_div(K, kps);
  dim3 grid = sym ? dim3((unsigned)tile_count(M, N, true), 1, (unsigned)splits)
                  : dim3((unsigned)ceil_div(M, TM), (unsigned)ceil_div(N, TN), (unsigned)splits);
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
  const int direct = splits == 1;
  if (trans_a)
    dgemm_kernel<true><<<grid, 256, smem_t, st>>>(M, N, K, A, lda, B, ldb, out, ldo, kps, M * N, ep, direct);
  else
    dgemm_kernel<false><<<grid, 256, smem_n, st>>>(M, N, K, A, lda, B, ldb, out, ldo, kps, M * N, ep, direct);
  LRAMM_LAUNCH_CHECK();
  if (splits > 1) {
    const unsigned gy = (unsigned)std::min<int64_t>(M, 4LL * num_sms());
    splitk_reduce_kernel<<<dim3((unsigned)ceil_div(N, 256), gy), 256, 0, st>>>((const double *)ws, splits, M, N, C,
                                                                                 ldc, ep);
    LRAMM_LAUNCH_CHECK();
  }
  return LRAMM_OK;
}

int dgemm_device(int trans_a, int64_t M, int64_t N, int64_t K, const double *A, int64_t lda, const double *B,
                 int64_t ldb, double *C, int64_t ldc, void *ws, size_t ws_bytes, cudaStream_t st) {
  return dgemm_device_ex(trans_a, M, N, K, A, lda, B, ldb, C, ldc, ws, ws_bytes, st, DgemmOptions{});
}

}  // namespace lramm
