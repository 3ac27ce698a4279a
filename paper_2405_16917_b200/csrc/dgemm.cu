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
#include <cstdlib>
#include <algorithm>
#include <mutex>

#include "common.cuh"
#include "sm100.cuh"

namespace lramm {
namespace {

constexpr int TM = 64, TN = 64;

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
  const int *gate;   // non-null: skip everything when *gate != 0 (== 0 with gate_inv)
  int gate_inv;
};
__device__ __forceinline__ bool gated_off(const DgemmEpi &ep) {
  return ep.gate && ((*ep.gate != 0) != (ep.gate_inv != 0));
}

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

// 64 x 64 CTA tile, 4 warps each owning a 32 x 32 sub-tile (4 x 4 DMMA 8x8 tiles: 8 fragment
// loads per 16 DMMA), K staged 16 doubles at a time through a 3-deep cp.async ring (16-byte
// copies through L2 when the operands are 16-byte aligned with even leading dimensions, 8-byte
// otherwise).  Shared-memory strides == 4 (mod 16) doubles: conflict-free fragment loads.
constexpr int KT = 16, NSTAGE = 3;
constexpr int LDA_N = KT + 4;   // As[m][k] (NN): 20
constexpr int LDA_T = TM + 4;   // As[k][m] (TN): 68
constexpr int LDB = TN + 4;     // Bs[k][n]: 68
constexpr int A_STAGE = TM * LDA_N > KT * LDA_T ? TM * LDA_N : KT * LDA_T;  // doubles
constexpr int B_STAGE = KT * LDB;
constexpr size_t kDgemmSmem = (size_t)NSTAGE * (A_STAGE + B_STAGE) * sizeof(double);

__device__ __forceinline__ void cp16(double *dst, const double *src, int nvalid) {
  // nvalid doubles (0..2) copied, the rest zero-filled
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"(sm100::smem_u32(dst)), "l"(src),
               "r"(nvalid * 8)
               : "memory");
}

template <bool TRANS_A, bool VEC>
__global__ void __launch_bounds__(128) dgemm_kernel(int64_t M, int64_t N, int64_t K, const double *__restrict__ A,
                                                    int64_t lda, const double *__restrict__ B, int64_t ldb,
                                                    double *__restrict__ C, int64_t ldc, int64_t k_per_split,
                                                    int64_t split_stride, DgemmEpi ep, int direct) {
  if (gated_off(ep)) return;
  extern __shared__ __align__(16) double dg_smem[];
  double *As = dg_smem;                    // [NSTAGE][A_STAGE]
  double *Bs = dg_smem + NSTAGE * A_STAGE;  // [NSTAGE][B_STAGE]
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int g = lane >> 2, t4 = lane & 3;
  const int wm = warp >> 1, wn = warp & 1;
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
  const int nkt = kend > kbeg ? (int)((kend - kbeg + KT - 1) / KT) : 0;

  auto stage = [&](int buf, int64_t k0) {
    double *as = As + buf * A_STAGE;
    double *bs = Bs + buf * B_STAGE;
    if (VEC) {
      if (TRANS_A) {  // A: K x M, chunks along m
        for (int e = tid; e < KT * TM / 2; e += 128) {
          const int kk = e / (TM / 2), mm = 2 * (e % (TM / 2));
          const int64_t gk = k0 + kk, gm = m0 + mm;
          const int nv = (gk < kend) ? (int)max((int64_t)0, min((int64_t)2, M - gm)) : 0;
          cp16(as + kk * LDA_T + mm, A + (nv ? gk * lda + gm : 0), nv);
        }
      } else {  // A: M x K, chunks along k
        for (int e = tid; e < TM * KT / 2; e += 128) {
          const int mm = e / (KT / 2), kk = 2 * (e % (KT / 2));
          const int64_t gk = k0 + kk, gm = m0 + mm;
          const int nv = (gm < M) ? (int)max((int64_t)0, min((int64_t)2, kend - gk)) : 0;
          cp16(as + mm * LDA_N + kk, A + (nv ? gm * lda + gk : 0), nv);
        }
      }
      for (int e = tid; e < KT * TN / 2; e += 128) {
        const int kk = e / (TN / 2), nn = 2 * (e % (TN / 2));
        const int64_t gk = k0 + kk, gn = n0 + nn;
        const int nv = (gk < kend) ? (int)max((int64_t)0, min((int64_t)2, N - gn)) : 0;
        cp16(bs + kk * LDB + nn, B + (nv ? gk * ldb + gn : 0), nv);
      }
    } else {
      if (TRANS_A) {
        for (int e = tid; e < KT * TM; e += 128) {
          const int kk = e / TM, mm = e % TM;
          const int64_t gk = k0 + kk, gm = m0 + mm;
          const bool v = gk < kend && gm < M;
          sm100::cp_async8(as + kk * LDA_T + mm, A + (v ? gk * lda + gm : 0), v);
        }
      } else {
        for (int e = tid; e < TM * KT; e += 128) {
          const int mm = e / KT, kk = e % KT;
          const int64_t gk = k0 + kk, gm = m0 + mm;
          const bool v = gk < kend && gm < M;
          sm100::cp_async8(as + mm * LDA_N + kk, A + (v ? gm * lda + gk : 0), v);
        }
      }
      for (int e = tid; e < KT * TN; e += 128) {
        const int kk = e / TN, nn = e % TN;
        const int64_t gk = k0 + kk, gn = n0 + nn;
        const bool v = gk < kend && gn < N;
        sm100::cp_async8(bs + kk * LDB + nn, B + (v ? gk * ldb + gn : 0), v);
      }
    }
  };
  double acc[4][4][2];
#pragma unroll
  for (int i = 0; i < 4; ++i)
#pragma unroll
    for (int j = 0; j < 4; ++j) acc[i][j][0] = acc[i][j][1] = 0.0;
#pragma unroll
  for (int s0 = 0; s0 < NSTAGE - 1; ++s0) {
    if (s0 < nkt) stage(s0, kbeg + (int64_t)s0 * KT);
    asm volatile("cp.async.commit_group;" ::: "memory");
  }
  for (int kt = 0; kt < nkt; ++kt) {
    asm volatile("cp.async.wait_group %0;" ::"n"(NSTAGE - 2) : "memory");
    __syncthreads();
    const int buf = kt % NSTAGE;
    const double *as = As + buf * A_STAGE;
    const double *bs = Bs + buf * B_STAGE;
#pragma unroll
    for (int kk = 0; kk < KT; kk += 4) {
      double a[4], b[4];
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        const int m = wm * 32 + i * 8 + g;
        a[i] = TRANS_A ? as[(kk + t4) * LDA_T + m] : as[m * LDA_N + kk + t4];
      }
#pragma unroll
      for (int j = 0; j < 4; ++j) b[j] = bs[(kk + t4) * LDB + wn * 32 + j * 8 + g];
#pragma unroll
      for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j) dmma(acc[i][j], a[i], b[j]);
    }
    const int nxt = kt + NSTAGE - 1;
    if (nxt < nkt) stage(nxt % NSTAGE, kbeg + (int64_t)nxt * KT);
    asm volatile("cp.async.commit_group;" ::: "memory");
  }
  asm volatile("cp.async.wait_group 0;" ::: "memory");
  double *Cz = C + (int64_t)blockIdx.z * split_stride;
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    const int64_t r = m0 + wm * 32 + i * 8 + g;
    if (r >= M) continue;
#pragma unroll
    for (int j = 0; j < 4; ++j)
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        const int64_t c = n0 + wn * 32 + j * 8 + 2 * t4 + h;
        if (c >= N) continue;
        if (ep.sym && c < r) continue;  // lower half: mirrored from the upper element
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
  if (gated_off(ep)) return;
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
  // ~4 waves of 4 resident CTAs per SM when K is long enough (wave quantisation stays small);
  // each split keeps >= 256 of K (max_by_k)
  if (tiles >= 4LL * num_sms()) return 1;  // already a full wave of tiles: no partials
  int64_t want = ceil_div(16LL * num_sms(), tiles);
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
  DgemmEpi ep{sym ? 1 : 0, opt.b_upper, opt.alpha, opt.beta, opt.cin, opt.ldci, opt.gate, opt.gate_run_if_nonzero};
  int splits = choose_splits(trans_a, M, N, K, sym);
  if (splits > 1 && (ws == nullptr || ws_bytes < dgemm_ws_bytes(trans_a, M, N, K))) splits = 1;
  int64_t kps = round_up(ceil_div(K, splits), KT);
  splits = (int)ceil_div(K, kps);
  dim3 grid = sym ? dim3((unsigned)tile_count(M, N, true), 1, (unsigned)splits)
                  : dim3((unsigned)ceil_div(M, TM), (unsigned)ceil_div(N, TN), (unsigned)splits);
  double *out = splits > 1 ? (double *)ws : C;
  int64_t ldo = splits > 1 ? N : ldc;
  static PerDeviceOnce once;
  LRAMM_CUDA_TRY(once.run([] {
    cudaError_t e = cudaSuccess;
    for (auto k : {dgemm_kernel<true, true>, dgemm_kernel<true, false>, dgemm_kernel<false, true>,
                   dgemm_kernel<false, false>})
      if (e == cudaSuccess) e = cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kDgemmSmem);
    return e;
  }));
  const int direct = splits == 1;
  const bool vec = ((lda | ldb) % 2 == 0) && (((uintptr_t)A | (uintptr_t)B) % 16 == 0);
  auto kern = trans_a ? (vec ? dgemm_kernel<true, true> : dgemm_kernel<true, false>)
                      : (vec ? dgemm_kernel<false, true> : dgemm_kernel<false, false>);
  kern<<<grid, 128, kDgemmSmem, st>>>(M, N, K, A, lda, B, ldb, out, ldo, kps, M * N, ep, direct);
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
