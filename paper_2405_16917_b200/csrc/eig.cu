// Eigenvector preconditioner for the one-sided Jacobi SVD (svd_tall_device, factor.cu).
//
// The reference computes the small SVD of the projection Bs (rsvd.py:78) with one-sided cyclic
// Jacobi sweeps to tol 1e-13 (_jacobi.py:14-50, _core.pyx:72-133).  On the device that is a
// chain of ~10 sweeps x (w - 1) dependent rotation steps.  Here the right singular vectors of
// W = R^T are first obtained to working accuracy from the symmetric eigenproblem of the Gram
// G = W^T W = R R^T, and W is rotated by them once (W' = W V0, V0 orthogonal) -- a Jacobi
// preconditioner: W' has columns orthogonal to ~1e-15 relative, so the Jacobi run that follows
// (same kernel, same tolerance, same convergence test) has nothing left to rotate and is
// skipped by a device-side gate; when it is not (clustered / rank-deficient spectra, any failed
// check), the same Jacobi runs on W' -- or on the untouched W when the preconditioner itself
// failed -- and converges as before.  The singular values and left vectors are read from W'
// exactly as from the Jacobi result (column norms, normalised columns), so the multiplicative
// perturbation of an orthogonal V0 leaves them within ~eps relative (one-sided accuracy).
//
//   G = R R^T (DMMA GEMM)  ->  tridiagonalisation G = Q T Q^T      (sytrd_cluster_kernel)
//   eigenvalues of T by multisection Sturm counts                  (tridiag_bisect_kernel)
//   eigenvectors of T by one twisted factorisation each            (tridiag_twisted_kernel)
//   Z <- Z (Z^T Z)^-1/2 to first order (Lowdin)                    (GEMMs + eig_defect_kernel)
//   V0 = Q Z by the stored Householder reflectors                  (backtransform_kernel)
//   P = W V0 ; E_ij = S_ij / (S_jj - S_ii), S = P^T P ; P <- P + P E   (one-sided refinement)
//   gate = any S_ij^2 > tol^2 S_ii S_jj (S = P^T P)  -> Jacobi runs only if set
#include <cooperative_groups.h>

#include <algorithm>
#include <cfloat>
#include <cstdlib>

#include "common.cuh"
#include "sm100.cuh"

namespace cg = cooperative_groups;

#ifdef LRAMM_SYTRD_TRACE
__device__ long long sytrd_trace[16];
#define STR_MARK(v) long long v = clock64();
#define STR_ADD(slot, a, b) \
  if (threadIdx.x == 0 && blockIdx.x == 0) sytrd_trace[slot] += (b) - (a);
#else
#define STR_MARK(v)
#define STR_ADD(slot, a, b)
#endif

namespace lramm {
int dgemm_device_ex(int trans_a, int64_t M, int64_t N, int64_t K, const double *A, int64_t lda, const double *B,
                    int64_t ldb, double *C, int64_t ldc, void *ws, size_t ws_bytes, cudaStream_t st,
                    const DgemmOptions &opt);
size_t dgemm_ws_bytes(int trans_a, int64_t M, int64_t N, int64_t K);
int transpose_device(const double *a, int64_t rows, int64_t cols, int64_t lda, double *b, int64_t ldb,
                     cudaStream_t st);

using sm100::cp_async8;
using sm100::cp_async_wait_all;
namespace {

// 1/x to ~1 ulp: MUFU reciprocal seed + two Newton steps (x normal, |x| >= pivmin)
__device__ __forceinline__ double rcp_nr(double x) {
  double r;
  asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(r) : "d"(x));
  double e = fma(-x, r, 1.0);
  r = fma(r, e, r);
  e = fma(-x, r, 1.0);
  return fma(r, e, r);
}

// ------------------------------------------------------------------ CTA reductions
template <int NW>
__device__ __forceinline__ double cta_sum(double v, double *red) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  if (lane == 0) red[warp] = v;
  __syncthreads();
  double s = 0.0;
  const int nw = blockDim.x >> 5;
  for (int i = 0; i < nw; ++i) s += red[i];
  return s;
}

__device__ __forceinline__ double cta_max(double v, double *red) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v = fmax(v, __shfl_xor_sync(0xffffffffu, v, o));
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  if (lane == 0) red[warp] = v;
  __syncthreads();
  double s = 0.0;
  const int nw = blockDim.x >> 5;
  for (int i = 0; i < nw; ++i) s = fmax(s, red[i]);
  return s;
}

// ------------------------------------------------------------------ tridiagonalisation
// LAPACK dsytd2 (lower) semantics: reflector k = I - tau_k v_k v_k^T acts on indices k+1..n-1,
// v_k[k+1] = 1; d_k = T_kk, e_k = T_{k+1,k} = beta_k.  Rows of the n x n matrix are spread
// cyclically over the C CTAs of a cluster (row i on CTA i mod C).  Step k:
//   every CTA knows v_k, tau_k (derived redundantly) and holds its rows of A_k;
//   it has received from every CTA (p_j, A_k[j, k+1]) for j > k, p = tau_k A_k v_k: each CTA
//   pushes those pairs for its own rows into every CTA's receive buffer with st.async, whose
//   bytes complete a transaction count on the receiver's mbarrier (one per buffer parity), so a
//   CTA starts step k as soon as all rows of that step have landed -- no cluster barrier and no
//   gather per step;
//   s = p . v_k and w = p - (tau_k / 2) s v_k (every warp, redundantly); warp 0 updates column
//   k+1 (= row k+1) to A_{k+1} and derives reflector k+1 from it while the other warps apply
//   A -= v w^T + w v^T to their rows; after one CTA barrier the next p_i and A[i, k+2] of the own
//   rows are formed and pushed.
// Row storage per CTA: RM rows per row warp in registers (lane owns columns lane + 32 e), then
// nsm rows in shared memory, then the rest in L2-resident global scratch (w = 1056); the
// shared-memory / global rows are updated in one fused pass once the reflector is known.
struct SytrdArgs {
  const double *G;  // n x n row-major (ldg), symmetric; problem stride g_stride
  int64_t ldg, g_stride;
  int n;
  double *d, *e, *tau;  // per problem: n, n, n (stride n)
  double *V;            // per problem n x n row-major: row k = v_k at columns k+1..n-1
  int ldr;              // row stride (doubles) of the shared-memory / global row storage
  int nsm;              // rows per CTA held in shared memory (after the register rows)
  double *Ag;           // rows beyond those: global scratch, [batch * C][ag_rows][ldr]
  int64_t ag_rows;      // rows per CTA in Ag
};

__device__ __forceinline__ double warp_allsum(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

// reflector from x = (alpha, r[j0+1..n-1]): beta, tau, 1/(alpha - beta) (LAPACK dlarfg without the
// rescaling loop; the operand is prescaled to an O(1) range)
__device__ __forceinline__ void householder(double alpha, double s2, double &beta, double &tau, double &scl) {
  if (s2 == 0.0) {
    tau = 0.0;
    beta = alpha;
    scl = 0.0;
  } else {
    beta = -copysign(sqrt(fma(alpha, alpha, s2)), alpha);
    tau = (beta - alpha) / beta;
    scl = 1.0 / (alpha - beta);
  }
}

// dlarfg without division or square root on the chain: rs = 1/sqrt(alpha^2 + s2) (MUFU seed +
// third-order correction), beta = -sign(alpha)/rs, tau = 1 + |alpha| rs, 1/(alpha - beta) =
// sign(alpha) / (|alpha| + 1/rs); out-of-range operands take the exact library path
__device__ __forceinline__ void householder_fast(double alpha, double s2, double &beta, double &tau, double &scl) {
  const double t = fma(alpha, alpha, s2);
  if (s2 == 0.0) {
    tau = 0.0;
    beta = alpha;
    scl = 0.0;
    return;
  }
  if (!(t >= 0x1p-900 && t <= 0x1p900)) {
    householder(alpha, s2, beta, tau, scl);
    return;
  }
  double y;
  asm("rsqrt.approx.ftz.f64 %0, %1;" : "=d"(y) : "d"(t));
  const double e = fma(-(y * y), t, 1.0);
  const double rs = fma(fma(e, 0.375, 0.5), y * e, y);
  const double nrm = t * rs;
  const double aa = fabs(alpha);
  beta = -copysign(nrm, alpha);
  tau = fma(aa, rs, 1.0);
  scl = copysign(rcp_nr(aa + nrm), alpha);
}

__device__ __forceinline__ uint32_t mapa_u32(uint32_t saddr, int rank) {
  uint32_t r;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(r) : "r"(saddr), "r"(rank));
  return r;
}
__device__ __forceinline__ void mbar_wait_acq_cluster(uint32_t bar, uint32_t parity) {
  asm volatile(
      "{\n\t.reg .pred p;\n"
      "W_%=:\n\t"
      "mbarrier.try_wait.parity.acquire.cluster.shared::cta.b64 p, [%0], %1;\n\t"
      "@!p bra W_%=;\n}\n" ::"r"(bar),
      "r"(parity)
      : "memory");
}
__device__ __forceinline__ void st_async_v2(uint32_t raddr, double a, double b, uint32_t rbar) {
  asm volatile("st.async.shared::cluster.mbarrier::complete_tx::bytes.v2.f64 [%0], {%1, %2}, [%3];" ::"r"(raddr),
               "d"(a), "d"(b), "r"(rbar)
               : "memory");
}

constexpr int kSytrdRegMaxE = 12;   // register rows up to n = 384
constexpr int kSytrdMaxE = 33;      // n <= 1056
constexpr int kSytrdWarps = 8;

template <int E, int RM>
__global__ void __launch_bounds__(32 * kSytrdWarps, 1) sytrd_push_kernel(SytrdArgs a) {
  constexpr int RR = RM > 0 ? RM : 1;
  cg::cluster_group cl = cg::this_cluster();
  const int C = (int)cl.num_blocks();  // a power of two
  const int lgC = __ffs(C) - 1;
  const int me = (int)cl.block_rank();
  const int prob = blockIdx.x >> lgC;
  const int n = a.n, ldr = a.ldr;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5, nwarp = blockDim.x >> 5, nth = blockDim.x;
  // row warps: all but warp 0 (the reflector) and warp 4, which shares warp 0's SM sub-partition
  // (its fp64 pipe) -- the reflector chain is the critical path of a step
  const int nrw = nwarp - 2;
  const int rwi = warp == 0 || warp == 4 ? -1 : (warp < 4 ? warp - 1 : warp - 2);
  const int nl = (n - me + C - 1) >> lgC;  // local rows: global i = me + li * C
  const int nlmax = (n + C - 1) >> lgC;
  const int nreg = RM > 0 ? nrw * RM : 0;   // local rows li < nreg: registers (li = rwi + r * nrw)
  const int nsm = a.nsm;                     // then shared memory, then global
  extern __shared__ __align__(16) double sm[];
  double2 *rbuf = reinterpret_cast<double2 *>(sm);  // [2][n] received (p_j, A[j, k+1])
  double2 *stage = rbuf + 2 * (size_t)n;            // [nlmax] prologue pushes behind a barrier
  double *vb = reinterpret_cast<double *>(stage + nlmax);  // [2][ldr]
  double *rk = vb + 2 * (size_t)ldr;                // [ldr] row 0 at start
  double *As = rk + ldr;                            // [nsm][ldr]
  double *Ag = a.Ag ? a.Ag + (size_t)blockIdx.x * a.ag_rows * ldr : nullptr;
  __shared__ double red[2][32];
  __shared__ double hh[4];
  __shared__ __align__(8) uint64_t bars[2];
  auto row_ptr = [&](int li) {  // storage of a non-register local row
    const int t = li - nreg;
    return t < nsm ? As + (size_t)t * ldr : Ag + (size_t)(t - nsm) * ldr;
  };

  const double *G = a.G + (size_t)prob * a.g_stride;
  double *dout = a.d + (size_t)prob * n, *eout = a.e + (size_t)prob * n, *tout = a.tau + (size_t)prob * n;
  double *Vout = a.V + (size_t)prob * n * n;

  if (tid == 0) {
    sm100::mbar_init(&bars[0], 1);
    sm100::mbar_init(&bars[1], 1);
    sm100::fence_barrier_init();
  }
  // exact power-of-two prescale: largest diagonal into [1, 4)
  double dm = 0.0;
  for (int i = tid; i < n; i += nth) dm = fmax(dm, fabs(G[(int64_t)i * a.ldg + i]));
  dm = cta_max(dm, red[0]);
  double scale = 1.0;
  if (dm > 0.0 && dm <= DBL_MAX) scale = ldexp(1.0, -2 * (ilogb(dm) >> 1));
  double x[RR][E];
  int gi[RR];
#pragma unroll
  for (int r = 0; r < RR; ++r) {
    const int li = rwi + r * nrw;
    gi[r] = (RM > 0 && rwi >= 0 && li < nl) ? me + (li << lgC) : -1;
    const double *src = G + (int64_t)(gi[r] < 0 ? 0 : gi[r]) * a.ldg;
#pragma unroll
    for (int e = 0; e < E; ++e) {
      const int j = lane + 32 * e;
      x[r][e] = (gi[r] >= 0 && j < n) ? src[j] * scale : 0.0;
    }
  }
  for (int li = nreg + warp; li < nl; li += nwarp) {
    const double *src = G + (int64_t)(me + (li << lgC)) * a.ldg;
    double *dst = row_ptr(li);
    for (int j = lane; j < 32 * E; j += 32) dst[j] = j < n ? src[j] * scale : 0.0;
  }
  for (int j = tid; j < n; j += nth) rk[j] = G[j] * scale;
  __syncthreads();
  double *v = vb, *vn = vb + ldr;
  double tau;
  {  // row 0 (redundant in every CTA) -> d_0, reflector 0
    double s2 = 0.0;
    for (int j = 2 + tid; j < n; j += nth) s2 = fma(rk[j], rk[j], s2);
    s2 = cta_sum<32>(s2, red[1]);
    double beta, scl;
    householder(rk[1], s2, beta, tau, scl);
    for (int j = tid; j < ldr; j += nth) {
      const double vj = (j < 1 || j >= n) ? 0.0 : (j == 1 ? 1.0 : rk[j] * scl);
      v[j] = vj;
      vn[j] = 0.0;
      if (me == 0 && j >= 1 && j < n) Vout[j] = vj;
    }
    if (me == 0 && tid == 0) {
      dout[0] = rk[0];
      eout[0] = beta;
      tout[0] = tau;
    }
  }
  const uint32_t rbuf_s = sm100::smem_u32(rbuf), bar_s = sm100::smem_u32(bars);
  cl.sync();  // barriers initialised everywhere before any remote push
  if (tid == 0) sm100::mbar_arrive_expect_tx(&bars[0], 16u * (uint32_t)(n - 1));
  // push (p_i, A[i, j]) of local row i to every CTA's receive buffer (parity bp)
  auto push = [&](int i, double pv, double cv, int bp) {
    if (lane < C) {
      const uint32_t ra = mapa_u32(rbuf_s + (uint32_t)(bp * n + i) * 16u, lane);
      const uint32_t rb = mapa_u32(bar_s + (uint32_t)bp * 8u, lane);
      st_async_v2(ra, pv, cv, rb);
    }
  };
  {  // p_0 and the column-1 entries of own rows i >= 1 (once: dots staged, a barrier, then pushes)
    for (int li = warp; li < nl; li += nwarp) {
      const int i = me + (li << lgC);
      if (i < 1) continue;
      double dot = 0.0;
      for (int j = lane; j < n; j += 32) dot = fma(G[(int64_t)i * a.ldg + j] * scale, v[j], dot);
      dot = warp_allsum(dot);
      if (lane == 0) stage[li] = make_double2(tau * dot, G[(int64_t)i * a.ldg + 1] * scale);
    }
    __syncthreads();
    for (int li = warp; li < nl; li += nwarp) {
      const int i = me + (li << lgC);
      if (i >= 1) push(i, stage[li].x, stage[li].y, 0);
    }
  }

  for (int k = 0; k <= n - 3; ++k) {
    const int par = k & 1, npar = par ^ 1;
    const bool last = (k == n - 3);
    STR_MARK(t0);
    mbar_wait_acq_cluster(bar_s + par * 8, (uint32_t)((k >> 1) & 1));
    if (tid == 0 && !last) sm100::mbar_arrive_expect_tx(&bars[npar], 16u * (uint32_t)(n - k - 2));
    STR_MARK(t1);
    const double2 *rb = rbuf + (size_t)par * n;
    // s = p . v; w_j = p_j - c v_j on this lane's columns (zero for j <= k)
    double wr[E], vr[E];
#pragma unroll
    for (int e = 0; e < E; ++e) {
      const int j = lane + 32 * e;
      const bool in = j > k && j < n;
      wr[e] = in ? rb[j].x : 0.0;
      vr[e] = in ? v[j] : 0.0;
    }
    double sacc = 0.0;
#pragma unroll
    for (int e = 0; e < E; ++e) sacc = fma(wr[e], vr[e], sacc);
    const double c = 0.5 * tau * warp_allsum(sacc);
#pragma unroll
    for (int e = 0; e < E; ++e) wr[e] = fma(-c, vr[e], wr[e]);
    STR_MARK(t2);
    if (warp == 0) {
      // column k+1 of A_{k+1}: r_j = A_k[j, k+1] - v_j w_{k+1} - w_j   (v_{k+1} = 1)
      const double wk1 = rb[k + 1].x - c;
      double rr[E];
      double s2 = 0.0;
#pragma unroll
      for (int e = 0; e < E; ++e) {
        const int j = lane + 32 * e;
        rr[e] = (j > k && j < n) ? rb[j].y - wr[e] - wk1 * vr[e] : 0.0;
        if (j >= k + 3) s2 = fma(rr[e], rr[e], s2);
      }
      s2 = warp_allsum(s2);
      double al = 0.0, dk = 0.0;
#pragma unroll
      for (int e = 0; e < E; ++e) {
        if (e == ((k + 2) >> 5)) al = rr[e];
        if (e == ((k + 1) >> 5)) dk = rr[e];
      }
      const double alpha = __shfl_sync(0xffffffffu, al, (k + 2) & 31);
      const double dk1 = __shfl_sync(0xffffffffu, dk, (k + 1) & 31);
      if (!last) {
        double beta, tn, scl;
        householder_fast(alpha, s2, beta, tn, scl);
#pragma unroll
        for (int e = 0; e < E; ++e) vn[lane + 32 * e] = rr[e] * scl;  // zero below k+1; padded to 32 E
        __syncwarp();
        if (lane == 0) {
          vn[k + 1] = 0.0;
          vn[k + 2] = 1.0;
          hh[0] = tn;
          hh[1] = dk1;
          hh[2] = beta;
        }
      } else if (me == 0 && lane == 0) {
        dout[n - 2] = dk1;
        eout[n - 2] = alpha;
      }
    } else if (RM > 0) {
      // own register rows i >= k+2: A -= v w^T + w v^T
#pragma unroll
      for (int r = 0; r < RR; ++r) {
        if (gi[r] >= k + 2) {
          const double vi = v[gi[r]], wi = rb[gi[r]].x - c * vi;
#pragma unroll
          for (int e = 0; e < E; ++e) x[r][e] = fma(-wi, vr[e], fma(-vi, wr[e], x[r][e]));
        }
      }
      if (last) {
#pragma unroll
        for (int r = 0; r < RR; ++r)
          if (gi[r] == n - 1) {
#pragma unroll
            for (int e = 0; e < E; ++e)
              if (lane + 32 * e == n - 1) dout[n - 1] = x[r][e];
          }
      }
    }
    if (last && warp == 1 && lane == 0 && ((n - 1) & (C - 1)) == me && ((n - 1) >> lgC) >= nreg) {
      // row n-1 outside the registers: a_{n-1,n-1} - 2 v_{n-1} w_{n-1}
      const double vl = v[n - 1], wl = rb[n - 1].x - c * vl;
      dout[n - 1] = row_ptr((n - 1) >> lgC)[n - 1] - 2.0 * vl * wl;
    }
    if (last) break;
    STR_MARK(t3);
    __syncthreads();
    STR_MARK(t4);
    // ---- p_{k+1} and the column-(k+2) entry of own rows i >= k+2, pushed to every CTA
    const double tn = hh[0];
    if (warp == 4 && me == 0) {  // outputs, off the reflector chain
      double *vrow = Vout + (size_t)(k + 1) * n;
      for (int j = k + 2 + lane; j < n; j += 32) vrow[j] = vn[j];
      if (lane == 0) {
        dout[k + 1] = hh[1];
        eout[k + 1] = hh[2];
        tout[k + 1] = tn;
      }
    }
    double vv[E];
#pragma unroll
    for (int e = 0; e < E; ++e) vv[e] = vn[lane + 32 * e];  // zero below k+2 and beyond n
    const int ek2 = (k + 2) >> 5, lk2 = (k + 2) & 31;
    if (RM > 0 && rwi >= 0) {
      double dots[RR], cols[RR];
#pragma unroll
      for (int r = 0; r < RR; ++r) {
        double dot = 0.0, ce = 0.0;
#pragma unroll
        for (int e = 0; e < E; ++e) {
          dot = fma(x[r][e], vv[e], dot);
          if (e == ek2) ce = x[r][e];
        }
        dots[r] = dot;
        cols[r] = ce;
      }
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) {
#pragma unroll
        for (int r = 0; r < RR; ++r) dots[r] += __shfl_xor_sync(0xffffffffu, dots[r], o);
      }
#pragma unroll
      for (int r = 0; r < RR; ++r) {
        const double ck2 = __shfl_sync(0xffffffffu, cols[r], lk2);
        if (gi[r] >= k + 2) push(gi[r], tn * dots[r], ck2, npar);
      }
    }
    {  // shared-memory / global rows: update fused with the dot product
      int li0 = (k + 2 - me + C - 1) >> lgC;
      if (li0 < nreg) li0 = nreg;
      for (int li = li0 + warp; li < nl; li += nwarp) {
        const int i = me + (li << lgC);
        double *ar = row_ptr(li);
        const double vi = v[i], wi = rb[i].x - c * vi;
        // rows are padded to 32 E columns with zeros and w, v, vv vanish outside (k, n): the
        // update and the dot run over every column without guards
        double dot = 0.0;
#pragma unroll
        for (int e = 0; e < E; ++e) {
          if (32 * e + 31 <= k) continue;  // chunk finished (warp-uniform)
          const int j = lane + 32 * e;
          const double xv = fma(-wi, vr[e], fma(-vi, wr[e], ar[j]));
          ar[j] = xv;
          dot = fma(xv, vv[e], dot);
        }
        dot = warp_allsum(dot);
        __syncwarp();
        push(i, tn * dot, ar[k + 2], npar);
      }
    }
    tau = tn;
    {
      double *t = v;
      v = vn;
      vn = t;
    }
    STR_MARK(t5);
    STR_ADD(0, t0, t1);
    STR_ADD(1, t1, t2);
    STR_ADD(2, t2, t3);
    STR_ADD(3, t3, t4);
    STR_ADD(4, t4, t5);
    STR_ADD(6, t0, t5);
  }
  cl.sync();  // no CTA leaves while peers may still push into it
}

// ------------------------------------------------------------------ eigenvalues of T
// Multisection on Sturm counts: one warp per eigenvalue index i (ascending), each lane follows
// NCH shifts; a round splits the bracket into 32*NCH+1 parts.  Counts come from the
// leading-minor recurrence p_j = (d_j - x) p_{j-1} - e_{j-1}^2 p_{j-2} (no division; the
// critical path per step is one FMA), rescaled by a power of two every 8 steps; the count is
// the number of sign changes (sign bits; an exact zero is vanishingly rare at these shifts and
// only moves the bracket by the point spacing).
constexpr int kBisRounds = 9;  // 65-section: 65^9 > 2^54
constexpr int kBisWpe = 2;     // warps per eigenvalue (each lane follows one shift)

__device__ __forceinline__ int sgnbit(double x) { return (int)((unsigned)__double2hiint(x) >> 31); }
__device__ __forceinline__ int bexp(double x) { return (__double2hiint(x) >> 20) & 0x7ff; }

// Multisection on Sturm counts: kBisWpe warps per eigenvalue index i (ascending), one shift per
// lane; a round splits the bracket into 32 kBisWpe + 1 parts.  Counts come from the
// leading-minor recurrence p_j = (d_j - x) p_{j-1} - e_{j-1}^2 p_{j-2} (no division; the
// critical path per step is one FMA), rescaled by a power of two every 8 steps; the count is
// the number of sign changes (sign bits; an exact zero is vanishingly rare at these shifts and
// only moves the bracket by the point spacing).  Two warps per eigenvalue put two latency-bound
// chains on each SM sub-partition.
__global__ void __launch_bounds__(256) tridiag_bisect_kernel(const double *__restrict__ dall,
                                                             const double *__restrict__ eall, int n,
                                                             double *__restrict__ lamall) {
  extern __shared__ __align__(16) double sh[];
  double2 *sde = reinterpret_cast<double2 *>(sh);  // (d_j, e_{j-1}^2)
  __shared__ double red[32];
  __shared__ int cnt_part[8];
  const int prob = blockIdx.y;
  const double *d = dall + (size_t)prob * n, *e = eall + (size_t)prob * n;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  double lo_b = DBL_MAX, hi_b = -DBL_MAX;
  for (int j = tid; j < n; j += blockDim.x) {
    const double dj = d[j];
    const double el = j > 0 ? fabs(e[j - 1]) : 0.0, er = j < n - 1 ? fabs(e[j]) : 0.0;
    sde[j] = make_double2(dj, j > 0 ? e[j - 1] * e[j - 1] : 0.0);
    lo_b = fmin(lo_b, dj - el - er);
    hi_b = fmax(hi_b, dj + el + er);
  }
  lo_b = -cta_max(-lo_b, red);
  __syncthreads();
  hi_b = cta_max(hi_b, red);
  const double span = fmax(hi_b - lo_b, DBL_MIN);
  lo_b -= 4.0 * DBL_EPSILON * span + DBL_MIN;
  hi_b += 4.0 * DBL_EPSILON * span + DBL_MIN;
  const int epb = (blockDim.x >> 5) / kBisWpe;  // eigenvalues per block
  const int slot = warp / kBisWpe, h = warp % kBisWpe;
  const int i = blockIdx.x * epb + slot;
  const bool active = i < n;
  double lo = lo_b, hi = hi_b;
  constexpr int NP = 32 * kBisWpe;  // interior points per round
  for (int round = 0; round < kBisRounds; ++round) {
    const double hs = (hi - lo) / (double)(NP + 1);
    const double nx = -fma((double)(1 + kBisWpe * lane + h), hs, lo);
    double p2 = 1.0, p1 = sde[0].x + nx;
    int ng = sgnbit(p1), cnt = ng;
    if (active) {
#pragma unroll 8
      for (int j = 1; j < n; ++j) {
        const double2 de = sde[j];
        const double pn = fma(de.x + nx, p1, -de.y * p2);
        const int g = sgnbit(pn);
        cnt += g ^ ng;
        ng = g;
        p2 = p1;
        p1 = pn;
        if ((j & 7) == 0) {
          const int ex = max(bexp(p1), bexp(p2));
          const double f = __hiloint2double((2046 - ex) << 20, 0);
          p1 *= f;
          p2 *= f;
        }
      }
    }
    // points with count <= i (monotone in the point index 1 + kBisWpe lane + h)
    const int mine = __popc(__ballot_sync(0xffffffffu, cnt <= i));
    if (lane == 0) cnt_part[warp] = mine;
    __syncthreads();
    int m = 0;
#pragma unroll
    for (int q = 0; q < kBisWpe; ++q) m += cnt_part[slot * kBisWpe + q];
    __syncthreads();
    const double nlo = m >= 1 ? fma((double)m, hs, lo) : lo;
    const double nhi = m < NP ? fma((double)(m + 1), hs, lo) : hi;
    lo = nlo;
    hi = fmax(nhi, nlo);
  }
  if (active && h == 0 && lane == 0) lamall[(size_t)prob * n + i] = 0.5 * (lo + hi);
}

// ------------------------------------------------------------------ eigenvectors of T
// One thread per eigenvalue: stationary (L+ D+ L+^T) and progressive (U- D- U-^T) factorisations
// of T - lambda I, twist index r = argmin |gamma_r|, gamma_r = D+_r + D-_r - (d_r - lambda);
// z_r = 1, z_j = -L+_j z_{j+1} (j < r), z_{j+1} = -U-_{j+1} z_j (j >= r); normalised.
// The multipliers of the CTA's threads live in shared memory laid out [j][thread]; T in shared
// memory too.  The eigenvector is written as column i of Z (row-major n x n).
__global__ void __launch_bounds__(32) tridiag_twisted_kernel(const double *__restrict__ dall,
                                                             const double *__restrict__ eall, int n,
                                                             const double *__restrict__ lamall,
                                                             double *__restrict__ Zall) {
  extern __shared__ __align__(16) double tw[];
  const int nt = blockDim.x;
  double *sd = tw, *se = tw + n;                 // d, e
  double *Lp = se + n, *Um = Lp + (size_t)n * nt;  // [j][nt]
  const int prob = blockIdx.y;
  const double *d = dall + (size_t)prob * n, *e = eall + (size_t)prob * n;
  double emax = 0.0;
  for (int j = threadIdx.x; j < n; j += nt) {
    sd[j] = d[j];
    se[j] = j < n - 1 ? e[j] : 0.0;
  }
  __syncthreads();
  for (int j = 0; j < n - 1; ++j) emax = fmax(emax, fabs(se[j]));
  const int i = blockIdx.x * nt + threadIdx.x;
  if (i >= n) return;
  const int tx = threadIdx.x;
  const double lam = lamall[(size_t)prob * n + i];
  double *Z = Zall + (size_t)prob * n * n;
  const double pivmin = DBL_MIN * fmax(1.0, emax * emax);
  // forward D+ / L+ and backward D- / U-, interleaved (independent division chains)
  double dp = sd[0] - lam, dmn = sd[n - 1] - lam;
  for (int j = 0; j < n - 1; ++j) {
    if (fabs(dp) < pivmin) dp = -pivmin;
    const double l = se[j] * rcp_nr(dp);
    Lp[(size_t)j * nt + tx] = l;
    dp = (sd[j + 1] - lam) - l * se[j];
    const int jb = n - 2 - j;
    if (fabs(dmn) < pivmin) dmn = -pivmin;
    const double u = se[jb] * rcp_nr(dmn);
    Um[(size_t)(jb + 1) * nt + tx] = u;
    dmn = (sd[jb] - lam) - u * se[jb];
  }
  // gamma_r = (d_r - lam) - L+_{r-1} e_{r-1} - U-_{r+1} e_r
  int r = 0;
  double gbest = DBL_MAX;
  for (int j = 0; j < n; ++j) {
    double g = sd[j] - lam;
    if (j > 0) g -= Lp[(size_t)(j - 1) * nt + tx] * se[j - 1];
    if (j < n - 1) g -= Um[(size_t)(j + 1) * nt + tx] * se[j];
    if (fabs(g) < gbest) {
      gbest = fabs(g);
      r = j;
    }
  }
  // vector (unnormalised; the components reuse the multiplier slots), then scaled into Z
  double nrm2 = 1.0, z = 1.0;
  for (int j = r - 1; j >= 0; --j) {
    z = -Lp[(size_t)j * nt + tx] * z;
    if (!(fabs(z) <= 1e150)) z = 0.0;  // guard runaway growth from an unusable pivot
    Lp[(size_t)j * nt + tx] = z;
    nrm2 = fma(z, z, nrm2);
  }
  z = 1.0;
  for (int j = r; j < n - 1; ++j) {
    z = -Um[(size_t)(j + 1) * nt + tx] * z;
    if (!(fabs(z) <= 1e150)) z = 0.0;
    Um[(size_t)(j + 1) * nt + tx] = z;
    nrm2 = fma(z, z, nrm2);
  }
  const double inv = 1.0 / sqrt(nrm2);
  for (int j = 0; j < n; ++j) {
    const double zj = j < r ? Lp[(size_t)j * nt + tx] : (j == r ? 1.0 : Um[(size_t)j * nt + tx]);
    Z[(size_t)j * n + i] = zj * inv;
  }
}

// ------------------------------------------------------------------ checks and small updates
// D <- Z^T Z - I in place; flags[0] |= (max |D| > limit or non-finite)
__global__ void eig_defect_kernel(double *__restrict__ D, int n, int64_t stride, double limit, int *flags) {
  const int prob = blockIdx.y;
  double *Dp = D + (size_t)prob * stride;
  bool bad = false;
  for (int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; t < (int64_t)n * n;
       t += (int64_t)gridDim.x * blockDim.x) {
    const int r = (int)(t / n), c = (int)(t % n);
    double x = Dp[t];
    if (r == c) x -= 1.0;
    Dp[t] = x;
    if (!(fabs(x) <= limit)) bad = true;
  }
  if (__any_sync(0xffffffffu, bad) && (threadIdx.x & 31) == 0) atomicOr(flags + prob * 4, 1);
}

// V0 = Q Z, Q = H_0 H_1 ... H_{n-3}, applied in WY blocks of kNB reflectors:
//   H_{k0} ... H_{k0+nb-1} = I - V_b T_b V_b^T   (T_b upper triangular, reflector_t_kernel)
//   Z <- Z - V_b (T_b (V_b^T Z)) for the blocks from last to first, on strips of kBtCols
//   columns of Z held in shared memory (backtransform_kernel).
constexpr int kNB = 32;
constexpr int kBtCols = 8;

// T_b of every block (one CTA each): G_ac = v_a . v_c (a < c), then row a of T by the forward
// recurrence T[a][c] = -tau_c sum_{a <= b < c} T[a][b] G_bc, T[a][a] = tau_a
__global__ void __launch_bounds__(256) reflector_t_kernel(const double *__restrict__ Vall,
                                                          const double *__restrict__ tauall, int n, int jchunk,
                                                          double *__restrict__ Tall) {
  extern __shared__ __align__(16) double vs[];  // [kNB][jchunk] columns of the block's vectors
  __shared__ double Gs[kNB][kNB + 1];
  __shared__ double Ts[kNB][kNB + 1];
  const int prob = blockIdx.y, blk = blockIdx.x;
  const int nblk = (n - 2 + kNB - 1) / kNB;
  const double *V = Vall + (size_t)prob * n * n;
  const double *tau = tauall + (size_t)prob * n;
  double *T = Tall + ((size_t)prob * nblk + blk) * kNB * kNB;
  const int k0 = blk * kNB, nb = min(kNB, n - 2 - k0);
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5, nwarp = blockDim.x >> 5;
  for (int t = tid; t < kNB * (kNB + 1); t += blockDim.x) Gs[t / (kNB + 1)][t % (kNB + 1)] = 0.0;
  // G_ac = v_a . v_c (a < c) over column chunks of the vectors (zero left of each start)
  for (int j0 = k0; j0 < n; j0 += jchunk) {
    const int len = min(jchunk, n - j0);
    __syncthreads();
    for (int r = warp; r < kNB; r += nwarp) {  // warp per vector row, lanes along j
      const double *src = V + (size_t)(k0 + r) * n;
      double *dst = vs + (size_t)r * jchunk - j0;
      for (int j = j0 + lane; j < j0 + len; j += 32) dst[j] = (r < nb && j > k0 + r) ? __ldcg(src + j) : 0.0;
    }
    __syncthreads();
    for (int pr = warp; pr < kNB * kNB; pr += nwarp) {
      const int aa = pr / kNB, cc = pr % kNB;
      if (aa >= cc || cc >= nb) continue;
      const double *va = vs + (size_t)aa * jchunk, *vc = vs + (size_t)cc * jchunk;
      double sacc = 0.0;
      for (int j = lane; j < len; j += 32) sacc = fma(va[j], vc[j], sacc);
      sacc = warp_allsum(sacc);
      if (lane == 0) Gs[aa][cc] += sacc;  // the same warp owns this pair in every chunk
    }
  }
  __syncthreads();
  if (tid < kNB) {
    const int ar = tid;
    for (int c = 0; c < kNB; ++c) Ts[ar][c] = 0.0;
    if (ar < nb) {
      Ts[ar][ar] = tau[k0 + ar];
      for (int c = ar + 1; c < nb; ++c) {
        double acc = 0.0;
        for (int bb = ar; bb < c; ++bb) acc = fma(Ts[ar][bb], Gs[bb][c], acc);
        Ts[ar][c] = -tau[k0 + c] * acc;
      }
    }
  }
  __syncthreads();
  for (int t = tid; t < kNB * kNB; t += blockDim.x) T[t] = Ts[t / kNB][t % kNB];
}

// identity when the preconditioner failed (flags[0] != 0)
__global__ void __launch_bounds__(256) backtransform_kernel(const double *__restrict__ Zall,
                                                            const double *__restrict__ Vall,
                                                            const double *__restrict__ Tall, int n, int jchunk,
                                                            const int *__restrict__ flags,
                                                            double *__restrict__ V0all) {
  extern __shared__ __align__(16) double zs[];  // [n][kBtCols], then vsb[kNB][jchunk]
  double *vsb = zs + (size_t)n * kBtCols;
  __shared__ double w1[kNB][kBtCols];
  __shared__ double w2[kNB][kBtCols];
  __shared__ double ts[kNB][kNB + 1];
  const int prob = blockIdx.y;
  const int nblk = (n - 2 + kNB - 1) / kNB;
  const double *Z = Zall + (size_t)prob * n * n;
  const double *V = Vall + (size_t)prob * n * n;
  const double *Tb = Tall + (size_t)prob * nblk * kNB * kNB;
  double *V0 = V0all + (size_t)prob * n * n;
  const int c0 = blockIdx.x * kBtCols;
  const int tid = threadIdx.x;
  const bool bad = flags[prob * 4] != 0;
  if (bad) {
    for (int t = tid; t < n * kBtCols; t += blockDim.x) {
      const int j = t / kBtCols, c = c0 + t % kBtCols;
      if (c < n) V0[(size_t)j * n + c] = (j == c) ? 1.0 : 0.0;
    }
    return;
  }
  for (int t = tid; t < n * kBtCols; t += blockDim.x) {
    const int j = t / kBtCols, c = c0 + t % kBtCols;
    zs[t] = c < n ? Z[(size_t)j * n + c] : 0.0;
  }
  const int sc = tid % kBtCols, rc = tid / kBtCols;  // 256 threads: 32 x kBtCols
  // stage columns [j0, j0 + len) of the block's vectors (zero left of each vector's start)
  const int lane = tid & 31, warp = tid >> 5;
  auto stage = [&](int k0, int nb, int j0, int len) {  // warp per vector row, lanes along j
    for (int r = warp; r < kNB; r += 8) {
      const double *src = V + (size_t)(k0 + r) * n;
      double *dst = vsb + (size_t)r * jchunk - j0;
      for (int j = j0 + lane; j < j0 + len; j += 32) dst[j] = (r < nb && j > k0 + r) ? __ldcg(src + j) : 0.0;
    }
  };
  for (int blk = nblk - 1; blk >= 0; --blk) {
    const int k0 = blk * kNB, nb = min(kNB, n - 2 - k0);
    for (int t = tid; t < kNB * kNB; t += blockDim.x) ts[t / kNB][t % kNB] = Tb[(size_t)blk * kNB * kNB + t];
    // W1[c][s] = v_{k0+c} . Z[:, s]
    double a0 = 0.0, a1 = 0.0, a2 = 0.0, a3 = 0.0;
    for (int j0 = k0 + 1; j0 < n; j0 += jchunk) {
      const int len = min(jchunk, n - j0);
      __syncthreads();
      stage(k0, nb, j0, len);
      __syncthreads();
      const double *vr = vsb + (size_t)rc * jchunk;
      const double *zc = zs + (size_t)j0 * kBtCols + sc;
      int j = max(0, k0 + rc + 1 - j0);  // v_{k0+rc} is zero before column k0 + rc + 1
#pragma unroll 2
      for (; j + 3 < len; j += 4) {
        a0 = fma(vr[j], zc[j * kBtCols], a0);
        a1 = fma(vr[j + 1], zc[(j + 1) * kBtCols], a1);
        a2 = fma(vr[j + 2], zc[(j + 2) * kBtCols], a2);
        a3 = fma(vr[j + 3], zc[(j + 3) * kBtCols], a3);
      }
      for (; j < len; ++j) a0 = fma(vr[j], zc[j * kBtCols], a0);
    }
    w1[rc][sc] = (a0 + a1) + (a2 + a3);
    __syncthreads();
    // W2 = T_b W1
    {
      double acc = 0.0;
      for (int c = rc; c < nb; ++c) acc = fma(ts[rc][c], w1[c][sc], acc);
      w2[rc][sc] = acc;
    }
    // Z[j][s] -= sum_c v_{k0+c}[j] W2[c][s]   (a block whose vectors fit one chunk is still staged
    // from the W1 pass: half the L2 traffic of the kernel at w <= 657)
    const bool single = k0 + 1 + jchunk >= n;
    for (int j0 = k0 + 1; j0 < n; j0 += jchunk) {
      const int len = min(jchunk, n - j0);
      __syncthreads();
      if (!single) {
        stage(k0, nb, j0, len);
        __syncthreads();
      }
      double w2r[kNB];
#pragma unroll
      for (int c = 0; c < kNB; ++c) w2r[c] = w2[c][sc];  // zero beyond nb (T_b is)
      for (int jj = rc; jj < len; jj += kNB) {
        // vsb is zero where v_{k0+c}[j] is (j <= k0 + c, c >= nb): a fixed-length sum
        double s0 = 0.0, s1 = 0.0;
#pragma unroll
        for (int c = 0; c < kNB; c += 2) {
          s0 = fma(vsb[(size_t)c * jchunk + jj], w2r[c], s0);
          s1 = fma(vsb[(size_t)(c + 1) * jchunk + jj], w2r[c + 1], s1);
        }
        zs[(j0 + jj) * kBtCols + sc] -= s0 + s1;
      }
    }
    __syncthreads();
  }
  for (int t = tid; t < n * kBtCols; t += blockDim.x) {
    const int j = t / kBtCols, c = c0 + t % kBtCols;
    if (c < n) V0[(size_t)j * n + c] = zs[t];
  }
}

// E_ij = S_ij / (S_jj - S_ii) (i != j), 0 on the diagonal; runs only when flags[2] (the first
// orthogonality check failed); flags[1] = 1 when any |E_ij| > limit or is not finite
__global__ void refine_e_kernel(const double *__restrict__ S, int n, int64_t stride, double limit,
                                double *__restrict__ E, int *flags) {
  const int prob = blockIdx.y;
  if (flags[prob * 4 + 2] == 0) return;
  const double *Sp = S + (size_t)prob * stride;
  double *Ep = E + (size_t)prob * stride;
  bool bad = false;
  for (int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; t < (int64_t)n * n;
       t += (int64_t)gridDim.x * blockDim.x) {
    const int r = (int)(t / n), c = (int)(t % n);
    double x = 0.0;
    if (r != c) {
      const double den = Sp[(size_t)c * n + c] - Sp[(size_t)r * n + r];
      const double sij = Sp[t];
      x = sij == 0.0 ? 0.0 : sij / den;
      if (!(fabs(x) <= limit)) bad = true;
    }
    Ep[t] = x;
  }
  if (__any_sync(0xffffffffu, bad) && (threadIdx.x & 31) == 0) atomicOr(flags + prob * 4 + 1, 1);
}

// after the E kernels of all blocks: zero E when any block flagged it (P + P F == P exactly)
__global__ void refine_gate_kernel(double *__restrict__ E, int n, int64_t stride, const int *flags) {
  const int prob = blockIdx.y;
  if (flags[prob * 4 + 2] == 0 || flags[prob * 4 + 1] == 0) return;
  double *Ep = E + (size_t)prob * stride;
  for (int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; t < (int64_t)n * n;
       t += (int64_t)gridDim.x * blockDim.x)
    Ep[t] = 0.0;
}

// dst <- src when the refinement did not run (flags[2] == 0)
__global__ void copy_if_converged_kernel(const double *__restrict__ src, double *__restrict__ dst, int64_t count,
                                         int64_t stride, const int *flags) {
  const int prob = blockIdx.y;
  if (flags[prob * 4 + 2] != 0) return;
  const double *sp = src + (size_t)prob * stride;
  double *dp = dst + (size_t)prob * stride;
  for (int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; t < count; t += (int64_t)gridDim.x * blockDim.x)
    dp[t] = sp[t];
}

// orthogonality check: flags[slot] = 1 when some column pair of W' fails the reference's test
// |apq| <= tol sqrt(app aqq) (_core.pyx:104) or anything is not finite; with gate_slot >= 0 it
// runs only when flags[gate_slot] != 0
__global__ void offrel_check_kernel(const double *__restrict__ S, int n, int64_t stride, double tol2, int *flags,
                                    int slot, int gate_slot) {
  const int prob = blockIdx.y;
  if (gate_slot >= 0 && flags[prob * 4 + gate_slot] == 0) return;
  const double *Sp = S + (size_t)prob * stride;
  bool need = false;
  for (int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; t < (int64_t)n * n;
       t += (int64_t)gridDim.x * blockDim.x) {
    const int r = (int)(t / n), c = (int)(t % n);
    if (r == c) continue;
    const double sij = Sp[t], sii = Sp[(size_t)r * n + r], sjj = Sp[(size_t)c * n + c];
    if (!(sij * sij <= tol2 * (sii * sjj))) need = true;
  }
  if (__any_sync(0xffffffffu, need) && (threadIdx.x & 31) == 0) atomicOr(flags + prob * 4 + slot, 1);
}

// the Jacobi sweeps still run when the first check failed and the refined one failed too
__global__ void jacobi_gate_kernel(const int *flags, int *gate, int batch) {
  const int prob = blockIdx.x * blockDim.x + threadIdx.x;
  if (prob < batch) gate[prob] = (flags[prob * 4 + 2] != 0 && flags[prob * 4 + 3] != 0) ? 1 : 0;
}

}  // namespace

// ================================================================== host side
struct EigPlan {
  int C = 0, threads = 0, ldr = 0, rm = 0, nsm = 0;
  int64_t ag_rows = 0;  // rows per CTA in global scratch
  size_t smem = 0;
  bool ok = false;
};

// sytrd_push_kernel<E, RM>: RM rows per row warp in registers (0: none)
static void (*sytrd_push_pick(int n, int rm))(SytrdArgs) {
  const int E = (n + 31) / 32;
#define LRAMM_SP(EE, RR) \
  if (E == EE && rm == RR) return sytrd_push_kernel<EE, RR>;
  LRAMM_SP(1, 3) LRAMM_SP(2, 3) LRAMM_SP(3, 3) LRAMM_SP(4, 3) LRAMM_SP(5, 3) LRAMM_SP(6, 3) LRAMM_SP(7, 3)
  LRAMM_SP(8, 3) LRAMM_SP(9, 3) LRAMM_SP(10, 3) LRAMM_SP(11, 3) LRAMM_SP(12, 3)
  LRAMM_SP(1, 6) LRAMM_SP(2, 6) LRAMM_SP(3, 6) LRAMM_SP(4, 6) LRAMM_SP(5, 6) LRAMM_SP(6, 6) LRAMM_SP(7, 6)
  LRAMM_SP(8, 6) LRAMM_SP(9, 6) LRAMM_SP(10, 6) LRAMM_SP(11, 6) LRAMM_SP(12, 6)
  LRAMM_SP(13, 0) LRAMM_SP(14, 0) LRAMM_SP(15, 0) LRAMM_SP(16, 0) LRAMM_SP(17, 0) LRAMM_SP(18, 0)
  LRAMM_SP(19, 0) LRAMM_SP(20, 0) LRAMM_SP(21, 0) LRAMM_SP(22, 0) LRAMM_SP(23, 0) LRAMM_SP(24, 0)
  LRAMM_SP(25, 0) LRAMM_SP(26, 0) LRAMM_SP(27, 0) LRAMM_SP(28, 0) LRAMM_SP(29, 0) LRAMM_SP(30, 0)
  LRAMM_SP(31, 0) LRAMM_SP(32, 0) LRAMM_SP(33, 0)
#undef LRAMM_SP
  return nullptr;
}

static size_t sytrd_fixed_smem(int n, int C, int ldr) {
  return (size_t)(4 * (int64_t)n + 2 * ceil_div(n, C) + 3 * (int64_t)ldr) * sizeof(double);
}

// Row placement: up to n = 384 every row lives in registers (3 or 6 per row warp, the cluster
// the smallest power of two that allows it; batched problems prefer fewer CTAs each); wider
// problems use a 16-CTA cluster with the rows in shared memory, spilling to L2-resident global
// scratch when they do not fit (w = 1056: 66 rows per CTA, ~20 in shared memory).
static EigPlan plan_sytrd(int n, int batch) {
  EigPlan p;
  static const int env_c = [] {
    const char *s = getenv("LRAMM_EIG_CLUSTER");
    return s ? atoi(s) : 0;
  }();
  const int E = (n + 31) / 32, nrw = kSytrdWarps - 2;
  if (E > kSytrdMaxE) return p;
  int optin = 0, dev = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev);
  const size_t budget = (size_t)optin - 4096;
  p.ldr = 32 * E + 1;  // rows padded to 32 E columns (odd stride)
  auto rows_per_warp = [&](int C) { return (int)ceil_div(ceil_div(n, C), nrw); };
  const int cands[5] = {1, 2, 4, 8, 16};
  int pick = 0, rm = 0;
  if (E <= kSytrdRegMaxE) {
    for (int want : {3, 6}) {
      for (int C : cands) {
        if (env_c > 0 && C != env_c) continue;
        if (batch < 16 && want == 3 && C < 16 && rows_per_warp(C) > 3) continue;
        if (rows_per_warp(C) <= want && sytrd_fixed_smem(n, C, p.ldr) <= budget) {
          pick = C;
          rm = want;
          break;
        }
      }
      if (pick) break;
    }
  }
  if (!pick) {
    pick = env_c > 0 ? env_c : 16;
    rm = 0;
  }
  const size_t fixed = sytrd_fixed_smem(n, pick, p.ldr);
  if (fixed > budget) return p;
  const int64_t rows = ceil_div(n, pick) - (int64_t)nrw * rm;
  p.nsm = (int)std::max<int64_t>(0, std::min<int64_t>(rows, (int64_t)((budget - fixed) / (p.ldr * sizeof(double)))));
  p.ag_rows = std::max<int64_t>(0, rows - p.nsm);
  p.C = pick;
  p.rm = rm;
  p.threads = 32 * kSytrdWarps;
  p.smem = fixed + (size_t)p.nsm * p.ldr * sizeof(double);
  p.ok = sytrd_push_pick(n, rm) != nullptr;
  return p;
}

static size_t twisted_smem(int n, int tpb) { return (size_t)(2 * n + 2 * (size_t)n * tpb) * sizeof(double); }
static int twisted_threads(int n) {
  int t = 32;
  while (t > 1 && twisted_smem(n, t) > 200 * 1024) t >>= 1;
  return t;
}

// whether the preconditioner runs for an n x n Jacobi (LRAMM_EIG_PRE = 0 / 1 overrides)
bool eig_precondition_enabled(int n, int batch) {
  static const int env = [] {
    const char *s = getenv("LRAMM_EIG_PRE");
    return s ? atoi(s) : -1;
  }();
  if (env == 0) return false;
  if (n < 3) return false;
  if (env != 1 && n < 48) return false;
  return plan_sytrd(n, batch).ok;
}

struct EigWs {
  double *Rt, *G, *V, *Z, *D, *Zo, *V0, *P, *S, *E, *P2, *d, *e, *tau, *lam, *T, *gemm, *Ag;
  int *flags;
  size_t gemm_bytes;
};
static EigWs carve_eig(Arena &ar, int n, int batch) {
  EigWs w;
  const int64_t nn = (int64_t)n * n * batch;
  w.Rt = ar.take<double>(nn);
  w.G = ar.take<double>(nn);
  w.V = ar.take<double>(nn);
  w.Z = ar.take<double>(nn);
  w.D = ar.take<double>(nn);
  w.Zo = ar.take<double>(nn);
  w.V0 = ar.take<double>(nn);
  w.P = ar.take<double>(nn);
  w.S = ar.take<double>(nn);
  w.E = ar.take<double>(nn);
  w.P2 = ar.take<double>(nn);
  w.d = ar.take<double>((int64_t)n * batch);
  w.e = ar.take<double>((int64_t)n * batch);
  w.tau = ar.take<double>((int64_t)n * batch);
  w.lam = ar.take<double>((int64_t)n * batch);
  w.T = ar.take<double>(ceil_div(n - 2, kNB) * kNB * kNB * batch);
  w.flags = ar.take<int>(4 * batch);
  w.gemm_bytes = std::max(dgemm_ws_bytes(1, n, n, n), dgemm_ws_bytes(0, n, n, n));
  w.gemm = ar.take<double>((int64_t)(w.gemm_bytes / 8 + 1));
  const EigPlan pl = plan_sytrd(n, batch);
  w.Ag = pl.ag_rows > 0 ? ar.take<double>((int64_t)batch * pl.C * pl.ag_rows * pl.ldr) : nullptr;
  return w;
}

size_t eig_precondition_ws_bytes(int n, int batch) {
  Arena ar;
  ar.dry = true;
  carve_eig(ar, n, batch);
  return ar.off + 256;
}

// R: n x n row-major (the Jacobi operand W = R^T, column-major), one problem (batch == 1).
// On return R holds R' = (W V0)^T (or R unchanged when the preconditioner failed) and
// *jac_gate (device int) is nonzero when the Jacobi sweeps still have to run.
int eig_precondition_device(double *R, int n, int *jac_gate, void *ws, size_t ws_bytes, cudaStream_t st) {
  const int batch = 1;
  EigPlan p = plan_sytrd(n, batch);
  if (!p.ok) return fail(LRAMM_ERR_UNSUPPORTED, "eig preconditioner: n = %d does not fit", n);
  Arena ar(ws, ws_bytes);
  EigWs w = carve_eig(ar, n, batch);
  if (!ar.ok()) return fail(LRAMM_ERR_WORKSPACE, "eig preconditioner: workspace too small");
  LRAMM_CUDA_TRY(cudaMemsetAsync(w.flags, 0, 4 * sizeof(int) * batch, st));
  LRAMM_CUDA_TRY(cudaMemsetAsync(w.V, 0, (size_t)n * n * sizeof(double) * batch, st));
  // G = R R^T = Rt^T Rt
  LRAMM_TRY(transpose_device(R, n, n, n, w.Rt, n, st));
  DgemmOptions sym;
  sym.sym = 1;
  LRAMM_TRY(dgemm_device_ex(1, n, n, n, w.Rt, n, w.Rt, n, w.G, n, w.gemm, w.gemm_bytes, st, sym));
  // tridiagonalisation
  {
    void (*kern)(SytrdArgs) = sytrd_push_pick(n, p.rm);
    if (!kern) return fail(LRAMM_ERR_UNSUPPORTED, "eig preconditioner: n = %d too wide", n);
    static PerDeviceOnce once;
    LRAMM_CUDA_TRY(once.run([] {
      cudaError_t e = cudaSuccess;
      for (int E = 1; E <= kSytrdMaxE && e == cudaSuccess; ++E)
        for (int rm : {0, 3, 6}) {
          void (*k)(SytrdArgs) = sytrd_push_pick(32 * E, rm);
          if (!k) continue;
          e = allow_max_dyn_smem(k);
          if (e == cudaSuccess) e = cudaFuncSetAttribute(k, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
        }
      if (e == cudaSuccess) e = allow_max_dyn_smem(backtransform_kernel);
      if (e == cudaSuccess) e = allow_max_dyn_smem(reflector_t_kernel);
      if (e == cudaSuccess) e = allow_max_dyn_smem(tridiag_twisted_kernel);
      return e;
    }));
    SytrdArgs a;
    a.G = w.G;
    a.ldg = n;
    a.g_stride = (int64_t)n * n;
    a.n = n;
    a.d = w.d;
    a.e = w.e;
    a.tau = w.tau;
    a.V = w.V;
    a.ldr = p.ldr;
    a.nsm = p.nsm;
    a.Ag = p.ag_rows > 0 ? w.Ag : nullptr;
    a.ag_rows = p.ag_rows;
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3((unsigned)(p.C * batch));
    cfg.blockDim = dim3((unsigned)p.threads);
    cfg.dynamicSmemBytes = p.smem;
    cfg.stream = st;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = (unsigned)p.C;
    attr[0].val.clusterDim.y = 1;
    attr[0].val.clusterDim.z = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    LRAMM_CUDA_TRY(cudaLaunchKernelEx(&cfg, kern, a));
  }
  // eigenvalues, eigenvectors of T
  {
    const int wpb = 2 * kBisWpe;  // two eigenvalues per block: the warps spread over the SMs
    tridiag_bisect_kernel<<<dim3((unsigned)ceil_div(n, wpb / kBisWpe), batch), 32 * wpb, (size_t)2 * n * sizeof(double), st>>>(
        w.d, w.e, n, w.lam);
    LRAMM_LAUNCH_CHECK();
    const int tpb = twisted_threads(n);
    tridiag_twisted_kernel<<<dim3((unsigned)ceil_div(n, tpb), batch), tpb, twisted_smem(n, tpb), st>>>(w.d, w.e, n,
                                                                                                  w.lam, w.Z);
    LRAMM_LAUNCH_CHECK();
  }
  const unsigned eblocks = (unsigned)std::min<int64_t>(ceil_div((int64_t)n * n, 256), 4LL * num_sms());
  // Lowdin: D = Z^T Z - I; Zo = Z - Z D / 2; a defect above 1e-4 (clustered eigenvalues) means
  // the preconditioner failed -> identity (Jacobi on the untouched W)
  LRAMM_TRY(dgemm_device_ex(1, n, n, n, w.Z, n, w.Z, n, w.D, n, w.gemm, w.gemm_bytes, st, sym));
  eig_defect_kernel<<<dim3(eblocks, batch), 256, 0, st>>>(w.D, n, (int64_t)n * n, 1e-4, w.flags);
  LRAMM_LAUNCH_CHECK();
  {
    DgemmOptions lo;
    lo.alpha = -0.5;
    lo.beta = 1.0;
    lo.cin = w.Z;
    lo.ldci = n;
    LRAMM_TRY(dgemm_device_ex(0, n, n, n, w.Z, n, w.D, n, w.Zo, n, w.gemm, w.gemm_bytes, st, lo));
  }
  {
    const int nblk = (int)ceil_div(n - 2, kNB);
    int optin = 0, dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev);
    const int64_t budget = optin - 24 * 1024;  // static shared memory of the two kernels: < 17 KB
    const int jt = (int)std::min<int64_t>(n, budget / (kNB * 8));
    reflector_t_kernel<<<dim3((unsigned)nblk, batch), 256, (size_t)kNB * jt * sizeof(double), st>>>(w.V, w.tau, n, jt,
                                                                                                 w.T);
    LRAMM_LAUNCH_CHECK();
    const int jb = (int)std::min<int64_t>(n, (budget - (int64_t)n * kBtCols * 8) / (kNB * 8));
    backtransform_kernel<<<dim3((unsigned)ceil_div(n, kBtCols), batch), 256,
                           (size_t)(n * kBtCols + kNB * jb) * sizeof(double), st>>>(w.Zo, w.V, w.T, n, jb, w.flags,
                                                                                    w.V0);
    LRAMM_LAUNCH_CHECK();
  }
  // P = W V0 = Rt V0 (row-major P == W' as a plain matrix); check; one-sided refinement only
  // when the check failed: P2 = P + P F, F = E + E^2 / 2 (orthogonal to O(|E|^3))
  LRAMM_TRY(dgemm_device_ex(0, n, n, n, w.Rt, n, w.V0, n, w.P, n, w.gemm, w.gemm_bytes, st, DgemmOptions{}));
  LRAMM_TRY(dgemm_device_ex(1, n, n, n, w.P, n, w.P, n, w.S, n, w.gemm, w.gemm_bytes, st, sym));
  offrel_check_kernel<<<dim3(eblocks, batch), 256, 0, st>>>(w.S, n, (int64_t)n * n, 1e-26, w.flags, 2, -1);
  LRAMM_LAUNCH_CHECK();
  // P2 = P when the first check passed; otherwise the refinement below (mutually exclusive writers of
  // P2).  The refinement and its second check are one IF node of a captured graph (batch == 1).
  copy_if_converged_kernel<<<dim3(eblocks, batch), 256, 0, st>>>(w.P, w.P2, (int64_t)n * n, (int64_t)n * n, w.flags);
  LRAMM_LAUNCH_CHECK();
  {
    CondIf sec;
    if (batch == 1) LRAMM_TRY(sec.begin(st, w.flags + 2, true));
    cudaStream_t s2 = sec.stream();
    refine_e_kernel<<<dim3(eblocks, batch), 256, 0, s2>>>(w.S, n, (int64_t)n * n, 1e-4, w.E, w.flags);
    LRAMM_LAUNCH_CHECK();
    refine_gate_kernel<<<dim3(eblocks, batch), 256, 0, s2>>>(w.E, n, (int64_t)n * n, w.flags);
    LRAMM_LAUNCH_CHECK();
    DgemmOptions f;  // F = E + E E / 2   (into D: free after the Lowdin step)
    f.alpha = 0.5;
    f.beta = 1.0;
    f.cin = w.E;
    f.ldci = n;
    f.gate = w.flags + 2;
    f.gate_run_if_nonzero = 1;
    LRAMM_TRY(dgemm_device_ex(0, n, n, n, w.E, n, w.E, n, w.D, n, w.gemm, w.gemm_bytes, s2, f));
    DgemmOptions rf;  // P2 = P + P F
    rf.alpha = 1.0;
    rf.beta = 1.0;
    rf.cin = w.P;
    rf.ldci = n;
    rf.gate = w.flags + 2;
    rf.gate_run_if_nonzero = 1;
    LRAMM_TRY(dgemm_device_ex(0, n, n, n, w.P, n, w.D, n, w.P2, n, w.gemm, w.gemm_bytes, s2, rf));
    DgemmOptions sg = sym;
    sg.gate = w.flags + 2;
    sg.gate_run_if_nonzero = 1;
    LRAMM_TRY(dgemm_device_ex(1, n, n, n, w.P2, n, w.P2, n, w.S, n, w.gemm, w.gemm_bytes, s2, sg));
    offrel_check_kernel<<<dim3(eblocks, batch), 256, 0, s2>>>(w.S, n, (int64_t)n * n, 1e-26, w.flags, 3, 2);
    LRAMM_LAUNCH_CHECK();
    LRAMM_TRY(sec.end());
  }
  // R' = P2^T (the Jacobi operand, column-major W')
  LRAMM_TRY(transpose_device(w.P2, n, n, n, R, n, st));
  jacobi_gate_kernel<<<1, 32, 0, st>>>(w.flags, jac_gate, batch);
  LRAMM_LAUNCH_CHECK();
  return LRAMM_OK;
}

}  // namespace lramm
