// Warp-block one-sided Jacobi (the reference's _core.jacobi_sweeps semantics, _core.pyx:72-133:
// tol 1e-13, <= 60 sweeps, per-sweep column-norm refresh, tau/t/c/s rotation, norm update,
// stop after a sweep without rotations) for widths whose columns fit in registers.
//
// Layout: 2N column blocks of BS (even) columns; warp g of the cluster keeps the blocks at
// circle positions g (top, X) and 2N-1-g (bottom, Y) in REGISTERS, rows spread over the 32
// lanes (row = lane + 32 r, r < NR).  A round pairs every X column with every Y column in BS
// steps of BS disjoint rotations (X_i with Y_(i+s) mod BS, unrolled: static registers); the first
// round of a sweep also pairs the columns inside each block (circle method inside the block,
// BS-1 steps).  A step is register-local: the BS dot products are reduce-scattered over the
// warp, lane group i evaluates the angle and new norms of rotation i (one evaluation per step
// instead of one per lane per rotation), the results are broadcast with shuffles, and every
// lane applies the rotations to its rows.  No shared-memory traffic and no barrier inside a round.
// Between rounds the blocks move one circle position (top -> warp g+1, bottom -> warp g-1):
// to a warp of the same CTA with st.shared + an mbarrier arrive by every lane, to a warp of a
// neighbouring CTA of the cluster with st.async completing on the receiver's mbarrier (the
// bytes are the transaction count).  Warps synchronise only with their two neighbours; one
// cluster barrier per sweep combines the "rotated" flags.
//
// OPT-IN (LRAMM_JACOBI_WB=1), measured slower than the shared-memory cluster kernel on B200:
// at w = 272 (c2) the SVD takes 3.56 ms (BS 4, 4 warps/CTA, 9 CTAs) / 3.60 ms (BS 2, 8
// warps/CTA) against 3.17 ms, at w = 74 0.79 vs 0.59 ms (scripts/jac_wb_check.py).  ncu
// (BS 4): ~470 instructions per step per warp (DP core 180; reduce-scatter, angle, broadcasts,
// selects and moves the rest) at ~4.5 cycles per instruction with one warp per scheduler
// (fixed-latency dependency and shuffle stalls), plus the neighbour waits of the exchange
// wavefront; the step is not cheaper than the smem kernel's ~1.7k cycles.  Kept as the
// documented experiment; the dispatcher uses it only when asked.
#include <cooperative_groups.h>

#include <algorithm>
#include <cstdlib>

#include "common.cuh"
#include "sm100.cuh"

namespace cg = cooperative_groups;

namespace lramm {
namespace {

struct WbArgs {
  double *W;  // column-major, ncols columns of `rows` (ld = ldw) per problem
  int64_t ldw, batch_stride;
  int rows, ncols;
  int N;   // block pairs (= working warps) per problem
  int Wc;  // warps per CTA
  double tol;
  int max_sweeps;
  int *info;  // per problem: sweeps, or -1 when max_sweeps was reached
};

__device__ __forceinline__ uint32_t mapa_u32(uint32_t addr, uint32_t rank) {
  uint32_t r;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(r) : "r"(addr), "r"(rank));
  return r;
}
__device__ __forceinline__ void st_async_b64(uint32_t addr, double v, uint32_t mbar) {
  asm volatile("st.async.shared::cluster.mbarrier::complete_tx::bytes.b64 [%0], %1, [%2];" ::"r"(addr),
               "l"(__double_as_longlong(v)), "r"(mbar)
               : "memory");
}
__device__ __forceinline__ void st_async_v2(uint32_t addr, double v0, double v1, uint32_t mbar) {
  asm volatile("st.async.shared::cluster.mbarrier::complete_tx::bytes.v2.b64 [%0], {%1, %2}, [%3];" ::"r"(addr),
               "l"(__double_as_longlong(v0)), "l"(__double_as_longlong(v1)), "r"(mbar)
               : "memory");
}
__device__ __forceinline__ void mbar_arrive_local(uint64_t *bar) {
  asm volatile("mbarrier.arrive.release.cta.shared::cta.b64 _, [%0];" ::"r"(sm100::smem_u32(bar)) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t *bar, uint32_t parity) {
  asm volatile(
      "{\n\t.reg .pred p;\n"
      "WB_WAIT_%=:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
      "@!p bra WB_WAIT_%=;\n}\n" ::"r"(sm100::smem_u32(bar)),
      "r"(parity)
      : "memory");
}

constexpr int kWbThreads = 256;  // <= 2 warps per SMSP, each with the full 255 registers
constexpr int kWbMaxWarps = 8;

template <int NR>
__device__ __forceinline__ double dot_lane(const double (&a)[NR], const double (&b)[NR]) {
  double s0 = 0.0, s1 = 0.0;
#pragma unroll
  for (int i = 0; i < NR; ++i) {
    if (i & 1)
      s1 = fma(a[i], b[i], s1);
    else
      s0 = fma(a[i], b[i], s0);
  }
  return s0 + s1;
}

template <int K>
__device__ __forceinline__ void butterfly(double (&v)[K]) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
#pragma unroll
    for (int k = 0; k < K; ++k) v[k] += __shfl_xor_sync(0xffffffffu, v[k], o);
  }
}

template <int K>
__device__ __forceinline__ double pick(const double (&v)[K], int j) {
  double r = v[0];
#pragma unroll
  for (int k = 1; k < K; ++k) r = j == k ? v[k] : r;
  return r;
}

// (c, s) of the reference's rotation of the pair (p, q) (_core.pyx:114-119: tau = (aqq - app) /
// (2 apq), t = sign(tau)/(|tau| + sqrt(1 + tau^2)), c = 1/sqrt(1 + t^2), s = c t), evaluated
// through the double angle without a division:
//   r1 = 1/sqrt(d^2 + 4 apq^2), cos2 = |d| r1, sin2 = 2|apq| r1, r2 = 1/sqrt(2 (1 + cos2)),
//   c = (1 + cos2) r2, s = sign(tau) sin2 r2.
// Safe for any input (a skipped pair evaluates the identity).
__device__ __forceinline__ void rot_cs(double app, double aqq, double apq, bool go, double &c, double &s) {
  const double d = go ? aqq - app : 1.0;
  const double g = go ? apq : 0.0;
  const double r1 = rsqrt(fma(d, d, 4.0 * g * g));
  const double cos2 = fabs(d) * r1, sin2 = 2.0 * fabs(g) * r1;
  const double opc = 1.0 + cos2;
  const double r2 = rsqrt(2.0 * opc);
  const double sgn = (d == 0.0) ? 1.0 : ((d > 0.0) == (g > 0.0) ? 1.0 : -1.0);
  c = opc * r2;
  s = sgn * sin2 * r2;
}

// Sum over the warp of v[k] for k = lane / (32 / K), by recursive halving (each of the first
// log2 K levels sends half of the remaining values) and a butterfly on the last value:
// 2 (K - 1 + 5 - log2 K) shuffles instead of 10 K.
template <int K>
__device__ __forceinline__ double reduce_scatter(const double (&v)[K], int lane) {
  static_assert(K == 1 || K == 2 || K == 4 || K == 8 || K == 16, "K must be a power of two <= 16");
  double cur[K];
#pragma unroll
  for (int k = 0; k < K; ++k) cur[k] = v[k];
  int o = 16;
#pragma unroll
  for (int M = K; M > 1; M >>= 1, o >>= 1) {
    const bool up = (lane & o) != 0;
#pragma unroll
    for (int j = 0; j < M / 2; ++j) {
      const double send = up ? cur[j] : cur[j + M / 2];
      const double keep = up ? cur[j + M / 2] : cur[j];
      cur[j] = keep + __shfl_xor_sync(0xffffffffu, send, o);
    }
  }
  double r = cur[0];
#pragma unroll
  for (; o > 0; o >>= 1) r += __shfl_xor_sync(0xffffffffu, r, o);
  return r;
}

// K rotations of the pairs (A_k, B_k): apq reduce-scattered over the warp, lane group k
// (32/K lanes) evaluates the decision, angle and new norms of rotation k, the results are
// broadcast with shuffles and every lane applies the rotations to its rows.  pf(k): A_k is the
// reference's p column (lower index).  A, B, an, bn are accessors into the caller's register
// arrays (static indices after unrolling).
template <int NR, int K, class GetA, class GetB, class NA, class NB, class PF>
__device__ __forceinline__ void rotate_pairs(GetA A, GetB B, NA an, NB bn, PF pf, double tol2, int lane,
                                             bool &rotated) {
  constexpr int GS = 32 / K;
  double apq[K], av[K], bv[K];
#pragma unroll
  for (int k = 0; k < K; ++k) {
    apq[k] = dot_lane<NR>(A(k), B(k));
    av[k] = an(k);
    bv[k] = bn(k);
  }
  const int kk = lane / GS;
  const double g = reduce_scatter<K>(apq, lane);
  bool pk = pf(0);
#pragma unroll
  for (int k = 1; k < K; ++k) pk = kk == k ? pf(k) : pk;
  const double na = pick<K>(av, kk), nb = pick<K>(bv, kk);
  const double app = pk ? na : nb, aqq = pk ? nb : na;
  const bool go = app != 0.0 && aqq != 0.0 && g * g > tol2 * (app * aqq);
  double c, s;
  rot_cs(app, aqq, g, go, c, s);
  double se = pk ? s : -s;  // applied as A' = c A - se B, B' = se A + c B
  const double npn = c * c * app - 2.0 * c * s * g + s * s * aqq;
  const double nqn = s * s * app + 2.0 * c * s * g + c * c * aqq;
  double nA = pk ? npn : nqn, nB = pk ? nqn : npn;
  if (!go) {
    c = 1.0;
    se = 0.0;
    nA = na;
    nB = nb;
  }
  double C[K], S[K];
#pragma unroll
  for (int k = 0; k < K; ++k) {  // convergent shuffles, outside the branches
    C[k] = __shfl_sync(0xffffffffu, c, k * GS);
    S[k] = __shfl_sync(0xffffffffu, se, k * GS);
    an(k) = __shfl_sync(0xffffffffu, nA, k * GS);
    bn(k) = __shfl_sync(0xffffffffu, nB, k * GS);
  }
  bool any = false;
#pragma unroll
  for (int k = 0; k < K; ++k) any |= S[k] != 0.0;
  if (any) {  // warp-uniform; a skipped pair (_core.pyx:104-109) applies the identity (c 1, s 0)
    rotated = true;
#pragma unroll
    for (int k = 0; k < K; ++k) {
      double(&a)[NR] = A(k);
      double(&b)[NR] = B(k);
#pragma unroll
      for (int i = 0; i < NR; ++i) {
        const double x = a[i], y = b[i];
        a[i] = C[k] * x - S[k] * y;
        b[i] = S[k] * x + C[k] * y;
      }
    }
  }
}

template <int NR, int BS>
__device__ __forceinline__ void norms(const double (&V)[BS][NR], double (&vn)[BS]) {
#pragma unroll
  for (int c = 0; c < BS; ++c) vn[c] = dot_lane<NR>(V[c], V[c]);
  butterfly<BS>(vn);
}

// rotate register slots lo..BS-1 by one: V[j] <- V[j+1], V[BS-1] <- V[lo]
template <int NR, int BS>
__device__ __forceinline__ void cycle(double (&V)[BS][NR], double (&vn)[BS], int lo) {
  double t[NR];
  const double tn = vn[lo];
#pragma unroll
  for (int i = 0; i < NR; ++i) t[i] = V[lo][i];
#pragma unroll
  for (int j = 0; j + 1 < BS; ++j) {
    if (j < lo) continue;
    vn[j] = vn[j + 1];
#pragma unroll
    for (int i = 0; i < NR; ++i) V[j][i] = V[j + 1][i];
  }
  vn[BS - 1] = tn;
#pragma unroll
  for (int i = 0; i < NR; ++i) V[BS - 1][i] = t[i];
}
template <int BS>
__device__ __forceinline__ void cycle_idx(int (&ix)[BS]) {
  const int t = ix[1];
#pragma unroll
  for (int j = 1; j + 1 < BS; ++j) ix[j] = ix[j + 1];
  ix[BS - 1] = t;
}

// slot layout: column c, row pair p -> double2 index (c NP + p) 32 + lane (odd last row padded),
// then the BS norms
template <int NR, int BS>
__host__ __device__ constexpr int wb_slot_doubles() { return BS * ((NR + 1) / 2) * 64 + 32; }
template <int NR, int BS>
__host__ __device__ constexpr uint32_t wb_tx_bytes() {
  return (uint32_t)((BS * (NR / 2) * 64 + (NR & 1) * BS * 32 + BS) * 8);
}

template <int NR, int BS>
__device__ __forceinline__ void push_remote(const double (&V)[BS][NR], const double (&vn)[BS], uint32_t b,
                                            uint32_t m, int lane) {
  constexpr int NP = (NR + 1) / 2;
#pragma unroll
  for (int c = 0; c < BS; ++c) {
#pragma unroll
    for (int r = 0; r + 1 < NR; r += 2)
      st_async_v2(b + (uint32_t)(((c * NP + r / 2) * 32 + lane) * 16), V[c][r], V[c][r + 1], m);
    if (NR & 1) st_async_b64(b + (uint32_t)(((c * NP + NR / 2) * 64 + lane) * 8), V[c][NR - 1], m);
  }
#pragma unroll
  for (int c = 0; c < BS; ++c)
    if (lane == c) st_async_b64(b + (uint32_t)((BS * NP * 64 + c) * 8), vn[c], m);
}

template <int NR, int BS>
__device__ __forceinline__ void push_local(const double (&V)[BS][NR], const double (&vn)[BS], double *buf,
                                           uint64_t *bar, int lane) {
  constexpr int NP = (NR + 1) / 2;
#pragma unroll
  for (int c = 0; c < BS; ++c) {
#pragma unroll
    for (int r = 0; r + 1 < NR; r += 2)
      reinterpret_cast<double2 *>(buf)[(c * NP + r / 2) * 32 + lane] = make_double2(V[c][r], V[c][r + 1]);
    if (NR & 1) buf[(c * NP + NR / 2) * 64 + lane] = V[c][NR - 1];
  }
#pragma unroll
  for (int c = 0; c < BS; ++c)
    if (lane == c) buf[BS * NP * 64 + c] = vn[c];
  mbar_arrive_local(bar);  // every lane: releases its own stores (barrier count 32)
}

template <int NR, int BS>
__device__ __forceinline__ void pull(double (&V)[BS][NR], double (&vn)[BS], const double *buf, int lane) {
  constexpr int NP = (NR + 1) / 2;
#pragma unroll
  for (int c = 0; c < BS; ++c) {
#pragma unroll
    for (int r = 0; r + 1 < NR; r += 2) {
      const double2 v = reinterpret_cast<const double2 *>(buf)[(c * NP + r / 2) * 32 + lane];
      V[c][r] = v.x;
      V[c][r + 1] = v.y;
    }
    if (NR & 1) V[c][NR - 1] = buf[(c * NP + NR / 2) * 64 + lane];
  }
#pragma unroll
  for (int c = 0; c < BS; ++c) vn[c] = buf[BS * NP * 64 + c];
}

template <int NR, int BS>
__global__ void __launch_bounds__(kWbThreads, 1) jacobi_wb_kernel(WbArgs a) {
  static_assert(BS % 2 == 0, "block width must be even");
  cg::cluster_group cl = cg::this_cluster();
  const int C = (int)cl.num_blocks();
  const int me = (int)cl.block_rank();
  const int prob = blockIdx.x / C;
  const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
  const int Wc = a.Wc, N = a.N;
  const int g = me * Wc + wid;
  const bool active = g < N;
  constexpr int SLOT = wb_slot_doubles<NR, BS>();
  constexpr uint32_t TX = wb_tx_bytes<NR, BS>();
  extern __shared__ __align__(16) double smem[];
  __shared__ __align__(8) uint64_t bars[kWbMaxWarps * 4];  // [warp][slot: 0 top-in, 1 bottom-in][parity]
  __shared__ int lf[2];
  __shared__ int gf[2][16];
  auto slot_buf = [&](int w, int s, int par) { return smem + (size_t)((w * 2 + s) * 2 + par) * SLOT; };
  auto slot_bar = [&](int w, int s, int par) { return &bars[(w * 2 + s) * 2 + par]; };
  // sources: top-in of warp g comes from warp g-1, bottom-in from warp g+1
  auto same_cta = [&](int w1, int w2) { return w1 / Wc == w2 / Wc; };
  const bool top_in = active && g >= 1;
  const bool bot_in = active && g <= N - 2;
  const bool top_remote = top_in && !same_cta(g - 1, g);
  const bool bot_remote = bot_in && !same_cta(g + 1, g);

  if (tid < Wc * 4) {
    const int w = tid >> 2, s = (tid >> 1) & 1;
    const int dst = me * Wc + w, src = s == 0 ? dst - 1 : dst + 1;
    sm100::mbar_init(&bars[tid], (src >= 0 && same_cta(src, dst)) ? 32 : 1);
  }
  if (tid < 2) lf[tid] = 0;
  if (tid == 0) sm100::fence_barrier_init();
  __syncthreads();
  if (lane == 0 && N > 1) {
#pragma unroll
    for (int par = 0; par < 2; ++par) {
      if (top_remote) sm100::mbar_arrive_expect_tx(slot_bar(wid, 0, par), TX);
      if (bot_remote) sm100::mbar_arrive_expect_tx(slot_bar(wid, 1, par), TX);
    }
  }
  cl.sync();  // every barrier initialised and armed before the first push

  double X[BS][NR], Y[BS][NR], xn[BS], yn[BS];
  double *Wp = a.W + (size_t)prob * a.batch_stride;
  const int R2 = 2 * N;
  const int home_t = g, home_b = R2 - 1 - g;
  auto load = [&](double (&V)[BS][NR], int blk) {
#pragma unroll
    for (int c = 0; c < BS; ++c) {
      const int col = blk * BS + c;
#pragma unroll
      for (int r = 0; r < NR; ++r) {
        const int row = lane + 32 * r;
        V[c][r] = (col < a.ncols && row < a.rows) ? Wp[(int64_t)col * a.ldw + row] : 0.0;
      }
    }
  };
  if (active) {
    load(X, home_t);
    load(Y, home_b);
  }
  // exchange destinations (fixed for the whole run): bottom -> warp g-1's bottom slot (warp 0:
  // warp 1's top slot), top -> warp g+1's top slot (interior warps)
  const bool send_top = active && g >= 1 && g <= N - 2;
  const int db = g >= 1 ? g - 1 : 1, sb = g >= 1 ? 1 : 0, dt = g + 1;
  const bool b_local = !active || N < 2 || same_cta(db, g), t_local = !send_top || same_cta(dt, g);
  double *b_buf = slot_buf(db % Wc, sb, 0), *t_buf = slot_buf(dt % Wc, 0, 0);
  uint64_t *b_bar = slot_bar(db % Wc, sb, 0), *t_bar = slot_bar(dt % Wc, 0, 0);
  const uint32_t b_rbuf = b_local ? 0u : mapa_u32(sm100::smem_u32(b_buf), (uint32_t)(db / Wc));
  const uint32_t b_rbar = b_local ? 0u : mapa_u32(sm100::smem_u32(b_bar), (uint32_t)(db / Wc));
  const uint32_t t_rbuf = t_local ? 0u : mapa_u32(sm100::smem_u32(t_buf), (uint32_t)(dt / Wc));
  const uint32_t t_rbar = t_local ? 0u : mapa_u32(sm100::smem_u32(t_bar), (uint32_t)(dt / Wc));
  const double tol2 = a.tol * a.tol;
  int G = 0;  // exchanges so far: exchange G uses slot parity G & 1, phase (G >> 1) & 1
  int sweeps_done = -1;
  for (int sw = 0; sw < a.max_sweeps; ++sw) {
    bool rotated = false;
    if (active) {
      norms<NR, BS>(X, xn);  // per-sweep refresh (_core.pyx:88-93)
      norms<NR, BS>(Y, yn);
      // pairs inside both home blocks: circle method on the BS slots (slot 0 fixed), BS-1 steps
      {
        int ix[BS];
#pragma unroll
        for (int c = 0; c < BS; ++c) ix[c] = c;
        constexpr int H = BS / 2;
#pragma unroll 1
        for (int t = 0; t < BS - 1; ++t) {
          rotate_pairs<NR, BS>(
              [&](int k) -> double(&)[NR] { return k < H ? X[k] : Y[k - H]; },
              [&](int k) -> double(&)[NR] { return k < H ? X[BS - 1 - k] : Y[BS - 1 - (k - H)]; },
              [&](int k) -> double & { return k < H ? xn[k] : yn[k - H]; },
              [&](int k) -> double & { return k < H ? xn[BS - 1 - k] : yn[BS - 1 - (k - H)]; },
              [&](int k) { return k < H ? ix[k] < ix[BS - 1 - k] : ix[k - H] < ix[BS - 1 - (k - H)]; }, tol2, lane,
              rotated);
          cycle<NR, BS>(X, xn, 1);
          cycle<NR, BS>(Y, yn, 1);
          cycle_idx<BS>(ix);
        }
      }
#pragma unroll 1
      for (int r = 0; r < R2 - 1; ++r) {
        // blocks at my two positions in round r: position j holds 1 + (j - 1 - r) mod (2N - 1)
        const int tb = home_t == 0 ? 0 : 1 + ((home_t - 1 - r) % (R2 - 1) + (R2 - 1)) % (R2 - 1);
        const int bb = 1 + ((home_b - 1 - r) % (R2 - 1) + (R2 - 1)) % (R2 - 1);
        const bool x_first = tb < bb;
#pragma unroll
        for (int s = 0; s < BS; ++s) {
          rotate_pairs<NR, BS>([&](int k) -> double(&)[NR] { return X[k]; },
                               [&](int k) -> double(&)[NR] { return Y[(k + s) % BS]; },
                               [&](int k) -> double & { return xn[k]; },
                               [&](int k) -> double & { return yn[(k + s) % BS]; }, [&](int) { return x_first; },
                               tol2, lane, rotated);
        }
        if (N > 1) {
          const int par = G & 1;
          const uint32_t ph = (uint32_t)(G >> 1) & 1u;
          // bottom -> position +1: warp g-1's bottom, or warp 1's top from warp 0
          if (b_local)
            push_local<NR, BS>(Y, yn, b_buf + par * SLOT, b_bar + par, lane);
          else
            push_remote<NR, BS>(Y, yn, b_rbuf + par * SLOT * 8, b_rbar + par * 8, lane);
          // top -> warp g+1's top (interior warps); warp N-1 moves its top to its own bottom
          if (send_top) {
            if (t_local)
              push_local<NR, BS>(X, xn, t_buf + par * SLOT, t_bar + par, lane);
            else
              push_remote<NR, BS>(X, xn, t_rbuf + par * SLOT * 8, t_rbar + par * 8, lane);
          }
          if (g == N - 1) {
#pragma unroll
            for (int c = 0; c < BS; ++c) {
              yn[c] = xn[c];
#pragma unroll
              for (int i = 0; i < NR; ++i) Y[c][i] = X[c][i];
            }
          }
          if (top_in) {
            mbar_wait(slot_bar(wid, 0, par), ph);
            pull<NR, BS>(X, xn, slot_buf(wid, 0, par), lane);
          }
          if (bot_in) {
            mbar_wait(slot_bar(wid, 1, par), ph);
            pull<NR, BS>(Y, yn, slot_buf(wid, 1, par), lane);
          }
          __syncwarp();
          if (lane == 0) {  // re-arm the remote slots of this parity for exchange G + 2
            if (top_remote) sm100::mbar_arrive_expect_tx(slot_bar(wid, 0, par), TX);
            if (bot_remote) sm100::mbar_arrive_expect_tx(slot_bar(wid, 1, par), TX);
          }
          ++G;
        }
      }
    }
    // cluster-wide "any rotation this sweep?" (_core.pyx:130-132)
    if (active && lane == 0 && rotated) lf[sw & 1] = 1;
    __syncthreads();
    if (tid < C) *cl.map_shared_rank(&gf[sw & 1][me], tid) = lf[sw & 1];
    cl.sync();
    int any = 0;
    for (int c = 0; c < C; ++c) any |= gf[sw & 1][c];
    if (tid == 0) lf[sw & 1] = 0;
    if (!any) {
      sweeps_done = sw + 1;
      break;
    }
  }
  // after whole sweeps every block is back at its home position (and in home slot order)
  if (active) {
    auto store = [&](const double (&V)[BS][NR], int blk) {
#pragma unroll
      for (int c = 0; c < BS; ++c) {
        const int col = blk * BS + c;
        if (col >= a.ncols) continue;
#pragma unroll
        for (int r = 0; r < NR; ++r) {
          const int row = lane + 32 * r;
          if (row < a.rows) Wp[(int64_t)col * a.ldw + row] = V[c][r];
        }
      }
    };
    store(X, home_t);
    store(Y, home_b);
  }
  if (me == 0 && tid == 0) a.info[prob] = sweeps_done;
}

// block width (power of two) per rows-per-lane: 2 BS NR <= ~72 doubles of columns per lane
constexpr int wb_bs(int nr) { return nr <= 4 ? 4 : 2; }

template <int NR>
struct WbPick {
  static constexpr int BS = wb_bs(NR);
  static void (*kernel())(WbArgs) { return jacobi_wb_kernel<NR, BS>; }
  static size_t slot_bytes() { return (size_t)wb_slot_doubles<NR, BS>() * 8; }
};

}  // namespace

// Returns LRAMM_OK when launched, 1 when the shape is outside this kernel's range (caller falls
// back to the shared-memory cluster / grid kernels), or an error status.
int jacobi_wb_device(double *W, int64_t ldw, int64_t batch_stride, int rows, int ncols, int batch, int *info,
                     cudaStream_t st) {
  static const int env = getenv("LRAMM_JACOBI_WB") ? atoi(getenv("LRAMM_JACOBI_WB")) : 0;  // opt-in: measured slower, see header
  if (!env || rows < 1 || ncols < 2) return 1;
  const int NR = (int)ceil_div(rows, 32);
  void (*kern)(WbArgs) = nullptr;
  int BS = 0;
  size_t slot = 0;
  switch (NR) {
#define LRAMM_WB(n)                 \
  case n:                           \
    kern = WbPick<n>::kernel();     \
    BS = WbPick<n>::BS;             \
    slot = WbPick<n>::slot_bytes(); \
    break;
    LRAMM_WB(1) LRAMM_WB(2) LRAMM_WB(3) LRAMM_WB(4) LRAMM_WB(5) LRAMM_WB(6) LRAMM_WB(7) LRAMM_WB(8) LRAMM_WB(9)
    LRAMM_WB(10) LRAMM_WB(11) LRAMM_WB(12)
#undef LRAMM_WB
    default: return 1;
  }
  const int N = (int)ceil_div(ncols, 2 * BS);
  static const int wmax = getenv("LRAMM_JACOBI_WB_W") ? atoi(getenv("LRAMM_JACOBI_WB_W")) : 8;
  const int Wc = std::min(N, std::max(1, std::min(wmax, kWbMaxWarps)));
  const int C = (int)ceil_div(N, Wc);
  if (C > 16 || (size_t)Wc * 4 * slot > 200 * 1024) return 1;
  WbArgs a;
  a.W = W;
  a.ldw = ldw;
  a.batch_stride = batch_stride;
  a.rows = rows;
  a.ncols = ncols;
  a.N = N;
  a.Wc = Wc;
  a.tol = 1e-13;      // _jacobi.py:10
  a.max_sweeps = 60;  // _jacobi.py:11
  a.info = info;
  const size_t smem = (size_t)Wc * 4 * slot;
  static bool attr_done[13] = {false};
  if (!attr_done[NR]) {
    LRAMM_CUDA_TRY(allow_max_dyn_smem(kern));
    LRAMM_CUDA_TRY(cudaFuncSetAttribute(kern, cudaFuncAttributeNonPortableClusterSizeAllowed, 1));
    attr_done[NR] = true;
  }
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3((unsigned)(C * batch));
  cfg.blockDim = dim3((unsigned)(32 * Wc));
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = (unsigned)C;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  LRAMM_CUDA_TRY(cudaLaunchKernelEx(&cfg, kern, a));
  return LRAMM_OK;
}

}  // namespace lramm
