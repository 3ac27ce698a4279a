// Fused absmax + symmetric quantisation (quant.py:55-71, _core.pyx:53-69) for
// per-tensor, per-row and per-column scales, int8 / int32 / packed-int4 output,
// optionally transposed so that every tensor-core operand is K-major.
//
// HBM-bound: absmax reads x once (fp32: 4 B/elem), quantize reads it again (the
// second read is usually an L2 hit for the operand sizes of the BASELINE configs)
// and writes 1 B/elem (0.5 for int4).  Loads are 128-bit where alignment allows.
#include "common.cuh"

namespace lramm {

namespace {

constexpr int kTile = 32;

// ---- vectorised tile kernels (the int8 operands of every sketch / E-product) ----
// x is read in 16-byte vectors when the base and ldx allow (VEC = 16 / sizeof(T)), else VEC = 1.

template <class T, int VEC>
__device__ __forceinline__ void load_vec(const T *__restrict__ p, int64_t c, int64_t cols, T (&v)[VEC]) {
  if (VEC > 1 && c + VEC <= cols) {
    if constexpr (VEC * sizeof(T) == 16) {
      uint4 u = __ldg(reinterpret_cast<const uint4 *>(p + c));
      memcpy(v, &u, 16);
      return;
    }
  }
#pragma unroll
  for (int k = 0; k < VEC; ++k) v[k] = c + k < cols ? p[c + k] : T(0);
}

template <class T>
__device__ __forceinline__ T vmax(T a, T b) { return fmax(a, b); }
template <>
__device__ __forceinline__ float vmax(float a, float b) { return fmaxf(a, b); }

// Tile 64 rows x (64 VEC) columns per 256-thread block; warp w covers rows w, w+8, ...; each lane two
// VEC-column chunks, loaded four rows at a time so eight 16-byte loads are in flight per thread.
// MASK selects the maxima produced in the one pass (1 per tensor, 2 per row, 4 per column), each
// combined with an atomic max into caller-zeroed outputs.  fmax drops NaN; the non-finite flag
// reports it (the reference refuses non-finite input, quant.py:59-60).
template <class T, int VEC, int MASK>
__global__ void __launch_bounds__(256, 4) absmax_tile_kernel(const T *__restrict__ x, int64_t rows, int64_t cols,
                                                             int64_t ldx, double *amax_t, double *amax_r,
                                                             double *amax_c, int *nonfinite, unsigned nbx) {
  constexpr int TC = 64 * VEC, TR = 64, RB = 4;
  constexpr bool kT = MASK & 1, kR = MASK & 2, kC = MASK & 4;
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  const int64_t r0 = (int64_t)(blockIdx.x / nbx) * TR, c0 = (int64_t)(blockIdx.x % nbx) * TC;
  T cm[2][VEC];
#pragma unroll
  for (int h = 0; h < 2; ++h)
#pragma unroll
    for (int k = 0; k < VEC; ++k) cm[h][k] = T(0);
  bool bad = false;
  T tm = T(0);
#pragma unroll 1
  for (int i0 = 0; i0 < TR / 8; i0 += RB) {
    T v[RB][2][VEC];
#pragma unroll
    for (int j = 0; j < RB; ++j) {
      const int64_t r = r0 + (int64_t)(i0 + j) * 8 + wid;
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        const int64_t c = c0 + (int64_t)(h * 32 + lane) * VEC;
        if (r < rows && c < cols) {
          load_vec<T, VEC>(x + r * ldx, c, cols, v[j][h]);
        } else {
#pragma unroll
          for (int k = 0; k < VEC; ++k) v[j][h][k] = T(0);
        }
      }
    }
#pragma unroll
    for (int j = 0; j < RB; ++j) {
      T rm = T(0);
#pragma unroll
      for (int h = 0; h < 2; ++h)
#pragma unroll
        for (int k = 0; k < VEC; ++k) {
          bad |= !isfinite(v[j][h][k]);
          T a = fabs(v[j][h][k]);
          rm = vmax(rm, a);
          if (kC) cm[h][k] = vmax(cm[h][k], a);
        }
      if (kT) tm = vmax(tm, rm);
      if (kR) {
        const int64_t r = r0 + (int64_t)(i0 + j) * 8 + wid;
        double m = warp_max((double)rm);
        if (lane == 0 && r < rows) atomic_max_nonneg(amax_r + r, m);
      }
    }
  }
  __shared__ double red[kC ? 8 : 1][kC ? 2 * 32 * VEC : 1];
  if (kC) {
#pragma unroll
    for (int h = 0; h < 2; ++h)
#pragma unroll
      for (int k = 0; k < VEC; ++k) red[wid][(h * 32 + lane) * VEC + k] = (double)cm[h][k];
  }
  __shared__ double tred[8];
  if (kT) {
    double m = warp_max((double)tm);
    if (lane == 0) tred[wid] = m;
  }
  const bool any_bad = __syncthreads_or(bad);
  if (any_bad && threadIdx.x == 0 && nonfinite) *nonfinite = 1;
  if (kC) {
    for (int j = threadIdx.x; j < TC; j += blockDim.x) {
      const int64_t c = c0 + j;
      if (c >= cols) continue;
      double m = red[0][j];
#pragma unroll
      for (int w = 1; w < 8; ++w) m = fmax(m, red[w][j]);
      atomic_max_nonneg(amax_c + c, m);
    }
  }
  if (kT && threadIdx.x == 0) {
    double m = tred[0];
#pragma unroll
    for (int w = 1; w < 8; ++w) m = fmax(m, tred[w]);
    atomic_max_nonneg(amax_t, m);
  }
}

// one side of a quantisation: int8 output, scale per tensor / input row / input column
struct QSide {
  int8_t *q;  // NULL = side not wanted
  int64_t ld;  // bytes per output row
  const double *scale;
  int gran, cap;
  int packed = 0;  // row-major side only: two's-complement nibbles, column 2j in the low nibble of byte j
  // non-NULL: the kernel derives the scales from these maxima itself (quant_scale) and writes
  // them to `scale` (no separate scales kernel)
  const double *amax = nullptr;
};

// quant_round (quant.py:70-71) in three fp64 instructions.  With scales from the true maxima
// (scale = cap / amax, |x| <= amax) |x * scale| <= cap (1 + 3 ulp) rounds into [-cap, cap] without
// a clamp; CLAMP (caller-supplied maxima) clamps first, which gives the same integer as rounding
// first since cap is an integer.  Adding 1.5 * 2^52 rounds half-to-even (the sum's ulp is 1) and
// leaves the integer in the low mantissa word; __dmul_rn / __dadd_rn keep the roundings separate.
template <bool CLAMP>
__device__ __forceinline__ uint32_t qround(double a, double scale, double capd) {
  double t = __dmul_rn(a, scale);
  if (CLAMP) t = fmin(fmax(t, -capd), capd);
  return (uint32_t)__double2loint(__dadd_rn(t, 6755399441055744.0));
}

// low bytes of four ints -> one word, a in byte 0
__device__ __forceinline__ uint32_t pack4(uint32_t a, uint32_t b, uint32_t c, uint32_t d) {
  return __byte_perm(__byte_perm(a, b, 0x0040), __byte_perm(c, d, 0x0040), 0x5410);
}

// four consecutive elements of a row (16 B for fp32, 2 x 16 B for fp64), zero past `cols`
template <class T>
__device__ __forceinline__ void load4(const T *__restrict__ row, int64_t c, int64_t cols, T (&v)[4]) {
  if (c + 4 <= cols) {
    if constexpr (sizeof(T) == 4) {
      uint4 u = __ldg(reinterpret_cast<const uint4 *>(row + c));
      memcpy(v, &u, 16);
    } else {
      uint4 u0 = __ldg(reinterpret_cast<const uint4 *>(row + c));
      uint4 u1 = __ldg(reinterpret_cast<const uint4 *>(row + c + 2));
      memcpy(v, &u0, 16);
      memcpy(v + 2, &u1, 16);
    }
    return;
  }
#pragma unroll
  for (int k = 0; k < 4; ++k) v[k] = c + k < cols ? row[c + k] : T(0);
}

// scale of element (j, k) of a thread's 4x4 micro-tile: G = 1 per input row (j), 2 per input column
// or tensor (k)
template <int G>
__device__ __forceinline__ void side_scales(const QSide &s, int64_t rb, int64_t c, int64_t rows, int64_t cols,
                                            double (&sc)[4]) {
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    if (s.amax) {  // scales derived here from the maxima (published by publish_scales)
      if (G == 1) sc[i] = rb + i < rows ? quant_scale(s.amax[rb + i], s.cap) : 0.0;
      else if (G == 2)
        sc[i] = s.gran == LRAMM_GRAN_TENSOR ? quant_scale(s.amax[0], s.cap)
                                            : (c + i < cols ? quant_scale(s.amax[c + i], s.cap) : 0.0);
    } else {
      if (G == 1) sc[i] = rb + i < rows ? s.scale[rb + i] : 0.0;
      else if (G == 2) sc[i] = s.gran == LRAMM_GRAN_TENSOR ? s.scale[0] : (c + i < cols ? s.scale[c + i] : 0.0);
    }
  }
}

// With QSide::amax the kernel writes the scales it derived: row scales by the first tile column
// (c0 == 0, one thread per micro-tile row), column scales by the first tile row, the tensor
// scale by thread 0 of block 0.
template <int G>
__device__ __forceinline__ void publish_scales(const QSide &s, int64_t rb, int64_t c, int64_t rows, int64_t cols,
                                               const double (&sc)[4]) {
  if (!s.amax) return;
  double *out = const_cast<double *>(s.scale);
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    if (G == 1) {
      if (rb + i < rows && (threadIdx.x & 15) == 0 && c < 64) out[rb + i] = sc[i];
    } else if (G == 2) {
      if (s.gran == LRAMM_GRAN_TENSOR) {
        if (i == 0 && blockIdx.x == 0 && threadIdx.x == 0) out[0] = sc[0];
      } else if (c + i < cols && (threadIdx.x >> 4) == 0 && rb < 64) {
        out[c + i] = sc[i];
      }
    }
  }
}

// Tile 64 x 64 of x per 256-thread block, a 4x4 micro-tile per thread (rows 4*tr4.., columns
// 4*tc4..).  GR / GT: the row-major side R and the transposed side T (0 absent, 1 row scales,
// 2 column / tensor scales); SAME: both sides share scales and cap, so rounding is done once.
// R is written from registers (one word per micro-tile row); T through a shared-memory tile (one
// word per micro-tile column, i.e. four input rows of one output row) and read out 64 bytes per
// output row.  Elements past rows / cols load as zero and quantise to zero, so the tile grid
// spans max(rows, T.ld) x max(cols, R.ld) and zero-fills both outputs' padding.
template <class T, int GR, int GT, bool SAME, bool CLAMP>
__global__ void __launch_bounds__(256) quantize_tile_kernel(const T *__restrict__ x, int64_t rows, int64_t cols,
                                                            int64_t ldx, QSide R, QSide Tq, unsigned nbx) {
  __shared__ uint32_t tile[GT ? 64 : 1][17];  // [input column][word of four input rows]
  const int64_t r0 = (int64_t)(blockIdx.x / nbx) * 64, c0 = (int64_t)(blockIdx.x % nbx) * 64;
  const int tc4 = threadIdx.x & 15, tr4 = threadIdx.x >> 4;
  const int64_t c = c0 + 4 * tc4, rb = r0 + 4 * tr4;
  // interior tiles (all but the last tile row / column): no bounds checks
  const bool interior = r0 + 64 <= rows && c0 + 64 <= cols;
  T v[4][4];
  if (interior) {
    const T *p = x + rb * ldx + c;
#pragma unroll
    for (int j = 0; j < 4; ++j) load4<T>(p + j * ldx, 0, 4, v[j]);
  } else {
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      if (rb + j < rows) {
        load4<T>(x + (rb + j) * ldx, c, cols, v[j]);
      } else {
#pragma unroll
        for (int k = 0; k < 4; ++k) v[j][k] = T(0);
      }
    }
  }
  double sr[4], st[4];
  if (GR) side_scales<GR>(R, rb, c, rows, cols, sr);
  if (GT && !SAME) side_scales<GT>(Tq, rb, c, rows, cols, st);
  if (GR) publish_scales<GR>(R, rb, c, rows, cols, sr);
  if (GT) publish_scales<GT>(Tq, rb, c, rows, cols, SAME ? sr : st);
  const double capr = (double)R.cap, capt = (double)Tq.cap;
  uint32_t qr[4][4], qt[4][4];
#pragma unroll
  for (int j = 0; j < 4; ++j)
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      if (GR) qr[j][k] = qround<CLAMP>((double)v[j][k], GR == 1 ? sr[j] : sr[k], capr);
      if (GT) qt[j][k] = SAME ? qr[j][k] : qround<CLAMP>((double)v[j][k], GT == 1 ? st[j] : st[k], capt);
    }
  if (GR) {
    if (R.packed) {  // four nibbles = 2 bytes per micro-tile row
      int8_t *o = R.q + rb * R.ld + c / 2;
#pragma unroll
      for (int j = 0; j < 4; ++j)
        if (interior || (rb + j < rows && c / 2 < R.ld))
          *reinterpret_cast<uint16_t *>(o + j * R.ld) =
              (uint16_t)((qr[j][0] & 0xF) | ((qr[j][1] & 0xF) << 4) | ((qr[j][2] & 0xF) << 8) | ((qr[j][3] & 0xF) << 12));
    } else {
      int8_t *o = R.q + rb * R.ld + c;
#pragma unroll
      for (int j = 0; j < 4; ++j)
        if (interior || (rb + j < rows && c < R.ld))
          *reinterpret_cast<uint32_t *>(o + j * R.ld) = pack4(qr[j][0], qr[j][1], qr[j][2], qr[j][3]);
    }
  }
  if (GT) {
#pragma unroll
    for (int k = 0; k < 4; ++k) tile[4 * tc4 + k][tr4] = pack4(qt[0][k], qt[1][k], qt[2][k], qt[3][k]);
    __syncthreads();
    const bool t_full = interior && r0 + 64 <= Tq.ld;
    const int w = threadIdx.x & 15, orow0 = threadIdx.x >> 4;
    int8_t *o = Tq.q + (c0 + orow0) * Tq.ld + r0 + 4 * w;
#pragma unroll
    for (int it = 0; it < 4; ++it) {
      const int orow = orow0 + 16 * it;
      if (t_full || (c0 + orow < cols && r0 + 4 * w < Tq.ld))
        *reinterpret_cast<uint32_t *>(o + 16 * it * Tq.ld) = tile[orow][w];
    }
  }
}

// x rows must allow 16-byte loads of four-element groups
template <class T>
bool x_vec_ok(const T *x, int64_t ldx) {
  return (uintptr_t)x % 16 == 0 && (ldx * (int64_t)sizeof(T)) % 16 == 0;
}

// absmax on the quantiser's 64 x 64 tile / 4 x 4 micro-tile layout (all four rows' loads in flight
// before any compare); per-row maxima reduce over the 16 lanes of a half-warp, per-column maxima
// over the 16 thread rows through shared memory.  Used for fp64 operands (the tall w-column Q and
// E-stage matrices), where it runs at the quantiser's bandwidth.
template <class T, int MASK>
__global__ void __launch_bounds__(256) absmax_micro_kernel(const T *__restrict__ x, int64_t rows, int64_t cols,
                                                           int64_t ldx, double *amax_t, double *amax_r,
                                                           double *amax_c, int *nonfinite, unsigned nbx) {
  constexpr bool kT = MASK & 1, kR = MASK & 2, kC = MASK & 4;
  const int64_t r0 = (int64_t)(blockIdx.x / nbx) * 64, c0 = (int64_t)(blockIdx.x % nbx) * 64;
  const int tc4 = threadIdx.x & 15, tr4 = threadIdx.x >> 4, lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  const int64_t c = c0 + 4 * tc4, rb = r0 + 4 * tr4;
  const bool interior = r0 + 64 <= rows && c0 + 64 <= cols;
  T v[4][4];
  if (interior) {
    const T *p = x + rb * ldx + c;
#pragma unroll
    for (int j = 0; j < 4; ++j) load4<T>(p + j * ldx, 0, 4, v[j]);
  } else {
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      if (rb + j < rows) {
        load4<T>(x + (rb + j) * ldx, c, cols, v[j]);
      } else {
#pragma unroll
        for (int k = 0; k < 4; ++k) v[j][k] = T(0);
      }
    }
  }
  bool bad = false;
  T rm[4], cm[4];
#pragma unroll
  for (int k = 0; k < 4; ++k) cm[k] = T(0);
#pragma unroll
  for (int j = 0; j < 4; ++j) {
    rm[j] = T(0);
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      bad |= !isfinite(v[j][k]);
      const T a = fabs(v[j][k]);
      rm[j] = vmax(rm[j], a);
      if (kC) cm[k] = vmax(cm[k], a);
    }
  }
  if (kR) {
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      double m = (double)rm[j];
#pragma unroll
      for (int o = 8; o > 0; o >>= 1) m = fmax(m, __shfl_xor_sync(0xffffffffu, m, o));
      if (tc4 == 0 && rb + j < rows) atomic_max_nonneg(amax_r + rb + j, m);
    }
  }
  __shared__ double cred[kC ? 16 : 1][kC ? 65 : 1];
  if (kC) {
#pragma unroll
    for (int k = 0; k < 4; ++k) cred[tr4][4 * tc4 + k] = (double)cm[k];
  }
  __shared__ double tred[8];
  if (kT) {
    double m = (double)vmax(vmax(rm[0], rm[1]), vmax(rm[2], rm[3]));
    m = warp_max(m);
    if (lane == 0) tred[wid] = m;
  }
  const bool any_bad = __syncthreads_or(bad);
  if (any_bad && threadIdx.x == 0 && nonfinite) *nonfinite = 1;
  if (kC && threadIdx.x < 64 && c0 + threadIdx.x < cols) {
    double m = cred[0][threadIdx.x];
#pragma unroll
    for (int i = 1; i < 16; ++i) m = fmax(m, cred[i][threadIdx.x]);
    atomic_max_nonneg(amax_c + c0 + threadIdx.x, m);
  }
  if (kT && threadIdx.x == 0) {
    double m = tred[0];
#pragma unroll
    for (int w = 1; w < 8; ++w) m = fmax(m, tred[w]);
    atomic_max_nonneg(amax_t, m);
  }
}

template <class T, int MASK>
void absmax_micro_go(const T *x, int64_t rows, int64_t cols, int64_t ldx, double *at, double *ar, double *ac, int *nf,
                     cudaStream_t st) {
  const int64_t nbx = ceil_div(cols, 64), blocks = nbx * ceil_div(rows, 64);
  absmax_micro_kernel<T, MASK><<<(unsigned)blocks, 256, 0, st>>>(x, rows, cols, ldx, at, ar, ac, nf, (unsigned)nbx);
}

template <class T, int VEC, int MASK>
void absmax_go(const T *x, int64_t rows, int64_t cols, int64_t ldx, double *at, double *ar, double *ac, int *nf,
               int64_t blocks, int64_t nbx, cudaStream_t st) {
  absmax_tile_kernel<T, VEC, MASK><<<(unsigned)blocks, 256, 0, st>>>(x, rows, cols, ldx, at, ar, ac, nf, (unsigned)nbx);
}

template <class T, int VEC>
void absmax_mask(int mask, const T *x, int64_t rows, int64_t cols, int64_t ldx, double *at, double *ar, double *ac,
                 int *nf, int64_t blocks, int64_t nbx, cudaStream_t st) {
  switch (mask) {
    case 1: absmax_go<T, VEC, 1>(x, rows, cols, ldx, at, ar, ac, nf, blocks, nbx, st); break;
    case 2: absmax_go<T, VEC, 2>(x, rows, cols, ldx, at, ar, ac, nf, blocks, nbx, st); break;
    case 3: absmax_go<T, VEC, 3>(x, rows, cols, ldx, at, ar, ac, nf, blocks, nbx, st); break;
    case 4: absmax_go<T, VEC, 4>(x, rows, cols, ldx, at, ar, ac, nf, blocks, nbx, st); break;
    case 5: absmax_go<T, VEC, 5>(x, rows, cols, ldx, at, ar, ac, nf, blocks, nbx, st); break;
    case 6: absmax_go<T, VEC, 6>(x, rows, cols, ldx, at, ar, ac, nf, blocks, nbx, st); break;
    default: absmax_go<T, VEC, 7>(x, rows, cols, ldx, at, ar, ac, nf, blocks, nbx, st); break;
  }
}

template <class T>
int absmax_tile_launch(const T *x, int64_t rows, int64_t cols, int64_t ldx, double *amax_t, double *amax_r,
                       double *amax_c, int *nonfinite, cudaStream_t st) {
  const int mask = (amax_t ? 1 : 0) | (amax_r ? 2 : 0) | (amax_c ? 4 : 0);
  if (!mask) return LRAMM_OK;
  constexpr int VV = 16 / sizeof(T);
  const int V = (uintptr_t)x % 16 == 0 && ldx % VV == 0 ? VV : 1;
  const int64_t nbx = ceil_div(cols, 64LL * V), blocks = nbx * ceil_div(rows, 64);
  if (ceil_div(cols, 64) * ceil_div(rows, 64) >= (1LL << 31))
    return fail(LRAMM_ERR_SHAPE, "absmax: %lld x %lld exceeds the tile grid", (long long)rows, (long long)cols);
  const bool micro = x_vec_ok(x, ldx) && sizeof(T) == 8;
  if (micro) {
    switch (mask) {
      case 1: absmax_micro_go<T, 1>(x, rows, cols, ldx, amax_t, amax_r, amax_c, nonfinite, st); break;
      case 2: absmax_micro_go<T, 2>(x, rows, cols, ldx, amax_t, amax_r, amax_c, nonfinite, st); break;
      case 3: absmax_micro_go<T, 3>(x, rows, cols, ldx, amax_t, amax_r, amax_c, nonfinite, st); break;
      case 4: absmax_micro_go<T, 4>(x, rows, cols, ldx, amax_t, amax_r, amax_c, nonfinite, st); break;
      case 5: absmax_micro_go<T, 5>(x, rows, cols, ldx, amax_t, amax_r, amax_c, nonfinite, st); break;
      case 6: absmax_micro_go<T, 6>(x, rows, cols, ldx, amax_t, amax_r, amax_c, nonfinite, st); break;
      default: absmax_micro_go<T, 7>(x, rows, cols, ldx, amax_t, amax_r, amax_c, nonfinite, st); break;
    }
  } else if (V == 1)
    absmax_mask<T, 1>(mask, x, rows, cols, ldx, amax_t, amax_r, amax_c, nonfinite, blocks, nbx, st);
  else
    absmax_mask<T, VV>(mask, x, rows, cols, ldx, amax_t, amax_r, amax_c, nonfinite, blocks, nbx, st);
  LRAMM_LAUNCH_CHECK();
  return LRAMM_OK;
}

// both sides' outputs must allow 4-byte stores (ld % 4, base alignment)
bool tile_ok(const QSide &s) { return !s.q || (s.ld % 4 == 0 && (uintptr_t)s.q % 4 == 0); }
// output columns a side spans (packed int4: two per byte)
inline int64_t side_cols(const QSide &s) { return s.packed ? 2 * s.ld : s.ld; }

inline int side_kind(const QSide &s) { return !s.q ? 0 : (s.gran == LRAMM_GRAN_ROW ? 1 : 2); }

template <class T, int GR, int GT, bool SAME, bool CLAMP>
void qtile_go(const T *x, int64_t rows, int64_t cols, int64_t ldx, const QSide &R, const QSide &Tq, int64_t blocks,
              int64_t nbx, cudaStream_t st) {
  quantize_tile_kernel<T, GR, GT, SAME, CLAMP><<<(unsigned)blocks, 256, 0, st>>>(x, rows, cols, ldx, R, Tq,
                                                                                  (unsigned)nbx);
}

// requires x_vec_ok and tile_ok on both sides; `clamp` for caller-supplied maxima (single side only)
template <class T>
int quantize_tile_launch(const T *x, int64_t rows, int64_t cols, int64_t ldx, const QSide &R, const QSide &Tq,
                         bool clamp, cudaStream_t st) {
  const int64_t ext_r = std::max(rows, Tq.q ? Tq.ld : 0), ext_c = std::max(cols, R.q ? side_cols(R) : 0);
  const int64_t nbx = ceil_div(ext_c, 64), blocks = nbx * ceil_div(ext_r, 64);
  if (blocks >= (1LL << 31)) return fail(LRAMM_ERR_SHAPE, "quantize: %lld x %lld exceeds the tile grid",
                                         (long long)rows, (long long)cols);
  const int gr = side_kind(R), gt = side_kind(Tq);
  // equal granularity and cap: both sides' scales come from the same maxima (quantize_pair_device)
  const bool same = gr && gt && R.gran == Tq.gran && R.cap == Tq.cap;
  if (clamp && gr && gt) return fail(LRAMM_ERR_UNSUPPORTED, "quantize: clamped pair");
#define QG(a, b, s, c) qtile_go<T, a, b, s, c>(x, rows, cols, ldx, R, Tq, blocks, nbx, st)
  switch (gr * 3 + gt) {
    case 1: if (clamp) QG(0, 1, false, true); else QG(0, 1, false, false); break;
    case 2: if (clamp) QG(0, 2, false, true); else QG(0, 2, false, false); break;
    case 3: if (clamp) QG(1, 0, false, true); else QG(1, 0, false, false); break;
    case 6: if (clamp) QG(2, 0, false, true); else QG(2, 0, false, false); break;
    case 4: if (same) QG(1, 1, true, false); else QG(1, 1, false, false); break;
    case 5: QG(1, 2, false, false); break;
    case 7: QG(2, 1, false, false); break;
    case 8: if (same) QG(2, 2, true, false); else QG(2, 2, false, false); break;
    default: return fail(LRAMM_ERR_PARAM, "quantize: no output side");
  }
#undef QG
  LRAMM_LAUNCH_CHECK();
  return LRAMM_OK;
}


__global__ void scales_from_amax_kernel(const double *amax, int64_t n, int cap, double *scales) {
  int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) scales[i] = quant_scale(amax[i], cap);
}

template <class OutT>
__device__ __forceinline__ void store_q(OutT *q, int64_t idx, int v) { q[idx] = (OutT)v; }

// 32x32 tiles.  gran: 0 tensor, 1 row, 2 col.  The output index space covers
// [0, out_rows) x [0, ldq) so padding columns are zeroed.
template <class T, class OutT>
__global__ void quantize_kernel(const T *__restrict__ x, int64_t rows, int64_t cols, int64_t ldx,
                                const double *__restrict__ scales, int gran, int cap, int transpose,
                                OutT *__restrict__ q, int64_t ldq) {
  __shared__ int tile[kTile][kTile + 1];
  const int64_t out_rows = transpose ? cols : rows;
  // this block's output tile origin
  const int64_t orow0 = (int64_t)blockIdx.y * kTile;
  const int64_t ocol0 = (int64_t)blockIdx.x * kTile;
  if (!transpose) {
    for (int i = threadIdx.y; i < kTile; i += blockDim.y) {
      int64_t r = orow0 + i, c = ocol0 + threadIdx.x;
      if (r >= out_rows || c >= ldq) continue;
      int v = 0;
      if (c < cols) {
        double s = gran == 0 ? scales[0] : (gran == 1 ? scales[r] : scales[c]);
        v = quant_round((double)x[r * ldx + c], s, cap);
      }
      store_q(q, r * ldq + c, v);
    }
  } else {
    // input tile rows [ocol0, +32) (input rows = output cols), input cols [orow0, +32)
    for (int i = threadIdx.y; i < kTile; i += blockDim.y) {
      int64_t r = ocol0 + i, c = orow0 + threadIdx.x;
      int v = 0;
      if (r < rows && c < cols) {
        double s = gran == 0 ? scales[0] : (gran == 1 ? scales[r] : scales[c]);
        v = quant_round((double)x[r * ldx + c], s, cap);
      }
      tile[i][threadIdx.x] = v;
    }
    __syncthreads();
    for (int i = threadIdx.y; i < kTile; i += blockDim.y) {
      int64_t orow = orow0 + i, ocol = ocol0 + threadIdx.x;
      if (orow >= out_rows || ocol >= ldq) continue;
      store_q(q, orow * ldq + ocol, tile[threadIdx.x][i]);
    }
  }
}

// packed int4: output byte j of a row holds logical columns 2j (low nibble) and 2j+1.
template <class T>
__global__ void quantize_int4_kernel(const T *__restrict__ x, int64_t rows, int64_t cols, int64_t ldx,
                                     const double *__restrict__ scales, int gran, int cap,
                                     int transpose, uint8_t *__restrict__ q, int64_t ldq_bytes) {
  const int64_t out_rows = transpose ? cols : rows;
  const int64_t out_cols = transpose ? rows : cols;
  int64_t orow = (int64_t)blockIdx.y * blockDim.y + threadIdx.y;
  int64_t ob = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;  // output byte
  if (orow >= out_rows || ob >= ldq_bytes) return;
  int nib[2];
#pragma unroll
  for (int h = 0; h < 2; ++h) {
    int64_t ocol = 2 * ob + h;
    int v = 0;
    if (ocol < out_cols) {
      int64_t r = transpose ? ocol : orow, c = transpose ? orow : ocol;
      double s = gran == 0 ? scales[0] : (gran == 1 ? scales[r] : scales[c]);
      v = quant_round((double)x[r * ldx + c], s, cap);
    }
    nib[h] = v & 0xF;
  }
  q[orow * ldq_bytes + ob] = (uint8_t)(nib[0] | (nib[1] << 4));
}

__global__ void scale_round_clip_kernel(const double *__restrict__ a, int64_t rows, int64_t cols,
                                        int64_t lda, double scale, int cap, int32_t *__restrict__ out,
                                        int64_t ldo) {
  int64_t n = rows * cols;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    int64_t r = i / cols, c = i - r * cols;
    out[r * ldo + c] = quant_round(a[r * lda + c], scale, cap);
  }
}

template <class T>
int absmax_launch(const T *x, int64_t rows, int64_t cols, int64_t ldx, int gran, double *amax, int *nonfinite,
                  cudaStream_t st) {
  return absmax_tile_launch<T>(x, rows, cols, ldx, gran == LRAMM_GRAN_TENSOR ? amax : nullptr,
                               gran == LRAMM_GRAN_ROW ? amax : nullptr, gran == LRAMM_GRAN_COL ? amax : nullptr,
                               nonfinite, st);
}

template <class T>
int quantize_from_amax(const T *x, int64_t rows, int64_t cols, int64_t ldx, int bits, int gran, int transpose,
                       const double *amax, void *q, int q_dtype, int64_t ldq, double *scales, bool clamp,
                       cudaStream_t st) {
  const int cap = bit_cap(bits);
  const int64_t nscale = gran == LRAMM_GRAN_TENSOR ? 1 : (gran == LRAMM_GRAN_ROW ? rows : cols);
  const int64_t out_rows = transpose ? cols : rows;
  // the tile kernel derives and publishes the scales itself
  if (q_dtype == LRAMM_I4 && !transpose && ldq % 2 == 0 && (uintptr_t)q % 2 == 0 && x_vec_ok(x, ldx)) {
    QSide side{(int8_t *)q, ldq, scales, gran, cap, 1, amax}, none{nullptr, 0, nullptr, 0, 0};
    return quantize_tile_launch<T>(x, rows, cols, ldx, side, none, clamp, st);
  }
  if (q_dtype == LRAMM_I8 && tile_ok(QSide{(int8_t *)q, ldq, scales, gran, cap}) && x_vec_ok(x, ldx)) {
    QSide side{(int8_t *)q, ldq, scales, gran, cap, 0, amax}, none{nullptr, 0, nullptr, 0, 0};
    return quantize_tile_launch<T>(x, rows, cols, ldx, transpose ? none : side, transpose ? side : none, clamp, st);
  }
  scales_from_amax_kernel<<<(unsigned)ceil_div(nscale, 256), 256, 0, st>>>(amax, nscale, cap, scales);
  LRAMM_LAUNCH_CHECK();
  if (q_dtype == LRAMM_I4) {
    dim3 blk(32, 8);
    dim3 grid((unsigned)ceil_div(ldq, 32), (unsigned)ceil_div(out_rows, 8));
    quantize_int4_kernel<T><<<grid, blk, 0, st>>>(x, rows, cols, ldx, scales, gran, cap, transpose,
                                                  (uint8_t *)q, ldq);
  } else {
    dim3 blk(32, 8);
    dim3 grid((unsigned)ceil_div(ldq, kTile), (unsigned)ceil_div(out_rows, kTile));
    if (q_dtype == LRAMM_I8)
      quantize_kernel<T, int8_t><<<grid, blk, 0, st>>>(x, rows, cols, ldx, scales, gran, cap, transpose,
                                                      (int8_t *)q, ldq);
    else
      quantize_kernel<T, int32_t><<<grid, blk, 0, st>>>(x, rows, cols, ldx, scales, gran, cap, transpose,
                                                       (int32_t *)q, ldq);
  }
  LRAMM_LAUNCH_CHECK();
  return LRAMM_OK;
}

template <class T>
int quantize_impl(const T *x, int64_t rows, int64_t cols, int64_t ldx, int bits, int gran, int transpose,
                  void *q, int q_dtype, int64_t ldq, double *scales, int *nonfinite, void *ws,
                  size_t ws_bytes, cudaStream_t st, const AmaxSync *sync) {
  const int64_t nscale = gran == LRAMM_GRAN_TENSOR ? 1 : (gran == LRAMM_GRAN_ROW ? rows : cols);
  Arena ar(ws, ws_bytes);
  double *amax = ar.take<double>(nscale);
  if (!ar.ok() || amax == nullptr) return fail(LRAMM_ERR_WORKSPACE, "quantize: workspace too small");
  LRAMM_CUDA_TRY(cudaMemsetAsync(amax, 0, nscale * sizeof(double), st));
  LRAMM_TRY(absmax_launch<T>(x, rows, cols, ldx, gran, amax, nonfinite, st));
  if (sync && sync->wants(gran)) LRAMM_TRY(sync->coll->max_f64(amax, (size_t)nscale, st));
  return quantize_from_amax<T>(x, rows, cols, ldx, bits, gran, transpose, amax, q, q_dtype, ldq, scales, false, st);
}

template <class T>
int quantize_pair_impl(const T *x, int64_t rows, int64_t cols, int64_t ldx, int bits_r, int gran_r, int8_t *qr,
                       int64_t ldqr, double *scales_r, int bits_t, int gran_t, int8_t *qt, int64_t ldqt,
                       double *scales_t, int *nonfinite, void *ws, size_t ws_bytes, cudaStream_t st, int r_packed,
                       const AmaxSync *sync) {
  Arena ar(ws, ws_bytes);
  const bool need[3] = {gran_r == LRAMM_GRAN_TENSOR || gran_t == LRAMM_GRAN_TENSOR,
                        gran_r == LRAMM_GRAN_ROW || gran_t == LRAMM_GRAN_ROW,
                        gran_r == LRAMM_GRAN_COL || gran_t == LRAMM_GRAN_COL};
  const int64_t n[3] = {1, rows, cols};
  double *amax[3] = {nullptr, nullptr, nullptr};
  int64_t total = 0;
  for (int g = 0; g < 3; ++g) total += need[g] ? round_up(n[g], 32) : 0;
  double *base = ar.take<double>(total);
  if (!ar.ok() || base == nullptr) return fail(LRAMM_ERR_WORKSPACE, "quantize: workspace too small");
  for (int g = 0, off = 0; g < 3; ++g)
    if (need[g]) amax[g] = base + off, off += (int)round_up(n[g], 32);
  LRAMM_CUDA_TRY(cudaMemsetAsync(base, 0, total * sizeof(double), st));
  LRAMM_TRY(absmax_tile_launch<T>(x, rows, cols, ldx, amax[0], amax[1], amax[2], nonfinite, st));
  for (int g = 0; g < 3; ++g)  // maxima over a sharded dimension: combined across the ranks
    if (need[g] && sync && sync->wants(g)) LRAMM_TRY(sync->coll->max_f64(amax[g], (size_t)n[g], st));
  const int cap_r = bit_cap(bits_r), cap_t = bit_cap(bits_t);
  QSide R{qr, ldqr, scales_r, gran_r, cap_r, r_packed, amax[gran_r]}, Tq{qt, ldqt, scales_t, gran_t, cap_t, 0, amax[gran_t]};
  const bool r_ok = r_packed ? (ldqr % 2 == 0 && (uintptr_t)qr % 2 == 0) : tile_ok(R);
  if (r_ok && tile_ok(Tq) && x_vec_ok(x, ldx)) return quantize_tile_launch<T>(x, rows, cols, ldx, R, Tq, false, st);
  scales_from_amax_kernel<<<(unsigned)ceil_div(n[gran_r], 256), 256, 0, st>>>(amax[gran_r], n[gran_r], cap_r, scales_r);
  LRAMM_LAUNCH_CHECK();
  scales_from_amax_kernel<<<(unsigned)ceil_div(n[gran_t], 256), 256, 0, st>>>(amax[gran_t], n[gran_t], cap_t, scales_t);
  LRAMM_LAUNCH_CHECK();
  LRAMM_TRY(quantize_from_amax<T>(x, rows, cols, ldx, bits_r, gran_r, 0, amax[gran_r], qr, r_packed ? LRAMM_I4 : LRAMM_I8,
                                  ldqr, scales_r, false, st));
  return quantize_from_amax<T>(x, rows, cols, ldx, bits_t, gran_t, 1, amax[gran_t], qt, LRAMM_I8, ldqt, scales_t, false, st);
}

}  // namespace

int quantize_device(const void *x, int x_dtype, int64_t rows, int64_t cols, int64_t ldx, int bits,
                    int gran, int transpose, void *q, int q_dtype, int64_t ldq, double *scales,
                    int *nonfinite, void *ws, size_t ws_bytes, cudaStream_t st, const AmaxSync *sync) {
  if (rows < 1 || cols < 1 || ldx < cols) return fail(LRAMM_ERR_SHAPE, "quantize: bad shape %lldx%lld ld %lld",
                                                      (long long)rows, (long long)cols, (long long)ldx);
  if (bits < 2 || bits > 24) return fail(LRAMM_ERR_PARAM, "bits must be an integer in [2, 24], got %d", bits);
  if (q_dtype == LRAMM_I8 && bits > 8) return fail(LRAMM_ERR_UNSUPPORTED, "int8 output needs bits <= 8");
  if (q_dtype == LRAMM_I4 && bits > 4) return fail(LRAMM_ERR_UNSUPPORTED, "int4 output needs bits <= 4");
  const int64_t out_cols = transpose ? rows : cols;
  if (q_dtype == LRAMM_I4 ? ldq * 2 < out_cols : ldq < out_cols)
    return fail(LRAMM_ERR_SHAPE, "quantize: ldq too small");
  if (gran < 0 || gran > 2) return fail(LRAMM_ERR_PARAM, "bad granularity %d", gran);
  if (x_dtype == LRAMM_F32)
    return quantize_impl<float>((const float *)x, rows, cols, ldx, bits, gran, transpose, q, q_dtype, ldq,
                                scales, nonfinite, ws, ws_bytes, st, sync);
  if (x_dtype == LRAMM_F64)
    return quantize_impl<double>((const double *)x, rows, cols, ldx, bits, gran, transpose, q, q_dtype, ldq,
                                 scales, nonfinite, ws, ws_bytes, st, sync);
  return fail(LRAMM_ERR_PARAM, "quantize: input dtype must be F32 or F64");
}

int absmax_device(const void *x, int x_dtype, int64_t rows, int64_t cols, int64_t ldx, int gran, double *amax,
                  int *nonfinite, cudaStream_t st) {
  if (rows < 1 || cols < 1 || ldx < cols) return fail(LRAMM_ERR_SHAPE, "absmax: bad shape");
  if (gran < 0 || gran > 2) return fail(LRAMM_ERR_PARAM, "bad granularity %d", gran);
  if (x_dtype == LRAMM_F32) return absmax_launch<float>((const float *)x, rows, cols, ldx, gran, amax, nonfinite, st);
  if (x_dtype == LRAMM_F64) return absmax_launch<double>((const double *)x, rows, cols, ldx, gran, amax, nonfinite, st);
  return fail(LRAMM_ERR_PARAM, "absmax: input dtype must be F32 or F64");
}

int quantize_amax_device(const void *x, int x_dtype, int64_t rows, int64_t cols, int64_t ldx, int bits, int gran,
                         int transpose, const double *amax, void *q, int q_dtype, int64_t ldq, double *scales,
                         cudaStream_t st) {
  if (rows < 1 || cols < 1 || ldx < cols) return fail(LRAMM_ERR_SHAPE, "quantize: bad shape");
  if (bits < 2 || bits > 24) return fail(LRAMM_ERR_PARAM, "bits must be an integer in [2, 24], got %d", bits);
  if (q_dtype == LRAMM_I8 && bits > 8) return fail(LRAMM_ERR_UNSUPPORTED, "int8 output needs bits <= 8");
  if (x_dtype == LRAMM_F32)
    return quantize_from_amax<float>((const float *)x, rows, cols, ldx, bits, gran, transpose, amax, q, q_dtype, ldq,
                                     scales, true, st);
  if (x_dtype == LRAMM_F64)
    return quantize_from_amax<double>((const double *)x, rows, cols, ldx, bits, gran, transpose, amax, q, q_dtype,
                                      ldq, scales, true, st);
  return fail(LRAMM_ERR_PARAM, "quantize: input dtype must be F32 or F64");
}

// one quantisation of x into two int8 layouts (row-major at bits_r / gran_r, transposed at bits_t /
// gran_t; gran in input coordinates) from a single absmax pass and a single read of x
int quantize_pair_device(const void *x, int x_dtype, int64_t rows, int64_t cols, int64_t ldx, int bits_r, int gran_r,
                         int8_t *qr, int64_t ldqr, double *scales_r, int bits_t, int gran_t, int8_t *qt, int64_t ldqt,
                         double *scales_t, int *nonfinite, void *ws, size_t ws_bytes, cudaStream_t st, int r_packed,
                         const AmaxSync *sync) {
  if (rows < 1 || cols < 1 || ldx < cols) return fail(LRAMM_ERR_SHAPE, "quantize: bad shape");
  if (bits_r < 2 || bits_r > 8 || bits_t < 2 || bits_t > 8)
    return fail(LRAMM_ERR_UNSUPPORTED, "quantize pair: int8 outputs need bits in [2, 8]");
  if (r_packed && bits_r > 4) return fail(LRAMM_ERR_UNSUPPORTED, "quantize pair: packed int4 needs bits <= 4");
  if (gran_r < 0 || gran_r > 2 || gran_t < 0 || gran_t > 2) return fail(LRAMM_ERR_PARAM, "bad granularity");
  if ((r_packed ? 2 * ldqr : ldqr) < cols || ldqt < rows) return fail(LRAMM_ERR_SHAPE, "quantize pair: ldq too small");
  if (x_dtype == LRAMM_F32)
    return quantize_pair_impl<float>((const float *)x, rows, cols, ldx, bits_r, gran_r, qr, ldqr, scales_r, bits_t,
                                     gran_t, qt, ldqt, scales_t, nonfinite, ws, ws_bytes, st, r_packed, sync);
  if (x_dtype == LRAMM_F64)
    return quantize_pair_impl<double>((const double *)x, rows, cols, ldx, bits_r, gran_r, qr, ldqr, scales_r, bits_t,
                                      gran_t, qt, ldqt, scales_t, nonfinite, ws, ws_bytes, st, r_packed, sync);
  return fail(LRAMM_ERR_PARAM, "quantize: input dtype must be F32 or F64");
}

size_t quantize_ws_bytes(int64_t rows, int64_t cols) {
  return (size_t)(round_up(rows, 32) + round_up(cols, 32) + 32) * sizeof(double) + 512;
}

int scale_round_clip_device(const double *a, int64_t rows, int64_t cols, int64_t lda, double scale, int cap,
                            int32_t *out, int64_t ldo, cudaStream_t st) {
  if (rows < 1 || cols < 1) return fail(LRAMM_ERR_SHAPE, "scale_round_clip: empty");
  int grid = (int)std::min<int64_t>(ceil_div(rows * cols, 256), 16LL * num_sms());
  scale_round_clip_kernel<<<grid, 256, 0, st>>>(a, rows, cols, lda, scale, cap, out, ldo);
  LRAMM_LAUNCH_CHECK();
  return LRAMM_OK;
}

}  // namespace lramm
