// Integer GEMM on the 5th-generation tensor cores: C = A . B^T, A: M x K int8,
// B: N x K int8 (both K-major), int32 accumulators in TMEM (tcgen05.mma.kind::i8),
// operands streamed by TMA into a STAGES-deep shared-memory ring, and the
// reference's dequantisation acc / (sa * sb) (quant.py:116) applied in the
// epilogue in IEEE fp64 (bit-exact), optionally followed by alpha/beta
// (quant.py:117-121, pipeline.py:205-210) and a transposed store so the next
// GEMM's operand is K-major.
//
// Warp roles (192 threads, one CTA per SM):
//   warp 0     TMA producer (one elected lane)
//   warp 1     TMEM allocator + MMA issuer (one elected lane)
//   warps 2-5  epilogue: TMEM -> registers -> global (warp w reads TMEM lanes 32*(w%4)..+31)
#include <cudaTypedefs.h>

#include <algorithm>
#include <cstdlib>
#include <mutex>

#include "common.cuh"
#include "sm100.cuh"

namespace lramm {

struct EpiDev {
  int out_dtype, accumulate, transpose_out, c_dtype;
  void *out;
  int64_t ldo;
  const double *row_scale;
  int64_t row_scale_inc;
  const double *col_scale;
  int64_t col_scale_inc;
  double alpha, beta;
  const void *c;
  int64_t ldc;
  int shift;  // EK_I64_ADD: out += acc * 2^shift (limb-pair products of multi-limb operands)
  int signs;  // bit 0: A int8 signed, bit 1: B int8 signed (unsigned limbs otherwise)
  int nfast;  // grid laid out with N tiles fastest (see igemm_device)
  int a4;     // A arrives as packed int4 (two's-complement nibbles) and is unpacked to int8 in smem
};

// Correctly rounded a / s for |a| < 2^53 integer-valued a and normal s > 0, given y = RN(1/s):
// Markstein step q1 = RN(q0 + r y), r = a - q0 s (exact by FMA), then an exact residual check
// against the neighbour in the direction of the residual (ties to even).  Bit-identical to
// IEEE division (__ddiv_rn), ~10 instructions instead of the iterative divide.
__device__ __forceinline__ double next_toward(double x, bool up) {
  if (x == 0.0) return up ? __longlong_as_double(1LL) : -__longlong_as_double(1LL);
  const long long b = __double_as_longlong(x);
  return __longlong_as_double(((x > 0.0) == up) ? b + 1 : b - 1);
}

__device__ __forceinline__ double div_exact(double a, double s, double y) {
  const double q0 = __dmul_rn(a, y);
  const double r0 = __fma_rn(-q0, s, a);
  const double q1 = __fma_rn(r0, y, q0);
  const double r1 = __fma_rn(-q1, s, a);
  // q1 is the correctly rounded quotient iff |r1| <= s ulp(q1) / 2 (strictly < : no tie to resolve)
  const long long eb = __double_as_longlong(q1) & 0x7FF0000000000000LL;
  if (eb > (53LL << 52)) {
    const double half_ulp = __longlong_as_double(eb - (53LL << 52));  // ulp(q1) / 2 for normal q1
    if (fabs(r1) < __dmul_rn(s, half_ulp)) return q1;
  } else if (r1 == 0.0) {
    return q1;
  }
  const double qn = next_toward(q1, r1 > 0.0);
  const double rn = __fma_rn(-qn, s, a);
  const double e1 = fabs(r1), en = fabs(rn);
  if (en < e1) return qn;
  if (en == e1) return (__double_as_longlong(qn) & 1) ? q1 : qn;  // tie: even mantissa
  return q1;
}

// a / s for an output that is rounded to fp32 next (and used for nothing else): a double whose
// fp32 rounding equals that of the correctly rounded fp64 quotient.  q0 = RN(a y), y = RN(1/s), lies
// within 2.5 ulp64 of RN(a / s); the two round to the same float unless q0 sits within a few ulp64
// of a midpoint between adjacent floats (the 29 mantissa bits below fp32 precision near 2^28) or
// outside the normal fp32 range -- only then the exact division runs (~2^-24 of the elements).
// The fp32-output epilogue is fp64-pipe bound otherwise: 15 fp64 instructions per element.
__device__ __forceinline__ double div_for_f32(double a, double s, double y) {
  const double q0 = __dmul_rn(a, y);
  const long long b = __double_as_longlong(q0);
  const int ex = (int)((b >> 52) & 0x7FF);
  const unsigned lo = (unsigned)b & 0x1FFFFFFFu;
  if (ex >= 1023 - 120 && ex <= 1023 + 120 && (lo - 0x0FFFFFF8u) > 16u) return q0;
  return div_exact(a, s, y);
}

// reference dequantisation + alpha/beta on one accumulator (bit-exact IEEE fp64)
template <typename AccT>
__device__ __forceinline__ double epi_value(const EpiDev &e, AccT acc, int64_t row, int64_t col) {
  double rs = e.row_scale ? e.row_scale[row * e.row_scale_inc] : 1.0;
  double cs = e.col_scale ? e.col_scale[col * e.col_scale_inc] : 1.0;
  double v = __ddiv_rn((double)acc, __dmul_rn(rs, cs));  // acc.astype(f64) / (sa*sb) (int64: RN convert)
  if (e.beta != 0.0 && e.c != nullptr) {
    double cv = e.c_dtype == LRAMM_F32 ? (double)((const float *)e.c)[row * e.ldc + col]
                                       : ((const double *)e.c)[row * e.ldc + col];
    v = __dadd_rn(__dmul_rn(e.alpha, v), __dmul_rn(e.beta, cv));
  } else if (e.alpha != 1.0) {
    v = __dmul_rn(e.alpha, v);
  }
  return v;
}

__device__ __forceinline__ double epi_alpha_beta(const EpiDev &e, double v, int64_t row, int64_t col) {
  if (e.beta != 0.0 && e.c != nullptr) {
    double cv = e.c_dtype == LRAMM_F32 ? (double)((const float *)e.c)[row * e.ldc + col]
                                       : ((const double *)e.c)[row * e.ldc + col];
    return __dadd_rn(__dmul_rn(e.alpha, v), __dmul_rn(e.beta, cv));
  }
  if (e.alpha != 1.0) return __dmul_rn(e.alpha, v);
  return v;
}

__device__ __forceinline__ void epi_store(const EpiDev &e, int32_t acc, int64_t row, int64_t col) {
  int64_t idx = e.transpose_out ? col * e.ldo + row : row * e.ldo + col;
  if (e.out_dtype == LRAMM_I32) {
    int32_t *o = (int32_t *)e.out;
    if (e.accumulate)
      atomicAdd(o + idx, acc);
    else
      o[idx] = acc;
    return;
  }
  double v = epi_value(e, acc, row, col);
  if (e.out_dtype == LRAMM_F64)
    ((double *)e.out)[idx] = v;
  else
    ((float *)e.out)[idx] = __double2float_rn(v);
}

namespace {

constexpr int BM = 128;
constexpr int BK = 128;  // bytes == int8 elements == one 128-B swizzle row
constexpr int kThreads = 320;  // warp 0 TMA, warp 1 MMA, warps 2-9 epilogue
constexpr int kSmemBudget = 200 * 1024;

// epilogue kinds (compile time): raw int32 store / atomic add, or dequantised f32 / f64
enum { EK_I32 = 0, EK_I32_ATOMIC = 1, EK_F32 = 2, EK_F64 = 3, EK_I64_ADD = 4 };

template <int EK, bool TRANS, bool AB>
__global__ void __launch_bounds__(kThreads, 2)  // two CTAs per SM in the shallow-ring mode: registers stay <= 96
    igemm_tn_kernel(const __grid_constant__ CUtensorMap tma_a, const __grid_constant__ CUtensorMap tma_b,
                    int64_t M, int64_t N, int64_t K, int BN, int stages, int kb_per_split, EpiDev epi) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t *smem = reinterpret_cast<uint8_t *>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  const uint32_t a_bytes = BM * BK;
  const uint32_t b_bytes = (uint32_t)BN * BK;
  const bool a4 = epi.a4 != 0;
  const uint32_t a4_bytes = a4 ? BM * (BK / 2) : 0u;  // packed staging tile (64 B per row, no swizzle)
  uint8_t *sA = smem;
  uint8_t *sB = smem + (size_t)stages * a_bytes;
  uint8_t *sA4 = sB + (size_t)stages * b_bytes;
  uint64_t *full = reinterpret_cast<uint64_t *>(sA4 + (size_t)stages * a4_bytes);
  uint64_t *empty = full + stages;
  uint64_t *unpacked = empty + stages;  // a4: the int8 A tile of the stage is in sA
  uint64_t *tmem_full = unpacked + stages;
  uint32_t *tmem_slot = reinterpret_cast<uint32_t *>(tmem_full + 1);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  // tile order: blockIdx.x runs over N tiles when the grid was laid out N-fastest (nfast), so
  // consecutive CTAs share the A tile and the (smaller) B operand is what gets re-read
  const bool nfast = epi.nfast != 0;
  const int64_t m0 = (int64_t)(nfast ? blockIdx.y : blockIdx.x) * BM;
  const int64_t n0 = (int64_t)(nfast ? blockIdx.x : blockIdx.y) * BN;
  const int kb_total = (int)((K + BK - 1) / BK);
  const int kb0 = blockIdx.z * kb_per_split;
  const int kb1 = min(kb0 + kb_per_split, kb_total);
  const int nkb = max(kb1 - kb0, 0);
  const uint32_t tmem_cols = BN <= 32 ? 32u : (BN <= 64 ? 64u : (BN <= 128 ? 128u : 256u));

  if (warp == 0 && lane == 0) {
    sm100::prefetch_tmap(&tma_a);
    sm100::prefetch_tmap(&tma_b);
    for (int s = 0; s < stages; ++s) {
      sm100::mbar_init(&full[s], 1);
      sm100::mbar_init(&empty[s], 1);
      sm100::mbar_init(&unpacked[s], 256);  // every epilogue thread unpacks a quarter of a row band
    }
    sm100::mbar_init(tmem_full, 1);
    sm100::fence_barrier_init();
  }
  if (warp == 1) sm100::tmem_alloc(tmem_slot, tmem_cols);
  sm100::tc_fence_before();
  __syncthreads();
  sm100::tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;

  if (warp == 0) {
    if (lane == 0) {
      for (int i = 0; i < nkb; ++i) {
        const int s = i % stages;
        const uint32_t ph = (uint32_t)(i / stages) & 1u;
        sm100::mbar_wait(&empty[s], ph ^ 1u);
        sm100::mbar_arrive_expect_tx(&full[s], (a4 ? a4_bytes : a_bytes) + b_bytes);
        const int32_t kx = (kb0 + i) * BK;
        if (a4)
          sm100::tma_load_2d(&tma_a, &full[s], sA4 + (size_t)s * a4_bytes, kx / 2, (int32_t)m0);
        else
          sm100::tma_load_2d(&tma_a, &full[s], sA + (size_t)s * a_bytes, kx, (int32_t)m0);
        sm100::tma_load_2d(&tma_b, &full[s], sB + (size_t)s * b_bytes, kx, (int32_t)n0);
      }
    }
  } else if (warp == 1) {
    if (lane == 0) {
      const uint32_t idesc = (sm100::idesc_i8(BM, BN) & ~((1u << 7) | (1u << 10))) | ((uint32_t)(epi.signs & 1) << 7) |
                             ((uint32_t)((epi.signs >> 1) & 1) << 10);
      for (int i = 0; i < nkb; ++i) {
        const int s = i % stages;
        const uint32_t ph = (uint32_t)(i / stages) & 1u;
        sm100::mbar_wait(a4 ? &unpacked[s] : &full[s], ph);
        sm100::tc_fence_after();
        const uint64_t ad = sm100::sdesc_k_sw128(sm100::smem_u32(sA + (size_t)s * a_bytes));
        const uint64_t bd = sm100::sdesc_k_sw128(sm100::smem_u32(sB + (size_t)s * b_bytes));
#pragma unroll
        for (int k = 0; k < BK / 32; ++k)  // K = 32 int8 per MMA: advance 32 B = 2 descriptor units
          sm100::mma_i8(tmem_base, ad + 2 * k, bd + 2 * k, idesc, (i > 0 || k > 0) ? 1u : 0u);
        sm100::mma_commit(&empty[s]);
      }
      sm100::mma_commit(tmem_full);
    }
  } else {
    // epilogue warps 2..9: TMEM -> registers (thread = row; the two warps of a TMEM lane quarter
    // take alternate 16-column halves) -> dequant -> shared tile (32-column chunks in the drained
    // pipeline buffers) -> coalesced stores (warp = rows, lanes = columns)
    constexpr bool RAW = EK == EK_I32 || EK == EK_I32_ATOMIC || EK == EK_I64_ADD;
    const int ew = warp - 2;               // 0..7
    const int quarter = warp & 3;          // TMEM lane quarter (hardware: warp id mod 4)
    const int half = ew >> 2;              // column half of each 32-column chunk
    const int etid = threadIdx.x - 64;     // 0..255
    const int rloc = quarter * 32 + lane;
    const int64_t row = m0 + rloc;
    // per-column scales of this tile -> shared memory while the mainloop runs (the epilogue used to
    // read them from global memory per element: 83.9 -> 74.1 us at the c3 sketch shape, 37.5 -> 30.5 us
    // at c2's)
    __shared__ double cs_sh[256];
    constexpr bool RAW0 = EK == EK_I32 || EK == EK_I32_ATOMIC || EK == EK_I64_ADD;
    if (!RAW0 && epi.col_scale != nullptr && epi.col_scale_inc != 0) {
      for (int cidx = etid; cidx < BN; cidx += 256)
        cs_sh[cidx] = epi.col_scale[min(n0 + cidx, N - 1) * epi.col_scale_inc];
      asm volatile("bar.sync 1, 256;" ::: "memory");
    }
    if (a4) {
      // mainloop role of the epilogue warps: unpack each stage's packed A tile (BM rows x 64 B of
      // nibbles) into the int8 tile the MMA reads, in the TMA SWIZZLE_128B layout (16-byte chunk c
      // of row r at chunk c ^ (r & 7)); one 16-byte chunk = 8 packed bytes per step
      for (int i = 0; i < nkb; ++i) {
        const int s = i % stages;
        sm100::mbar_wait(&full[s], (uint32_t)(i / stages) & 1u);
        const uint8_t *src = sA4 + (size_t)s * a4_bytes;
        uint8_t *dst = sA + (size_t)s * a_bytes;
#pragma unroll
        for (int t = 0; t < (BM * 8) / 256; ++t) {
          const int idx = etid + 256 * t, r = idx >> 3, c = idx & 7;
          const uint2 pk = *reinterpret_cast<const uint2 *>(src + r * (BK / 2) + 8 * c);
          uint32_t w[4];
#pragma unroll
          for (int h = 0; h < 2; ++h) {
            const uint32_t v = h ? pk.y : pk.x;  // 4 packed bytes -> 8 int8 (2 words)
#pragma unroll
            for (int q = 0; q < 2; ++q) {
              const uint32_t b2 = v >> (16 * q);  // two packed bytes -> four nibbles
              uint32_t out = 0;
#pragma unroll
              for (int n = 0; n < 4; ++n) {
                const int32_t nib = (int32_t)((b2 >> (4 * n)) & 0xF);
                out |= (uint32_t)(uint8_t)(int8_t)((nib ^ 8) - 8) << (8 * n);
              }
              w[2 * h + q] = out;
            }
          }
          *reinterpret_cast<uint4 *>(dst + r * BK + ((c ^ (r & 7)) * 16)) = make_uint4(w[0], w[1], w[2], w[3]);
        }
        sm100::fence_proxy_async_smem();  // generic stores -> the tensor core's async-proxy reads
        asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(sm100::smem_u32(&unpacked[s])) : "memory");
      }
    }
    if (nkb > 0) {
      sm100::mbar_wait(tmem_full, 0);
      sm100::tc_fence_after();
    }
    double rs = 1.0;
    if (!RAW && epi.row_scale) rs = epi.row_scale[(row < M ? row : M - 1) * epi.row_scale_inc];
    const bool tensor_scale = epi.col_scale == nullptr || epi.col_scale_inc == 0;
    double s_t = 1.0, y_t = 1.0;
    if (!RAW && tensor_scale) {
      s_t = __dmul_rn(rs, epi.col_scale ? epi.col_scale[0] : 1.0);
      y_t = __drcp_rn(s_t);
    }
    if constexpr (!TRANS && (EK == EK_F32 || EK == EK_F64)) {
      // direct stores: thread = output row, 16 consecutive columns per TMEM load (64 B of fp32 /
      // 128 B of fp64 per thread per chunk: whole sectors), no shared-memory staging or barriers
      const bool vec = ((reinterpret_cast<uintptr_t>(epi.out) & 15) == 0) && (epi.ldo % 4 == 0);
      for (int c0 = 0; c0 < BN; c0 += 32) {
        const int cb = c0 + half * 16;
        if (cb >= BN) continue;
        uint32_t r[16];
        if (nkb > 0) {
          sm100::tmem_ld16(tmem_base + ((uint32_t)(quarter * 32) << 16) + (uint32_t)cb, r);
          sm100::tmem_wait_ld();
        } else {
#pragma unroll
          for (int j = 0; j < 16; ++j) r[j] = 0;
        }
        if (row >= M) continue;
        const int64_t col0 = n0 + cb;
        double v[16];
#pragma unroll
        for (int j = 0; j < 16; ++j) {
          if (tensor_scale) {
            if constexpr (EK == EK_F32 && !AB)
              v[j] = div_for_f32((double)(int32_t)r[j], s_t, y_t);
            else
              v[j] = div_exact((double)(int32_t)r[j], s_t, y_t);
          } else {
            const double sc = __dmul_rn(rs, cs_sh[cb + j]);
            v[j] = div_exact((double)(int32_t)r[j], sc, __drcp_rn(sc));
          }
          if constexpr (AB) v[j] = epi_alpha_beta(epi, v[j], row, min(col0 + j, N - 1));
        }
        const int64_t base = row * epi.ldo + col0;
        if (vec && col0 + 16 <= N) {
          if constexpr (EK == EK_F32) {
            float4 *o = reinterpret_cast<float4 *>((float *)epi.out + base);
#pragma unroll
            for (int q = 0; q < 4; ++q)
              o[q] = make_float4(__double2float_rn(v[4 * q]), __double2float_rn(v[4 * q + 1]),
                                 __double2float_rn(v[4 * q + 2]), __double2float_rn(v[4 * q + 3]));
          } else {
            double2 *o = reinterpret_cast<double2 *>((double *)epi.out + base);
#pragma unroll
            for (int q = 0; q < 8; ++q) o[q] = make_double2(v[2 * q], v[2 * q + 1]);
          }
        } else {
#pragma unroll
          for (int j = 0; j < 16; ++j)
            if (col0 + j < N) {
              if constexpr (EK == EK_F32) ((float *)epi.out)[base + j] = __double2float_rn(v[j]);
              else ((double *)epi.out)[base + j] = v[j];
            }
        }
      }
    } else {
    double *tile = reinterpret_cast<double *>(smem);  // 128 x 33
    int32_t *itile = reinterpret_cast<int32_t *>(smem);
    for (int c0 = 0; c0 < BN; c0 += 32) {
      const int cb = c0 + half * 16;
      uint32_t r[16];
      if (nkb > 0 && cb < BN) {
        sm100::tmem_ld16(tmem_base + ((uint32_t)(quarter * 32) << 16) + (uint32_t)cb, r);
        sm100::tmem_wait_ld();
      } else {
#pragma unroll
        for (int j = 0; j < 16; ++j) r[j] = 0;
      }
      if (RAW) {
#pragma unroll
        for (int j = 0; j < 16; ++j) itile[rloc * 33 + half * 16 + j] = (int32_t)r[j];
      } else if (tensor_scale) {
#pragma unroll
        for (int j = 0; j < 16; ++j) tile[rloc * 33 + half * 16 + j] = div_exact((double)(int32_t)r[j], s_t, y_t);
      } else {
#pragma unroll
        for (int j = 0; j < 16; ++j) {
          const double s = __dmul_rn(rs, cs_sh[min(cb + j, BN - 1)]);
          tile[rloc * 33 + half * 16 + j] = div_exact((double)(int32_t)r[j], s, __drcp_rn(s));
        }
      }
      asm volatile("bar.sync 1, 256;" ::: "memory");
      const int nc = min(32, BN - c0);
      if (!TRANS) {
        const int64_t gcol = n0 + c0 + lane;
        const bool colok = lane < nc && gcol < N;
        for (int rr = etid >> 5; rr < 128; rr += 8) {
          const int64_t grow = m0 + rr;
          if (grow < M && colok) {
            const int64_t idx = grow * epi.ldo + gcol;
            if constexpr (EK == EK_I32) {
              ((int32_t *)epi.out)[idx] = itile[rr * 33 + lane];
            } else if constexpr (EK == EK_I32_ATOMIC) {
              atomicAdd((int32_t *)epi.out + idx, itile[rr * 33 + lane]);
            } else if constexpr (EK == EK_I64_ADD) {
              ((int64_t *)epi.out)[idx] += (int64_t)itile[rr * 33 + lane] * ((int64_t)1 << epi.shift);
            } else {
              double v = tile[rr * 33 + lane];
              if constexpr (AB) v = epi_alpha_beta(epi, v, grow, gcol);
              if constexpr (EK == EK_F64) ((double *)epi.out)[idx] = v;
              else ((float *)epi.out)[idx] = __double2float_rn(v);
            }
          }
        }
      } else {
        // out^T: tile column j is a contiguous output row; lanes run over tile rows
        for (int jj = etid >> 5; jj < nc; jj += 8) {
          const int64_t gcol = n0 + c0 + jj;
          if (gcol >= N) continue;
          for (int rr = lane; rr < 128; rr += 32) {
            const int64_t grow = m0 + rr;
            if (grow >= M) continue;
            const int64_t idx = gcol * epi.ldo + grow;
            if constexpr (EK == EK_I32) {
              ((int32_t *)epi.out)[idx] = itile[rr * 33 + jj];
            } else if constexpr (EK == EK_I32_ATOMIC) {
              atomicAdd((int32_t *)epi.out + idx, itile[rr * 33 + jj]);
            } else if constexpr (EK == EK_I64_ADD) {
              ((int64_t *)epi.out)[idx] += (int64_t)itile[rr * 33 + jj] * ((int64_t)1 << epi.shift);
            } else {
              double v = tile[rr * 33 + jj];
              if constexpr (AB) v = epi_alpha_beta(epi, v, grow, gcol);
              if constexpr (EK == EK_F64) ((double *)epi.out)[idx] = v;
              else ((float *)epi.out)[idx] = __double2float_rn(v);
            }
          }
        }
      }
      asm volatile("bar.sync 1, 256;" ::: "memory");
    }
    }
  }
  sm100::tc_fence_before();
  __syncthreads();
  if (warp == 1) sm100::tmem_dealloc(tmem_base, tmem_cols);
}

// stand-alone epilogue over an int32 accumulator matrix (after split-K)
// dequantised value of one int32 accumulator: acc / (rs cs) correctly rounded through the
// reciprocal + exact residual check (div_exact; __ddiv_rn for a non-normal scale product)
__device__ __forceinline__ double epi_dequant_fast(const EpiDev &e, int32_t acc, int64_t row, int64_t col) {
  const double rs = e.row_scale ? e.row_scale[row * e.row_scale_inc] : 1.0;
  const double cs = e.col_scale ? e.col_scale[col * e.col_scale_inc] : 1.0;
  const double sc = __dmul_rn(rs, cs);
  const double v = (sc >= 2.2250738585072014e-308 && sc <= 1.7976931348623157e308)
                       ? div_exact((double)acc, sc, __drcp_rn(sc))
                       : __ddiv_rn((double)acc, sc);
  return epi_alpha_beta(e, v, row, col);
}

// int32 outputs (raw copy / accumulate) of lramm_dequant: the generic per-element store
__global__ void epilogue_generic_kernel(const int32_t *__restrict__ acc, int64_t M, int64_t N, int64_t lda,
                                        EpiDev epi) {
  for (int64_t r = blockIdx.y; r < M; r += gridDim.y)
    for (int64_t c = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; c < N; c += (int64_t)gridDim.x * blockDim.x)
      epi_store(epi, acc[r * lda + c], r, c);
}

// split-K epilogue (int32 accumulator -> dequantised f32 / f64): a warp per row, lanes over the
// columns (no 64-bit index division); transposed outputs go through a 32 x 32
// shared-memory tile so both the accumulator reads and the output writes are coalesced
template <bool TRANS>
__global__ void __launch_bounds__(256) epilogue_kernel(const int32_t *__restrict__ acc, int64_t M, int64_t N,
                                                       int64_t lda, EpiDev epi) {
  if constexpr (!TRANS) {
    // one warp per row, lanes over the columns (every lane busy for any N >= 32)
    const int lane = threadIdx.x & 31;
    const int64_t wstep = (int64_t)gridDim.x * (blockDim.x >> 5);
    for (int64_t r = (int64_t)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5); r < M; r += wstep)
      for (int64_t c = lane; c < N; c += 32) {
        const double v = epi_dequant_fast(epi, acc[r * lda + c], r, c);
        if (epi.out_dtype == LRAMM_F64)
          ((double *)epi.out)[r * epi.ldo + c] = v;
        else
          ((float *)epi.out)[r * epi.ldo + c] = __double2float_rn(v);
      }
  } else {
    __shared__ double t[32][33];
    const int tx = threadIdx.x & 31, ty = threadIdx.x >> 5;  // 32 x 8
    for (int64_t r0 = (int64_t)blockIdx.y * 32; r0 < M; r0 += (int64_t)gridDim.y * 32)
      for (int64_t c0 = (int64_t)blockIdx.x * 32; c0 < N; c0 += (int64_t)gridDim.x * 32) {
        for (int rr = ty; rr < 32; rr += 8) {
          const int64_t r = r0 + rr, c = c0 + tx;
          t[rr][tx] = (r < M && c < N) ? epi_dequant_fast(epi, acc[r * lda + c], r, c) : 0.0;
        }
        __syncthreads();
        for (int cc = ty; cc < 32; cc += 8) {
          const int64_t c = c0 + cc, r = r0 + tx;
          if (r < M && c < N) {
            if (epi.out_dtype == LRAMM_F64)
              ((double *)epi.out)[c * epi.ldo + r] = t[tx][cc];
            else
              ((float *)epi.out)[c * epi.ldo + r] = __double2float_rn(t[tx][cc]);
          }
        }
        __syncthreads();
      }
  }
}

// epilogue over an exact int64 accumulator (multi-limb products): float output only, or the
// raw int64 (imatmul)
__global__ void epilogue64_kernel(const int64_t *__restrict__ acc, int64_t M, int64_t N, int64_t lda, EpiDev e) {
  for (int64_t r = blockIdx.y; r < M; r += gridDim.y)
    for (int64_t c = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; c < N; c += (int64_t)gridDim.x * blockDim.x) {
      const int64_t a = acc[r * lda + c];
      const int64_t idx = e.transpose_out ? c * e.ldo + r : r * e.ldo + c;
      if (e.out_dtype == LRAMM_I64) {
        ((int64_t *)e.out)[idx] = a;
        continue;
      }
      const double v = epi_value(e, a, r, c);
      if (e.out_dtype == LRAMM_F64)
        ((double *)e.out)[idx] = v;
      else
        ((float *)e.out)[idx] = __double2float_rn(v);
    }
}

// 8-bit limb planes of int32 values (K-major rows x ld): v = sum_l limb_l 256^l with unsigned low
// limbs and a signed top limb (floor division), L = 2 for |v| < 2^15, 3 for |v| < 2^23
__global__ void split_limbs_kernel(const int32_t *__restrict__ src, int64_t rows, int64_t cols, int64_t lds,
                                   int nlimb, int8_t *__restrict__ dst, int64_t ldd, int64_t plane) {
  for (int64_t r = blockIdx.y; r < rows; r += gridDim.y)
    for (int64_t c = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; c < ldd; c += (int64_t)gridDim.x * blockDim.x) {
      int32_t v = c < cols ? src[r * lds + c] : 0;
      for (int l = 0; l < nlimb; ++l) {
        int8_t d;
        if (l == nlimb - 1) {
          d = (int8_t)v;  // |v| <= 127 here by construction
        } else {
          d = (int8_t)(uint8_t)(v & 0xFF);
          v = v >> 8;  // arithmetic shift = floor division by 256
        }
        dst[l * plane + r * ldd + c] = d;
      }
    }
}

PFN_cuTensorMapEncodeTiled_v12000 encode_fn() {
  static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
  static std::once_flag once;
  std::call_once(once, [] {
    void *p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(p);
  });
  return fn;
}

int make_tmap_i8(CUtensorMap *m, const int8_t *ptr, int64_t rows, int64_t k, int64_t ld, int box_rows) {
  auto fn = encode_fn();
  if (!fn) return fail(LRAMM_ERR_CUDA, "cuTensorMapEncodeTiled unavailable");
  cuuint64_t dims[2] = {(cuuint64_t)k, (cuuint64_t)rows};
  cuuint64_t strides[1] = {(cuuint64_t)ld};
  cuuint32_t box[2] = {(cuuint32_t)BK, (cuuint32_t)box_rows};
  cuuint32_t estr[2] = {1, 1};
  CUresult r = fn(m, CU_TENSOR_MAP_DATA_TYPE_UINT8, 2, const_cast<int8_t *>(ptr), dims, strides, box, estr,
                  CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                  CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) return fail(LRAMM_ERR_CUDA, "cuTensorMapEncodeTiled failed (%d)", (int)r);
  return LRAMM_OK;
}

// packed-int4 A: rows of ceil(K/2) bytes, box 64 bytes (one 128-element k-block) x box_rows,
// no swizzle (the kernel's unpack step writes the swizzled int8 tile)
int make_tmap_i4(CUtensorMap *m, const int8_t *ptr, int64_t rows, int64_t k, int64_t ld_bytes, int box_rows) {
  auto fn = encode_fn();
  if (!fn) return fail(LRAMM_ERR_CUDA, "cuTensorMapEncodeTiled unavailable");
  cuuint64_t dims[2] = {(cuuint64_t)ceil_div(k, 2), (cuuint64_t)rows};
  cuuint64_t strides[1] = {(cuuint64_t)ld_bytes};
  cuuint32_t box[2] = {(cuuint32_t)(BK / 2), (cuuint32_t)box_rows};
  cuuint32_t estr[2] = {1, 1};
  CUresult r = fn(m, CU_TENSOR_MAP_DATA_TYPE_UINT8, 2, const_cast<int8_t *>(ptr), dims, strides, box, estr,
                  CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                  CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) return fail(LRAMM_ERR_CUDA, "cuTensorMapEncodeTiled (int4) failed (%d)", (int)r);
  return LRAMM_OK;
}

EpiDev to_dev(const lramm_epilogue_t &e) {
  EpiDev d;
  d.out_dtype = e.out_dtype;
  d.accumulate = e.accumulate;
  d.transpose_out = e.transpose_out;
  d.c_dtype = e.c_dtype;
  d.out = e.out;
  d.ldo = e.ldo;
  d.row_scale = e.row_scale;
  d.row_scale_inc = e.row_scale_inc;
  d.col_scale = e.col_scale;
  d.col_scale_inc = e.col_scale_inc;
  d.alpha = e.alpha;
  d.beta = e.beta;
  d.c = e.c;
  d.ldc = e.ldc;
  d.shift = 0;
  d.signs = 3;
  d.nfast = 0;
  d.a4 = 0;
  return d;
}

}  // namespace

// limb-pair launch parameters (set only around igemm_limbs_device's launches; thread-local so
// concurrent host threads do not interfere)
static thread_local int g_limb_shift = 0;
static thread_local int g_limb_signs = 3;

// BN: multiple of 16 in [16, 256] covering N with the fewest tiles and least padding
int pick_bn(int64_t N) {
  int64_t tiles = ceil_div(N, 256);
  int64_t bn = round_up(ceil_div(N, tiles), 16);
  return (int)std::max<int64_t>(16, std::min<int64_t>(256, bn));
}

int igemm_device(int64_t M, int64_t N, int64_t K, const int8_t *a, int64_t lda, const int8_t *b, int64_t ldb,
                 const lramm_epilogue_t &epi, int split_k, cudaStream_t st, int a4 = 0) {
  if (M < 1 || N < 1 || K < 1) return fail(LRAMM_ERR_SHAPE, "igemm: empty shape");
  // a4: A is packed int4, lda in bytes (>= ceil(K/2))
  if ((a4 ? 2 * lda < K : lda < K) || ldb < K || (lda % 16) || (ldb % 16))
    return fail(LRAMM_ERR_SHAPE, "igemm: leading dims must cover K and be multiples of 16");
  if ((reinterpret_cast<uintptr_t>(a) | reinterpret_cast<uintptr_t>(b)) & 15)
    return fail(LRAMM_ERR_SHAPE, "igemm: operands must be 16-byte aligned");
  if (M > INT32_MAX || N > INT32_MAX || K > INT32_MAX) return fail(LRAMM_ERR_SHAPE, "igemm: dims exceed int32");
  const int kb_total = (int)ceil_div(K, BK);
  split_k = std::max(1, std::min(split_k, kb_total));
  if (split_k > 1 && !(epi.out_dtype == LRAMM_I32 && epi.accumulate))
    return fail(LRAMM_ERR_PARAM, "igemm: split-K needs an accumulating int32 output");
  const int kb_per = (int)ceil_div(kb_total, split_k);
  split_k = (int)ceil_div(kb_total, kb_per);
  const int BN = pick_bn(N);
  const int stage_bytes = BM * BK + BN * BK + (a4 ? BM * BK / 2 : 0);
  // no more stages than k-blocks: short-K products (E2, E3) then fit two CTAs per SM
  int stages = std::max(2, std::min(std::min(8, kb_total), (kSmemBudget - 2048) / stage_bytes));
  // more than one wave: a shallower ring that fits two CTAs per SM (and two TMEM accumulators),
  // so one CTA's epilogue overlaps the other's loads and MMAs (c5 E3 131072x8192x1024: 4.1 ->
  // 2.7 ms; c3 E3: 239 -> 143 us); single-wave grids keep the deep ring
  const int64_t ctas = ceil_div(M, BM) * ceil_div(N, BN) * split_k;
  const int two_per_sm = (109 * 1024) / stage_bytes;  // + barriers, alignment slack and 2 KB static (cs_sh) <= 113 KB
  if (ctas > num_sms() && two_per_sm >= 2) stages = std::min(stages, two_per_sm);
  const int smem = stages * stage_bytes + (3 * stages + 2) * 8 + 1024 + 64;
  CUtensorMap ta, tb;
  if (a4)
    LRAMM_TRY(make_tmap_i4(&ta, a, M, K, lda, BM));
  else
    LRAMM_TRY(make_tmap_i8(&ta, a, M, K, lda, BM));
  LRAMM_TRY(make_tmap_i8(&tb, b, N, K, ldb, BN));
  const int ek = epi.out_dtype == LRAMM_I64 ? EK_I64_ADD
                 : epi.out_dtype == LRAMM_I32 ? (epi.accumulate ? EK_I32_ATOMIC : EK_I32)
                                              : (epi.out_dtype == LRAMM_F64 ? EK_F64 : EK_F32);
  if (ek == EK_I64_ADD && split_k > 1) return fail(LRAMM_ERR_PARAM, "igemm: int64 accumulation runs without split-K");
  const bool ab = (ek == EK_F32 || ek == EK_F64) && (epi.alpha != 1.0 || (epi.beta != 0.0 && epi.c != nullptr));
  using KernT = void (*)(CUtensorMap, CUtensorMap, int64_t, int64_t, int64_t, int, int, int, EpiDev);
  KernT kern = nullptr;
#define LRAMM_IG_PICK(EKV, TR, ABV) \
  if (ek == EKV && (epi.transpose_out != 0) == TR && ab == ABV) kern = igemm_tn_kernel<EKV, TR, ABV>;
  LRAMM_IG_PICK(EK_I32, false, false) LRAMM_IG_PICK(EK_I32, true, false)
  LRAMM_IG_PICK(EK_I32_ATOMIC, false, false) LRAMM_IG_PICK(EK_I32_ATOMIC, true, false)
  LRAMM_IG_PICK(EK_F32, false, false) LRAMM_IG_PICK(EK_F32, true, false)
  LRAMM_IG_PICK(EK_F32, false, true) LRAMM_IG_PICK(EK_F32, true, true)
  LRAMM_IG_PICK(EK_F64, false, false) LRAMM_IG_PICK(EK_F64, true, false)
  LRAMM_IG_PICK(EK_F64, false, true) LRAMM_IG_PICK(EK_F64, true, true)
  LRAMM_IG_PICK(EK_I64_ADD, false, false)
#undef LRAMM_IG_PICK
  if (!kern) return fail(LRAMM_ERR_PARAM, "igemm: unsupported epilogue");
  LRAMM_CUDA_TRY(allow_max_dyn_smem(kern));
  // rasterisation: M-fastest keeps one B tile hot while A tiles stream; when A is the larger
  // operand and does not fit in L2 (c5: A 134 MB-1 GB, B 8 MB) that re-reads A from HBM once per
  // N tile, so the grid goes N-fastest instead and B is the operand re-read (from L2)
  const int64_t mt = ceil_div(M, BM), nt = ceil_div(N, BN);
  const bool nfast = nt > 1 && M * K > N * K && M * K > (int64_t)48 << 20 && mt <= 65535;
  dim3 grid = nfast ? dim3((unsigned)nt, (unsigned)mt, (unsigned)split_k)
                    : dim3((unsigned)mt, (unsigned)nt, (unsigned)split_k);
  EpiDev ed = to_dev(epi);
  ed.shift = g_limb_shift;
  ed.signs = g_limb_signs;
  ed.nfast = nfast ? 1 : 0;
  ed.a4 = a4 ? 1 : 0;
  kern<<<grid, kThreads, smem, st>>>(ta, tb, M, N, K, BN, stages, kb_per, ed);
  LRAMM_LAUNCH_CHECK();
  return LRAMM_OK;
}

// C = dequant(A . B^T) for multi-limb operands: A has la limb planes (rows x lda each, plane
// stride pa bytes), B lb planes; the la x lb int8 products accumulate exactly into acc64
// (int64, M x N) with the shifts 8(i + j), then the fp64 dequant epilogue (or raw int64 out)
int igemm_limbs_device(int64_t M, int64_t N, int64_t K, const int8_t *a, int64_t lda, int64_t pa, int la,
                       const int8_t *b, int64_t ldb, int64_t pb, int lb, int64_t *acc64,
                       const lramm_epilogue_t &epi, cudaStream_t st) {
  if (la < 1 || lb < 1 || la > 4 || lb > 4) return fail(LRAMM_ERR_PARAM, "igemm_limbs: 1..4 limbs per operand");
  LRAMM_CUDA_TRY(cudaMemsetAsync(acc64, 0, (size_t)M * N * sizeof(int64_t), st));
  lramm_epilogue_t e = {};
  e.out_dtype = LRAMM_I64;
  e.out = acc64;
  e.ldo = N;
  // each limb product accumulates exactly in int32 while K * 255^2 < 2^31: longer K in chunks
  const int64_t kc = 33024;  // multiple of 128, 33024 * 255^2 < 2^31
  for (int64_t k0 = 0; k0 < K; k0 += kc) {
    const int64_t kk = std::min(kc, K - k0);
    for (int i = 0; i < la; ++i)
      for (int j = 0; j < lb; ++j) {
        g_limb_shift = 8 * (i + j);
        g_limb_signs = (i == la - 1 ? 1 : 0) | (j == lb - 1 ? 2 : 0);
        const int rc = igemm_device(M, N, kk, a + i * pa + k0, lda, b + j * pb + k0, ldb, e, 1, st);
        g_limb_shift = 0;
        g_limb_signs = 3;
        if (rc) return rc;
      }
  }
  const unsigned gy = (unsigned)std::min<int64_t>(M, 8LL * num_sms());
  epilogue64_kernel<<<dim3((unsigned)ceil_div(N, 256), gy), 256, 0, st>>>(acc64, M, N, N, to_dev(epi));
  LRAMM_LAUNCH_CHECK();
  return LRAMM_OK;
}

int split_limbs_device(const int32_t *src, int64_t rows, int64_t cols, int64_t lds, int nlimb, int8_t *dst,
                       int64_t ldd, cudaStream_t st) {
  const unsigned gy = (unsigned)std::min<int64_t>(rows, 8LL * num_sms());
  split_limbs_kernel<<<dim3((unsigned)ceil_div(ldd, 256), gy), 256, 0, st>>>(src, rows, cols, lds, nlimb, dst, ldd,
                                                                             rows * ldd);
  LRAMM_LAUNCH_CHECK();
  return LRAMM_OK;
}

int epilogue_device(const int32_t *acc, int64_t M, int64_t N, int64_t lda, const lramm_epilogue_t &epi,
                    cudaStream_t st) {
  if (epi.out_dtype != LRAMM_F64 && epi.out_dtype != LRAMM_F32) {
    const dim3 grid((unsigned)ceil_div(N, 256),
                    (unsigned)std::min<int64_t>(M, std::max<int64_t>(1, 16LL * num_sms() / ceil_div(N, 256))));
    epilogue_generic_kernel<<<grid, 256, 0, st>>>(acc, M, N, lda, to_dev(epi));
  } else if (epi.transpose_out) {
    const dim3 grid((unsigned)std::min<int64_t>(ceil_div(N, 32), 4096),
                    (unsigned)std::min<int64_t>(ceil_div(M, 32), std::max<int64_t>(1, 8LL * num_sms() / ceil_div(N, 32))));
    epilogue_kernel<true><<<grid, 256, 0, st>>>(acc, M, N, lda, to_dev(epi));
  } else {
    const unsigned grid = (unsigned)std::min<int64_t>(ceil_div(M, 8), 16LL * num_sms());
    epilogue_kernel<false><<<grid, 256, 0, st>>>(acc, M, N, lda, to_dev(epi));
  }
  LRAMM_LAUNCH_CHECK();
  return LRAMM_OK;
}

}  // namespace lramm
