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
};

// reference dequantisation + alpha/beta on one accumulator (bit-exact IEEE fp64)
__device__ __forceinline__ double epi_value(const EpiDev &e, int32_t acc, int64_t row, int64_t col) {
  double rs = e.row_scale ? e.row_scale[row * e.row_scale_inc] : 1.0;
  double cs = e.col_scale ? e.col_scale[col * e.col_scale_inc] : 1.0;
  double v = __ddiv_rn((double)acc, __dmul_rn(rs, cs));  // acc.astype(f64) / (sa*sb)
  if (e.beta != 0.0 && e.c != nullptr) {
    double cv = e.c_dtype == LRAMM_F32 ? (double)((const float *)e.c)[row * e.ldc + col]
                                       : ((const double *)e.c)[row * e.ldc + col];
    v = __dadd_rn(__dmul_rn(e.alpha, v), __dmul_rn(e.beta, cv));
  } else if (e.alpha != 1.0) {
    v = __dmul_rn(e.alpha, v);
  }
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
constexpr int kThreads = 192;
constexpr int kSmemBudget = 200 * 1024;

__global__ void __launch_bounds__(kThreads, 1)
    igemm_tn_kernel(const __grid_constant__ CUtensorMap tma_a, const __grid_constant__ CUtensorMap tma_b,
                    int64_t M, int64_t N, int64_t K, int BN, int stages, int kb_per_split, EpiDev epi) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t *smem = reinterpret_cast<uint8_t *>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  const uint32_t a_bytes = BM * BK;
  const uint32_t b_bytes = (uint32_t)BN * BK;
  uint8_t *sA = smem;
  uint8_t *sB = smem + (size_t)stages * a_bytes;
  uint64_t *full = reinterpret_cast<uint64_t *>(sB + (size_t)stages * b_bytes);
  uint64_t *empty = full + stages;
  uint64_t *tmem_full = empty + stages;
  uint32_t *tmem_slot = reinterpret_cast<uint32_t *>(tmem_full + 1);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int64_t m0 = (int64_t)blockIdx.x * BM;
  const int64_t n0 = (int64_t)blockIdx.y * BN;
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
        sm100::mbar_arrive_expect_tx(&full[s], a_bytes + b_bytes);
        const int32_t kx = (kb0 + i) * BK;
        sm100::tma_load_2d(&tma_a, &full[s], sA + (size_t)s * a_bytes, kx, (int32_t)m0);
        sm100::tma_load_2d(&tma_b, &full[s], sB + (size_t)s * b_bytes, kx, (int32_t)n0);
      }
    }
  } else if (warp == 1) {
    if (lane == 0) {
      const uint32_t idesc = sm100::idesc_i8(BM, BN);
      for (int i = 0; i < nkb; ++i) {
        const int s = i % stages;
        const uint32_t ph = (uint32_t)(i / stages) & 1u;
        sm100::mbar_wait(&full[s], ph);
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
    // epilogue warps 2..5
    const int quarter = warp & 3;
    const int64_t row = m0 + quarter * 32 + lane;
    if (nkb > 0) {
      sm100::mbar_wait(tmem_full, 0);
      sm100::tc_fence_after();
    }
    for (int c0 = 0; c0 < BN; c0 += 16) {
      uint32_t r[16];
      if (nkb > 0) {
        sm100::tmem_ld16(tmem_base + ((uint32_t)(quarter * 32) << 16) + (uint32_t)c0, r);
        sm100::tmem_wait_ld();
      } else {
#pragma unroll
        for (int j = 0; j < 16; ++j) r[j] = 0;
      }
      if (row < M) {
#pragma unroll
        for (int j = 0; j < 16; ++j) {
          const int64_t col = n0 + c0 + j;
          if (col < N) epi_store(epi, (int32_t)r[j], row, col);
        }
      }
    }
  }
  sm100::tc_fence_before();
  __syncthreads();
  if (warp == 1) sm100::tmem_dealloc(tmem_base, tmem_cols);
}

// stand-alone epilogue over an int32 accumulator matrix (after split-K)
__global__ void epilogue_kernel(const int32_t *__restrict__ acc, int64_t M, int64_t N, int64_t lda, EpiDev epi) {
  int64_t n = M * N;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    int64_t r = i / N, c = i - r * N;
    epi_store(epi, acc[r * lda + c], r, c);
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
  return d;
}

}  // namespace

// BN: multiple of 16 in [16, 256] covering N with the fewest tiles and least padding
int pick_bn(int64_t N) {
  int64_t tiles = ceil_div(N, 256);
  int64_t bn = round_up(ceil_div(N, tiles), 16);
  return (int)std::max<int64_t>(16, std::min<int64_t>(256, bn));
}

int igemm_device(int64_t M, int64_t N, int64_t K, const int8_t *a, int64_t lda, const int8_t *b, int64_t ldb,
                 const lramm_epilogue_t &epi, int split_k, cudaStream_t st) {
  if (M < 1 || N < 1 || K < 1) return fail(LRAMM_ERR_SHAPE, "igemm: empty shape");
  if (lda < K || ldb < K || (lda % 16) || (ldb % 16))
    return fail(LRAMM_ERR_SHAPE, "igemm: leading dims must be >= K and multiples of 16");
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
  const int stage_bytes = BM * BK + BN * BK;
  const int stages = std::max(2, std::min(8, (kSmemBudget - 2048) / stage_bytes));
  const int smem = stages * stage_bytes + (2 * stages + 2) * 8 + 1024 + 64;
  CUtensorMap ta, tb;
  LRAMM_TRY(make_tmap_i8(&ta, a, M, K, lda, BM));
  LRAMM_TRY(make_tmap_i8(&tb, b, N, K, ldb, BN));
  static std::once_flag attr_once;
  cudaError_t attr_err = cudaSuccess;
  std::call_once(attr_once, [&] {
    attr_err = allow_max_dyn_smem(igemm_tn_kernel);
  });
  LRAMM_CUDA_TRY(attr_err);
  dim3 grid((unsigned)ceil_div(M, BM), (unsigned)ceil_div(N, BN), (unsigned)split_k);
  igemm_tn_kernel<<<grid, kThreads, smem, st>>>(ta, tb, M, N, K, BN, stages, kb_per, to_dev(epi));
  LRAMM_LAUNCH_CHECK();
  return LRAMM_OK;
}

int epilogue_device(const int32_t *acc, int64_t M, int64_t N, int64_t lda, const lramm_epilogue_t &epi,
                    cudaStream_t st) {
  int grid = (int)std::min<int64_t>(ceil_div(M * N, 256), 16LL * num_sms());
  epilogue_kernel<<<grid, 256, 0, st>>>(acc, M, N, lda, to_dev(epi));
  LRAMM_LAUNCH_CHECK();
  return LRAMM_OK;
}

}  // namespace lramm
