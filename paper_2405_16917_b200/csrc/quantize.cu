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

template <class T>
__global__ void absmax_tensor_kernel(const T *__restrict__ x, int64_t rows, int64_t cols, int64_t ldx,
                                     double *amax, int *nonfinite) {
  double m = 0.0;
  bool bad = false;
  for (int64_t r = blockIdx.x; r < rows; r += gridDim.x) {
    const T *row = x + r * ldx;
    for (int64_t c = threadIdx.x; c < cols; c += blockDim.x) {
      double v = (double)row[c];
      bad |= !isfinite(v);
      m = fmax(m, fabs(v));
    }
  }
  __shared__ double red[32];
  m = warp_max(m);
  int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  if (lane == 0) red[wid] = m;
  if (__syncthreads_or(bad) && threadIdx.x == 0 && nonfinite) *nonfinite = 1;
  if (wid == 0) {
    m = lane < (int)(blockDim.x >> 5) ? red[lane] : 0.0;
    m = warp_max(m);
    if (lane == 0) atomic_max_nonneg(amax, m);
  }
}

// one warp per row; 4 rows per 128-thread block
template <class T>
__global__ void absmax_rows_kernel(const T *__restrict__ x, int64_t rows, int64_t cols, int64_t ldx,
                                   double *amax_row, int *nonfinite) {
  int lane = threadIdx.x & 31;
  int64_t r = (int64_t)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  if (r >= rows) return;
  const T *row = x + r * ldx;
  double m = 0.0;
  bool bad = false;
  for (int64_t c = lane; c < cols; c += 32) {
    double v = (double)row[c];
    bad |= !isfinite(v);
    m = fmax(m, fabs(v));
  }
  m = warp_max(m);
  if (__any_sync(0xffffffffu, bad) && lane == 0 && nonfinite) *nonfinite = 1;
  if (lane == 0) amax_row[r] = m;
}

// 32-column tile x row chunk; block (32, 8)
template <class T>
__global__ void absmax_cols_kernel(const T *__restrict__ x, int64_t rows, int64_t cols, int64_t ldx,
                                   int64_t row_chunk, double *amax_col, int *nonfinite) {
  int64_t c = (int64_t)blockIdx.x * 32 + threadIdx.x;
  int64_t r0 = (int64_t)blockIdx.y * row_chunk;
  int64_t r1 = r0 + row_chunk < rows ? r0 + row_chunk : rows;
  double m = 0.0;
  bool bad = false;
  if (c < cols)
    for (int64_t r = r0 + threadIdx.y; r < r1; r += blockDim.y) {
      double v = (double)x[r * ldx + c];
      bad |= !isfinite(v);
      m = fmax(m, fabs(v));
    }
  __shared__ double red[8][33];
  red[threadIdx.y][threadIdx.x] = m;
  if (__syncthreads_or(bad) && threadIdx.x == 0 && threadIdx.y == 0 && nonfinite) *nonfinite = 1;
  if (threadIdx.y == 0 && c < cols) {
    for (int i = 1; i < (int)blockDim.y; ++i) m = fmax(m, red[i][threadIdx.x]);
    atomic_max_nonneg(amax_col + c, m);
  }
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
  const int sms = num_sms();
  if (gran == LRAMM_GRAN_TENSOR) {
    int grid = (int)std::min<int64_t>(rows, 8LL * sms);
    absmax_tensor_kernel<T><<<grid, 256, 0, st>>>(x, rows, cols, ldx, amax, nonfinite);
  } else if (gran == LRAMM_GRAN_ROW) {
    absmax_rows_kernel<T><<<(unsigned)ceil_div(rows, 4), 128, 0, st>>>(x, rows, cols, ldx, amax, nonfinite);
  } else {
    int64_t chunk = std::max<int64_t>(256, ceil_div(rows * ceil_div(cols, 32), 8LL * sms));
    dim3 grid((unsigned)ceil_div(cols, 32), (unsigned)ceil_div(rows, chunk));
    absmax_cols_kernel<T><<<grid, dim3(32, 8), 0, st>>>(x, rows, cols, ldx, chunk, amax, nonfinite);
  }
  LRAMM_LAUNCH_CHECK();
  return LRAMM_OK;
}

template <class T>
int quantize_from_amax(const T *x, int64_t rows, int64_t cols, int64_t ldx, int bits, int gran, int transpose,
                       const double *amax, void *q, int q_dtype, int64_t ldq, double *scales, cudaStream_t st) {
  const int cap = bit_cap(bits);
  const int64_t nscale = gran == LRAMM_GRAN_TENSOR ? 1 : (gran == LRAMM_GRAN_ROW ? rows : cols);
  scales_from_amax_kernel<<<(unsigned)ceil_div(nscale, 256), 256, 0, st>>>(amax, nscale, cap, scales);
  LRAMM_LAUNCH_CHECK();
  const int64_t out_rows = transpose ? cols : rows;
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
                  size_t ws_bytes, cudaStream_t st) {
  const int64_t nscale = gran == LRAMM_GRAN_TENSOR ? 1 : (gran == LRAMM_GRAN_ROW ? rows : cols);
  Arena ar(ws, ws_bytes);
  double *amax = ar.take<double>(nscale);
  if (!ar.ok() || amax == nullptr) return fail(LRAMM_ERR_WORKSPACE, "quantize: workspace too small");
  LRAMM_CUDA_TRY(cudaMemsetAsync(amax, 0, nscale * sizeof(double), st));
  LRAMM_TRY(absmax_launch<T>(x, rows, cols, ldx, gran, amax, nonfinite, st));
  return quantize_from_amax<T>(x, rows, cols, ldx, bits, gran, transpose, amax, q, q_dtype, ldq, scales, st);
}

}  // namespace

int quantize_device(const void *x, int x_dtype, int64_t rows, int64_t cols, int64_t ldx, int bits,
                    int gran, int transpose, void *q, int q_dtype, int64_t ldq, double *scales,
                    int *nonfinite, void *ws, size_t ws_bytes, cudaStream_t st) {
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
                                scales, nonfinite, ws, ws_bytes, st);
  if (x_dtype == LRAMM_F64)
    return quantize_impl<double>((const double *)x, rows, cols, ldx, bits, gran, transpose, q, q_dtype, ldq,
                                 scales, nonfinite, ws, ws_bytes, st);
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
                                     scales, st);
  if (x_dtype == LRAMM_F64)
    return quantize_from_amax<double>((const double *)x, rows, cols, ldx, bits, gran, transpose, amax, q, q_dtype,
                                      ldq, scales, st);
  return fail(LRAMM_ERR_PARAM, "quantize: input dtype must be F32 or F64");
}

size_t quantize_ws_bytes(int64_t rows, int64_t cols) {
  return (size_t)round_up(std::max(rows, cols) * (int64_t)sizeof(double), 256) + 256;
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
