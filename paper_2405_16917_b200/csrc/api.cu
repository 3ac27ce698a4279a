// extern "C" entry points of liblramm_cuda.so (include/lramm_cuda.h).
#include <algorithm>
#include <mutex>
#include <vector>

#include "common.cuh"

namespace lramm {

static thread_local std::string g_err;

void set_error(const char *fmt, ...) {
  char buf[1024];
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(buf, sizeof(buf), fmt, ap);
  va_end(ap);
  g_err = buf;
}

int fail(int code, const char *fmt, ...) {
  char buf[1024];
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(buf, sizeof(buf), fmt, ap);
  va_end(ap);
  g_err = buf;
  return code;
}

int num_sms() {
  static int cache[64] = {0};
  int dev = 0;
  cudaGetDevice(&dev);
  if (dev < 0 || dev >= 64) dev = 0;
  if (!cache[dev]) {
    int n = 0;
    cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev);
    cache[dev] = n > 0 ? n : 148;
  }
  return cache[dev];
}

// internal entry points
int quantize_device(const void *, int, int64_t, int64_t, int64_t, int, int, int, void *, int, int64_t, double *, int *,
                    void *, size_t, cudaStream_t, const AmaxSync *sync = nullptr);
size_t quantize_ws_bytes(int64_t, int64_t);
int quantize_pair_device(const void *, int, int64_t, int64_t, int64_t, int, int, int8_t *, int64_t, double *, int, int,
                         int8_t *, int64_t, double *, int *, void *, size_t, cudaStream_t, int r_packed = 0,
                         const AmaxSync *sync = nullptr);
int absmax_device(const void *, int, int64_t, int64_t, int64_t, int, double *, int *, cudaStream_t);
int quantize_amax_device(const void *, int, int64_t, int64_t, int64_t, int, int, int, const double *, void *, int, int64_t,
                         double *, cudaStream_t);
int cholqr_pass_device(const double *, int64_t, int64_t, int64_t, const double *, double *, int64_t, double *, int *,
                       void *, size_t, cudaStream_t);
size_t cholqr_pass_ws_bytes(int64_t, int64_t);
int epilogue_device(const int32_t *, int64_t, int64_t, int64_t, const lramm_epilogue_t &, cudaStream_t);
int scale_round_clip_device(const double *, int64_t, int64_t, int64_t, double, int, int32_t *, int64_t, cudaStream_t);
int igemm_device(int64_t, int64_t, int64_t, const int8_t *, int64_t, const int8_t *, int64_t, const lramm_epilogue_t &,
                 int, cudaStream_t, int a4 = 0);
int dgemm_device(int, int64_t, int64_t, int64_t, const double *, int64_t, const double *, int64_t, double *, int64_t,
                 void *, size_t, cudaStream_t);
size_t dgemm_ws_bytes(int, int64_t, int64_t, int64_t);
int qr_device(const double *, int64_t, int64_t, int64_t, double *, int64_t, double *, void *, size_t, cudaStream_t,
              bool q_needed = true, bool fast = false, const double *gram_in = nullptr,
              const Coll *rows_coll = nullptr);
size_t qr_ws_bytes(int64_t, int64_t);
int svd_tall_device(const double *, int64_t, int64_t, int64_t, double *, int64_t, double *, double *, int64_t, int *,
                    int *, void *, size_t, cudaStream_t, const Coll *rows_coll = nullptr, bool fast = false);
size_t svd_tall_ws_bytes(int64_t, int64_t);
int transpose_device(const double *, int64_t, int64_t, int64_t, double *, int64_t, cudaStream_t);
size_t rsvd_ws_bytes(int64_t, int64_t, const lramm_params_t &, int);
int rsvd_device(const void *, int, int64_t, int64_t, const lramm_params_t &, const double *, double *, double *,
                double *, int *, void *, size_t, cudaStream_t);
size_t lramm_ws_bytes(int64_t, int64_t, int64_t, const lramm_params_t &, int);
size_t lramm_sharded_ws_bytes(int64_t, int64_t, int64_t, const lramm_params_t &, int, int, int);
void shard_bounds_host(int64_t, int, int, int64_t *, int64_t *);
int lramm_sharded_device(const void *, const void *, int, int64_t, int64_t, int64_t, const lramm_params_t &,
                         const double *, const double *, const void *, int, void *, int, int *, void *, size_t,
                         const lramm_comm_t *, cudaStream_t);
int omega_device(uint64_t key0, uint64_t key1, int64_t n, int64_t w, double *out, void *ws, size_t ws_bytes,
                 cudaStream_t st);
size_t omega_ws_bytes(int64_t n, int64_t w);
int igemm_limbs_device(int64_t M, int64_t N, int64_t K, const int8_t *a, int64_t lda, int64_t pa, int la,
                       const int8_t *b, int64_t ldb, int64_t pb, int lb, int64_t *acc64,
                       const lramm_epilogue_t &epi, cudaStream_t st);
int split_limbs_device(const int32_t *src, int64_t rows, int64_t cols, int64_t lds, int nlimb, int8_t *dst,
                       int64_t ldd, cudaStream_t st);
int lramm_device(const void *, const void *, int, int64_t, int64_t, int64_t, const lramm_params_t &, const double *,
                 const double *, const void *, int, void *, int, int *, void *, size_t, lramm_timings_t *,
                 cudaStream_t, cudaEvent_t b_ready = nullptr, cudaEvent_t *stage_events = nullptr);

// ---------------------------------------------------------------- host-side device memory
// One cached device arena + stream for the host-pointer entry points (grow-only,
// serialised by a mutex; the device-pointer API never allocates).
struct HostCtx {
  std::mutex mu;
  char *buf = nullptr;
  size_t cap = 0;
  cudaStream_t st = nullptr;
  cudaStream_t copy = nullptr;  // upload stream (A, then B, Omega_B, C): A's chain starts first
  cudaStream_t down = nullptr;  // download stream of lramm_host_lramm (D), behind ev_done
  cudaEvent_t ev_a = nullptr, ev_b = nullptr, ev_done = nullptr;
  cudaEvent_t ev_t[6] = {};  // stage boundaries of lramm_host_lramm (timing events)
  int *status = nullptr;
  int *h_status = nullptr;  // pinned copy of the status word (read without another D2H copy)
  int dev = -1;
};
// Host entry points lease one context (streams + device buffer) for the duration of a call:
// concurrent host threads run on their own contexts and streams (the reference's kernels are
// thread-safe and reentrant and its sweeps call them from a thread pool, cli.py:415-419);
// contexts are reused, so device memory stays bounded by the peak number of concurrent calls.
struct CtxLease {
  static std::mutex &mu() {
    static std::mutex m;
    return m;
  }
  static std::vector<HostCtx *> &pool() {
    static std::vector<HostCtx *> p;
    return p;
  }
  HostCtx *c;
  CtxLease() {
    std::lock_guard<std::mutex> g(mu());
    if (pool().empty()) {
      c = new HostCtx();
    } else {
      c = pool().back();
      pool().pop_back();
    }
  }
  ~CtxLease() {
    std::lock_guard<std::mutex> g(mu());
    pool().push_back(c);
  }
};
static int host_reserve(HostCtx &c, size_t bytes) {
  int dev = 0;
  LRAMM_CUDA_TRY(cudaGetDevice(&dev));
  if (c.dev != dev) {  // new device: drop the old cache
    c.buf = nullptr;
    c.cap = 0;
    c.st = nullptr;
    c.copy = nullptr;
    c.down = nullptr;
    c.ev_a = c.ev_b = c.ev_done = nullptr;
    for (auto &e : c.ev_t) e = nullptr;
    c.status = nullptr;
    c.h_status = nullptr;
    c.dev = dev;
  }
  if (!c.st) LRAMM_CUDA_TRY(cudaStreamCreateWithFlags(&c.st, cudaStreamNonBlocking));
  if (!c.copy) LRAMM_CUDA_TRY(cudaStreamCreateWithFlags(&c.copy, cudaStreamNonBlocking));
  if (!c.down) LRAMM_CUDA_TRY(cudaStreamCreateWithFlags(&c.down, cudaStreamNonBlocking));
  if (!c.ev_a) LRAMM_CUDA_TRY(cudaEventCreateWithFlags(&c.ev_a, cudaEventDisableTiming));
  if (!c.ev_b) LRAMM_CUDA_TRY(cudaEventCreateWithFlags(&c.ev_b, cudaEventDisableTiming));
  if (!c.ev_done) LRAMM_CUDA_TRY(cudaEventCreateWithFlags(&c.ev_done, cudaEventDisableTiming));
  for (auto &e : c.ev_t)
    if (!e) LRAMM_CUDA_TRY(cudaEventCreate(&e));
  if (!c.status) LRAMM_CUDA_TRY(cudaMalloc(&c.status, 64));
  if (!c.h_status) LRAMM_CUDA_TRY(cudaMallocHost(&c.h_status, 64));
  if (bytes > c.cap) {
    if (c.buf) LRAMM_CUDA_TRY(cudaFree(c.buf));
    c.buf = nullptr;
    size_t want = round_up((int64_t)bytes, 1 << 20);
    LRAMM_CUDA_TRY(cudaMalloc(&c.buf, want));
    c.cap = want;
  }
  return LRAMM_OK;
}

}  // namespace lramm

using namespace lramm;

extern "C" {

const char *lramm_last_error(void) { return g_err.c_str(); }
const char *lramm_version(void) { return "lramm-b200 0.1.0 (sm_100a)"; }

int lramm_device_check(void) {
  int dev = 0, major = 0, minor = 0;
  if (cudaGetDevice(&dev) != cudaSuccess) return fail(LRAMM_ERR_UNSUPPORTED, "no CUDA device");
  cudaDeviceGetAttribute(&major, cudaDevAttrComputeCapabilityMajor, dev);
  cudaDeviceGetAttribute(&minor, cudaDevAttrComputeCapabilityMinor, dev);
  if (major != 10 || minor != 0)
    return fail(LRAMM_ERR_UNSUPPORTED, "liblramm_cuda is built for sm_100a; device is sm_%d%d", major, minor);
  return LRAMM_OK;
}

int lramm_quantize(const void *x, int x_dtype, int64_t rows, int64_t cols, int64_t ldx, int bits, int granularity,
                   int transpose_out, void *q, int q_dtype, int64_t ldq, double *scales, int *nonfinite_flag, void *ws,
                   size_t ws_bytes, lramm_stream_t stream) {
  return quantize_device(x, x_dtype, rows, cols, ldx, bits, granularity, transpose_out, q, q_dtype, ldq, scales,
                         nonfinite_flag, ws, ws_bytes, (cudaStream_t)stream);
}
size_t lramm_quantize_ws(int64_t rows, int64_t cols) { return quantize_ws_bytes(rows, cols); }

int lramm_quantize_pair(const void *x, int x_dtype, int64_t rows, int64_t cols, int64_t ldx, int bits_r,
                        int granularity_r, int8_t *q_r, int64_t ldq_r, double *scales_r, int bits_t,
                        int granularity_t, int8_t *q_t, int64_t ldq_t, double *scales_t, int *nonfinite_flag,
                        void *ws, size_t ws_bytes, lramm_stream_t stream) {
  return quantize_pair_device(x, x_dtype, rows, cols, ldx, bits_r, granularity_r, q_r, ldq_r, scales_r, bits_t,
                              granularity_t, q_t, ldq_t, scales_t, nonfinite_flag, ws, ws_bytes, (cudaStream_t)stream);
}

int lramm_absmax(const void *x, int x_dtype, int64_t rows, int64_t cols, int64_t ldx, int granularity, double *amax,
                 int *nonfinite_flag, lramm_stream_t stream) {
  return absmax_device(x, x_dtype, rows, cols, ldx, granularity, amax, nonfinite_flag, (cudaStream_t)stream);
}

int lramm_quantize_amax(const void *x, int x_dtype, int64_t rows, int64_t cols, int64_t ldx, int bits,
                        int granularity, int transpose_out, const double *amax, void *q, int q_dtype, int64_t ldq,
                        double *scales, lramm_stream_t stream) {
  return quantize_amax_device(x, x_dtype, rows, cols, ldx, bits, granularity, transpose_out, amax, q, q_dtype, ldq,
                              scales, (cudaStream_t)stream);
}

int lramm_cholqr_pass(const double *y, int64_t m, int64_t w, int64_t ldy, const double *gram, double *q, int64_t ldq,
                      double *l, int *info, void *ws, size_t ws_bytes, lramm_stream_t stream) {
  return cholqr_pass_device(y, m, w, ldy, gram, q, ldq, l, info, ws, ws_bytes, (cudaStream_t)stream);
}
size_t lramm_cholqr_pass_ws(int64_t m, int64_t w) { return cholqr_pass_ws_bytes(m, w); }

int lramm_dequant(const int32_t *acc, int64_t M, int64_t N, int64_t lda, const lramm_epilogue_t *epi,
                  lramm_stream_t stream) {
  if (!epi) return fail(LRAMM_ERR_PARAM, "dequant: epilogue is NULL");
  return epilogue_device(acc, M, N, lda, *epi, (cudaStream_t)stream);
}

int lramm_scale_round_clip(const double *a, int64_t rows, int64_t cols, int64_t lda, double scale, int cap, int32_t *out,
                           int64_t ldo, lramm_stream_t stream) {
  return scale_round_clip_device(a, rows, cols, lda, scale, cap, out, ldo, (cudaStream_t)stream);
}

int lramm_igemm(int64_t M, int64_t N, int64_t K, const int8_t *a, int64_t lda, const int8_t *b, int64_t ldb,
                const lramm_epilogue_t *epi, int split_k, lramm_stream_t stream) {
  if (!epi) return fail(LRAMM_ERR_PARAM, "igemm: epilogue is NULL");
  return igemm_device(M, N, K, a, lda, b, ldb, *epi, split_k, (cudaStream_t)stream);
}

int lramm_igemm_i4(int64_t M, int64_t N, int64_t K, const uint8_t *a4, int64_t lda, const int8_t *b, int64_t ldb,
                   const lramm_epilogue_t *epi, int split_k, lramm_stream_t stream) {
  if (!epi) return fail(LRAMM_ERR_PARAM, "igemm_i4: epilogue is NULL");
  return igemm_device(M, N, K, (const int8_t *)a4, lda, b, ldb, *epi, split_k, (cudaStream_t)stream, 1);
}

int lramm_omega(uint64_t key0, uint64_t key1, int64_t ncols, int64_t w, double *out, void *ws, size_t ws_bytes,
                lramm_stream_t stream) {
  return omega_device(key0, key1, ncols, w, out, ws, ws_bytes, (cudaStream_t)stream);
}
size_t lramm_omega_ws(int64_t ncols, int64_t w) { return omega_ws_bytes(ncols, w); }

int lramm_split_limbs(const int32_t *src, int64_t rows, int64_t cols, int64_t lds, int nlimb, int8_t *dst,
                      int64_t ldd, lramm_stream_t stream) {
  if (nlimb < 1 || nlimb > 4) return fail(LRAMM_ERR_PARAM, "split_limbs: 1..4 limbs");
  if (rows < 1 || cols < 1 || ldd < cols || (ldd % 16)) return fail(LRAMM_ERR_SHAPE, "split_limbs: bad shape");
  return split_limbs_device(src, rows, cols, lds, nlimb, dst, ldd, (cudaStream_t)stream);
}

int lramm_igemm_limbs(int64_t M, int64_t N, int64_t K, const int8_t *a, int64_t lda, int64_t pa, int la,
                      const int8_t *b, int64_t ldb, int64_t pb, int lb, int64_t *acc64, const lramm_epilogue_t *epi,
                      lramm_stream_t stream) {
  if (!epi) return fail(LRAMM_ERR_PARAM, "igemm_limbs: epilogue is NULL");
  if (!acc64) return fail(LRAMM_ERR_PARAM, "igemm_limbs: acc64 is NULL");
  return igemm_limbs_device(M, N, K, a, lda, pa, la, b, ldb, pb, lb, acc64, *epi, (cudaStream_t)stream);
}

int lramm_dgemm(int trans_a, int64_t M, int64_t N, int64_t K, const double *a, int64_t lda, const double *b,
                int64_t ldb, double *c, int64_t ldc, void *ws, size_t ws_bytes, lramm_stream_t stream) {
  return dgemm_device(trans_a, M, N, K, a, lda, b, ldb, c, ldc, ws, ws_bytes, (cudaStream_t)stream);
}
size_t lramm_dgemm_ws(int trans_a, int64_t M, int64_t N, int64_t K) { return dgemm_ws_bytes(trans_a, M, N, K); }

int lramm_qr(const double *y, int64_t m, int64_t w, int64_t ldy, double *q, int64_t ldq, double *r, void *ws,
             size_t ws_bytes, lramm_stream_t stream) {
  return qr_device(y, m, w, ldy, q, ldq, r, ws, ws_bytes, (cudaStream_t)stream);
}
size_t lramm_qr_ws(int64_t m, int64_t w) { return qr_ws_bytes(m, w); }

// SVD (matcore.oracle_svd contract).  Tall: u = A H S^-1, v = H.  Wide: work on A^T.
size_t lramm_svd_ws(int64_t m, int64_t n) {
  int64_t t = std::min(m, n), l = std::max(m, n);
  return svd_tall_ws_bytes(l, t) + (size_t)round_up(l * t * 8, 256) + 512;
}
int lramm_svd(const double *a, int64_t m, int64_t n, double *u, double *s, double *v, int *info, void *ws,
              size_t ws_bytes, lramm_stream_t stream) {
  cudaStream_t st = (cudaStream_t)stream;
  if (m < 1 || n < 1) return fail(LRAMM_ERR_SHAPE, "svd: empty matrix");
  const int64_t t = std::min(m, n), l = std::max(m, n);
  if (ws_bytes < lramm_svd_ws(m, n)) return fail(LRAMM_ERR_WORKSPACE, "svd: workspace too small");
  Arena ar(ws, ws_bytes);
  double *at = ar.take<double>(l * t);
  int *st_compl = ar.take<int>(4);
  size_t rest = ws_bytes - ar.off;
  void *inner = (char *)ws + ar.off;
  LRAMM_CUDA_TRY(cudaMemsetAsync(st_compl, 0, 16, st));
  if (m >= n)
    return svd_tall_device(a, m, n, n, u, n, s, v, n, info, st_compl, inner, rest, st);
  // wide: A^T (n x m) = P S H^T  =>  A = H S P^T : u = H, v = P
  LRAMM_TRY(transpose_device(a, m, n, n, at, m, st));
  return svd_tall_device(at, n, m, m, v, m, s, u, m, info, st_compl, inner, rest, st);
}

size_t lramm_rsvd_ws(int64_t rows, int64_t cols, const lramm_params_t *params) {
  return params ? rsvd_ws_bytes(rows, cols, *params, LRAMM_F32) : 0;
}
int lramm_rsvd(const void *x, int x_dtype, int64_t rows, int64_t cols, const lramm_params_t *params,
               const double *omega, double *u, double *s, double *v, int *status, void *ws, size_t ws_bytes,
               lramm_stream_t stream) {
  if (!params) return fail(LRAMM_ERR_PARAM, "rsvd: params is NULL");
  return rsvd_device(x, x_dtype, rows, cols, *params, omega, u, s, v, status, ws, ws_bytes, (cudaStream_t)stream);
}

size_t lramm_lramm_ws(int64_t m, int64_t k, int64_t n, const lramm_params_t *params) {
  return params ? lramm_ws_bytes(m, k, n, *params, LRAMM_F32) : 0;
}
int lramm_lramm(const void *a, const void *b, int in_dtype, int64_t m, int64_t k, int64_t n,
                const lramm_params_t *params, const double *omega_a, const double *omega_b, const void *c, int c_dtype,
                void *d, int d_dtype, int *status, void *ws, size_t ws_bytes, lramm_timings_t *timings,
                lramm_stream_t stream) {
  if (!params) return fail(LRAMM_ERR_PARAM, "lramm: params is NULL");
  return lramm_device(a, b, in_dtype, m, k, n, *params, omega_a, omega_b, c, c_dtype, d, d_dtype, status, ws, ws_bytes,
                      timings, (cudaStream_t)stream);
}

void lramm_shard_bounds(int64_t total, int32_t world, int32_t rank, int64_t *lo, int64_t *hi) {
  shard_bounds_host(total, world, rank, lo, hi);
}
size_t lramm_lramm_sharded_ws(int64_t m, int64_t k, int64_t n, const lramm_params_t *params, int32_t world,
                              int32_t rank) {
  return params ? lramm_sharded_ws_bytes(m, k, n, *params, LRAMM_F32, world, rank) : 0;
}
int lramm_lramm_sharded(const void *a_rows, const void *b_cols, int in_dtype, int64_t m, int64_t k, int64_t n,
                        const lramm_params_t *params, const double *omega_a, const double *omega_b,
                        const void *c_rows, int c_dtype, void *d_rows, int d_dtype, int *status, void *ws,
                        size_t ws_bytes, const lramm_comm_t *comm, lramm_stream_t stream) {
  if (!params) return fail(LRAMM_ERR_PARAM, "lramm_sharded: params is NULL");
  return lramm_sharded_device(a_rows, b_cols, in_dtype, m, k, n, *params, omega_a, omega_b, c_rows, c_dtype, d_rows,
                              d_dtype, status, ws, ws_bytes, comm, (cudaStream_t)stream);
}

// ---------------------------------------------------------------- host API
static int status_to_rc(int s) {
  if (s == LRAMM_ERR_NONCONVERGENCE) return fail(s, "jacobi sweeps did not converge within 60");
  if (s == LRAMM_ERR_NONFINITE) return fail(s, "cannot quantize non-finite entries");
  if (s) return fail(s, "device status %d", s);
  return LRAMM_OK;
}

static int finish(HostCtx &c) {
  LRAMM_CUDA_TRY(cudaStreamSynchronize(c.st));
  int s = 0;
  LRAMM_CUDA_TRY(cudaMemcpy(&s, c.status, sizeof(int), cudaMemcpyDeviceToHost));
  if (s == LRAMM_ERR_NONCONVERGENCE) return fail(s, "jacobi sweeps did not converge within 60");
  if (s == LRAMM_ERR_NONFINITE) return fail(s, "cannot quantize non-finite entries");
  if (s) return fail(s, "device status %d", s);
  return LRAMM_OK;
}

int lramm_host_matmul(const double *a, const double *b, double *out, int64_t m, int64_t k, int64_t n) {
  if (m < 1 || k < 1 || n < 1) return fail(LRAMM_ERR_SHAPE, "inner dimensions differ");
  CtxLease lease;
  HostCtx &c = *lease.c;
  size_t gw = dgemm_ws_bytes(0, m, n, k);
  size_t need = (size_t)round_up((m * k + k * n + m * n) * 8, 256) * 1 + gw + 4096;
  LRAMM_TRY(host_reserve(c, need));
  Arena ar(c.buf, c.cap);
  double *da = ar.take<double>(m * k), *db = ar.take<double>(k * n), *dc = ar.take<double>(m * n);
  void *w = ar.take<char>((int64_t)gw + 8);
  LRAMM_CUDA_TRY(cudaMemcpyAsync(da, a, m * k * 8, cudaMemcpyHostToDevice, c.st));
  LRAMM_CUDA_TRY(cudaMemcpyAsync(db, b, k * n * 8, cudaMemcpyHostToDevice, c.st));
  LRAMM_TRY(dgemm_device(0, m, n, k, da, k, db, n, dc, n, w, gw, c.st));
  LRAMM_CUDA_TRY(cudaMemcpyAsync(out, dc, m * n * 8, cudaMemcpyDeviceToHost, c.st));
  LRAMM_CUDA_TRY(cudaMemsetAsync(c.status, 0, 4, c.st));
  return finish(c);
}

namespace {
// out (cols x rows) = x^T through 32 x 32 tiles
__global__ void transpose_i32_kernel(const int32_t *__restrict__ x, int64_t rows, int64_t cols,
                                     int32_t *__restrict__ out) {
  __shared__ int32_t t[32][33];
  const int64_t c0 = (int64_t)blockIdx.x * 32, r0 = (int64_t)blockIdx.y * 32;
  for (int i = threadIdx.y; i < 32; i += 8)
    if (r0 + i < rows && c0 + threadIdx.x < cols) t[i][threadIdx.x] = x[(r0 + i) * cols + c0 + threadIdx.x];
  __syncthreads();
  for (int i = threadIdx.y; i < 32; i += 8)
    if (c0 + i < cols && r0 + threadIdx.x < rows) out[(c0 + i) * rows + r0 + threadIdx.x] = t[threadIdx.x][i];
}
__global__ void max_abs_i32_kernel(const int32_t *x, int64_t n, unsigned *out) {
  unsigned m = 0;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    int v = x[i];
    unsigned a = v < 0 ? (unsigned)(-(int64_t)v) : (unsigned)v;
    m = a > m ? a : m;
  }
  atomicMax(out, m);
}
}  // namespace

// exact int32 x int32 -> int64 for |entries| <= 127 (bit budgets <= 8) on the int8 tensor cores
int lramm_host_imatmul(const int32_t *a, const int32_t *b, int64_t *out, int64_t m, int64_t k, int64_t n) {
  // exact int64 product of arbitrary int32 matrices (_core.pyx:35-50): each operand is split
  // into 1..4 8-bit limbs (as many as its largest magnitude needs) and the limb products run
  // on the int8 tensor cores, accumulated exactly in int64
  if (m < 1 || k < 1 || n < 1) return fail(LRAMM_ERR_SHAPE, "inner dimensions differ");
  CtxLease lease;
  HostCtx &c = *lease.c;
  const int64_t ldk = round_up(k, 16);
  size_t need = (size_t)round_up((m * k + 2 * k * n) * 4, 256) + round_up(4 * (m + n) * ldk, 256) +
                round_up(2 * m * n * 8, 256) + 8192;
  LRAMM_TRY(host_reserve(c, need));
  Arena ar(c.buf, c.cap);
  int32_t *da = ar.take<int32_t>(m * k), *db = ar.take<int32_t>(k * n), *dbt = ar.take<int32_t>(n * k);
  int8_t *qa = ar.take<int8_t>(4 * m * ldk), *qb = ar.take<int8_t>(4 * n * ldk);
  int64_t *acc = ar.take<int64_t>(m * n), *o64 = ar.take<int64_t>(m * n);
  unsigned *mx = ar.take<unsigned>(4);
  LRAMM_CUDA_TRY(cudaMemcpyAsync(da, a, m * k * 4, cudaMemcpyHostToDevice, c.st));
  LRAMM_CUDA_TRY(cudaMemcpyAsync(db, b, k * n * 4, cudaMemcpyHostToDevice, c.st));
  LRAMM_CUDA_TRY(cudaMemsetAsync(mx, 0, 16, c.st));
  const int grid = 4 * num_sms();
  max_abs_i32_kernel<<<grid, 256, 0, c.st>>>(da, m * k, mx);
  max_abs_i32_kernel<<<grid, 256, 0, c.st>>>(db, k * n, mx + 1);
  transpose_i32_kernel<<<dim3((unsigned)ceil_div(n, 32), (unsigned)ceil_div(k, 32)), dim3(32, 8), 0, c.st>>>(
      db, k, n, dbt);  // B^T: n x k, K-major
  LRAMM_LAUNCH_CHECK();
  unsigned hmx[2] = {0, 0};
  LRAMM_CUDA_TRY(cudaMemcpyAsync(hmx, mx, 8, cudaMemcpyDeviceToHost, c.st));
  LRAMM_CUDA_TRY(cudaStreamSynchronize(c.st));
  auto limbs = [](unsigned v) { return v <= 127u ? 1 : (v <= 32767u ? 2 : (v <= 8388607u ? 3 : 4)); };
  const int la = limbs(hmx[0]), lb = limbs(hmx[1]);
  LRAMM_TRY(split_limbs_device(da, m, k, k, la, qa, ldk, c.st));
  LRAMM_TRY(split_limbs_device(dbt, n, k, k, lb, qb, ldk, c.st));
  lramm_epilogue_t e = {};
  e.out_dtype = LRAMM_I64;
  e.out = o64;
  e.ldo = n;
  LRAMM_TRY(igemm_limbs_device(m, n, k, qa, ldk, m * ldk, la, qb, ldk, n * ldk, lb, acc, e, c.st));
  LRAMM_CUDA_TRY(cudaMemcpyAsync(out, o64, m * n * 8, cudaMemcpyDeviceToHost, c.st));
  LRAMM_CUDA_TRY(cudaMemsetAsync(c.status, 0, 4, c.st));
  return finish(c);
}

int lramm_host_scale_round_clip(const double *a, int64_t m, int64_t n, double scale, int cap, int32_t *out) {
  if (m < 1 || n < 1) return fail(LRAMM_ERR_SHAPE, "empty matrix");
  CtxLease lease;
  HostCtx &c = *lease.c;
  LRAMM_TRY(host_reserve(c, (size_t)round_up(m * n * 8, 256) + round_up(m * n * 4, 256) + 4096));
  Arena ar(c.buf, c.cap);
  double *da = ar.take<double>(m * n);
  int32_t *dq = ar.take<int32_t>(m * n);
  LRAMM_CUDA_TRY(cudaMemcpyAsync(da, a, m * n * 8, cudaMemcpyHostToDevice, c.st));
  LRAMM_TRY(scale_round_clip_device(da, m, n, n, scale, cap, dq, n, c.st));
  LRAMM_CUDA_TRY(cudaMemcpyAsync(out, dq, m * n * 4, cudaMemcpyDeviceToHost, c.st));
  LRAMM_CUDA_TRY(cudaMemsetAsync(c.status, 0, 4, c.st));
  return finish(c);
}

int lramm_host_svd(const double *a, int64_t m, int64_t n, double *u, double *s, double *v) {
  if (m < 1 || n < 1) return fail(LRAMM_ERR_SHAPE, "empty matrix");
  CtxLease lease;
  HostCtx &c = *lease.c;
  const int64_t t = std::min(m, n);
  size_t ws = lramm_svd_ws(m, n);
  LRAMM_TRY(host_reserve(c, (size_t)round_up((m * n + m * t + t + n * t) * 8, 256) + ws + 8192));
  Arena ar(c.buf, c.cap);
  double *da = ar.take<double>(m * n), *du = ar.take<double>(m * t), *ds = ar.take<double>(t),
         *dv = ar.take<double>(n * t);
  void *w = ar.take<char>((int64_t)ws);
  LRAMM_CUDA_TRY(cudaMemcpyAsync(da, a, m * n * 8, cudaMemcpyHostToDevice, c.st));
  LRAMM_CUDA_TRY(cudaMemsetAsync(c.status, 0, 16, c.st));
  LRAMM_TRY(lramm_svd(da, m, n, du, ds, dv, c.status + 1, w, ws, (lramm_stream_t)c.st));
  LRAMM_CUDA_TRY(cudaMemcpyAsync(u, du, m * t * 8, cudaMemcpyDeviceToHost, c.st));
  LRAMM_CUDA_TRY(cudaMemcpyAsync(s, ds, t * 8, cudaMemcpyDeviceToHost, c.st));
  LRAMM_CUDA_TRY(cudaMemcpyAsync(v, dv, n * t * 8, cudaMemcpyDeviceToHost, c.st));
  LRAMM_CUDA_TRY(cudaStreamSynchronize(c.st));
  int info = 0;
  LRAMM_CUDA_TRY(cudaMemcpy(&info, c.status + 1, sizeof(int), cudaMemcpyDeviceToHost));
  if (info < 0) return fail(LRAMM_ERR_NONCONVERGENCE, "jacobi sweeps did not converge within 60");
  return LRAMM_OK;
}

int lramm_host_lramm(const void *a, const void *b, int in_dtype, int64_t m, int64_t k, int64_t n,
                     const lramm_params_t *params, const double *omega_a, const double *omega_b, const void *cmat,
                     int c_dtype, void *d, int d_dtype, lramm_timings_t *timings) {
  if (!params) return fail(LRAMM_ERR_PARAM, "lramm: params is NULL");
  if (in_dtype != LRAMM_F32 && in_dtype != LRAMM_F64) return fail(LRAMM_ERR_PARAM, "inputs must be F32 or F64");
  CtxLease lease;
  HostCtx &c = *lease.c;
  const int64_t es = in_dtype == LRAMM_F32 ? 4 : 8, ds = d_dtype == LRAMM_F32 ? 4 : 8,
                cs = c_dtype == LRAMM_F32 ? 4 : 8;
  const int64_t wa = std::min<int64_t>(params->rank + params->oversample, std::min(m, k));
  const int64_t wb = std::min<int64_t>(params->rank + params->oversample, std::min(k, n));
  size_t ws = lramm_ws_bytes(m, k, n, *params, in_dtype);
  size_t need = (size_t)round_up((m * k + k * n) * es, 256) + round_up((k * wa + n * wb) * 8, 256) +
                round_up(m * n * ds, 256) + (cmat ? round_up(m * n * cs, 256) : 0) + ws + 8192;
  LRAMM_TRY(host_reserve(c, need));
  Arena ar(c.buf, c.cap);
  char *da = ar.take<char>(m * k * es), *db = ar.take<char>(k * n * es);
  double *oa = ar.take<double>(k * wa), *ob = ar.take<double>(n * wb);
  char *dd = ar.take<char>(m * n * ds);
  char *dc = cmat ? ar.take<char>(m * n * cs) : nullptr;
  void *w = ar.take<char>((int64_t)ws);
  // uploads overlap the factorisation: A's chain starts as soon as A (and Omega_A) have landed,
  // B's chain waits only for its own operands (b_ready); both uploads run on the copy stream
  // Omega may already live on this device (the device generator's cache): used in place
  auto on_device = [&](const void *p) {
    cudaPointerAttributes at;
    if (cudaPointerGetAttributes(&at, p) != cudaSuccess) {
      cudaGetLastError();
      return false;
    }
    return at.type == cudaMemoryTypeDevice && at.device == c.dev;
  };
  const double *oa_use = oa, *ob_use = ob;
  const bool oa_dev = on_device(omega_a), ob_dev = on_device(omega_b);
  if (oa_dev) oa_use = omega_a;
  if (ob_dev) ob_use = omega_b;
  {
    // one call's uploads are submitted as a unit (A, then B), all on the copy stream: with several
    // host threads in flight the copy engine then serves A1 B1 A2 B2 ... instead of A1 A2 .. B1 B2 ..,
    // so call i's factorisation overlaps call i+1's upload and call i-1's download
    static std::mutex upload_mu;
    std::lock_guard<std::mutex> g(upload_mu);
    if (!oa_dev) LRAMM_CUDA_TRY(cudaMemcpyAsync(oa, omega_a, k * wa * 8, cudaMemcpyHostToDevice, c.copy));
    LRAMM_CUDA_TRY(cudaMemcpyAsync(da, a, m * k * es, cudaMemcpyHostToDevice, c.copy));
    LRAMM_CUDA_TRY(cudaEventRecord(c.ev_a, c.copy));
    if (!ob_dev) LRAMM_CUDA_TRY(cudaMemcpyAsync(ob, omega_b, n * wb * 8, cudaMemcpyHostToDevice, c.copy));
    LRAMM_CUDA_TRY(cudaMemcpyAsync(db, b, k * n * es, cudaMemcpyHostToDevice, c.copy));
    if (cmat) LRAMM_CUDA_TRY(cudaMemcpyAsync(dc, cmat, m * n * cs, cudaMemcpyHostToDevice, c.copy));
    LRAMM_CUDA_TRY(cudaEventRecord(c.ev_b, c.copy));
  }
  LRAMM_CUDA_TRY(cudaStreamWaitEvent(c.st, c.ev_a, 0));
  // (the rsvd stage time of a host call therefore includes the tail of B's upload)
  // Device-side FIFO of concurrent host calls: kernels of a large product fill the GPU, so calls
  // whose factorisations interleave all finish late and their downloads queue up behind one
  // another (measured at c3, three calls in flight: first download at 38 ms instead of 19 ms).
  // Each large call therefore waits, on the device, for the call before it in its slot; copies
  // are not gated, so call i+1 uploads and call i-1 downloads while call i computes.  Small
  // products (latency-bound, e.g. the batched 2048^3 pairs) keep running side by side.
  static const int slots_env = [] {
    const char *e = getenv("LRAMM_HOST_COMPUTE_SLOTS");
    return e ? atoi(e) : -1;
  }();
  const bool big = std::max(std::max(m, n), k) >= 4096;
  const int slots = slots_env >= 0 ? std::min(slots_env, 8) : (big ? 1 : 0);
  {
    static std::mutex gate_mu;
    static cudaEvent_t last_done[8][64] = {};  // [slot][device]
    static unsigned long long ticket = 0;
    std::unique_lock<std::mutex> g(gate_mu, std::defer_lock);
    int slot = 0;
    const int dv = c.dev & 63;
    if (slots > 0) {
      g.lock();
      slot = (int)(ticket++ % (unsigned)slots);
      if (last_done[slot][dv]) LRAMM_CUDA_TRY(cudaStreamWaitEvent(c.st, last_done[slot][dv], 0));
    }
    const int rc_dev = lramm_device(da, db, in_dtype, m, k, n, *params, oa_use, ob_use, dc, c_dtype, dd, d_dtype,
                                    c.status, w, ws, timings, c.st, c.ev_b, timings ? c.ev_t : nullptr);
    if (rc_dev != LRAMM_OK) {  // refused before or while issuing: the uploads still read the caller's buffers
      cudaStreamSynchronize(c.copy);
      cudaStreamSynchronize(c.st);
      return rc_dev;
    }
    LRAMM_CUDA_TRY(cudaEventRecord(c.ev_done, c.st));
    if (slots > 0) last_done[slot][dv] = c.ev_done;
  }
  // D goes down on its own stream behind ev_done: the compute stream ends with the event the next
  // call in the FIFO waits for (with the copy queued on the compute stream itself the next call's
  // kernels started only when the download had finished: scripts/e2e_timeline.py)
  // The status word travels on the same stream just before D, into pinned memory: a separate
  // synchronous read after the download would queue behind the other calls' pending downloads in
  // the copy engine's FIFO (measured: four calls in flight all returned together).
  LRAMM_CUDA_TRY(cudaStreamWaitEvent(c.down, c.ev_done, 0));
  LRAMM_CUDA_TRY(cudaMemcpyAsync(c.h_status, c.status, sizeof(int), cudaMemcpyDeviceToHost, c.down));
  LRAMM_CUDA_TRY(cudaMemcpyAsync(d, dd, m * n * ds, cudaMemcpyDeviceToHost, c.down));
  LRAMM_CUDA_TRY(cudaStreamSynchronize(c.down));
  const int rc = status_to_rc(*c.h_status);
  if (timings && rc == LRAMM_OK) {
    float t[5];
    for (int i = 0; i < 5; ++i) LRAMM_CUDA_TRY(cudaEventElapsedTime(&t[i], c.ev_t[i], c.ev_t[i + 1]));
    timings->rsvd_ms = t[0];
    timings->scaling_ms = t[1];
    timings->gemm1_ms = t[2];
    timings->gemm2_ms = t[3];
    timings->gemm3_ms = t[4];
  }
  return rc;
}

}  // extern "C"
