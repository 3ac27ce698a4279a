// Shared helpers: status handling, numeric conventions, sm_100a PTX wrappers.
#pragma once

#include <cuda.h>
#include <cuda_runtime.h>
#include <stdint.h>

#include <cstdarg>
#include <cstdio>
#include <map>
#include <mutex>
#include <string>

#include <nvtx3/nvToolsExt.h>  // header-only NVTX v3 (resolved lazily; a no-op without an attached tool)

#include "../../include/lramm_cuda.h"

namespace lramm {

// NVTX range over the host-side issue of one pipeline stage (the reference's stage names,
// pipeline.py:40: rsvd / scaling / gemm1 / gemm2 / gemm3); nsys / ncu attribute the kernels
// launched inside it
struct NvtxStages {
  bool open = false;
  void next(const char *name) {  // closes the running stage, opens `name` (nullptr: just close)
    if (open) nvtxRangePop();
    open = name != nullptr;
    if (open) nvtxRangePushA(name);
  }
  ~NvtxStages() { next(nullptr); }  // error returns leave no range open
};

// ------------------------------------------------------------------ status
void set_error(const char *fmt, ...);
int fail(int code, const char *fmt, ...);

#define LRAMM_CUDA_TRY(expr)                                                              \
  do {                                                                                     \
    cudaError_t _e = (expr);                                                               \
    if (_e != cudaSuccess)                                                                 \
      return ::lramm::fail(LRAMM_ERR_CUDA, "%s failed: %s (%s:%d)", #expr,                  \
                           cudaGetErrorString(_e), __FILE__, __LINE__);                     \
  } while (0)

#define LRAMM_TRY(expr)        \
  do {                         \
    int _s = (expr);           \
    if (_s != LRAMM_OK) return _s; \
  } while (0)

#define LRAMM_LAUNCH_CHECK() LRAMM_CUDA_TRY(cudaGetLastError())

inline int64_t ceil_div(int64_t a, int64_t b) { return (a + b - 1) / b; }
inline int64_t round_up(int64_t a, int64_t b) { return ceil_div(a, b) * b; }
inline int bit_cap(int bits) { return (1 << (bits - 1)) - 1; }  // quant.py:20-22

// fp64 GEMM options (dgemm.cu): symmetric Gram output, upper-triangular B, alpha/beta epilogue,
// device-side gate (skip when *gate != 0)
struct DgemmOptions {
  int sym = 0;
  int b_upper = 0;
  double alpha = 1.0, beta = 0.0;
  const double *cin = nullptr;
  int64_t ldci = 0;
  const int *gate = nullptr;
  int gate_run_if_nonzero = 0;  // invert the gate: run only when *gate != 0
};
int dgemm_device_ex(int trans_a, int64_t M, int64_t N, int64_t K, const double *A, int64_t lda, const double *B,
                    int64_t ldb, double *C, int64_t ldc, void *ws, size_t ws_bytes, cudaStream_t st,
                    const DgemmOptions &opt);
int num_sms();

// opt a kernel into the largest dynamic shared memory the device allows next to its static smem
template <class K>
inline cudaError_t allow_max_dyn_smem(K kernel) {
  cudaFuncAttributes fa;
  cudaError_t e = cudaFuncGetAttributes(&fa, kernel);
  if (e != cudaSuccess) return e;
  int dev = 0, optin = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev);
  return cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, optin - (int)fa.sharedSizeBytes);
}

// Run a setup step (kernel attributes, symbol uploads) once per device: function attributes
// such as the dynamic shared-memory limit are per device, so a process-wide call_once would
// leave the second device of a multi-GPU process with the default limit.
struct PerDeviceOnce {
  static constexpr int kMaxDev = 64;
  std::once_flag flags[kMaxDev];
  cudaError_t err[kMaxDev] = {};
  template <class F>
  cudaError_t run(F &&f) {
    int dev = 0;
    cudaError_t e = cudaGetDevice(&dev);
    if (e != cudaSuccess) return e;
    if (dev < 0 || dev >= kMaxDev) return f();
    std::call_once(flags[dev], [&] { err[dev] = f(); });
    return err[dev];
  }
};

// ------------------------------------------------------------------ conditional graph sections
// The rarely taken branches of the factorisations (second CholeskyQR pass, Cholesky path of the
// closed-form update) are sequences of ~10 kernels that each read a device flag and return at
// once: cheap as work, but every one is a graph node (~1-2.5 us of launch chain; c4 is bound by
// its node count).  While the caller's stream is being captured into a CUDA graph the sequence
// is recorded instead into the body of an IF node (CUDA 12.4 conditional nodes): a one-thread
// kernel sets the node's condition from the flag, the body is captured on an auxiliary stream
// into the node's body graph, and the caller's capture continues behind the node.  Outside a
// capture (eager launches, the host entry points) nothing changes: stream() is the caller's
// stream and the kernels gate themselves as before (they keep their gates inside the body too).
static __global__ void cond_set_kernel(cudaGraphConditionalHandle h, const int *flag, int run_if_nonzero) {
  cudaGraphSetConditional(h, ((*flag != 0) == (run_if_nonzero != 0)) ? 1u : 0u);
}

struct CondIf {
  cudaStream_t outer = nullptr, body = nullptr;
  cudaGraphNode_t node = nullptr;
  bool active = false;
  static bool enabled() {
    static const bool on = [] {
      const char *e = getenv("LRAMM_GRAPH_COND");
      return !e || atoi(e) != 0;
    }();
    return on;
  }
  static cudaStream_t aux_stream(cudaStream_t main) {
    static std::mutex mu;
    static std::map<std::pair<int, cudaStream_t>, cudaStream_t> table;
    int dev = 0;
    cudaGetDevice(&dev);
    std::lock_guard<std::mutex> g(mu);
    cudaStream_t &x = table[{dev, main}];
    if (!x) cudaStreamCreateWithFlags(&x, cudaStreamNonBlocking);
    return x;
  }
  int begin(cudaStream_t st, const int *flag, bool run_if_nonzero) {
    outer = st;
    if (!enabled()) return LRAMM_OK;
    cudaStreamCaptureStatus cs = cudaStreamCaptureStatusNone;
    cudaGraph_t g = nullptr;
    const cudaGraphNode_t *deps = nullptr;
    size_t nd = 0;
    if (cudaStreamGetCaptureInfo(st, &cs, nullptr, &g, &deps, &nd) != cudaSuccess || cs != cudaStreamCaptureStatusActive) {
      cudaGetLastError();
      return LRAMM_OK;  // not capturing: the kernels gate themselves
    }
    cudaGraphConditionalHandle h;
    if (cudaGraphConditionalHandleCreate(&h, g, 0, cudaGraphCondAssignDefault) != cudaSuccess) {
      cudaGetLastError();  // a driver without conditional nodes: the kernels gate themselves
      return LRAMM_OK;
    }
    cond_set_kernel<<<1, 1, 0, st>>>(h, flag, run_if_nonzero ? 1 : 0);
    LRAMM_LAUNCH_CHECK();
    LRAMM_CUDA_TRY(cudaStreamGetCaptureInfo(st, &cs, nullptr, &g, &deps, &nd));
    cudaGraphNodeParams p = {};
    p.type = cudaGraphNodeTypeConditional;
    p.conditional.handle = h;
    p.conditional.type = cudaGraphCondTypeIf;
    p.conditional.size = 1;
    LRAMM_CUDA_TRY(cudaGraphAddNode(&node, g, deps, nd, &p));
    body = aux_stream(st);
    LRAMM_CUDA_TRY(cudaStreamBeginCaptureToGraph(body, p.conditional.phGraph_out[0], nullptr, nullptr, 0,
                                                 cudaStreamCaptureModeRelaxed));
    active = true;
    return LRAMM_OK;
  }
  cudaStream_t stream() const { return active ? body : outer; }
  int end() {
    if (!active) return LRAMM_OK;
    active = false;
    cudaGraph_t out = nullptr;
    LRAMM_CUDA_TRY(cudaStreamEndCapture(body, &out));
    LRAMM_CUDA_TRY(cudaStreamUpdateCaptureDependencies(outer, &node, 1, cudaStreamSetCaptureDependencies));
    return LRAMM_OK;
  }
  ~CondIf() {
    if (active) {  // error return inside the section: close the body capture
      cudaGraph_t out = nullptr;
      cudaStreamEndCapture(body, &out);
      cudaStreamUpdateCaptureDependencies(outer, &node, 1, cudaStreamSetCaptureDependencies);
    }
  }
};

// Bump allocator over a caller-provided workspace (256-byte aligned slices).
struct Arena {
  char *base = nullptr;
  size_t cap = 0, off = 0;
  bool dry = false;  // sizing pass: count bytes only
  Arena() = default;
  Arena(void *p, size_t n) : base((char *)p), cap(n), dry(p == nullptr) {}
  template <class T>
  T *take(int64_t count) {
    size_t bytes = round_up((int64_t)(count * sizeof(T)), 256);
    size_t at = off;
    off += bytes;
    if (dry) return nullptr;
    if (off > cap) return nullptr;
    return reinterpret_cast<T *>(base + at);
  }
  bool ok() const { return dry || off <= cap; }
};

// ------------------------------------------------------------------ collectives (sharded pipeline)
// Thin wrapper over the caller's lramm_comm_t table (NCCL signatures and enum values,
// include/lramm_cuda.h).  `comm` selects the communicator of the chain that issues the call.
struct Coll {
  const lramm_comm_t *c = nullptr;
  void *comm = nullptr;
  bool on() const { return c && (c->world > 1 || (c->flags & LRAMM_COMM_FORCE)); }
  int world() const { return c ? c->world : 1; }
  int rank() const { return c ? c->rank : 0; }
  int reduce(void *x, size_t n, int dtype, int op, cudaStream_t st) const {
    if (!on() || n == 0) return LRAMM_OK;
    int rc = c->all_reduce(x, x, n, dtype, op, comm, (lramm_stream_t)st);
    return rc ? fail(LRAMM_ERR_CUDA, "all_reduce failed with code %d", rc) : LRAMM_OK;
  }
  // nccl.h: ncclInt8 0, ncclInt32 2, ncclInt64 4, ncclFloat64 8; ncclSum 0, ncclMax 2
  int sum_f64(double *x, size_t n, cudaStream_t st) const { return reduce(x, n, 8, 0, st); }
  int max_f64(double *x, size_t n, cudaStream_t st) const { return reduce(x, n, 8, 2, st); }
  int sum_i32(int32_t *x, size_t n, cudaStream_t st) const { return reduce(x, n, 2, 0, st); }
  int max_i32(int32_t *x, size_t n, cudaStream_t st) const { return reduce(x, n, 2, 2, st); }
  int gather_i8(const void *send, void *recv, size_t count, cudaStream_t st) const {
    if (!c) return fail(LRAMM_ERR_PARAM, "all_gather without a communicator");
    int rc = c->all_gather(send, recv, count, 0, comm, (lramm_stream_t)st);
    return rc ? fail(LRAMM_ERR_CUDA, "all_gather failed with code %d", rc) : LRAMM_OK;
  }
};
// which absmax vectors of a quantisation span a sharded dimension (allreduce(MAX) before the scales)
struct AmaxSync {
  const Coll *coll = nullptr;
  bool tensor = false, row = false, col = false;  // in the INPUT's coordinates
  bool wants(int gran) const {
    return coll && coll->on() &&
           (gran == LRAMM_GRAN_TENSOR ? tensor : (gran == LRAMM_GRAN_ROW ? row : col));
  }
};

// ------------------------------------------------------------------ device numerics
// Bit-exact conventions: every rounding step is an explicit
// IEEE round-to-nearest intrinsic so nvcc cannot contract it into an FMA.
__device__ __forceinline__ unsigned long long dbits(double x) { return __double_as_longlong(x); }

// non-negative doubles order like their bit patterns -> atomicMax on u64 is an exact max
__device__ __forceinline__ void atomic_max_nonneg(double *addr, double v) {
  atomicMax(reinterpret_cast<unsigned long long *>(addr), (unsigned long long)__double_as_longlong(v));
}

__device__ __forceinline__ double warp_max(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v = fmax(v, __shfl_xor_sync(0xffffffffu, v, o));
  return v;
}
__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v = __dadd_rn(v, __shfl_xor_sync(0xffffffffu, v, o));
  return v;
}

// rint(a*scale) (half-to-even), clamp to +-cap: _core.pyx:63-68
__device__ __forceinline__ int quant_round(double a, double scale, int cap) {
  double t = __dmul_rn(a, scale);
  double r = rint(t);
  if (r > (double)cap) r = (double)cap;
  if (r < -(double)cap) r = -(double)cap;
  return (int)r;
}

// scale = cap / amax (quant.py:69), all-zero sentinel 1.0 (quant.py:67-68)
__device__ __forceinline__ double quant_scale(double amax, int cap) {
  return amax == 0.0 ? 1.0 : __ddiv_rn((double)cap, amax);
}

template <class T>
__device__ __forceinline__ double to_f64(T v) { return (double)v; }

}  // namespace lramm
