// Jacobi phase timing (clock64 trace): nvcc ... scripts/jac_probe.cu
#define LRAMM_TRACE 1
#include "../paper_2405_16917_b200/csrc/factor.cu"
namespace lramm { void set_error(const char*, ...) {} int fail(int c, const char*, ...) { return c; } int num_sms() { return 148; }
int dgemm_device(int, int64_t, int64_t, int64_t, const double*, int64_t, const double*, int64_t, double*, int64_t, void*, size_t, cudaStream_t) { return 0; }
size_t dgemm_ws_bytes(int, int64_t, int64_t, int64_t) { return 0; } }
#include <vector>
#include <cstdlib>
int main(int argc, char** argv) {
  int w = argc > 1 ? atoi(argv[1]) : 272;
  std::vector<double> h((size_t)w * w);
  for (auto& v : h) v = (rand() / (double)RAND_MAX) - 0.5;
  double *W, *W0; int* info; cudaMalloc(&W, w*w*8); cudaMalloc(&W0, w*w*8); cudaMalloc(&info, 64);
  cudaMemcpy(W0, h.data(), w*w*8, cudaMemcpyHostToDevice);
  for (int rep = 0; rep < 2; ++rep) {
    cudaMemcpy(W, W0, w*w*8, cudaMemcpyDeviceToDevice);
    cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
    cudaEventRecord(a);
    int rc = lramm::jacobi_device(W, w, 0, w, w, 1, info, nullptr, 0, 0);
    cudaEventRecord(b); cudaEventSynchronize(b);
    float ms; cudaEventElapsedTime(&ms, a, b);
    int hi; cudaMemcpy(&hi, info, 4, cudaMemcpyDeviceToHost);
    long long t[4096]; cudaMemcpyFromSymbol(t, lramm_trace, sizeof(t));
    printf("w=%d rc=%d %.1f us sweeps=%d err=%s\n", w, rc, ms * 1e3, hi, cudaGetErrorString(cudaGetLastError()));
    if (rep == 1) for (int s = 0; s < hi; ++s) {
      long long total = (s + 1 < hi ? t[100 + (s+1)*4] : 0) - t[100 + s*4];
      printf("sweep %2d: total %8lld  inter-steps %8lld  exchange %8lld\n", s, total, t[101 + s*4] - (s ? t[101 + (s-1)*4] : 0), t[102 + s*4] - (s ? t[102 + (s-1)*4] : 0));
    }
  }
}
