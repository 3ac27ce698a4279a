// Phase timing of chol_kernel (clock64 trace) -- build: nvcc ... -DLRAMM_TRACE scripts/chol_probe.cu
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
  // SPD: G = X^T X + w I
  std::vector<double> x((size_t)w * w);
  for (auto& v : x) v = (rand() / (double)RAND_MAX) - 0.5;
  for (int i = 0; i < w; ++i) for (int j = 0; j < w; ++j) { double s = 0; for (int k = 0; k < w; ++k) s += x[k*w+i]*x[k*w+j]; h[i*w+j] = s + (i==j ? w : 0); }
  double *G, *L; int* info; cudaMalloc(&G, w*w*8); cudaMalloc(&L, w*w*8); cudaMalloc(&info, 4);
  cudaMemcpy(G, h.data(), w*w*8, cudaMemcpyHostToDevice);
  lramm::allow_max_dyn_smem(lramm::chol_kernel);
  for (int rep = 0; rep < 3; ++rep) {
    cudaMemset(L, 0, w*w*8);
    cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
    cudaEventRecord(a);
    lramm::chol_kernel<<<1, lramm::kCholThreads, lramm::kCholSmem>>>(G, w, w, L, info, nullptr);
    cudaEventRecord(b); cudaEventSynchronize(b);
    float ms; cudaEventElapsedTime(&ms, a, b);
    long long t[4096]; cudaMemcpyFromSymbol(t, lramm_trace, sizeof(t));
    printf("w=%d  %.1f us  err=%s\n", w, ms * 1e3, cudaGetErrorString(cudaGetLastError()));
    if (rep == 2) {
      long long t0 = t[0];
      for (int jb = 0; jb < (w + 31) / 32; ++jb) {
        long long s1 = t[1 + jb*4], s2 = t[2 + jb*4], s3 = t[3 + jb*4], nxt = (jb + 1 < (w+31)/32) ? t[1 + (jb+1)*4] : 0;
        printf("panel %2d: update %8lld  potrf %8lld  below %8lld cycles\n", jb, s2 - s1, s3 - s2, nxt ? nxt - s3 : -1);
      }
    }
  }
}
