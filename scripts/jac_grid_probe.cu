// Round timing of the grid-wide Jacobi (globaltimer trace of CTA 0).
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 scripts/jac_grid_probe.cu -o scripts/jac_grid_probe
#define LRAMM_TRACE 1
#include "../paper_2405_16917_b200/csrc/factor.cu"
namespace lramm {
void set_error(const char *, ...) {}
int fail(int c, const char *, ...) { return c; }
int num_sms() { return 148; }
int dgemm_device(int, int64_t, int64_t, int64_t, const double *, int64_t, const double *, int64_t, double *, int64_t,
                 void *, size_t, cudaStream_t) { return 0; }
int dgemm_device_ex(int, int64_t, int64_t, int64_t, const double *, int64_t, const double *, int64_t, double *,
                    int64_t, void *, size_t, cudaStream_t, const DgemmOptions &) { return 0; }
size_t dgemm_ws_bytes(int, int64_t, int64_t, int64_t) { return 0; }
}  // namespace lramm
#include <cstdio>
#include <cstdlib>
#include <vector>
int main(int argc, char **argv) {
  int n = argc > 1 ? atoi(argv[1]) : 1056;
  double tau = argc > 2 ? atof(argv[2]) : 256.0;
  // W = upper-triangular-ish with graded columns: R^T of a matrix with exp(-i/tau) spectrum
  std::vector<double> h((size_t)n * n);
  srand(1);
  for (int j = 0; j < n; ++j)
    for (int i = 0; i < n; ++i) h[(size_t)j * n + i] = (i >= j ? ((rand() / (double)RAND_MAX) - 0.5) : 0.0) * exp(-j / tau);
  double *W;
  int *info;
  cudaMalloc(&W, (size_t)n * n * 8);
  cudaMalloc(&info, 4);
  size_t wsb = lramm::jacobi_ws_bytes(n, n, 1);
  void *ws;
  cudaMalloc(&ws, wsb + 256);
  for (int rep = 0; rep < 2; ++rep) {
    cudaMemcpy(W, h.data(), (size_t)n * n * 8, cudaMemcpyHostToDevice);
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    cudaEventRecord(a);
    int rc = lramm::jacobi_device(W, n, 0, n, n, 1, info, ws, wsb, 0);
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    float ms;
    cudaEventElapsedTime(&ms, a, b);
    int sw;
    cudaMemcpy(&sw, info, 4, cudaMemcpyDeviceToHost);
    printf("n=%d rc=%d sweeps=%d %.3f ms err=%s\n", n, rc, sw, ms, cudaGetErrorString(cudaGetLastError()));
  }
  std::vector<unsigned long long> t(148 * 128);
  cudaMemcpyFromSymbol(t.data(), chol_trace, t.size() * 8);
  double ph[4] = {0, 0, 0, 0};
  int cnt = 0;
  for (int g = 0; g < 2000 && (g + 1) * 4 < (int)t.size(); ++g) {
    if (!t[g * 4] || !t[g * 4 + 1] || !t[g * 4 + 2] || !t[g * 4 + 3] || !t[(g + 1) * 4]) continue;
    for (int q = 0; q < 4; ++q) ph[q] += ((q < 3 ? t[g * 4 + q + 1] : t[(g + 1) * 4]) - t[g * 4 + q]) / 1e3;
    ++cnt;
  }
  {
    std::vector<unsigned long long> ct(148 * 16 * 4);
    cudaMemcpyFromSymbol(ct.data(), jac_cta_trace, ct.size() * 8);
    int C = 0;
    for (int b = 0; b < 148; ++b) if (ct[(b * 16) * 4]) C = b + 1;
    for (int rr = 0; rr < 6; ++rr) {
      unsigned long long s0 = ~0ull, s1 = 0, d0 = ~0ull, d1 = 0, e0 = ~0ull, e1 = 0;
      for (int b = 0; b < C; ++b) {
        auto *x = &ct[(b * 16 + rr) * 4];
        s0 = std::min(s0, x[0]); s1 = std::max(s1, x[0]);
        d0 = std::min(d0, x[1]); d1 = std::max(d1, x[1]);
        e0 = std::min(e0, x[2]); e1 = std::max(e1, x[2]);
      }
      printf("round %d over %d CTAs: start spread %.2f us, steps-done spread %.2f, sends-done spread %.2f; "
             "first start -> last steps done %.2f us\n", 100 + rr, C, (s1 - s0) / 1e3, (d1 - d0) / 1e3,
             (e1 - e0) / 1e3, (d1 - s0) / 1e3);
    }
  }
  printf("rounds %d: phase us (grid kernel: steps/send/recv/-; gram kernel: gram/steps/apply/exchange): "
         "%.2f %.2f %.2f %.2f\n", cnt, ph[0] / cnt, ph[1] / cnt, ph[2] / cnt, ph[3] / cnt);
}
