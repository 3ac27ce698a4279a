// Per-phase cycle counts inside one rotation of the cluster Jacobi (thread 0 of CTA 0):
// y loads + dot, shuffle reduction, angle, apply; plus whole steps (LRAMM_TRACE t_steps).
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 scripts/jac_step_probe.cu -o scripts/jac_step_probe
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
  int n = argc > 1 ? atoi(argv[1]) : 272;
  std::vector<double> h((size_t)n * n);
  srand(1);
  for (int j = 0; j < n; ++j)
    for (int i = 0; i < n; ++i) h[(size_t)j * n + i] = (i >= j ? ((rand() / (double)RAND_MAX) - 0.5) : 0.0) * exp(-j / 128.0);
  double *W;
  int *info;
  cudaMalloc(&W, (size_t)n * n * 8);
  cudaMalloc(&info, 4);
  long long z[8] = {0};
  cudaMemcpy(W, h.data(), (size_t)n * n * 8, cudaMemcpyHostToDevice);
  cudaMemcpyToSymbol(step_trace, z, sizeof(z));
  int rc = lramm::jacobi_device(W, n, 0, n, n, 1, info, nullptr, 0, 0);
  cudaDeviceSynchronize();
  long long t[8], lt[4096];
  cudaMemcpyFromSymbol(t, step_trace, sizeof(t));
  cudaMemcpyFromSymbol(lt, lramm_trace, sizeof(lt));
  int sw;
  cudaMemcpy(&sw, info, 4, cudaMemcpyDeviceToHost);
  double cnt = (double)t[5];
  printf("n=%d rc=%d sweeps=%d rotations traced %lld: loads+dot %.0f, shuffle %.0f, angle %.0f, apply %.0f cycles\n", n, rc,
         sw, t[5], t[1] / cnt, t[2] / cnt, t[3] / cnt, t[4] / cnt);
  long long st = 0, xc = 0;
  for (int s = 0; s < sw && s < 60; ++s) { st += lt[100 + s * 4 + 1]; xc += lt[100 + s * 4 + 2]; }
  printf("per sweep: steps %.0f cycles, exchange %.0f cycles\n", st / (double)sw, xc / (double)sw);
}
