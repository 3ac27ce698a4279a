// Phase timing of the dataflow tile Cholesky (globaltimer trace per CTA).
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -DLRAMM_TRACE -Ipaper_2405_16917_b200/csrc \
//        scripts/chol_probe.cu -o scripts/chol_probe
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
int jacobi_wb_device(double *, int64_t, int64_t, int, int, int, int *, cudaStream_t) { return 1; }
}  // namespace lramm
#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <vector>
int main(int argc, char **argv) {
  int w = argc > 1 ? atoi(argv[1]) : 272;
  int T = (w + 31) / 32;
  std::vector<double> h((size_t)w * w), x((size_t)w * w);
  for (auto &v : x) v = (rand() / (double)RAND_MAX) - 0.5;
  for (int i = 0; i < w; ++i)
    for (int j = 0; j < w; ++j) {
      double s = 0;
      for (int k = 0; k < w; ++k) s += x[k * w + i] * x[k * w + j];
      h[i * w + j] = s + (i == j ? w : 0);
    }
  double *G, *L, *dinv;
  int *info, *flags;
  cudaMalloc(&G, w * w * 8);
  cudaMalloc(&L, w * w * 8);
  cudaMalloc(&dinv, T * 1024 * 8);
  cudaMalloc(&info, 4);
  cudaMalloc(&flags, (T + 1) * 4);
  cudaMemcpy(G, h.data(), w * w * 8, cudaMemcpyHostToDevice);
  for (int rep = 0; rep < 4; ++rep) {
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    cudaEventRecord(a);
    int rc = lramm::chol_device(G, w, w, L, dinv, flags, info, nullptr, 0);
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    float ms;
    cudaEventElapsedTime(&ms, a, b);
    printf("w=%d rc=%d %.1f us err=%s\n", w, rc, ms * 1e3, cudaGetErrorString(cudaGetLastError()));
    if (rep == 0) {  // residual max |L L^T - G| / max |G| and max |Dinv_J L_JJ - I|
      std::vector<double> hl((size_t)w * w), hd((size_t)T * 1024);
      cudaMemcpy(hl.data(), L, (size_t)w * w * 8, cudaMemcpyDeviceToHost);
      cudaMemcpy(hd.data(), dinv, (size_t)T * 1024 * 8, cudaMemcpyDeviceToHost);
      double gm = 0, er = 0, ei = 0;
      for (int i = 0; i < w; ++i)
        for (int j = 0; j <= i; ++j) {
          double s = 0;
          for (int k = 0; k <= j; ++k) s += hl[(size_t)i * w + k] * hl[(size_t)j * w + k];
          er = std::max(er, std::fabs(s - h[(size_t)i * w + j]));
          gm = std::max(gm, std::fabs(h[(size_t)i * w + j]));
        }
      for (int J = 0; J < T; ++J) {
        const int nb = std::min(32, w - 32 * J);
        for (int r = 0; r < nb; ++r)
          for (int c = 0; c < nb; ++c) {
            double s = 0;
            for (int k = 0; k < 32 && 32 * J + k < w; ++k)
              s += hd[(size_t)J * 1024 + r * 32 + k] * hl[(size_t)(32 * J + k) * w + 32 * J + c];
            ei = std::max(ei, std::fabs(s - (r == c ? 1.0 : 0.0)));
          }
      }
      int hinfo = -7;
      cudaMemcpy(&hinfo, info, 4, cudaMemcpyDeviceToHost);
      printf("w=%d info=%d residual %.3e (rel to max|G| %.3e) dinv*L-I %.3e\n", w, hinfo, er / gm, gm, ei);
    }
    if (rep == 3) {
      std::vector<unsigned long long> t(148 * 128);
      cudaMemcpyFromSymbol(t.data(), chol_trace, t.size() * 8);
      unsigned long long t0 = ~0ull;
      for (int i = 0; i < T; ++i) t0 = std::min(t0, t[i * 128 + 0 < 1 ? 0 : i * 128 + (i > 0 ? 0 : 120)]);
      for (int i = 0; i < T; ++i) t0 = std::min(t0, i > 0 ? t[i * 128] : t[120]);
      for (int i = 0; i < T; ++i) {
        auto *r = &t[i * 128];
        printf("row %2d:", i);
        for (int j = 0; j < i; ++j)
          printf(" [j%d start %5.1f poll1 %4.1f panel %4.1f poll2 %4.1f fin %4.1f]", j, (r[4 * j] - t0) / 1e3,
                 j ? (r[4 * j + 1] - r[4 * j]) / 1e3 : 0.0, (r[4 * j + 2] - (j ? r[4 * j + 1] : r[4 * j])) / 1e3,
                 (r[4 * j + 3] - r[4 * j + 2]) / 1e3, ((j + 1 < i ? r[4 * j + 4] : r[120]) - r[4 * j + 3]) / 1e3);
        printf("\n        diag start %6.1f potrf+inverse %5.1f publish %5.1f end %6.1f us\n", (r[120] - t0) / 1e3,
               (r[121] - r[120]) / 1e3, (r[123] - r[121]) / 1e3, (r[123] - t0) / 1e3);
      }
    }
  }
}
