// Phase trace of sytrd_cluster_kernel (compile-time LRAMM_SYTRD_TRACE): cycles per step spent in
// gather / s / HH+row update / barrier / p dots / cluster barrier, on warp 0 of CTA 0.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -DLRAMM_SYTRD_TRACE -I../include \
//        sytrd_probe.cu -o sytrd_probe -L../paper_2405_16917_b200 -llramm_cuda
#define LRAMM_SYTRD_TRACE
#include "../paper_2405_16917_b200/csrc/eig.cu"
#include <cstdio>
#include <vector>
#include <random>
int main(int argc, char **argv) {
  int n = argc > 1 ? atoi(argv[1]) : 272;
  int C = argc > 2 ? atoi(argv[2]) : 16;
  int rm = argc > 3 ? atoi(argv[3]) : 3;  // rows per row warp in registers (0: shared memory)
  int warps = 8;
  std::vector<double> h((size_t)n * n);
  std::mt19937_64 g(1);
  std::normal_distribution<double> nd;
  for (int i = 0; i < n; ++i)
    for (int j = 0; j <= i; ++j) h[(size_t)i * n + j] = h[(size_t)j * n + i] = nd(g);
  double *G, *d, *e, *tau, *V;
  cudaMalloc(&G, 8ull * n * n); cudaMalloc(&V, 8ull * n * n);
  cudaMalloc(&d, 8 * n); cudaMalloc(&e, 8 * n); cudaMalloc(&tau, 8 * n);
  cudaMemcpy(G, h.data(), 8ull * n * n, cudaMemcpyHostToDevice);
  lramm::SytrdArgs a{G, n, (int64_t)n * n, n, d, e, tau, V, (int)(((n + 1) / 2) * 2 + 1)};
  const int nlmax = (n + C - 1) / C;
  const int srows = nlmax - 6 * rm > 0 ? nlmax - 6 * rm : 0;
  size_t smem = (size_t)(4 * n + 3 * a.ldr + 2 * (size_t)nlmax + (size_t)srows * a.ldr) * 8; a.nsm = srows; a.Ag = nullptr; a.ag_rows = 0;
  void (*kern)(lramm::SytrdArgs) = lramm::sytrd_push_pick(n, rm);
  if (!kern) { printf("no kernel for n=%d rm=%d\n", n, rm); return 1; }
  cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  cudaFuncSetAttribute(kern, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(C); cfg.blockDim = dim3(32 * warps); cfg.dynamicSmemBytes = smem;
  cudaLaunchAttribute at[1]; at[0].id = cudaLaunchAttributeClusterDimension;
  at[0].val.clusterDim.x = C; at[0].val.clusterDim.y = 1; at[0].val.clusterDim.z = 1;
  cfg.attrs = at; cfg.numAttrs = 1;
  for (int it = 0; it < 3; ++it) {
    long long z[16] = {0};
    cudaMemcpyToSymbol(sytrd_trace, z, sizeof(z));
    cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
    cudaEventRecord(e0);
    cudaError_t err = cudaLaunchKernelEx(&cfg, kern, a);
    cudaEventRecord(e1); cudaEventSynchronize(e1);
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    long long t[16]; cudaMemcpyFromSymbol(t, sytrd_trace, sizeof(t));
    double st = n - 3;
    printf("n=%d C=%d rm=%d err=%s  %.1f us (%.2f us/step)  cycles/step: wait %.0f  s %.0f  hh/rows %.0f  sync %.0f  dots+push %.0f  -  %.0f  total %.0f\n",
           n, C, rm, cudaGetErrorString(err), ms * 1e3, ms * 1e3 / st, t[0] / st, t[1] / st, t[2] / st, t[3] / st, t[4] / st, t[5] / st, t[6] / st);
    printf("   hh: rr %.0f  sig2 %.0f  shfl %.0f  householder %.0f\n", t[8] / st, t[9] / st, t[10] / st, t[11] / st);
  }
  return 0;
}
