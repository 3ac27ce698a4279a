// Dependent-chain latency of fp64 primitives on the B200 (cycles per op).
#include <cstdio>
#include <cuda_runtime.h>
__global__ void k(double* out, long long* cyc, double seed, int n) {
  __shared__ double sm[64];
  if (threadIdx.x < 64) sm[threadIdx.x] = seed + threadIdx.x;
  __syncwarp();
  double x = seed + threadIdx.x * 1e-9;
  long long t0, t1;
  // DFMA chain
  t0 = clock64(); for (int i = 0; i < n; ++i) x = fma(x, 0.999999, 1e-9); t1 = clock64(); cyc[0] = (t1 - t0) / n;
  // sqrt chain
  t0 = clock64(); for (int i = 0; i < n; ++i) x = sqrt(x + 1.0); t1 = clock64(); cyc[1] = (t1 - t0) / n;
  // div chain
  t0 = clock64(); for (int i = 0; i < n; ++i) x = 1.0 / (x + 1.5); t1 = clock64(); cyc[2] = (t1 - t0) / n;
  // rsqrt chain
  t0 = clock64(); for (int i = 0; i < n; ++i) x = rsqrt(x + 2.0); t1 = clock64(); cyc[3] = (t1 - t0) / n;
  // shfl double chain
  t0 = clock64(); for (int i = 0; i < n; ++i) x = __shfl_sync(0xffffffffu, x, (threadIdx.x + 1) & 31) + 1e-9; t1 = clock64(); cyc[4] = (t1 - t0) / n;
  // LDS chain (pointer chase on value)
  int idx = threadIdx.x & 31;
  t0 = clock64(); for (int i = 0; i < n; ++i) { double v = sm[idx]; idx = ((int)v + i) & 31; x += v; } t1 = clock64(); cyc[5] = (t1 - t0) / n;
  // DADD chain
  t0 = clock64(); for (int i = 0; i < n; ++i) x = x + 1e-9; t1 = clock64(); cyc[6] = (t1 - t0) / n;
  // __syncwarp cost
  t0 = clock64(); for (int i = 0; i < n; ++i) { __syncwarp(); x += 1e-9; } t1 = clock64(); cyc[7] = (t1 - t0) / n;
  // float rsqrt chain
  float xf = (float)x;
  t0 = clock64(); for (int i = 0; i < n; ++i) xf = rsqrtf(xf + 2.0f); t1 = clock64(); cyc[8] = (t1 - t0) / n;
  out[threadIdx.x] = x + xf;
}
__global__ void ksync(long long* cyc, int n) {
  long long t0 = clock64(); for (int i = 0; i < n; ++i) __syncthreads(); long long t1 = clock64();
  if (threadIdx.x == 0) cyc[9] = (t1 - t0) / n;
}
int main() {
  double* out; long long* cyc; cudaMalloc(&out, 1 << 16); cudaMallocManaged(&cyc, 128 * 8);
  for (int r = 0; r < 2; ++r) { k<<<1, 32>>>(out, cyc, 1.5, 1000); ksync<<<1, 512>>>(cyc, 1000); cudaDeviceSynchronize(); }
  const char* names[] = {"dfma", "dsqrt", "ddiv(1/x)", "drsqrt", "shfl.f64", "lds+dadd chase", "dadd", "syncwarp+dadd", "rsqrtf", "syncthreads(512)"};
  for (int i = 0; i < 10; ++i) printf("%-18s %lld cycles\n", names[i], cyc[i]);
}
