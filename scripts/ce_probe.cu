// Does a small cudaMemsetAsync / D2D cudaMemcpyAsync on one stream queue behind a large D2H copy
// that is running on another stream?  (time from the start of the D2H to the completion of the
// small operation; a kernel for comparison)
#include <cstdio>
#include <cuda_runtime.h>
__global__ void tiny(int *p) { p[0] = 1; }
int main() {
  const size_t n = 512ull << 20;
  char *h, *d; int *w, *w2;
  cudaMallocHost(&h, n); cudaMalloc(&d, n); cudaMalloc(&w, 1 << 20); cudaMalloc(&w2, 1 << 20);
  cudaStream_t s1, s2;
  cudaStreamCreateWithFlags(&s1, cudaStreamNonBlocking); cudaStreamCreateWithFlags(&s2, cudaStreamNonBlocking);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0); cudaEventCreate(&e1);
  const char *names[] = {"kernel", "memset 16 B", "memset 2.4 MB", "memcpy D2D 4 KB", "memcpy2D D2D 4 MB"};
  for (int rep = 0; rep < 2; ++rep)
    for (int kind = 0; kind < 5; ++kind) {
      cudaDeviceSynchronize();
      cudaEventRecord(e0, s2);
      cudaMemcpyAsync(h, d, n, cudaMemcpyDeviceToHost, s1);
      if (kind == 0) tiny<<<1, 32, 0, s2>>>(w);
      if (kind == 1) cudaMemsetAsync(w, 0, 16, s2);
      if (kind == 2) cudaMemsetAsync(w, 0, 544 * 544 * 8, s2);
      if (kind == 3) cudaMemcpyAsync(w2, w, 4096, cudaMemcpyDeviceToDevice, s2);
      if (kind == 4) cudaMemcpy2DAsync(w2, 512 * 8, w, 544 * 8, 512 * 8, 1024, cudaMemcpyDeviceToDevice, s2);
      cudaEventRecord(e1, s2);
      cudaDeviceSynchronize();
      float ms = 0;
      cudaEventElapsedTime(&ms, e0, e1);
      if (rep) printf("%-20s completes %.3f ms after the D2H started (D2H takes ~10 ms)\n", names[kind], ms);
    }
  return 0;
}
