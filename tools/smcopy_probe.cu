// SM-driven copies over the host link: a few CTAs read / write pinned
// (mapped) host memory directly. Times device->host (16 n bytes), host->device
// (8 n bytes), both at once, and both in 8 / 32 ranges per direction, against
// the DMA engines (cudaMemcpyAsync).   nvcc -O3 -arch=sm_100a smcopy_probe.cu
#include <cstdio>
#include <cuda_runtime.h>
#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("%s: %s\n", #x, cudaGetErrorString(e)); return 1; } } while (0)

__global__ void copy_kernel(const double2* __restrict__ src, double2* __restrict__ dst, size_t n2) {
  const size_t st = (size_t)gridDim.x * blockDim.x;
  size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
  for (; i + 3 * st < n2; i += 4 * st) {
    double2 a = src[i], b = src[i + st], c = src[i + 2 * st], d = src[i + 3 * st];
    dst[i] = a; dst[i + st] = b; dst[i + 2 * st] = c; dst[i + 3 * st] = d;
  }
  for (; i < n2; i += st) dst[i] = src[i];
}

int main() {
  const size_t n = 2356227 / 2 * 2;
  double *hx, *ho, *dx, *dout;
  CK(cudaHostAlloc(&hx, 8 * n, cudaHostAllocDefault));
  CK(cudaHostAlloc(&ho, 16 * n, cudaHostAllocDefault));
  CK(cudaMalloc(&dx, 8 * n));
  CK(cudaMalloc(&dout, 16 * n));
  for (size_t i = 0; i < n; ++i) hx[i] = (double)i;
  cudaStream_t s1, s2;
  CK(cudaStreamCreateWithFlags(&s1, cudaStreamNonBlocking));
  CK(cudaStreamCreateWithFlags(&s2, cudaStreamNonBlocking));
  cudaEvent_t e0, e1;
  CK(cudaEventCreate(&e0));
  CK(cudaEventCreate(&e1));
  for (int ctas : {8, 16, 32, 64}) {
    for (int mode = 0; mode < 5; ++mode) {
      const int K = 20;
      float best = 1e9f;
      for (int rep = 0; rep < 3; ++rep) {
        CK(cudaDeviceSynchronize());
        CK(cudaEventRecord(e0, 0));
        CK(cudaStreamWaitEvent(s1, e0, 0));
        CK(cudaStreamWaitEvent(s2, e0, 0));
        for (int k = 0; k < K; ++k) {
          const int parts = mode == 3 ? 8 : mode == 4 ? 32 : 1;
          for (int q = 0; q < parts; ++q) {
            const size_t a = n / 2 * q / parts, b = n / 2 * (q + 1) / parts;  // double2 units
            if (mode != 1)
              copy_kernel<<<ctas, 512, 0, s1>>>((const double2*)dout + 2 * a, (double2*)ho + 2 * a, 2 * (b - a));
            if (mode != 0)
              copy_kernel<<<ctas, 512, 0, s2>>>((const double2*)hx + a, (double2*)dx + a, b - a);
          }
        }
        CK(cudaEventRecord(e1, s1));
        CK(cudaStreamWaitEvent(0, e1, 0));
        CK(cudaEventRecord(e1, s2));
        CK(cudaStreamWaitEvent(0, e1, 0));
        CK(cudaEventRecord(e1, 0));
        CK(cudaEventSynchronize(e1));
        float ms;
        CK(cudaEventElapsedTime(&ms, e0, e1));
        best = ms / K < best ? ms / K : best;
      }
      const char* nm[] = {"d2h", "h2d", "both", "both/8", "both/32"};
      printf("sm ctas=%d %-8s %.3f ms\n", ctas, nm[mode], best);
    }
  }
  // DMA reference, same shapes
  for (int mode = 0; mode < 5; ++mode) {
    const int K = 20;
    CK(cudaDeviceSynchronize());
    CK(cudaEventRecord(e0, 0));
    CK(cudaStreamWaitEvent(s1, e0, 0));
    CK(cudaStreamWaitEvent(s2, e0, 0));
    for (int k = 0; k < K; ++k) {
      const int parts = mode == 3 ? 8 : mode == 4 ? 32 : 1;
      for (int q = 0; q < parts; ++q) {
        const size_t a = n * q / parts, b = n * (q + 1) / parts;
        if (mode != 1) CK(cudaMemcpyAsync(ho + 2 * a, dout + 2 * a, 16 * (b - a), cudaMemcpyDeviceToHost, s1));
        if (mode != 0) CK(cudaMemcpyAsync(dx + a, hx + a, 8 * (b - a), cudaMemcpyHostToDevice, s2));
      }
    }
    CK(cudaEventRecord(e1, s1));
    CK(cudaStreamWaitEvent(0, e1, 0));
    CK(cudaEventRecord(e1, s2));
    CK(cudaStreamWaitEvent(0, e1, 0));
    CK(cudaEventRecord(e1, 0));
    CK(cudaEventSynchronize(e1));
    float ms;
    CK(cudaEventElapsedTime(&ms, e0, e1));
    const char* nm[] = {"d2h", "h2d", "both", "both/8", "both/32"};
    printf("dma %-8s %.3f ms\n", nm[mode], ms / K);
  }
  return 0;
}
