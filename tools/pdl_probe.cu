// Launch-gap probe: a chain of N dependent small kernels (each reads the
// previous one's output, 197k doubles -- one scalar-hierarchy level of the
// SV mass projection) captured in a CUDA graph, launched plainly vs with
// programmatic dependent launch (griddepcontrol.wait in the kernel,
// cudaLaunchAttributeProgrammaticStreamSerialization on the launch).
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/pdl_probe tools/pdl_probe.cu
#include <cstdio>
#include <cuda_runtime.h>

__global__ void step(int n, const double* __restrict__ a, double* __restrict__ b, int wait) {
  if (wait) asm volatile("griddepcontrol.wait;" ::: "memory");
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x)
    b[i] = a[i] * 0.5 + 1.0;
}

static float run(int n, int N, bool pdl, int grid, double* x, double* y, cudaStream_t s) {
  cudaGraph_t g;
  cudaStreamBeginCapture(s, cudaStreamCaptureModeThreadLocal);
  for (int k = 0; k < N; ++k) {
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = grid;
    cfg.blockDim = 256;
    cfg.stream = s;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    at[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = at;
    cfg.numAttrs = pdl ? 1 : 0;
    cudaLaunchKernelEx(&cfg, step, n, (k & 1) ? y : x, (k & 1) ? x : y, pdl ? 1 : 0);
  }
  cudaStreamEndCapture(s, &g);
  cudaGraphExec_t e;
  cudaGraphInstantiate(&e, g, 0);
  cudaGraphLaunch(e, s);
  cudaStreamSynchronize(s);
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  cudaEventRecord(a, s);
  for (int r = 0; r < 5; ++r) cudaGraphLaunch(e, s);
  cudaEventRecord(b, s);
  cudaEventSynchronize(b);
  float ms = 0;
  cudaEventElapsedTime(&ms, a, b);
  cudaGraphExecDestroy(e);
  cudaGraphDestroy(g);
  return ms / 5 / N * 1000.0f;  // us per kernel
}

int main() {
  cudaStream_t s;
  cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking);
  for (int n : {1000, 197121, 2356227}) {
    double *x, *y;
    cudaMalloc(&x, 8 * (size_t)n);
    cudaMalloc(&y, 8 * (size_t)n);
    cudaMemset(x, 0, 8 * (size_t)n);
    int grid = (n + 255) / 256;
    if (grid > 148 * 8) grid = 148 * 8;
    const float plain = run(n, 1000, false, grid, x, y, s);
    const float pdl = run(n, 1000, true, grid, x, y, s);
    printf("{\"n\": %d, \"grid\": %d, \"plain_us_per_kernel\": %.3f, \"pdl_us_per_kernel\": %.3f}\n",
           n, grid, plain, pdl);
    cudaFree(x);
    cudaFree(y);
  }
  printf("err=%s\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}
