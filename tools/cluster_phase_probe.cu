// Microbenchmark: cost of one barrier-separated phase inside a 16-CTA
// cluster kernel (the scalar V-cycle tail's building block). Variants:
//   0 barrier only (release/acquire)      1 barrier only (relaxed)
//   2 + one L2 load and store per thread  3 + DSMEM partial-sum reduction
//   4 = 2 + 3 + thread-0 fp64 div/sqrt chain (a Krylov finisher)
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/cpp tools/cluster_phase_probe.cu
#include <cooperative_groups.h>
#include <cstdio>
namespace cg = cooperative_groups;

__device__ __forceinline__ void bar_rel() {
  asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}
__device__ __forceinline__ void bar_rlx() {
  asm volatile("barrier.cluster.arrive.relaxed.aligned;\n\tbarrier.cluster.wait.aligned;" ::: "memory");
}
__device__ __forceinline__ double wsum(double v) {
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

template <int V, int T>
__global__ void __launch_bounds__(T, 1) probe(int phases, double* buf, int n, double* out) {
  __shared__ double part[2], wp[32], tot, sc;
  cg::cluster_group cl = cg::this_cluster();
  const int q = cl.block_rank(), cs = cl.num_blocks();
  const int chunk = (n + cs - 1) / cs;
  const int i = q * chunk + threadIdx.x;
  double acc = 0.0;
  if (threadIdx.x == 0) sc = 1.0;
  __syncthreads();
  for (int p = 0; p < phases; ++p) {
    if (V >= 2 && V != 3 && threadIdx.x < chunk && i < n) {
      const double x = __ldcg(buf + ((i + 977 * p) % n));
      buf[i] = x * sc + 1.0;
      acc += x;
    }
    if (V >= 3) {
      double t = wsum(acc);
      if ((threadIdx.x & 31) == 0) wp[threadIdx.x >> 5] = t;
      __syncthreads();
      if (threadIdx.x < 32) {
        t = wsum(threadIdx.x < T / 32 ? wp[threadIdx.x] : 0.0);
        if (threadIdx.x == 0) part[p & 1] = t;
      }
    }
    if (V == 1) bar_rlx(); else bar_rel();
    if (V >= 3) {
      if (threadIdx.x < 32) {
        double t = threadIdx.x < cs ? *cl.map_shared_rank(&part[p & 1], threadIdx.x) : 0.0;
        t = wsum(t);
        if (threadIdx.x == 0) tot = t;
      }
      __syncthreads();
      if (V == 4 && threadIdx.x == 0) {
        double a = sqrt(fabs(tot) + 1.0);
        a = hypot(a, 2.0);
        sc = 1.0 / a + tot / (a + 3.0);
      }
      __syncthreads();
      acc = 0.0;
    }
  }
  if (threadIdx.x == 0 && q == 0) out[0] = acc + sc;
}

template <int V, int T>
float run(int phases, double* buf, int n, double* out) {
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3(16);
  cfg.blockDim = dim3(T);
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeClusterDimension;
  at[0].val.clusterDim.x = 16;
  at[0].val.clusterDim.y = 1;
  at[0].val.clusterDim.z = 1;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  cudaFuncSetAttribute(probe<V, T>, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  cudaLaunchKernelEx(&cfg, probe<V, T>, phases, buf, n, out);
  cudaEventRecord(e0);
  for (int k = 0; k < 10; ++k) cudaLaunchKernelEx(&cfg, probe<V, T>, phases, buf, n, out);
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  float ms = 0;
  cudaEventElapsedTime(&ms, e0, e1);
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) printf("error %s\n", cudaGetErrorString(e));
  return ms / 10 * 1e3f;
}

template <int V, int T>
void report(const char* name, double* buf, int n, double* out) {
  const float t0 = run<V, T>(1, buf, n, out), t1 = run<V, T>(201, buf, n, out);
  printf("%-34s threads %4d  n %6d: launch %.2f us, per phase %.3f us\n", name, T, n, t0,
         (t1 - t0) / 200);
}

int main() {
  const int n = 16384;
  double *buf, *out;
  cudaMalloc(&buf, sizeof(double) * n);
  cudaMalloc(&out, sizeof(double) * 8);
  cudaMemset(buf, 0, sizeof(double) * n);
  report<0, 1024>("barrier release/acquire", buf, n, out);
  report<1, 1024>("barrier relaxed", buf, n, out);
  report<2, 1024>("+ L2 load/store", buf, n, out);
  report<3, 1024>("+ DSMEM reduction", buf, n, out);
  report<4, 1024>("load/store + reduction + finisher", buf, n, out);
  report<0, 256>("barrier release/acquire", buf, n, out);
  report<2, 256>("+ L2 load/store", buf, n, out);
  report<4, 256>("load/store + reduction + finisher", buf, n, out);
  return 0;
}
