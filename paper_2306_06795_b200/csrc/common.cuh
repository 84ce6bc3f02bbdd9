// Internal infrastructure of libsag: error mapping, device buffers, the
// context (stream + deterministic-reduction workspace) and small device
// helpers shared by the kernels. sm_100a only.
#pragma once

#include <cuda_runtime.h>

#include <cstdint>
#include <cstdio>
#include <stdexcept>
#include <string>
#include <vector>

#include "../../include/sag.h"

namespace sag {

struct Error : std::runtime_error {
  int code;
  Error(int c, const std::string& m) : std::runtime_error(m), code(c) {}
};

[[noreturn]] inline void throw_cuda(cudaError_t e, const char* what, const char* file, int line) {
  throw Error(SAG_CUDA_ERROR, std::string(what) + ": " + cudaGetErrorString(e) + " (" + file +
                                  ":" + std::to_string(line) + ")");
}

#define SAG_CUDA(x)                                                  \
  do {                                                               \
    cudaError_t e_ = (x);                                            \
    if (e_ != cudaSuccess) ::sag::throw_cuda(e_, #x, __FILE__, __LINE__); \
  } while (0)

#define SAG_REQUIRE(cond, code, msg)                  \
  do {                                                \
    if (!(cond)) throw ::sag::Error((code), (msg));   \
  } while (0)

// Checks the launch and counts it (sag_launch_count).
#define SAG_LAUNCHED(ctx)                                   \
  do {                                                      \
    cudaError_t e_ = cudaGetLastError();                    \
    if (e_ != cudaSuccess) ::sag::throw_cuda(e_, "kernel launch", __FILE__, __LINE__); \
    (ctx).launches++;                                       \
  } while (0)

template <class T>
struct DevBuf {
  T* p = nullptr;
  size_t n = 0;
  DevBuf() = default;
  explicit DevBuf(size_t count) { alloc(count); }
  DevBuf(const DevBuf&) = delete;
  DevBuf& operator=(const DevBuf&) = delete;
  DevBuf(DevBuf&& o) noexcept : p(o.p), n(o.n) {
    o.p = nullptr;
    o.n = 0;
  }
  DevBuf& operator=(DevBuf&& o) noexcept {
    if (this != &o) {
      reset();
      p = o.p;
      n = o.n;
      o.p = nullptr;
      o.n = 0;
    }
    return *this;
  }
  ~DevBuf() { reset(); }
  void alloc(size_t count) {
    reset();
    if (count == 0) count = 1;
    SAG_CUDA(cudaMalloc(&p, count * sizeof(T)));
    n = count;
  }
  void reset() {
    if (p) cudaFree(p);
    p = nullptr;
    n = 0;
  }
  size_t bytes() const { return n * sizeof(T); }
};

// Fixed-grid deterministic reductions: every reduction kernel writes one
// partial per block, the last block to finish (ticket counter) sums the
// partials in index order. The grid depends only on n, so results are
// bitwise reproducible run to run.
constexpr int kRedBlock = 256;
constexpr int kMaxRedGrid = 148 * 8;

struct Ctx {
  int device = 0;
  int num_sms = 148;
  cudaStream_t stream = nullptr;
  bool own_stream = true;  // false: the stream belongs to the caller (sag_create_on_stream)
  long long launches = 0;
  DevBuf<double> partials;   // kMaxRedGrid * 2 (two independent sums per kernel)
  DevBuf<unsigned> ticket;   // reduction tickets
  DevBuf<double> scal;       // general device scalars (sag_dot/norm outputs)
  // second stream for device->host copies that overlap compute on `stream`
  // (created on first use, owned by the context)
  cudaStream_t copy_stream = nullptr;
  cudaEvent_t copy_ev = nullptr;
  // streams that capture the bodies of conditional graph nodes (by depth)
  cudaStream_t body_streams[4] = {nullptr, nullptr, nullptr, nullptr};
  int body_depth = 0;
  cudaStream_t copy() {
    if (!copy_stream) {
      SAG_CUDA(cudaStreamCreateWithFlags(&copy_stream, cudaStreamNonBlocking));
      SAG_CUDA(cudaEventCreateWithFlags(&copy_ev, cudaEventDisableTiming));
    }
    return copy_stream;
  }
  // staging for host vectors passed to the C-ABI
  std::vector<DevBuf<double>> stage;
  double* stage_buf(int slot, size_t n) {
    if ((int)stage.size() <= slot) stage.resize(slot + 1);
    if (stage[slot].n < n) stage[slot].alloc(n);
    return stage[slot].p;
  }
};

inline int red_grid(long long n) {
  long long g = (n + kRedBlock * 4 - 1) / (kRedBlock * 4);
  if (g < 1) g = 1;
  if (g > kMaxRedGrid) g = kMaxRedGrid;
  return (int)g;
}

inline bool is_device_ptr(const void* p) {
  if (!p) return false;
  cudaPointerAttributes a;
  if (cudaPointerGetAttributes(&a, p) != cudaSuccess) {
    cudaGetLastError();
    return false;
  }
  return a.type == cudaMemoryTypeDevice || a.type == cudaMemoryTypeManaged;
}

// Host-or-device input vector: device pointers are used in place, host
// vectors are copied into a context staging slot.
struct InVec {
  const double* d = nullptr;
  InVec(Ctx& c, const double* p, size_t n, int slot) {
    if (is_device_ptr(p) || n == 0) {
      d = p;
    } else {
      SAG_REQUIRE(p != nullptr, SAG_INVALID_ARGUMENT, "null vector");
      double* s = c.stage_buf(slot, n);
      SAG_CUDA(cudaMemcpyAsync(s, p, n * sizeof(double), cudaMemcpyHostToDevice, c.stream));
      d = s;
    }
  }
};

// Host-or-device output (or in/out) vector; call finish() to copy back.
struct OutVec {
  double* d = nullptr;
  double* host = nullptr;
  size_t n = 0;
  Ctx* c = nullptr;
  OutVec(Ctx& cx, double* p, size_t count, int slot, bool copy_in) : n(count), c(&cx) {
    SAG_REQUIRE(p != nullptr || count == 0, SAG_INVALID_ARGUMENT, "null vector");
    if (is_device_ptr(p) || count == 0) {
      d = p;
    } else {
      host = p;
      d = cx.stage_buf(slot, count);
      if (copy_in)
        SAG_CUDA(cudaMemcpyAsync(d, p, n * sizeof(double), cudaMemcpyHostToDevice, cx.stream));
    }
  }
  void finish() {
    if (host) {
      SAG_CUDA(cudaMemcpyAsync(host, d, n * sizeof(double), cudaMemcpyDeviceToHost, c->stream));
      SAG_CUDA(cudaStreamSynchronize(c->stream));
    }
  }
};

// ---------------------------------------------------------------- device --

__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

// Block reduction of one value (blockDim.x == kRedBlock); result valid in
// thread 0. Fixed order.
__device__ __forceinline__ double block_sum(double v, double* sh) {
  v = warp_sum(v);
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  if (lane == 0) sh[w] = v;
  __syncthreads();
  double s = 0.0;
  if (w == 0) {
    s = lane < (kRedBlock / 32) ? sh[lane] : 0.0;
    s = warp_sum(s);
  }
  __syncthreads();
  return s;
}

// Last-block ticket: after each block wrote its partial, returns true in the
// block that finishes last (all partials visible to it).
__device__ __forceinline__ bool last_block(unsigned* ticket) {
  __shared__ bool is_last;
  __threadfence();
  __syncthreads();
  if (threadIdx.x == 0) {
    unsigned t = atomicAdd(ticket, 1u);
    is_last = (t == gridDim.x - 1);
  }
  __syncthreads();
  if (is_last) {
    __threadfence();
  }
  return is_last;
}

// Sums partials[0..n) in a fixed order by the whole block; valid in thread 0.
__device__ __forceinline__ double sum_partials(const double* partials, int n, double* sh) {
  double s = 0.0;
  for (int i = threadIdx.x; i < n; i += blockDim.x) s += __ldcg(partials + i);
  return block_sum(s, sh);
}

// C-ABI boundary: exceptions -> status codes + thread-local message.
void set_last_error(const std::string& s);
template <class F>
int guard(F&& f) {
  try {
    f();
    return SAG_OK;
  } catch (const Error& e) {
    set_last_error(e.what());
    return e.code;
  } catch (const std::bad_alloc& e) {
    set_last_error(std::string("allocation failure: ") + e.what());
    return SAG_ERROR;
  } catch (const std::exception& e) {
    set_last_error(e.what());
    return SAG_ERROR;
  }
}

}  // namespace sag

#define SAG_NOTNULL(p)                                                                    \
  do {                                                                                    \
    if (!(p)) throw ::sag::Error(SAG_INVALID_ARGUMENT, std::string(#p) + " is null");     \
  } while (0)
