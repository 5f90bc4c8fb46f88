// Shared host/device plumbing for libnpcg_b200: error type, device buffers on
// the context stream, launch accounting, warp/block reductions.
#pragma once

#include <cuda_runtime.h>

#include <atomic>
#include <cstdint>
#include <cstdio>
#include <stdexcept>
#include <string>
#include <utility>

#include "../../include/npcg_capi.h"

namespace npcg {

using i64 = std::int64_t;

/// Carries a C-ABI status code up to the boundary (capi.cpp converts it).
struct Error : std::runtime_error {
  int code;
  Error(int c, const std::string& m) : std::runtime_error(m), code(c) {}
};
[[noreturn]] inline void fail(int code, const std::string& msg) { throw Error(code, msg); }
inline void invalid(const std::string& msg) { fail(NPCG_EINVAL, msg); }

#define NPCG_CUDA(call)                                                                 \
  do {                                                                                  \
    cudaError_t _e = (call);                                                            \
    if (_e != cudaSuccess)                                                              \
      ::npcg::fail(NPCG_ECUDA, std::string("CUDA error: ") + cudaGetErrorString(_e) +   \
                                   " at " + __FILE__ + ":" + std::to_string(__LINE__)); \
  } while (0)

constexpr i64 round_up(i64 x, i64 m) { return (x + m - 1) / m * m; }
constexpr i64 cdiv(i64 x, i64 m) { return (x + m - 1) / m; }
/// Leading dimension for device matrices: columns start on 128-byte lines
/// (TMA and 16-byte vector loads need 16-byte multiples; 128 B keeps every
/// column on its own cache lines).
constexpr i64 dev_ld(i64 rows) { return rows < 1 ? 16 : round_up(rows, 16); }

struct Ctx;

/// Stream-ordered device allocation owned by RAII (cudaMallocAsync pool).
template <class T>
struct DBuf {
  T* p = nullptr;
  i64 n = 0;
  cudaStream_t s = nullptr;
  DBuf() = default;
  DBuf(i64 count, cudaStream_t stream) { alloc(count, stream); }
  DBuf(const DBuf&) = delete;
  DBuf& operator=(const DBuf&) = delete;
  DBuf(DBuf&& o) noexcept { swap(o); }
  DBuf& operator=(DBuf&& o) noexcept {
    if (this != &o) {
      release();
      swap(o);
    }
    return *this;
  }
  ~DBuf() { release(); }
  void swap(DBuf& o) noexcept {
    std::swap(p, o.p);
    std::swap(n, o.n);
    std::swap(s, o.s);
  }
  void alloc(i64 count, cudaStream_t stream) {
    release();
    s = stream;
    n = count;
    if (count > 0) NPCG_CUDA(cudaMallocAsync(reinterpret_cast<void**>(&p), sizeof(T) * count, stream));
  }
  void zero() {
    if (n > 0) NPCG_CUDA(cudaMemsetAsync(p, 0, sizeof(T) * n, s));
  }
  void release() noexcept {
    if (p) cudaFreeAsync(p, s);
    p = nullptr;
    n = 0;
  }
};

/// Column-major FP64 matrix in device memory (ld >= rows, ld % 16 == 0).
struct DMat {
  DBuf<double> buf;
  i64 rows = 0, cols = 0, ld = 16;
  double* p() const { return buf.p; }
  double* col(i64 j) const { return buf.p + j * ld; }
  void alloc(i64 r, i64 c, cudaStream_t s, bool zero = true) {
    rows = r;
    cols = c;
    ld = dev_ld(r);
    buf.alloc(ld * (c < 1 ? 1 : c), s);
    if (zero) buf.zero();
  }
};

// ------------------------------------------------------------------ device
__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}
__device__ __forceinline__ double warp_max(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v = fmax(v, __shfl_xor_sync(0xffffffffu, v, o));
  return v;
}
/// Deterministic block sum (fixed tree); result valid in every thread.
/// `sh` needs blockDim.x/32 doubles.
__device__ __forceinline__ double block_sum(double v, double* sh) {
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5, nw = blockDim.x >> 5;
  v = warp_sum(v);
  __syncthreads();
  if (lane == 0) sh[wid] = v;
  __syncthreads();
  double t = 0.0;
  if (wid == 0) {
    t = lane < nw ? sh[lane] : 0.0;
    t = warp_sum(t);
    if (lane == 0) sh[0] = t;
  }
  __syncthreads();
  return sh[0];
}

/// Block max (result valid in every thread); `sh` needs blockDim.x/32 doubles.
__device__ __forceinline__ double block_max(double v, double* sh) {
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5, nw = blockDim.x >> 5;
  v = warp_max(v);
  __syncthreads();
  if (lane == 0) sh[wid] = v;
  __syncthreads();
  if (wid == 0) {
    double t = lane < nw ? sh[lane] : -1e308;
    t = warp_max(t);
    if (lane == 0) sh[0] = t;
  }
  __syncthreads();
  return sh[0];
}

}  // namespace npcg
