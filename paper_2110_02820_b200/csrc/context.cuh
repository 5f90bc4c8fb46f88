// Per-GPU context: device, the stream every call is ordered on, the
// stream-ordered memory pool, TMA descriptor encoder and launch accounting.
#pragma once

#include <cuda.h>
#include <cuda_runtime.h>

#include <atomic>
#include <mutex>

#include "common.cuh"

namespace npcg {

using EncodeTiledFn = CUresult (*)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*,
                                   const cuuint64_t*, const cuuint64_t*, const cuuint32_t*,
                                   const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle,
                                   CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

struct Ctx {
  int device = 0;
  int sm_count = 148;
  int max_smem_optin = 0;
  cudaStream_t stream = nullptr;
  std::atomic<int64_t> launches{0};
  EncodeTiledFn encode_tiled = nullptr;
  std::mutex mu;  // serialises public calls sharing this context

  explicit Ctx(int dev);
  ~Ctx();
  void sync() { NPCG_CUDA(cudaStreamSynchronize(stream)); }
  void count(int k = 1) { launches.fetch_add(k, std::memory_order_relaxed); }
  void check_launch(const char* what) {
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) fail(NPCG_ECUDA, std::string("kernel launch failed (") + what + "): " + cudaGetErrorString(e));
    count();
  }
  /// Make `dev` current for the calling thread.
  void activate() const { NPCG_CUDA(cudaSetDevice(device)); }
};

/// Launch helper: <<<>>> on the context stream + error check + accounting.
#define NPCG_LAUNCH(ctx, kernel, grid, block, smem, ...)                \
  do {                                                                  \
    kernel<<<(grid), (block), (smem), (ctx).stream>>>(__VA_ARGS__);     \
    (ctx).check_launch(#kernel);                                        \
  } while (0)

}  // namespace npcg
