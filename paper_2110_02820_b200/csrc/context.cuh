// Per-GPU context: device, the stream every call is ordered on, the
// stream-ordered memory pool, TMA descriptor encoder and launch accounting.
#pragma once

#include <cuda.h>
#include <cuda_runtime.h>

#include <atomic>
#include <memory>
#include <mutex>
#include <string>
#include <vector>

#include "comm.cuh"
#include "common.cuh"

namespace npcg {

using EncodeTiledFn = CUresult (*)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*,
                                   const cuuint64_t*, const cuuint64_t*, const cuuint32_t*,
                                   const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle,
                                   CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

/// Optional per-launch event timing (npcg_prof_enable): CUDA events recorded
/// on the context stream around every kernel this library launches.
struct ProfRec {
  const char* name;
  cudaEvent_t start, stop;
  double flops = 0.0;  // algorithmic work of this launch (when the caller knows it)
  double bytes = 0.0;
  std::string label;   // optional finer aggregation key (e.g. GEMM shape class)
};

struct Ctx {
  int device = 0;
  int sm_count = 148;
  int max_smem_optin = 0;
  cudaStream_t stream = nullptr;
  cudaStream_t aux = nullptr;   // side streams for pipelined host uploads (created on first use):
  cudaStream_t aux2 = nullptr;  // copies on aux, the per-block device work on aux2
  // Staging ring of pipelined host uploads, kept for the context's lifetime
  // (plain cudaMalloc: a stream-ordered free on the copy stream would let a
  // later allocation on the compute stream inherit a wait on the copies).
  static constexpr int kStageSlots = 4;
  double* stage = nullptr;
  i64 stage_slot = 0;  // doubles per slot
  cudaEvent_t stage_free[kStageSlots] = {};
  // Pinned host ring of large uploads from pageable memory (created on first
  // use): host threads fill one slot while the previous one crosses PCIe.
  static constexpr int kPinSlots = 8;  // 256 MB: the host packs ahead while earlier device work (e.g. the kernel-matrix build) still holds the stream
  static constexpr i64 kPinSlotBytes = i64{32} << 20;
  char* pin = nullptr;
  cudaEvent_t pin_free[kPinSlots] = {};
  std::atomic<int64_t> launches{0};
  EncodeTiledFn encode_tiled = nullptr;
  std::mutex mu;  // serialises public calls sharing this context
  // Row-sharded contexts (one process per GPU): the communicator every
  // operator dimension is split over (null = unsharded, one GPU).
  std::shared_ptr<Comm> comm;
  bool sharded() const { return comm && comm->world > 1; }
  int rank() const { return comm ? comm->rank : 0; }
  int world() const { return comm ? comm->world : 1; }
  /// The local row block of an n-dimensional operator / vector on this rank.
  RowSplit split(i64 n) const { return RowSplit(n, world()); }
  i64 local_rows(i64 n) const { return split(n).count(rank()); }
  i64 row_offset(i64 n) const { return split(n).offset(rank()); }
  bool prof = false;
  std::vector<ProfRec> prof_recs;

  explicit Ctx(int dev);
  ~Ctx();
  void sync() { NPCG_CUDA(cudaStreamSynchronize(stream)); }
  cudaStream_t aux_stream() {
    if (!aux) NPCG_CUDA(cudaStreamCreateWithFlags(&aux, cudaStreamNonBlocking));
    return aux;
  }
  cudaStream_t aux2_stream() {
    if (!aux2) NPCG_CUDA(cudaStreamCreateWithFlags(&aux2, cudaStreamNonBlocking));
    return aux2;
  }
  void count(int k = 1) { launches.fetch_add(k, std::memory_order_relaxed); }
  void check_launch(const char* what) {
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) fail(NPCG_ECUDA, std::string("kernel launch failed (") + what + "): " + cudaGetErrorString(e));
    count();
  }
  void prof_begin(const char* name) {
    if (!prof) return;
    ProfRec r{name, nullptr, nullptr};
    NPCG_CUDA(cudaEventCreate(&r.start));
    NPCG_CUDA(cudaEventCreate(&r.stop));
    NPCG_CUDA(cudaEventRecord(r.start, stream));
    prof_recs.push_back(r);
  }
  void prof_end() {
    if (!prof) return;
    NPCG_CUDA(cudaEventRecord(prof_recs.back().stop, stream));
  }
  /// Attach algorithmic flops / bytes to the most recent launch record.
  void prof_work(double flops, double bytes) {
    if (!prof || prof_recs.empty()) return;
    prof_recs.back().flops += flops;
    prof_recs.back().bytes += bytes;
  }
  void prof_label(std::string l) {
    if (!prof || prof_recs.empty()) return;
    prof_recs.back().label = std::move(l);
  }
  /// Make `dev` current for the calling thread.
  void activate() const { NPCG_CUDA(cudaSetDevice(device)); }
};

/// Launch helper: <<<>>> on the context stream + error check + accounting.
#define NPCG_LAUNCH(ctx, kernel, grid, block, smem, ...)                \
  do {                                                                  \
    (ctx).prof_begin(#kernel);                                          \
    kernel<<<(grid), (block), (smem), (ctx).stream>>>(__VA_ARGS__);     \
    (ctx).check_launch(#kernel);                                        \
    (ctx).prof_end();                                                   \
  } while (0)

}  // namespace npcg
