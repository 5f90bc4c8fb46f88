// Row-sharded data plane (see comm.cuh): NCCL driven from C++, a host
// callback transport, and the pack / unpack kernels around the collectives.
#include <dlfcn.h>
#include <nccl.h>

#include <algorithm>
#include <cstring>
#include <mutex>
#include <vector>

#include "comm.cuh"
#include "context.cuh"

namespace npcg {
namespace {

// ------------------------------------------------------------------ NCCL
// libnccl is opened at run time: the library links and runs without it, and
// inside a torch process the already-loaded copy (same soname) is reused.
struct NcclApi {
  void* h = nullptr;
  ncclResult_t (*GetUniqueId)(ncclUniqueId*) = nullptr;
  ncclResult_t (*CommInitRank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
  ncclResult_t (*CommDestroy)(ncclComm_t) = nullptr;
  ncclResult_t (*AllReduce)(const void*, void*, size_t, ncclDataType_t, ncclRedOp_t, ncclComm_t,
                            cudaStream_t) = nullptr;
  ncclResult_t (*AllGather)(const void*, void*, size_t, ncclDataType_t, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*ReduceScatter)(const void*, void*, size_t, ncclDataType_t, ncclRedOp_t, ncclComm_t,
                                cudaStream_t) = nullptr;
  const char* (*GetErrorString)(ncclResult_t) = nullptr;
};

const NcclApi& nccl() {
  static NcclApi api;
  static std::once_flag once;
  std::call_once(once, [] {
    for (const char* name : {"libnccl.so.2", "libnccl.so"}) {
      api.h = dlopen(name, RTLD_NOW | RTLD_GLOBAL);
      if (api.h) break;
    }
    if (!api.h) return;
    auto sym = [](const char* s) { return dlsym(api.h, s); };
    api.GetUniqueId = reinterpret_cast<decltype(api.GetUniqueId)>(sym("ncclGetUniqueId"));
    api.CommInitRank = reinterpret_cast<decltype(api.CommInitRank)>(sym("ncclCommInitRank"));
    api.CommDestroy = reinterpret_cast<decltype(api.CommDestroy)>(sym("ncclCommDestroy"));
    api.AllReduce = reinterpret_cast<decltype(api.AllReduce)>(sym("ncclAllReduce"));
    api.AllGather = reinterpret_cast<decltype(api.AllGather)>(sym("ncclAllGather"));
    api.ReduceScatter = reinterpret_cast<decltype(api.ReduceScatter)>(sym("ncclReduceScatter"));
    api.GetErrorString = reinterpret_cast<decltype(api.GetErrorString)>(sym("ncclGetErrorString"));
  });
  if (!api.h || !api.GetUniqueId || !api.CommInitRank || !api.AllReduce || !api.AllGather || !api.ReduceScatter)
    fail(NPCG_ENCCL, "libnccl.so.2 could not be loaded (needed for a sharded context)");
  return api;
}

void nccl_check(ncclResult_t r, const char* what) {
  if (r != ncclSuccess)
    fail(NPCG_ENCCL, std::string(what) + " failed: " + (nccl().GetErrorString ? nccl().GetErrorString(r) : "?"));
}

struct NcclComm final : Comm {
  ncclComm_t comm = nullptr;
  const char* name() const override { return "nccl"; }
  ~NcclComm() override {
    if (comm && nccl().CommDestroy) nccl().CommDestroy(comm);
  }
  void allreduce_sum(double* buf, i64 count, cudaStream_t s) override {
    if (count > 0)
      nccl_check(nccl().AllReduce(buf, buf, static_cast<size_t>(count), ncclFloat64, ncclSum, comm, s),
                 "ncclAllReduce");
  }
  void allgather(const double* send, double* recv, i64 count, cudaStream_t s) override {
    if (count > 0)
      nccl_check(nccl().AllGather(send, recv, static_cast<size_t>(count), ncclFloat64, comm, s), "ncclAllGather");
  }
  void reduce_scatter_sum(const double* send, double* recv, i64 count, cudaStream_t s) override {
    if (count > 0)
      nccl_check(nccl().ReduceScatter(send, recv, static_cast<size_t>(count), ncclFloat64, ncclSum, comm, s),
                 "ncclReduceScatter");
  }
};

// ------------------------------------------------------------- callback
struct CallbackComm final : Comm {
  npcg_exchange_fn fn = nullptr;
  void* user = nullptr;
  const char* name() const override { return "callback"; }
  void call(int kind, double* send, double* recv, i64 count, cudaStream_t s) {
    if (count > 0 && fn(user, kind, send, recv, count, s) != 0)
      fail(NPCG_ENCCL, std::string("exchange callback failed (kind ") + std::to_string(kind) + ")");
  }
  void allreduce_sum(double* buf, i64 count, cudaStream_t s) override { call(0, buf, buf, count, s); }
  void allgather(const double* send, double* recv, i64 count, cudaStream_t s) override {
    call(1, const_cast<double*>(send), recv, count, s);
  }
  void reduce_scatter_sum(const double* send, double* recv, i64 count, cudaStream_t s) override {
    call(2, const_cast<double*>(send), recv, count, s);
  }
};

// -------------------------------------------------------------- kernels
// send (nmax x k, contiguous) <- local rows (cnt x k, ld); pad rows are zero
__global__ void pack_rows_kernel(const double* __restrict__ src, i64 lds, i64 cnt, i64 nmax, i64 k,
                                 double* __restrict__ dst) {
  const i64 total = nmax * k;
  for (i64 idx = static_cast<i64>(blockIdx.x) * blockDim.x + threadIdx.x; idx < total;
       idx += static_cast<i64>(gridDim.x) * blockDim.x) {
    const i64 i = idx % nmax, s = idx / nmax;
    dst[idx] = i < cnt ? src[i + s * lds] : 0.0;
  }
}

__device__ __forceinline__ void owner_of(i64 row, i64 q, i64 r, i64* g, i64* i) {
  const i64 big = r * (q + 1);  // rows held by the ranks with q + 1 rows
  if (row < big) {
    *g = row / (q + 1);
    *i = row % (q + 1);
  } else {
    *g = r + (row - big) / q;
    *i = (row - big) % q;
  }
}

// out (n x k, ldo) <- gathered rank-major blocks recv[g][s][i] (nmax x k each)
__global__ void unpack_rows_kernel(const double* __restrict__ recv, i64 q, i64 r, i64 nmax, i64 k, i64 n,
                                   double* __restrict__ out, i64 ldo) {
  const i64 total = n * k;
  for (i64 idx = static_cast<i64>(blockIdx.x) * blockDim.x + threadIdx.x; idx < total;
       idx += static_cast<i64>(gridDim.x) * blockDim.x) {
    const i64 row = idx % n, s = idx / n;
    i64 g, i;
    owner_of(row, q, r, &g, &i);
    out[row + s * ldo] = recv[(g * k + s) * nmax + i];
  }
}

// send (world blocks of nmax x k, rank-major) <- full partial (n x k, ldp)
__global__ void pack_scatter_kernel(const double* __restrict__ partial, i64 ldp, i64 q, i64 r, i64 nmax, i64 k,
                                    int world, double* __restrict__ send) {
  const i64 total = static_cast<i64>(world) * nmax * k;
  for (i64 idx = static_cast<i64>(blockIdx.x) * blockDim.x + threadIdx.x; idx < total;
       idx += static_cast<i64>(gridDim.x) * blockDim.x) {
    const i64 i = idx % nmax, s = (idx / nmax) % k, g = idx / (nmax * k);
    const i64 cnt = q + (g < r ? 1 : 0), off = g * q + (g < r ? g : r);
    send[idx] = i < cnt ? partial[off + i + s * ldp] : 0.0;
  }
}

// local (cnt x k, ldl) <- recv (nmax x k)
__global__ void unpack_local_kernel(const double* __restrict__ recv, i64 cnt, i64 nmax, i64 k, double* __restrict__ out,
                                    i64 ldl) {
  const i64 total = cnt * k;
  for (i64 idx = static_cast<i64>(blockIdx.x) * blockDim.x + threadIdx.x; idx < total;
       idx += static_cast<i64>(gridDim.x) * blockDim.x) {
    const i64 i = idx % cnt, s = idx / cnt;
    out[i + s * ldl] = recv[i + s * nmax];
  }
}

unsigned grid_of(i64 total) { return static_cast<unsigned>(std::max<i64>(1, std::min<i64>(cdiv(total, 256), 4096))); }

}  // namespace

std::shared_ptr<Comm> make_nccl_comm(int device, int rank, int world, const void* unique_id128) {
  if (world < 1 || rank < 0 || rank >= world) invalid("sharded context: need 0 <= rank < world");
  if (!unique_id128) invalid("sharded context: NCCL unique id is null");
  const NcclApi& api = nccl();
  auto c = std::make_shared<NcclComm>();
  c->rank = rank;
  c->world = world;
  ncclUniqueId id;
  std::memcpy(&id, unique_id128, sizeof(id));
  NPCG_CUDA(cudaSetDevice(device));
  nccl_check(api.CommInitRank(&c->comm, world, id, rank), "ncclCommInitRank");
  return c;
}

void nccl_unique_id(void* out128) {
  ncclUniqueId id;
  nccl_check(nccl().GetUniqueId(&id), "ncclGetUniqueId");
  std::memcpy(out128, &id, sizeof(id));
}

std::shared_ptr<Comm> make_callback_comm(int rank, int world, npcg_exchange_fn fn, void* user) {
  if (world < 1 || rank < 0 || rank >= world) invalid("sharded context: need 0 <= rank < world");
  if (!fn) invalid("sharded context: exchange callback is null");
  auto c = std::make_shared<CallbackComm>();
  c->rank = rank;
  c->world = world;
  c->fn = fn;
  c->user = user;
  return c;
}

void rows_allreduce(Ctx& ctx, double* buf, i64 count) {
  if (!ctx.sharded() || count <= 0) return;
  ctx.comm->allreduce_sum(buf, count, ctx.stream);
}

double rows_allreduce_host(Ctx& ctx, double v, bool max) {
  if (!ctx.sharded()) return v;
  const int w = ctx.comm->world;
  DBuf<double> send(1, ctx.stream), recv(w, ctx.stream);
  NPCG_CUDA(cudaMemcpyAsync(send.p, &v, sizeof(double), cudaMemcpyHostToDevice, ctx.stream));
  ctx.comm->allgather(send.p, recv.p, 1, ctx.stream);
  std::vector<double> h(static_cast<size_t>(w));
  NPCG_CUDA(cudaMemcpyAsync(h.data(), recv.p, sizeof(double) * w, cudaMemcpyDeviceToHost, ctx.stream));
  ctx.sync();
  double acc = max ? -INFINITY : 0.0;
  for (const double x : h) acc = max ? std::max(acc, x) : acc + x;  // fixed rank order
  return acc;
}

void rows_allgather(Ctx& ctx, const RowSplit& sp, const double* local, i64 ldl, i64 k, double* full, i64 ldf) {
  if (k <= 0) return;
  const int g = ctx.comm ? ctx.comm->rank : 0;
  if (!ctx.sharded()) {
    NPCG_CUDA(cudaMemcpy2DAsync(full, ldf * 8, local, ldl * 8, sp.n * 8, k, cudaMemcpyDeviceToDevice, ctx.stream));
    return;
  }
  const i64 nmax = sp.nmax();
  DBuf<double> send(nmax * k, ctx.stream), recv(static_cast<i64>(sp.world) * nmax * k, ctx.stream);
  NPCG_LAUNCH(ctx, pack_rows_kernel, grid_of(nmax * k), 256, 0, local, ldl, sp.count(g), nmax, k, send.p);
  ctx.comm->allgather(send.p, recv.p, nmax * k, ctx.stream);
  NPCG_LAUNCH(ctx, unpack_rows_kernel, grid_of(sp.n * k), 256, 0, recv.p, sp.q, sp.r, nmax, k, sp.n, full, ldf);
}

void rows_reduce_scatter(Ctx& ctx, const RowSplit& sp, const double* partial, i64 ldp, i64 k, double* local,
                         i64 ldl) {
  if (k <= 0) return;
  const int g = ctx.comm ? ctx.comm->rank : 0;
  if (!ctx.sharded()) {
    NPCG_CUDA(cudaMemcpy2DAsync(local, ldl * 8, partial, ldp * 8, sp.n * 8, k, cudaMemcpyDeviceToDevice,
                                ctx.stream));
    return;
  }
  const i64 nmax = sp.nmax();
  DBuf<double> send(static_cast<i64>(sp.world) * nmax * k, ctx.stream), recv(nmax * k, ctx.stream);
  NPCG_LAUNCH(ctx, pack_scatter_kernel, grid_of(static_cast<i64>(sp.world) * nmax * k), 256, 0, partial, ldp, sp.q,
              sp.r, nmax, k, sp.world, send.p);
  ctx.comm->reduce_scatter_sum(send.p, recv.p, nmax * k, ctx.stream);
  NPCG_LAUNCH(ctx, unpack_local_kernel, grid_of(sp.count(g) * k), 256, 0, recv.p, sp.count(g), nmax, k, local, ldl);
}

}  // namespace npcg
