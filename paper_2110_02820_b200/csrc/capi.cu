// The C-ABI (include/npcg_capi.h): argument validation with the reference's
// messages, host<->device staging, and the orchestration loops (adaptive
// doubling, power method). Every compute step below is a CUDA kernel of this
// library; there is no CPU fallback.
#include <cuda.h>

#include <algorithm>
#include <atomic>
#include <chrono>
#include <cstdlib>
#include <future>
#include <random>
#include <thread>
#include <cmath>
#include <cstring>
#include <limits>
#include <memory>
#include <new>
#include <optional>
#include <string>
#include <vector>

#include "blas.cuh"
#include "factor.cuh"
#include "gemm.cuh"
#include "ozaki.cuh"
#include "ops.cuh"
#include "pcg.cuh"
#include "rng.hpp"

using namespace npcg;

// Handles made on a context (operators, sketches, preconditioners) hold a
// counted reference to it: npcg_ctx_destroy drops the caller's reference and
// the context (its stream, its pool) goes when the last handle does, whatever
// order a garbage collector destroys them in.
struct npcg_ctx {
  std::unique_ptr<Ctx> c;
  std::atomic<int> refs{1};
};
inline void ctx_release(npcg_ctx* p) {
  if (p && p->refs.fetch_sub(1) == 1) delete p;
}
struct CtxRef {
  npcg_ctx* p = nullptr;
  CtxRef() = default;
  CtxRef(npcg_ctx* c) : p(c) {  // NOLINT: implicit, handles are aggregate-initialised from npcg_ctx*
    if (p) p->refs.fetch_add(1);
  }
  CtxRef(const CtxRef& o) : CtxRef(o.p) {}
  CtxRef& operator=(const CtxRef& o) {
    if (o.p) o.p->refs.fetch_add(1);
    ctx_release(p);
    p = o.p;
    return *this;
  }
  ~CtxRef() { ctx_release(p); }
  operator npcg_ctx*() const { return p; }  // NOLINT
  npcg_ctx* operator->() const { return p; }
};
struct npcg_rng {
  HostRng r;
};
// (the context reference is the first member: destroyed last, after the device buffers)
struct npcg_op {
  CtxRef ctx;
  std::unique_ptr<Op> op;
};
struct npcg_nys {
  CtxRef ctx;
  Nys s;
};
struct npcg_pre {
  CtxRef ctx;
  Pre p;
};

namespace {
thread_local std::string g_err;

template <class F>
int guard(F&& f) {
  try {
    f();
    return NPCG_OK;
  } catch (const Error& e) {
    g_err = e.what();
    return e.code;
  } catch (const std::invalid_argument& e) {
    g_err = e.what();
    return NPCG_EINVAL;
  } catch (const std::bad_alloc&) {
    g_err = "out of host memory";
    return NPCG_ERUNTIME;
  } catch (const std::exception& e) {
    g_err = e.what();
    return NPCG_ERUNTIME;
  }
}

/// Re-raise the status of a nested C-ABI call inside guard().
void guard_rethrow(int rc) {
  if (rc != NPCG_OK) fail(rc, g_err);
}

void need(const void* p, const char* what) {
  if (!p) invalid(std::string(what) + ": null handle or pointer");
}

/// Device view of a caller matrix: uses the caller's device buffer when it is
/// already TMA/vector friendly, else stages a copy.
struct View {
  DMat owned;
  const double* p = nullptr;
  i64 ld = 0;
};
View view_in(Ctx& ctx, const double* src, i64 rows, i64 cols, i64 ld, int where) {
  View v;
  if (where == NPCG_DEVICE && ld % 2 == 0 && ld >= rows && (reinterpret_cast<uintptr_t>(src) & 15) == 0) {
    v.p = src;
    v.ld = ld;
    return v;
  }
  upload(ctx, v.owned, rows, cols, src, ld, where);
  v.p = v.owned.p();
  v.ld = v.owned.ld;
  return v;
}

double ulp_spacing_host(double x) {
  const double ax = std::abs(x);
  return std::nextafter(ax, std::numeric_limits<double>::infinity()) - ax;
}

/// Draw Omega blocks / power vectors with the GPU generator (rng_gpu.cu):
/// always on a row-sharded context (every rank walks the whole stream, on its
/// GPU instead of its host), and on request (NPCG_DEVICE_RNG=1) otherwise.
/// Engine words are bitwise the reference's; deviates differ by a few ulp.
bool use_device_rng(const Ctx& c) {
  static const bool env = std::getenv("NPCG_DEVICE_RNG") && std::string(std::getenv("NPCG_DEVICE_RNG")) == "1";
  return env || c.sharded();
}

Ctx& C(npcg_ctx* c) {
  need(c, "context");
  c->c->activate();
  return *c->c;
}
}  // namespace

// ============================== context =====================================
namespace npcg {
Ctx::Ctx(int dev) : device(dev) {
  int count = 0;
  if (cudaGetDeviceCount(&count) != cudaSuccess || count == 0)
    fail(NPCG_ECUDA, "no CUDA device available (libnpcg_b200 has no CPU fallback)");
  if (dev < 0 || dev >= count) invalid("npcg_ctx_create: device index out of range");
  NPCG_CUDA(cudaSetDevice(dev));
  cudaDeviceProp prop;
  NPCG_CUDA(cudaGetDeviceProperties(&prop, dev));
  if (prop.major < 10) fail(NPCG_ECUDA, std::string("libnpcg_b200 needs an sm_100 (B200) device, found ") + prop.name);
  sm_count = prop.multiProcessorCount;
  max_smem_optin = static_cast<int>(prop.sharedMemPerBlockOptin);
  NPCG_CUDA(cudaStreamCreateWithFlags(&stream, cudaStreamNonBlocking));
  cudaMemPool_t pool;
  NPCG_CUDA(cudaDeviceGetDefaultMemPool(&pool, dev));
  uint64_t thr = std::numeric_limits<uint64_t>::max();
  NPCG_CUDA(cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &thr));
  void* fn = nullptr;
  cudaDriverEntryPointQueryResult q;
  NPCG_CUDA(cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q));
  if (!fn || q != cudaDriverEntryPointSuccess) fail(NPCG_ECUDA, "cuTensorMapEncodeTiled unavailable");
  encode_tiled = reinterpret_cast<EncodeTiledFn>(fn);
}
Ctx::~Ctx() {
  if (stream || aux || aux2) cudaSetDevice(device);
  for (cudaStream_t* sp : {&aux, &aux2})
    if (*sp) {
      cudaStreamSynchronize(*sp);
      cudaStreamDestroy(*sp);
    }
  if (stage) cudaFree(stage);
  for (cudaEvent_t ev : stage_free)
    if (ev) cudaEventDestroy(ev);
  if (stream) cudaStreamSynchronize(stream);  // the pinned ring's last copies
  if (pin) cudaFreeHost(pin);
  for (cudaEvent_t ev : pin_free)
    if (ev) cudaEventDestroy(ev);
  if (stream) {
    cudaStreamSynchronize(stream);
    cudaStreamDestroy(stream);
  }
}
}  // namespace npcg

extern "C" {

const char* npcg_last_error(void) { return g_err.c_str(); }
const char* npcg_version(void) { return "npcg_b200 0.1 (sm_100a)"; }

int npcg_ctx_create(int device, npcg_ctx** out) {
  return guard([&] {
    need(out, "npcg_ctx_create");
    auto c = std::make_unique<npcg_ctx>();
    c->c = std::make_unique<Ctx>(device);
    *out = c.release();
  });
}
int npcg_nccl_unique_id(void* out128) {
  return guard([&] {
    need(out128, "npcg_nccl_unique_id");
    nccl_unique_id(out128);
  });
}
int npcg_ctx_create_sharded(int device, int rank, int world, const void* nccl_id128, npcg_ctx** out) {
  return guard([&] {
    need(out, "npcg_ctx_create_sharded");
    auto c = std::make_unique<npcg_ctx>();
    c->c = std::make_unique<Ctx>(device);
    c->c->comm = make_nccl_comm(device, rank, world, nccl_id128);
    *out = c.release();
  });
}
int npcg_ctx_create_exchange(int device, int rank, int world, npcg_exchange_fn fn, void* user, npcg_ctx** out) {
  return guard([&] {
    need(out, "npcg_ctx_create_exchange");
    auto c = std::make_unique<npcg_ctx>();
    c->c = std::make_unique<Ctx>(device);
    c->c->comm = make_callback_comm(rank, world, fn, user);
    *out = c.release();
  });
}
int npcg_ctx_layout(const npcg_ctx* ctx, int64_t n, int* rank, int* world, int64_t* offset, int64_t* count) {
  return guard([&] {
    need(ctx, "npcg_ctx_layout");
    const Ctx& c = *ctx->c;
    if (rank) *rank = c.rank();
    if (world) *world = c.world();
    if (offset) *offset = c.row_offset(n);
    if (count) *count = c.local_rows(n);
  });
}
int npcg_ctx_destroy(npcg_ctx* ctx) {
  return guard([&] { ctx_release(ctx); });
}
int npcg_ctx_sync(npcg_ctx* ctx) {
  return guard([&] { C(ctx).sync(); });
}
void* npcg_ctx_stream(npcg_ctx* ctx) { return ctx ? ctx->c->stream : nullptr; }
int64_t npcg_ctx_launches(npcg_ctx* ctx) { return ctx ? ctx->c->launches.load() : 0; }
int npcg_prof_enable(npcg_ctx* ctx, int on) {
  return guard([&] {
    Ctx& c = C(ctx);
    c.sync();
    for (auto& r : c.prof_recs) {
      cudaEventDestroy(r.start);
      cudaEventDestroy(r.stop);
    }
    c.prof_recs.clear();
    c.prof = on != 0;
  });
}
int npcg_prof_report(npcg_ctx* ctx, char* buf, int64_t cap) {
  return guard([&] {
    Ctx& c = C(ctx);
    c.sync();
    struct Agg {
      int64_t count = 0;
      double ms = 0.0, flops = 0.0, bytes = 0.0;
    };
    std::vector<std::pair<std::string, Agg>> agg;
    for (auto& r : c.prof_recs) {
      float ms = 0.f;
      NPCG_CUDA(cudaEventElapsedTime(&ms, r.start, r.stop));
      const std::string key = r.label.empty() ? std::string(r.name) : r.label;
      auto it = std::find_if(agg.begin(), agg.end(), [&](auto& p) { return p.first == key; });
      if (it == agg.end()) {
        agg.emplace_back(key, Agg{});
        it = agg.end() - 1;
      }
      it->second.count += 1;
      it->second.ms += ms;
      it->second.flops += r.flops;
      it->second.bytes += r.bytes;
    }
    std::string out;
    char line[512];
    for (auto& [name, a] : agg) {
      std::snprintf(line, sizeof(line), "%s\t%lld\t%.6f\t%.6e\t%.6e\n", name.c_str(),
                    static_cast<long long>(a.count), a.ms, a.flops, a.bytes);
      out += line;
    }
    if (static_cast<int64_t>(out.size()) + 1 > cap) invalid("npcg_prof_report: buffer too small");
    std::memcpy(buf, out.c_str(), out.size() + 1);
  });
}

int npcg_dev_alloc(npcg_ctx* ctx, int64_t bytes, void** out) {
  return guard([&] {
    Ctx& c = C(ctx);
    NPCG_CUDA(cudaMallocAsync(out, static_cast<size_t>(std::max<int64_t>(bytes, 16)), c.stream));
    c.sync();
  });
}
int npcg_dev_free(npcg_ctx* ctx, void* p) {
  return guard([&] {
    Ctx& c = C(ctx);
    NPCG_CUDA(cudaFreeAsync(p, c.stream));
  });
}
int npcg_memcpy(npcg_ctx* ctx, void* dst, int dst_where, const void* src, int src_where, int64_t bytes) {
  return guard([&] {
    Ctx& c = C(ctx);
    const cudaMemcpyKind k = dst_where == NPCG_DEVICE
                                 ? (src_where == NPCG_DEVICE ? cudaMemcpyDeviceToDevice : cudaMemcpyHostToDevice)
                                 : (src_where == NPCG_DEVICE ? cudaMemcpyDeviceToHost : cudaMemcpyHostToHost);
    NPCG_CUDA(cudaMemcpyAsync(dst, src, static_cast<size_t>(bytes), k, c.stream));
    c.sync();
  });
}

// =============================== random =====================================
int npcg_rng_create(uint64_t seed, npcg_rng** out) {
  return guard([&] { *out = new npcg_rng{HostRng(seed)}; });
}
int npcg_rng_clone(const npcg_rng* rng, npcg_rng** out) {
  return guard([&] { *out = new npcg_rng(*rng); });
}
int npcg_rng_destroy(npcg_rng* rng) {
  delete rng;
  return NPCG_OK;
}
double npcg_rng_normal(npcg_rng* rng) { return rng->r.normal(); }
double npcg_rng_uniform(npcg_rng* rng) { return rng->r.uniform(); }
uint64_t npcg_rng_word(npcg_rng* rng) { return rng->r.engine(); }
void npcg_rng_discard(npcg_rng* rng, uint64_t words) { rng->r.engine.discard(words); }
int npcg_rng_integer(npcg_rng* rng, uint64_t bound, uint64_t* out) {
  return guard([&] { *out = rng->r.integer(bound); });
}
int npcg_rng_gaussian(npcg_rng* rng, int64_t rows, int64_t cols, double* dst) {
  return guard([&] { rng->r.gaussian(rows, cols, dst); });
}
int npcg_rng_uniform_fill(npcg_rng* rng, int64_t count, double* dst) {
  return guard([&] {
    for (int64_t i = 0; i < count; ++i) dst[i] = rng->r.uniform();
  });
}
int npcg_rng_sample(npcg_rng* rng, int64_t n, int64_t k, int64_t* out) {
  return guard([&] {  // random.cpp:44-56
    if (k < 0 || k > n) invalid("sample_without_replacement: need 0 <= k <= n");
    std::vector<int64_t> pool(static_cast<size_t>(n));
    for (int64_t i = 0; i < n; ++i) pool[static_cast<size_t>(i)] = i;
    for (int64_t i = 0; i < k; ++i) {
      const int64_t j = i + static_cast<int64_t>(rng->r.integer(static_cast<uint64_t>(n - i)));
      std::swap(pool[static_cast<size_t>(i)], pool[static_cast<size_t>(j)]);
    }
    std::copy(pool.begin(), pool.begin() + k, out);
  });
}
int npcg_rng_words_device(npcg_ctx* ctx, npcg_rng* rng, int64_t count, uint64_t* dst) {
  return guard([&] {
    need(rng, "npcg_rng_words_device");
    Ctx& c = C(ctx);
    device_words(c, rng->r.engine, count, reinterpret_cast<unsigned long long*>(dst));
  });
}
int npcg_rng_gaussian_device(npcg_ctx* ctx, npcg_rng* rng, int64_t rows, int64_t cols, double* dst, int64_t ld) {
  return guard([&] {
    need(rng, "npcg_rng_gaussian_device");
    Ctx& c = C(ctx);
    if (rows < 0 || cols < 0) invalid("gaussian_matrix: dimensions must be >= 0");
    device_gaussian(c, rng->r.engine, rows, cols, c.row_offset(rows), c.local_rows(rows), dst, ld);
    c.sync();
  });
}
uint64_t npcg_splitmix64(uint64_t seed) {  // bench.cpp:180-185
  uint64_t z = seed + 0x9e3779b97f4a7c15ull;
  z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ull;
  z = (z ^ (z >> 27)) * 0x94d049bb133111ebull;
  return z ^ (z >> 31);
}
double npcg_ulp_spacing(double x) { return ulp_spacing_host(x); }

// ============================== operators ===================================
namespace {
/// The handle for a finished operator. On a sharded context `local` is the
/// rank's share (column block / row block of X / kernel work share) working on
/// full-length inputs and is wrapped in a ShardOp; otherwise it is the operator.
npcg_op* finish_op(npcg_ctx* ctx, std::unique_ptr<Op> local, i64 n, int kind) {
  Ctx& c = *ctx->c;
  if (c.sharded() && n < c.world()) invalid("sharded operator: dimension smaller than the number of ranks");
  local->set_dim(c, n);
  local->kind = kind;
  if (!c.sharded()) return new npcg_op{ctx, std::move(local)};
  auto op = std::make_unique<ShardOp>();
  op->set_dim(c, n);
  op->kind = kind;
  op->local = std::move(local);
  return new npcg_op{ctx, std::move(op)};
}

npcg_op* make_dense(npcg_ctx* ctx, DMat&& a, i64 n, int kind) {
  Ctx& c = *ctx->c;
  if (!c.sharded()) {
    auto op = std::make_unique<DenseOp>();
    op->a = std::move(a);
    return finish_op(ctx, std::move(op), n, kind);
  }
  // keep this rank's column block A[:, R_g] (= rows R_g, A symmetric)
  auto blk = std::make_unique<DenseColBlockOp>();
  blk->set_dim(c, n);
  blk->a.alloc(n, blk->nloc, c.stream, false);
  copy2d(c, n, blk->nloc, a.col(blk->off), a.ld, blk->a.p(), blk->a.ld);
  c.sync();
  a.buf.release();
  return finish_op(ctx, std::move(blk), n, kind);
}

npcg_op* make_colblock(npcg_ctx* ctx, DMat&& block, i64 n, int kind) {
  auto blk = std::make_unique<DenseColBlockOp>();
  blk->a = std::move(block);
  return finish_op(ctx, std::move(blk), n, kind);
}
}  // namespace

int npcg_op_dense_create(npcg_ctx* ctx, int64_t rows, int64_t cols, const double* a, int64_t lda, int where,
                         npcg_op** out) {
  return guard([&] {
    Ctx& c = C(ctx);
    if (rows != cols) invalid("DenseOperator: matrix must be square");  // operators.cpp:65
    DMat A;
    upload(c, A, rows, cols, a, lda, where);
    double asym = 0.0, amax = 0.0;
    symmetry_stats(c, A.p(), rows, A.ld, &asym, &amax);
    if (asym > 1e-12 * std::max(1.0, amax)) invalid("DenseOperator: matrix must be symmetric");  // :66-69
    *out = make_dense(ctx, std::move(A), rows, kDense);
  });
}

int npcg_op_gram_create(npcg_ctx* ctx, int64_t m, int64_t n, const double* g, int64_t ldg, int where, npcg_op** out) {
  return guard([&] {
    Ctx& c = C(ctx);
    if (m < 1 || n < 1) invalid("GramRidgeOperator: design matrix must be nonempty");  // operators.cpp:106-107
    auto op = std::make_unique<GramOp>();
    op->ctx = &c;
    op->n = n;
    op->div = static_cast<double>(m);
    if (c.sharded()) {  // this rank's rows of X (the m rows split like any dimension)
      const RowSplit sp = c.split(m);
      op->m = sp.count(c.rank());
      if (op->m < 1) invalid("GramRidgeOperator shard: more ranks than design rows");
      op->shard_partial = true;
      gram_upload(c, *op, g + sp.offset(c.rank()), ldg, where);
    } else {
      op->m = m;
      gram_upload(c, *op, g, ldg, where);
    }
    *out = finish_op(ctx, std::move(op), n, kGram);
  });
}

int npcg_op_gram_create_streamed(npcg_ctx* ctx, int64_t m, int64_t n, const double* g, int64_t ldg,
                                 npcg_op** out) {
  return guard([&] {
    Ctx& c = C(ctx);
    if (m < 1 || n < 1) invalid("GramRidgeOperator: design matrix must be nonempty");  // operators.cpp:106-107
    if (ldg < m) invalid("leading dimension smaller than the row count");
    if (c.sharded()) {  // sharded: the synchronous upload of this rank's rows
      guard_rethrow(npcg_op_gram_create(ctx, m, n, g, ldg, NPCG_HOST, out));
      return;
    }
    auto op = std::make_unique<GramOp>();
    op->ctx = &c;
    op->n = n;
    op->m = m;
    op->div = static_cast<double>(m);
    gram_upload_streamed(c, *op, g, ldg);
    *out = finish_op(ctx, std::move(op), n, kGram);
  });
}

int npcg_op_gram_shard_create(npcg_ctx* ctx, int64_t m_local, int64_t n, const double* g, int64_t ldg, int where,
                              int64_t m_total, npcg_op** out) {
  return guard([&] {
    Ctx& c = C(ctx);
    if (m_local < 1 || n < 1 || m_total < m_local) invalid("GramRidgeOperator shard: bad block dimensions");
    auto local = std::make_unique<GramOp>();
    local->ctx = &c;
    local->n = n;
    local->m = m_local;
    local->div = static_cast<double>(m_total);
    local->shard_partial = c.sharded();
    gram_upload(c, *local, g, ldg, where);
    *out = finish_op(ctx, std::move(local), n, kGram);
  });
}

int npcg_op_dense_shard_create(npcg_ctx* ctx, int64_t n, const double* a_block, int64_t lda, int where,
                               npcg_op** out) {
  return guard([&] {
    Ctx& c = C(ctx);
    if (n < 1) invalid("DenseOperator: matrix must be square");
    const i64 nloc = c.local_rows(n);
    DMat blk;
    upload(c, blk, n, nloc, a_block, lda, where);
    if (!all_finite(c, blk.p(), n, nloc, blk.ld)) invalid("DenseOperator: matrix has non-finite entries");
    *out = c.sharded() ? make_colblock(ctx, std::move(blk), n, kDense) : make_dense(ctx, std::move(blk), n, kDense);
  });
}

int npcg_op_kernel_create(npcg_ctx* ctx, int64_t n, int64_t d, const double* pts, int64_t ldp, double sigma,
                          int64_t dense_cap, int where, npcg_op** out) {
  return guard([&] {
    Ctx& c = C(ctx);
    if (n < 1) invalid("KernelOperator: need at least one point");   // operators.cpp:143
    if (!(sigma > 0.0)) invalid("KernelOperator: sigma must be > 0");  // :144
    DMat P;
    upload(c, P, n, d, pts, ldp, where);
    if (!all_finite(c, P.p(), n, d, P.ld)) invalid("KernelOperator: points have non-finite entries");
    if (n <= dense_cap) {  // :148-149
      DMat K;
      if (c.sharded()) {  // this rank's column block K[:, R_g], built from all points
        build_kernel_colblock(c, P, n, d, sigma, c.row_offset(n), c.local_rows(n), K);
        *out = make_colblock(ctx, std::move(K), n, kKernelStored);
      } else {
        build_kernel_matrix(c, P, n, d, sigma, K);
        *out = make_dense(ctx, std::move(K), n, kKernelStored);
      }
    } else {
      auto op = std::make_unique<KernelFreeOp>();
      op->ctx = &c;
      op->n = n;
      op->d = d;
      op->sigma = sigma;
      op->pts = std::move(P);
      op->shard_rank = c.rank();
      op->shard_world = c.world();
      op->shard_off = c.row_offset(n);
      op->shard_rows = c.local_rows(n);
      prepare_kernel_free(c, *op);
      *out = finish_op(ctx, std::move(op), n, kKernelFree);
    }
  });
}

int npcg_op_synthesize(npcg_ctx* ctx, int64_t n, const double* lambda, uint64_t seed, npcg_op** out) {
  return guard([&] {
    Ctx& c = C(ctx);
    // SpectrumProfile validation (operators.cpp:190-199)
    if (n < 1) invalid("SpectrumProfile: need at least one eigenvalue");
    for (int64_t i = 0; i < n; ++i) {
      if (!(lambda[i] >= 0.0) || !std::isfinite(lambda[i]))
        invalid("SpectrumProfile: eigenvalues must be finite and >= 0");
      if (i > 0 && lambda[i] > lambda[i - 1]) invalid("SpectrumProfile: eigenvalues must be nonincreasing");
    }
    // operators.cpp:211-219: Q from a seeded n x n Gaussian; A = Q diag(l) Q^T; (A + A^T)/2.
    // (A sharded context builds the whole A on every rank -- an O(n^3) input
    // generator -- and keeps its column block.)
    HostRng rng(seed);
    std::vector<double> g(static_cast<size_t>(n * n));
    rng.gaussian(n, n, g.data());
    DMat G, Q, A, S;
    upload(c, G, n, n, g.data(), n, NPCG_HOST);
    Q.alloc(n, n, c.stream, false);
    orthonormalize(c, G.p(), G.ld, n, n, Q.p(), Q.ld);  // replicated (not row-sharded) on every rank
    DBuf<double> lam(n, c.stream);
    NPCG_CUDA(cudaMemcpyAsync(lam.p, lambda, sizeof(double) * n, cudaMemcpyHostToDevice, c.stream));
    copy2d(c, n, n, Q.p(), Q.ld, G.p(), G.ld);  // G <- Q diag(lambda)
    scale_cols(c, G.p(), n, n, G.ld, lam.p);
    A.alloc(n, n, c.stream, false);
    gemm(c, n, n, n, 1.0, Operand{G.p(), G.ld, false}, Operand{Q.p(), Q.ld, false}, 0.0, A.p(), A.ld);
    S.alloc(n, n, c.stream, true);
    symmetrize(c, A.p(), n, A.ld, S.p(), S.ld);
    c.sync();
    *out = make_dense(ctx, std::move(S), n, kDense);
  });
}

int npcg_op_lowrank_create(npcg_ctx* ctx, int64_t n, int64_t r, const double* g, int64_t ldg, const double* lambda,
                           int where, npcg_op** out) {
  return guard([&] {
    Ctx& c = C(ctx);
    if (n < 1 || r < 1) invalid("lowrank operator: need n >= 1 and r >= 1");
    DMat G, GD, A;
    upload(c, G, n, r, g, ldg, where);
    GD.alloc(n, r, c.stream, false);
    copy2d(c, n, r, G.p(), G.ld, GD.p(), GD.ld);
    DBuf<double> lam(r, c.stream);
    NPCG_CUDA(cudaMemcpyAsync(lam.p, lambda, sizeof(double) * r, cudaMemcpyHostToDevice, c.stream));
    scale_cols(c, GD.p(), n, r, GD.ld, lam.p);
    if (c.sharded()) {  // A[:, R_g] = G diag(lambda) G[R_g, :]^T / r
      const i64 off = c.row_offset(n), nloc = c.local_rows(n);
      A.alloc(n, nloc, c.stream, false);
      gemm(c, n, nloc, r, 1.0, Operand{GD.p(), GD.ld, false}, Operand{G.p() + off, G.ld, false}, 0.0, A.p(), A.ld);
      divide(c, n, nloc, A.p(), A.ld, static_cast<double>(r));
      c.sync();
      *out = make_colblock(ctx, std::move(A), n, kDense);
      return;
    }
    A.alloc(n, n, c.stream, false);
    gemm(c, n, n, r, 1.0, Operand{GD.p(), GD.ld, false}, Operand{G.p(), G.ld, false}, 0.0, A.p(), A.ld);
    divide(c, n, n, A.p(), A.ld, static_cast<double>(r));
    symmetrize(c, A.p(), n, A.ld, A.p(), A.ld);  // in place: (A + A^T) / 2
    c.sync();
    *out = make_dense(ctx, std::move(A), n, kDense);
  });
}

int npcg_op_callback_create(npcg_ctx* ctx, int64_t n, npcg_apply_fn apply, npcg_column_fn column, void* user,
                            int where, npcg_op** out) {
  return guard([&] {
    Ctx& c = C(ctx);
    need(out, "npcg_op_callback_create");
    if (!apply) invalid("npcg_op_callback_create: apply callback is null");
    if (n < 1) invalid("LinearOperator: dimension must be positive");
    if (where != NPCG_HOST && where != NPCG_DEVICE) invalid("npcg_op_callback_create: where must be host or device");
    auto op = std::make_unique<CallbackOp>();
    op->set_dim(c, n);  // on a sharded context the callback sees this rank's row blocks
    op->kind = kCallback;
    op->fn = apply;
    op->col = column;
    op->user = user;
    op->where = where;
    *out = new npcg_op{ctx, std::move(op)};
  });
}

int npcg_op_regularize(npcg_op* base, double mu, npcg_op** out) {
  return guard([&] {
    need(base, "RegularizedOperator: base operator is null");  // operators.cpp:84-85
    need(out, "npcg_op_regularize");
    Ctx& c = C(base->ctx);
    if (!(mu >= 0.0)) invalid("RegularizedOperator: mu must be >= 0");  // operators.cpp:86
    auto op = std::make_unique<RegOp>();
    op->set_dim(c, base->op->n);
    op->kind = kRegularized;
    op->base = base->op.get();
    op->mu = mu;
    *out = new npcg_op{base->ctx, std::move(op)};
  });
}

int npcg_op_destroy(npcg_op* op) {
  return guard([&] {
    if (op) {
      op->ctx->c->activate();
      op->ctx->c->sync();
      delete op;
    }
  });
}
int npcg_op_dim(const npcg_op* op, int64_t* n) {
  return guard([&] {
    need(op, "npcg_op_dim");
    *n = op->op->n;
  });
}
int npcg_op_rows(const npcg_op* op, int64_t* offset, int64_t* count) {
  return guard([&] {
    need(op, "npcg_op_rows");
    if (offset) *offset = op->op->off;
    if (count) *count = op->op->nloc;
  });
}
int npcg_op_kind(const npcg_op* op) { return op ? op->op->kind : -1; }
int npcg_op_has_column_access(const npcg_op* op) { return op && op->op->has_column() ? 1 : 0; }

int npcg_op_apply(npcg_op* op, int64_t rows, int64_t k, const double* v, int64_t ldv, double* out, int64_t ldo,
                  int where) {
  return guard([&] {
    need(op, "npcg_op_apply");
    Ctx& c = C(op->ctx);
    const i64 n = op->op->nloc;  // this rank's rows (all of them unsharded)
    const bool single = k == 1;
    if (rows != n) {  // operators.cpp:14-19, 33-34
      if (single)
        invalid("LinearOperator - matvec: dimension mismatch (got " + std::to_string(rows) + ", operator dim " +
                std::to_string(n) + ")");
      invalid("LinearOperator - apply_block: dimension mismatch");
    }
    if (k <= 0) return;
    View in = view_in(c, v, n, k, ldv, where);
    if (!all_finite_rows(c, in.p, n, k, in.ld))
      invalid(single ? "LinearOperator - matvec: input has non-finite entries"
                     : "LinearOperator - apply_block: input has non-finite entries");
    DMat o;
    o.alloc(n, k, c.stream, false);
    op->op->apply(in.p, in.ld, k, o.p(), o.ld);
    download(c, o.p(), o.ld, n, k, out, ldo, where);
    c.sync();
  });
}

int npcg_op_column(npcg_op* op, int64_t j, double* out, int where) {
  return guard([&] {
    need(op, "npcg_op_column");
    Ctx& c = C(op->ctx);
    if (!op->op->has_column()) fail(NPCG_ERUNTIME, "LinearOperator - column: operator has no column access");
    if (j < 0 || j >= op->op->n) invalid("LinearOperator - column: index out of range");
    const i64 nl = op->op->nloc;  // sharded: this rank's rows of the column
    DMat o;
    o.alloc(nl, 1, c.stream, false);
    op->op->column(j, o.p());
    download(c, o.p(), o.ld, nl, 1, out, nl, where);
    c.sync();
  });
}

// =============================== Nyström ====================================
int npcg_nys_create(npcg_op* op, npcg_nys** out) {
  return guard([&] {
    need(op, "npcg_nys_create");
    Ctx& c = C(op->ctx);
    if (op->op->n < 1) invalid("make_empty_sketch: dimension must be positive");
    auto h = std::make_unique<npcg_nys>();
    h->ctx = op->ctx;
    h->s.ctx = &c;
    h->s.op = op->op.get();
    h->s.n = op->op->n;
    h->s.nloc = op->op->nloc;
    h->s.off = op->op->off;
    *out = h.release();
  });
}
int npcg_nys_bind(npcg_nys* nys, npcg_op* op) {
  return guard([&] {
    need(nys, "npcg_nys_bind");
    need(op, "npcg_nys_bind operator");
    if (op->op->n != nys->s.n) invalid("extend_sketch: dimension mismatch");
    nys->s.op = op->op.get();
  });
}
int npcg_nys_extend(npcg_nys* nys, int64_t extra, const double* omega_raw, int64_t ld, int where) {
  return guard([&] {
    need(nys, "npcg_nys_extend");
    C(nys->ctx);
    nys_extend(nys->s, omega_raw, ld, extra, where);
    nys->ctx->c->sync();
  });
}
int npcg_nys_extend_rng(npcg_nys* nys, int64_t extra, npcg_rng* rng) {
  return guard([&] {
    need(nys, "npcg_nys_extend_rng");
    C(nys->ctx);
    // nystrom.cpp:36-45: validate, then draw the n x extra Gaussian block.
    if (extra < 1) invalid("extend_sketch: extra must be >= 1");
    if (nys->s.size + extra > nys->s.n) invalid("extend_sketch: sketch size would exceed dimension");
    // the whole block is drawn (the reference's stream on every rank); this rank keeps its rows
    Ctx& c = *nys->ctx->c;
    if (use_device_rng(c)) {
      DMat raw;
      raw.alloc(nys->s.nloc, extra, c.stream, false);
      device_gaussian(c, rng->r.engine, nys->s.n, extra, nys->s.off, nys->s.nloc, raw.p(), raw.ld);
      nys_extend(nys->s, raw.p(), raw.ld, extra, NPCG_DEVICE);
    } else {
      std::vector<double> raw(static_cast<size_t>(nys->s.n * extra));
      rng->r.gaussian(nys->s.n, extra, raw.data());
      nys_extend(nys->s, raw.data() + nys->s.off, nys->s.n, extra, NPCG_HOST);
    }
    nys->ctx->c->sync();
  });
}
namespace {
// extend_sketch_columns' draw (nystrom.cpp:69-80): partial Fisher-Yates over the
// unused indices in increasing order, rng.integer(remaining - i).
std::vector<i64> draw_unused(HostRng& r, i64 n, const std::vector<i64>& used, i64 extra) {
  std::vector<bool> taken(static_cast<size_t>(n), false);
  for (const i64 j : used) taken[static_cast<size_t>(j)] = true;
  std::vector<i64> remaining;
  remaining.reserve(static_cast<size_t>(n) - used.size());
  for (i64 j = 0; j < n; ++j)
    if (!taken[static_cast<size_t>(j)]) remaining.push_back(j);
  for (i64 i = 0; i < extra; ++i) {
    const i64 pick = i + static_cast<i64>(r.integer(static_cast<uint64_t>(static_cast<i64>(remaining.size()) - i)));
    std::swap(remaining[static_cast<size_t>(i)], remaining[static_cast<size_t>(pick)]);
  }
  remaining.resize(static_cast<size_t>(extra));
  return remaining;
}
void extend_columns_rng(Nys& s, i64 extra, HostRng& r) {
  if (!s.op || !s.op->has_column())
    fail(NPCG_ERUNTIME, "extend_sketch_columns: operator has no column access");
  if (extra < 1) invalid("extend_sketch_columns: extra must be >= 1");
  if (static_cast<i64>(s.used.size()) + extra > s.n)
    invalid("extend_sketch_columns: sketch size would exceed dimension");
  const std::vector<i64> idx = draw_unused(r, s.n, s.used, extra);
  nys_extend_columns(s, idx);
  s.used.insert(s.used.end(), idx.begin(), idx.end());
}
}  // namespace

int npcg_nys_extend_columns(npcg_nys* nys, int64_t extra, npcg_rng* rng) {
  return guard([&] {
    need(nys, "npcg_nys_extend_columns");
    need(rng, "npcg_nys_extend_columns rng");
    C(nys->ctx);
    extend_columns_rng(nys->s, extra, rng->r);
  });
}

int npcg_nys_used(const npcg_nys* nys, int64_t* out, int64_t* count) {
  return guard([&] {
    need(nys, "npcg_nys_used");
    if (count) *count = static_cast<int64_t>(nys->s.used.size());
    if (out) std::copy(nys->s.used.begin(), nys->s.used.end(), out);
  });
}

int npcg_column_sampling_nystrom(npcg_op* op, int64_t ell, const int64_t* indices, npcg_rng* rng, npcg_nys** out) {
  return guard([&] {
    need(op, "npcg_column_sampling_nystrom");
    Ctx& c = C(op->ctx);
    const i64 n = op->op->n;
    std::vector<i64> idx;
    if (!indices) {  // nystrom.cpp:150-158
      need(rng, "npcg_column_sampling_nystrom rng");
      if (ell < 1 || ell > n) invalid("column_sampling_nystrom: need 1 <= ell <= dim");
      if (!op->op->has_column()) fail(NPCG_ERUNTIME, "column_sampling_nystrom: operator has no column access");
      std::vector<int64_t> pool(static_cast<size_t>(n));  // sample_without_replacement (random.cpp:44-56)
      for (i64 i = 0; i < n; ++i) pool[static_cast<size_t>(i)] = i;
      for (i64 i = 0; i < ell; ++i) {
        const i64 j = i + static_cast<i64>(rng->r.integer(static_cast<uint64_t>(n - i)));
        std::swap(pool[static_cast<size_t>(i)], pool[static_cast<size_t>(j)]);
      }
      idx.assign(pool.begin(), pool.begin() + ell);
    } else {  // nystrom.cpp:160-184
      if (ell < 1 || ell > n) invalid("column_sampling_nystrom: need 1 <= #indices <= dim");
      if (!op->op->has_column()) fail(NPCG_ERUNTIME, "column_sampling_nystrom: operator has no column access");
      std::vector<bool> seen(static_cast<size_t>(n), false);
      for (i64 i = 0; i < ell; ++i) {
        const i64 j = indices[i];
        if (j < 0 || j >= n) invalid("column_sampling_nystrom: index out of range");
        if (seen[static_cast<size_t>(j)]) invalid("column_sampling_nystrom: indices must be distinct");
        seen[static_cast<size_t>(j)] = true;
        idx.push_back(j);
      }
    }
    auto h = std::make_unique<npcg_nys>();
    h->ctx = op->ctx;
    h->s.ctx = &c;
    h->s.op = op->op.get();
    h->s.n = n;
    h->s.nloc = op->op->nloc;
    h->s.off = op->op->off;
    nys_extend_columns(h->s, idx);
    h->s.used = idx;
    nys_factor(h->s);
    *out = h.release();
  });
}

int npcg_nys_factor(npcg_nys* nys) {
  return guard([&] {
    need(nys, "npcg_nys_factor");
    C(nys->ctx);
    nys_factor(nys->s);
  });
}
int npcg_nys_from_factors(npcg_ctx* ctx, int64_t n, int64_t ell, const double* u, int64_t ldu, const double* lambda,
                          double shift_used, int where, npcg_nys** out) {
  return guard([&] {
    Ctx& c = C(ctx);
    auto h = std::make_unique<npcg_nys>();
    h->ctx = ctx;
    Nys& s = h->s;
    s.ctx = &c;
    s.n = n;
    s.nloc = c.local_rows(n);  // sharded: u holds this rank's rows
    s.off = c.row_offset(n);
    auto f = std::make_shared<Factors>();
    f->ell = ell;
    f->shift = shift_used;
    if (ell > 0) {
      upload(c, f->u, s.nloc, ell, u, ldu, where);
      f->lambda.alloc(ell, c.stream);
      NPCG_CUDA(cudaMemcpyAsync(f->lambda.p, lambda, sizeof(double) * ell,
                                where == NPCG_HOST ? cudaMemcpyHostToDevice : cudaMemcpyDeviceToDevice, c.stream));
      f->lambda_host.resize(static_cast<size_t>(ell));
      NPCG_CUDA(cudaMemcpyAsync(f->lambda_host.data(), f->lambda.p, sizeof(double) * ell, cudaMemcpyDeviceToHost,
                                c.stream));
    } else {
      f->u.alloc(s.nloc, 0, c.stream, false);
    }
    c.sync();
    s.fac = std::move(f);
    *out = h.release();
  });
}
int npcg_nys_info(const npcg_nys* nys, int64_t* n, int64_t* sketch_cols, int64_t* ell_factored, double* shift) {
  return guard([&] {
    need(nys, "npcg_nys_info");
    if (n) *n = nys->s.n;
    if (sketch_cols) *sketch_cols = nys->s.size;
    if (ell_factored) *ell_factored = nys->s.factored() ? nys->s.fac->ell : -1;
    if (shift) *shift = nys->s.factored() ? nys->s.fac->shift : 0.0;
  });
}
int npcg_nys_rows(const npcg_nys* nys, int64_t* offset, int64_t* count) {
  return guard([&] {
    need(nys, "npcg_nys_rows");
    if (offset) *offset = nys->s.off;
    if (count) *count = nys->s.nloc;
  });
}
int npcg_nys_get(npcg_nys* nys, double* lambda, double* u, int64_t ldu, int where) {
  return guard([&] {
    need(nys, "npcg_nys_get");
    Ctx& c = C(nys->ctx);
    if (!nys->s.factored()) fail(NPCG_ERUNTIME, "npcg_nys_get: approximation not factored (call npcg_nys_factor)");
    const Factors& f = *nys->s.fac;
    const i64 ell = f.ell;
    if (lambda && ell > 0) {
      if (where == NPCG_HOST) std::memcpy(lambda, f.lambda_host.data(), sizeof(double) * ell);
      else NPCG_CUDA(cudaMemcpyAsync(lambda, f.lambda.p, sizeof(double) * ell, cudaMemcpyDeviceToDevice, c.stream));
    }
    if (u && ell > 0) download(c, f.u.p(), f.u.ld, nys->s.nloc, ell, u, ldu, where);
    c.sync();
  });
}
int npcg_nys_get_sketch(npcg_nys* nys, double* omega, double* y, int64_t ld, int where) {
  return guard([&] {
    need(nys, "npcg_nys_get_sketch");
    Ctx& c = C(nys->ctx);
    if (nys->s.size == 0) return;
    if (omega) download(c, nys->s.omega().p(), nys->s.omega().ld, nys->s.nloc, nys->s.size, omega, ld, where);
    if (y) download(c, nys->s.y().p(), nys->s.y().ld, nys->s.nloc, nys->s.size, y, ld, where);
    c.sync();
  });
}
int npcg_nys_clone(const npcg_nys* nys, int factors_only, npcg_nys** out) {
  return guard([&] {
    need(nys, "npcg_nys_clone");
    need(out, "npcg_nys_clone");
    auto h = std::make_unique<npcg_nys>();
    h->ctx = nys->ctx;
    h->s.ctx = nys->s.ctx;
    h->s.n = nys->s.n;
    h->s.nloc = nys->s.nloc;
    h->s.off = nys->s.off;
    h->s.fac = nys->s.fac;
    if (!factors_only) {  // shares the sketch store; the first append by either handle past the other copies
      h->s.op = nys->s.op;
      h->s.sk = nys->s.sk;
      h->s.size = nys->s.size;
      h->s.used = nys->s.used;
    }
    *out = h.release();
  });
}
int npcg_nys_destroy(npcg_nys* nys) {
  return guard([&] {
    if (nys) {
      nys->ctx->c->activate();
      nys->ctx->c->sync();
      delete nys;
    }
  });
}

// ============================ preconditioner ================================
int npcg_pre_create(npcg_nys* nys, double mu, npcg_pre** out) {
  return guard([&] {
    need(nys, "npcg_pre_create");
    C(nys->ctx);
    auto h = std::make_unique<npcg_pre>();
    h->ctx = nys->ctx;
    pre_build(h->p, nys->s, mu);
    *out = h.release();
  });
}
namespace {
int pre_apply_common(npcg_pre* pre, int64_t s, const double* r, int64_t ldr, double* z, int64_t ldz, int where,
                     bool inverse) {
  return guard([&] {
    need(pre, "npcg_pre_apply");
    Ctx& c = C(pre->ctx);
    if (s <= 0) return;
    const i64 n = pre->p.nloc;
    View in = view_in(c, r, n, s, ldr, where);
    DMat o;
    o.alloc(n, s, c.stream, false);
    if (inverse) pre_apply_inverse(pre->p, in.p, in.ld, s, o.p(), o.ld);
    else pre_apply(pre->p, in.p, in.ld, s, o.p(), o.ld);
    download(c, o.p(), o.ld, n, s, z, ldz, where);
    c.sync();
  });
}
}  // namespace
int npcg_pre_apply_inverse(npcg_pre* pre, int64_t s, const double* r, int64_t ldr, double* z, int64_t ldz, int where) {
  return pre_apply_common(pre, s, r, ldr, z, ldz, where, true);
}
int npcg_pre_apply(npcg_pre* pre, int64_t s, const double* v, int64_t ldv, double* out, int64_t ldo, int where) {
  return pre_apply_common(pre, s, v, ldv, out, ldo, where, false);
}
int npcg_woodbury_inverse_apply(npcg_nys* nys, double mu, int64_t s, const double* b, int64_t ldb, double* x,
                                int64_t ldx, int where) {
  return guard([&] {
    need(nys, "npcg_woodbury_inverse_apply");
    Ctx& c = C(nys->ctx);
    if (!(mu > 0.0)) invalid("woodbury_inverse_apply: mu must be > 0");  // preconditioner.cpp:106-107
    if (!nys->s.factored()) fail(NPCG_ERUNTIME, "woodbury_inverse_apply: approximation not factored");
    if (s <= 0) return;
    const i64 n = nys->s.nloc;
    View B = view_in(c, b, n, s, ldb, where);
    DMat X;
    X.alloc(n, s, c.stream, false);
    woodbury_apply(c, *nys->s.fac, n, mu, B.p, B.ld, s, X.p(), X.ld);
    download(c, X.p(), X.ld, n, s, x, ldx, where);
    c.sync();
  });
}
int npcg_pre_destroy(npcg_pre* pre) {
  delete pre;
  return NPCG_OK;
}

// ================================ solvers ===================================
int npcg_pcg(npcg_op* op, npcg_pre* pre, double mu, int64_t s, const double* b, int64_t ldb, const double* x0,
             int64_t ldx0, const npcg_solve_opts* opts, double* x, int64_t ldx, npcg_solve_report* reports,
             double* history, double* iterates, int where) {
  bool diverged = false;
  std::string dmsg;
  int rc = guard([&] {
    need(op, "npcg_pcg");
    need(opts, "npcg_pcg options");
    Ctx& c = C(op->ctx);
    const char* context = pre ? "nystrom_pcg" : "cg";
    if (pre) {  // solvers.cpp:134-136
      if (!(mu >= 0.0)) invalid("nystrom_pcg: mu must be >= 0");
      if (pre->p.ell > 0) {
        if (pre->p.n != op->op->n) invalid("nystrom_pcg: preconditioner dimension mismatch");
        if (pre->p.mu != mu) invalid("nystrom_pcg: preconditioner built with a different mu");
      }
    } else if (!(mu >= 0.0)) {
      invalid("RegularizedOperator: mu must be >= 0");
    }
    if (!(opts->eta > 0.0)) invalid(std::string(context) + ": eta must be > 0");  // solvers.cpp:27-31
    if (opts->max_iter < 0) invalid(std::string(context) + ": max_iter must be >= 0");
    const i64 n = op->op->nloc;  // this rank's rows of b, x0, x (all of them unsharded)
    if (s <= 0) return;
    PcgOptions po{opts->eta, opts->max_iter, opts->relative != 0, opts->record_iterates != 0};
    View B = view_in(c, b, n, s, ldb, where);
    View X0;
    if (x0) {
      X0 = view_in(c, x0, n, s, ldx0, where);
      if (!all_finite_rows(c, X0.p, n, s, X0.ld)) invalid("LinearOperator - matvec: input has non-finite entries");
    }
    DMat X;
    X.alloc(n, s, c.stream, false);
    const bool rec = iterates && po.record_iterates;
    for (i64 s0 = 0; s0 < s; s0 += 8) {
      const i64 sb = std::min<i64>(8, s - s0);
      IterateRec its;
      PcgResult r = pcg_solve(c, *op->op, pre ? &pre->p : nullptr, mu, sb, B.p + s0 * B.ld, B.ld,
                              x0 ? X0.p + s0 * X0.ld : nullptr, X0.ld, po, X.p() + s0 * X.ld, X.ld,
                              rec ? &its : nullptr, context);
      i64 rows = 0;  // iterations recorded by any column of the batch
      for (i64 j = 0; j < sb; ++j) {
        const PcgColumnReport& cr = r.cols[static_cast<size_t>(j)];
        npcg_solve_report& rep = reports[s0 + j];
        rep.iterations = cr.iterations;
        rep.matvec_count = cr.matvec_count;
        rep.converged = cr.converged ? 1 : 0;
        rep.status = cr.status;
        rep.eta_used = cr.eta_used;
        rep.wall_time = r.wall_time;
        rep.history_len = static_cast<int64_t>(cr.history.size());
        rows = std::max<i64>(rows, rep.history_len);
        if (history)
          std::copy(cr.history.begin(), cr.history.end(), history + (s0 + j) * (po.max_iter + 1));
      }
      if (rec) {  // layout to caller: [t][col][n] for the whole s; only the rows the loop reached
        rows = std::min(rows, its.cap);
        for (i64 t = 0; t < rows; ++t) {
          const cudaMemcpyKind k = where == NPCG_HOST ? cudaMemcpyDeviceToHost : cudaMemcpyDeviceToDevice;
          NPCG_CUDA(cudaMemcpyAsync(iterates + (t * s + s0) * n, its.buf.p + t * n * sb, sizeof(double) * n * sb, k,
                                    c.stream));
        }
        c.sync();
      }
      if (r.diverged) {
        diverged = true;
        if (dmsg.empty()) dmsg = r.message;
      }
    }
    download(c, X.p(), X.ld, n, s, x, ldx, where);
    c.sync();
  });
  if (rc == NPCG_OK && diverged) {
    g_err = dmsg;
    return NPCG_EDIVERGED;
  }
  return rc;
}

int npcg_regularization_path(npcg_op* op, npcg_nys* nys, int64_t nmu, const double* mus, int64_t s,
                             const double* b, int64_t ldb, const npcg_solve_opts* opts, int warm_start,
                             double* x, int64_t ldx, npcg_solve_report* reports, int where) {
  return guard([&] {
    need(op, "npcg_regularization_path");
    need(nys, "npcg_regularization_path approximation");
    need(opts, "npcg_regularization_path options");
    Ctx& c = C(op->ctx);
    if (nmu < 0 || s < 0) invalid("regularization_path: counts must be >= 0");
    if (!nys->s.factored()) fail(NPCG_ERUNTIME, "build_preconditioner: approximation not factored");
    if (nys->s.fac->ell > 0 && nys->s.n != op->op->n) invalid("nystrom_pcg: preconditioner dimension mismatch");
    if (!(opts->eta > 0.0)) invalid("nystrom_pcg: eta must be > 0");
    if (opts->max_iter < 0) invalid("nystrom_pcg: max_iter must be >= 0");
    const i64 n = op->op->nloc;
    if (s == 0 || nmu == 0) return;
    PcgOptions po{opts->eta, opts->max_iter, opts->relative != 0, false};
    View B = view_in(c, b, n, s, ldb, where);
    DMat X, Xprev;
    X.alloc(n, s, c.stream, false);
    auto fill = [&](npcg_solve_report& rep, const PcgColumnReport& cr, double wall) {
      rep.iterations = cr.iterations;
      rep.matvec_count = cr.matvec_count;
      rep.converged = cr.converged ? 1 : 0;
      rep.status = cr.status;
      rep.eta_used = cr.eta_used;
      rep.wall_time = wall;
      rep.history_len = static_cast<int64_t>(cr.history.size());
    };
    // Cold starts: the systems of different mu are independent, so 8 / s
    // consecutive mu share one pass over A per iteration (8 columns with their
    // own shift and gains in the persistent loop); each column's arithmetic is
    // that of its own solve.
    const i64 group = (warm_start == 0 && s <= 4 && 8 % s == 0 && nys->s.fac->ell > 0 &&
                       pcg_mu_batch_eligible(c, *op->op, 8)) ? 8 / s : 1;
    i64 kbatched = 0;
    if (group > 1) {
      DMat Bg, Xg;
      Bg.alloc(n, 8, c.stream, false);
      Xg.alloc(n, 8, c.stream, false);
      for (i64 g = 0; g < group; ++g) copy2d(c, n, s, B.p, B.ld, Bg.p() + g * s * Bg.ld, Bg.ld);
      for (; kbatched + group <= nmu; kbatched += group) {
        std::vector<Pre> pres(static_cast<size_t>(group));
        PcgMuCols cols;
        for (i64 g = 0; g < group; ++g) {
          pre_build(pres[static_cast<size_t>(g)], nys->s, mus[kbatched + g]);  // rejects mu <= 0
          for (i64 j = 0; j < s; ++j) {
            cols.mu.push_back(mus[kbatched + g]);
            cols.pre.push_back(&pres[static_cast<size_t>(g)]);
          }
        }
        PcgResult r = pcg_solve(c, *op->op, cols.pre[0], cols.mu[0], 8, Bg.p(), Bg.ld, nullptr, 0, po, Xg.p(), Xg.ld,
                                nullptr, "nystrom_pcg", &cols);
        for (i64 g = 0; g < group; ++g) {
          for (i64 j = 0; j < s; ++j)
            fill(reports[(kbatched + g) * s + j], r.cols[static_cast<size_t>(g * s + j)], r.wall_time);
          if (x) download(c, Xg.p() + g * s * Xg.ld, Xg.ld, n, s, x + (kbatched + g) * s * ldx, ldx, where);
        }
        c.sync();  // the group's preconditioners go out of scope
      }
    }
    for (i64 k = kbatched; k < nmu; ++k) {
      const double mu = mus[k];
      Pre p;
      pre_build(p, nys->s, mu);  // rejects mu <= 0 (preconditioner.cpp:80-89)
      const bool warm = warm_start != 0 && k > 0;
      if (warm) copy2d(c, n, s, X.p(), X.ld, Xprev.p(), Xprev.ld);
      for (i64 s0 = 0; s0 < s; s0 += 8) {
        const i64 sb = std::min<i64>(8, s - s0);
        PcgResult r = pcg_solve(c, *op->op, &p, mu, sb, B.p + s0 * B.ld, B.ld,
                                warm ? Xprev.p() + s0 * Xprev.ld : nullptr, Xprev.ld, po, X.p() + s0 * X.ld, X.ld,
                                nullptr, "nystrom_pcg");
        for (i64 j = 0; j < sb; ++j) {
          fill(reports[k * s + s0 + j], r.cols[static_cast<size_t>(j)], r.wall_time);
        }
      }
      if (x) download(c, X.p(), X.ld, n, s, x + k * s * ldx, ldx, where);
      if (k == 0 && warm_start) Xprev.alloc(n, s, c.stream, false);
    }
    c.sync();
  });
}

int npcg_block_pcg(npcg_op* op, npcg_pre* pre, double mu, int64_t s, const double* b, int64_t ldb,
                   const npcg_solve_opts* opts, double* x, int64_t ldx, npcg_block_report* rep, int* converged,
                   int64_t* deflated, double* final_residual, double* history, int64_t* history_len, int where) {
  return guard([&] {
    need(op, "npcg_block_pcg");
    need(opts, "npcg_block_pcg options");
    Ctx& c = C(op->ctx);
    const i64 n = op->op->nloc;
    // solvers.cpp:156-165
    if (s < 1) invalid("block_nystrom_pcg: need at least one column");
    if (s > 32) invalid("block_nystrom_pcg: at most 32 right-hand sides per block in this build");
    if (!(opts->eta > 0.0)) invalid("block_nystrom_pcg: eta must be > 0");
    if (!(mu >= 0.0)) invalid("block_nystrom_pcg: mu must be >= 0");
    if (pre && pre->p.ell > 0 && pre->p.n != op->op->n) invalid("block_nystrom_pcg: preconditioner dimension mismatch");
    View B = view_in(c, b, n, s, ldb, where);
    DMat X;
    X.alloc(n, s, c.stream, false);
    PcgOptions po{opts->eta, opts->max_iter, opts->relative != 0, false};
    BlockPcgResult r = block_pcg_solve(c, *op->op, pre ? &pre->p : nullptr, mu, s, B.p, B.ld, po, X.p(), X.ld);
    download(c, X.p(), X.ld, n, s, x, ldx, where);
    rep->iterations = r.iterations;
    rep->fallback_count = r.fallback_count;
    rep->n_deflated = static_cast<int64_t>(r.deflated.size());
    rep->eta_used = r.eta_used;
    rep->wall_time = r.wall_time;
    for (i64 j = 0; j < s; ++j) {
      converged[j] = r.converged[static_cast<size_t>(j)] ? 1 : 0;
      const std::vector<double>& hj = r.history[static_cast<size_t>(j)];
      final_residual[j] = hj.back();
      const i64 len = std::min<i64>(static_cast<i64>(hj.size()), po.max_iter + 1);
      if (history_len) history_len[j] = len;
      if (history) std::copy(hj.begin(), hj.begin() + len, history + j * (po.max_iter + 1));
    }
    for (size_t i = 0; i < r.deflated.size(); ++i) deflated[i] = r.deflated[i];
  });
}

int npcg_iteration_bound(double kappa, double epsilon, int64_t* out) {
  return guard([&] {  // solvers.cpp:281-291
    if (!(kappa >= 1.0)) invalid("iteration_bound: kappa must be >= 1");
    if (!(epsilon > 0.0 && epsilon < 1.0)) invalid("iteration_bound: epsilon must lie in (0, 1)");
    if (kappa == 1.0) {
      *out = 1;
      return;
    }
    const double root = std::sqrt(kappa);
    const double rate = std::log((root + 1.0) / (root - 1.0));
    const double t = std::ceil(std::log(2.0 / epsilon) / rate);
    *out = std::max<int64_t>(1, static_cast<int64_t>(t));
  });
}

// =============================== adaptive ===================================
namespace {
double dot_dev(Ctx& c, const double* a, const double* b, i64 n) {
  // v.w through the coldot kernel (one column dotted with one vector); summed over the ranks when sharded
  DBuf<double> o(1, c.stream);
  coldot(c, a, dev_ld(n), n, 1, b, dev_ld(n), 1, o.p, 1);
  rows_allreduce(c, o.p, 1);
  double h = 0.0;
  NPCG_CUDA(cudaMemcpyAsync(&h, o.p, sizeof(double), cudaMemcpyDeviceToHost, c.stream));
  c.sync();
  return h;
}

// estimate_error_power (adaptive.cpp:83-109) from the raw start vector g
// (this rank's rows when sharded; norms, dots and U^T v are all-reduced).
double power_estimate(Ctx& c, Op& op, const Nys& s, i64 q, const double* g_dev) {
  const i64 n = op.nloc, ell = s.factored() ? s.fac->ell : 0;
  DMat v, w, t;
  v.alloc(n, 1, c.stream, true);
  w.alloc(n, 1, c.stream, true);
  copy2d(c, n, 1, g_dev, n, v.p(), v.ld);
  const double v0 = std::sqrt(sum_squares_rows(c, v.p(), n, 1, v.ld));
  if (v0 == 0.0) return 0.0;
  divide(c, n, 1, v.p(), v.ld, v0);
  double estimate = 0.0;
  if (ell > 0) t.alloc(ell, 1, c.stream, false);
  for (i64 i = 0; i < q; ++i) {
    op.apply(v.p(), v.ld, 1, w.p(), w.ld);
    if (ell > 0) {  // w -= U (lambda .* (U^T v))
      coldot(c, s.fac->u.p(), s.fac->u.ld, n, ell, v.p(), v.ld, 1, t.p(), t.ld);
      rows_allreduce(c, t.p(), ell);
      scale_cols(c, t.p(), 1, ell, 1, s.fac->lambda.p);  // t_j *= lambda_j (as a 1 x ell row)
      axpby(c, ell, 1, 0.0, t.p(), -1.0, t.p(), t.ld);  // t = -t (exact)
      rowdot(c, s.fac->u.p(), s.fac->u.ld, n, ell, t.p(), t.ld, 1, w.p(), w.ld, w.p(), w.ld);
    }
    estimate = dot_dev(c, v.p(), w.p(), n);
    const double nrm = std::sqrt(sum_squares_rows(c, w.p(), n, 1, w.ld));
    if (nrm == 0.0) return 0.0;
    copy2d(c, n, 1, w.p(), w.ld, v.p(), v.ld);
    divide(c, n, 1, v.p(), v.ld, nrm);
  }
  return estimate;
}
}  // namespace

int npcg_power_estimate(npcg_op* op, npcg_nys* nys, int64_t q, const double* g_raw, int where, double* est) {
  return guard([&] {
    need(op, "npcg_power_estimate");
    need(nys, "npcg_power_estimate");
    Ctx& c = C(op->ctx);
    if (q < 1) invalid("estimate_error_power: q must be >= 1");  // adaptive.cpp:86
    if (nys->s.factored() && nys->s.fac->ell > 0 && nys->s.n != op->op->n)
      invalid("estimate_error_power: factor shape mismatch");
    View g = view_in(c, g_raw, op->op->nloc, 1, op->op->nloc, where);
    *est = power_estimate(c, *op->op, nys->s, q, g.p);
  });
}
int npcg_power_estimate_rng(npcg_op* op, npcg_nys* nys, int64_t q, npcg_rng* rng, double* est) {
  return guard([&] {
    need(op, "npcg_power_estimate_rng");
    need(nys, "npcg_power_estimate_rng");
    Ctx& c = C(op->ctx);
    if (q < 1) invalid("estimate_error_power: q must be >= 1");
    if (nys->s.factored() && nys->s.fac->ell > 0 && nys->s.n != op->op->n)
      invalid("estimate_error_power: factor shape mismatch");
    std::vector<double> g(static_cast<size_t>(op->op->n));
    rng->r.gaussian(op->op->n, 1, g.data());  // gaussian_vector (adaptive.cpp:90); this rank keeps its rows
    View gv = view_in(c, g.data() + op->op->off, op->op->nloc, 1, op->op->nloc, NPCG_HOST);
    *est = power_estimate(c, *op->op, nys->s, q, gv.p);
  });
}

int npcg_posterior_condition(double lambda_ell, double mu, double err, double* out) {
  return guard([&] {  // adaptive.cpp:150-156
    if (!(mu > 0.0)) invalid("posterior_condition_estimate: mu must be > 0");
    if (lambda_ell < 0.0 || err < 0.0) invalid("posterior_condition_estimate: inputs must be >= 0");
    *out = (lambda_ell + mu + err) / mu;
  });
}

int npcg_adaptive(npcg_op* op, const npcg_adaptive_cfg* cfg, npcg_rng* rng, npcg_nys** out,
                  npcg_adaptive_outcome* outcome) {
  return guard([&] {
    need(op, "npcg_adaptive");
    need(cfg, "npcg_adaptive config");
    need(rng, "npcg_adaptive rng");
    Ctx& c = C(op->ctx);
    const i64 n = op->op->n;
    // mode checks (adaptive.cpp:113-114, 127-128, 137-138)
    // validate_config (adaptive.cpp:19-28)
    if (cfg->ell0 < 1 || cfg->ell0 > cfg->ell_max || cfg->ell_max > n)
      invalid("AdaptiveConfig: need 1 <= ell0 <= ell_max <= dim");
    if (!(cfg->mu > 0.0)) invalid("AdaptiveConfig: mu must be > 0");
    if (cfg->q < 1) invalid("AdaptiveConfig: q must be >= 1");
    double tau = cfg->tol_mode == 1 ? 10.0 : 30.0;  // resolved_tau (adaptive.cpp:9-15)
    if (cfg->has_tau) {
      if (!(cfg->tau > 0.0)) invalid("AdaptiveConfig: tau must be > 0");
      tau = cfg->tau;
    }
    if (cfg->sketch != 0 && !op->op->has_column())  // adaptive.cpp:26-27
      fail(NPCG_ERUNTIME, "AdaptiveConfig: column sampling needs column access");
    auto h = std::make_unique<npcg_nys>();
    h->ctx = op->ctx;
    Nys& s = h->s;
    s.ctx = &c;
    s.op = op->op.get();
    s.n = n;
    s.nloc = op->op->nloc;  // sharded: every draw is the whole block; this rank keeps its rows
    s.off = op->op->off;
    // Draw-ahead (error strategy, Gaussian sketch): the stream after an Omega
    // block is always the power vector g, then -- if the loop continues -- the
    // next block, whose size the doubling rule fixes in advance. A host thread
    // draws both from a copy of the engine while the GPU sketches and
    // factors; the caller's engine is advanced only by what the loop consumes
    // (g, then the block if used), so the stream is exactly the reference's.
    struct DrawAhead {
      std::thread th;
      std::promise<void> g_ready;
      std::future<void> g_fut;
      std::vector<double> g, raw;
      Mt64 after_g, after_raw;
      i64 extra = 0;
      bool active = false, g_taken = false;
      void finish() {
        if (th.joinable()) th.join();
        active = false;
      }
      ~DrawAhead() { finish(); }
    } ahead;
    const bool dev_rng = use_device_rng(c);
    const bool draw_ahead =
        !dev_rng && cfg->tol_mode == 0 && cfg->sketch == 0 && std::getenv("NPCG_NO_DRAW_AHEAD") == nullptr;
    auto start_ahead = [&](i64 size_after) {
      if (!draw_ahead) return;
      const i64 ex = size_after >= cfg->ell_max ? 0
                     : 2 * size_after <= cfg->ell_max ? size_after : cfg->ell_max - size_after;
      ahead.extra = (ex > 0 && n * ex <= (i64{2} << 30)) ? ex : 0;  // <= 16 GB of host staging
      ahead.g_ready = std::promise<void>();
      ahead.g_fut = ahead.g_ready.get_future();
      ahead.g_taken = false;
      ahead.active = true;
      ahead.th = std::thread([&ahead = ahead, eng = rng->r, n]() mutable {
        ahead.g.resize(static_cast<size_t>(n));
        eng.gaussian(n, 1, ahead.g.data());
        ahead.after_g = eng.engine;
        ahead.g_ready.set_value();
        if (ahead.extra > 0) {
          ahead.raw.resize(static_cast<size_t>(n * ahead.extra));
          eng.gaussian(n, ahead.extra, ahead.raw.data());
          ahead.after_raw = eng.engine;
        }
      });
    };
    auto grow = [&](i64 extra) {  // adaptive.cpp:30-35
      if (cfg->sketch != 0) {
        extend_columns_rng(s, extra, rng->r);
        return;
      }
      if (dev_rng) {  // the GPU generator continues the caller's engine
        DMat raw;
        raw.alloc(s.nloc, extra, c.stream, false);
        device_gaussian(c, rng->r.engine, n, extra, s.off, s.nloc, raw.p(), raw.ld);
        nys_extend(s, raw.p(), raw.ld, extra, NPCG_DEVICE);
        return;
      }
      std::vector<double> raw;
      if (ahead.active) {
        ahead.finish();
        if (ahead.g_taken && ahead.extra == extra) {
          raw.swap(ahead.raw);
          rng->r.engine = ahead.after_raw;
        }
      }
      if (raw.empty()) {
        raw.resize(static_cast<size_t>(n * extra));
        rng->r.gaussian(n, extra, raw.data());
      }
      start_ahead(s.size + extra);
      nys_extend(s, raw.data() + s.off, n, extra, NPCG_HOST);
    };
    auto estimate = [&]() {
      if (dev_rng) {
        DMat gd;
        gd.alloc(s.nloc, 1, c.stream, false);
        device_gaussian(c, rng->r.engine, n, 1, s.off, s.nloc, gd.p(), gd.ld);
        return power_estimate(c, *op->op, s, cfg->q, gd.p());
      }
      std::vector<double> g;
      if (ahead.active && !ahead.g_taken) {
        ahead.g_fut.wait();
        g = ahead.g;
        rng->r.engine = ahead.after_g;
        ahead.g_taken = true;
      } else {
        g.resize(static_cast<size_t>(n));
        rng->r.gaussian(n, 1, g.data());
      }
      View gv = view_in(c, g.data() + s.off, s.nloc, 1, s.nloc, NPCG_HOST);
      return power_estimate(c, *op->op, s, cfg->q, gv.p);
    };
    std::optional<double> err;
    i64 doublings = 0;
    bool hit_cap = false;
    if (cfg->tol_mode == 2) {  // fixed_rank_nystrom (adaptive.cpp:135-148)
      grow(cfg->ell_max);
      nys_factor(s);
      err = estimate();
    } else {  // doubling_loop (adaptive.cpp:50-79)
      const double tol = tau * cfg->mu;
      auto should_stop = [&]() -> bool {
        const double lmin = s.fac->lambda_min();
        if (cfg->tol_mode == 1) return lmin <= tau * cfg->mu;  // adaptive.cpp:129-132
        const double e = estimate();                           // adaptive.cpp:115-121
        err = e;
        if (e > tol) return false;
        return !cfg->secondary_criterion || lmin <= tol / 11.0;
      };
      grow(cfg->ell0);
      nys_factor(s);
      while (true) {
        if (should_stop()) break;
        const i64 ell = s.size;
        if (ell >= cfg->ell_max) {
          hit_cap = true;
          break;
        }
        const i64 extra = 2 * ell <= cfg->ell_max ? ell : cfg->ell_max - ell;
        grow(extra);
        ++doublings;
        nys_factor(s);
        if (s.size == cfg->ell_max && 2 * ell > cfg->ell_max) {
          hit_cap = true;
          break;
        }
      }
    }
    ahead.finish();  // an unused draw-ahead block is discarded (the engine never saw it)
    const double lmin = s.fac->lambda_min();
    const double e0 = err ? std::max(0.0, *err) : 0.0;
    outcome->ell_final = s.fac->ell;
    outcome->doublings = doublings;
    outcome->hit_cap = hit_cap ? 1 : 0;
    outcome->has_error_estimate = err ? 1 : 0;
    outcome->error_estimate = err.value_or(0.0);
    outcome->posterior_condition = (lmin + cfg->mu + e0) / cfg->mu;
    *out = h.release();
  });
}

// ============================ dense helpers =================================
int npcg_orthonormal_columns(npcg_ctx* ctx, int64_t m, int64_t n, const double* g, double* q, int where) {
  return guard([&] {
    Ctx& c = C(ctx);
    if (m < n) invalid("orthonormal_columns: expected a tall (m >= n) matrix");
    if (n <= 0) return;
    View G = view_in(c, g, m, n, m, where);
    DMat Q;
    Q.alloc(m, n, c.stream, false);
    orthonormalize(c, G.p, G.ld, m, n, Q.p(), Q.ld);
    download(c, Q.p(), Q.ld, m, n, q, m, where);
    c.sync();
  });
}
int npcg_gemm(npcg_ctx* ctx, int64_t m, int64_t n, int64_t k, double alpha, const double* a, int64_t lda,
              int a_kmajor, const double* b, int64_t ldb, int b_kmajor, double beta, double* c, int64_t ldc,
              int where) {
  return guard([&] {
    Ctx& cx = C(ctx);
    if (m < 0 || n < 0 || k < 0) invalid("npcg_gemm: negative dimension");
    if (m == 0 || n == 0) return;
    View A = view_in(cx, a, a_kmajor ? k : m, a_kmajor ? m : k, lda, where);
    View B = view_in(cx, b, b_kmajor ? k : n, b_kmajor ? n : k, ldb, where);
    View Cv = view_in(cx, c, m, n, ldc, where);
    gemm(cx, m, n, k, alpha, Operand{A.p, A.ld, a_kmajor != 0}, Operand{B.p, B.ld, b_kmajor != 0}, beta,
         const_cast<double*>(Cv.p), Cv.ld);
    if (Cv.owned.p() != nullptr || where == NPCG_HOST) download(cx, Cv.p, Cv.ld, m, n, c, ldc, where);
    cx.sync();
  });
}

int npcg_gemm_ozaki(npcg_ctx* ctx, int64_t m, int64_t n, int64_t k, const double* a, int64_t lda, int a_kmajor,
                    const double* b, int64_t ldb, int b_kmajor, double* c, int64_t ldc, int where) {
  return guard([&] {
    Ctx& cx = C(ctx);
    if (m < 0 || n < 0 || k < 0) invalid("npcg_gemm_ozaki: negative dimension");
    if (m == 0 || n == 0) return;
    View A = view_in(cx, a, a_kmajor ? k : m, a_kmajor ? m : k, lda, where);
    View B = view_in(cx, b, b_kmajor ? k : n, b_kmajor ? n : k, ldb, where);
    View Cv = view_in(cx, c, m, n, ldc, where);
    gemm_ozaki(cx, m, n, k, A.p, A.ld, a_kmajor != 0, B.p, B.ld, 0.0, const_cast<double*>(Cv.p), Cv.ld,
               b_kmajor != 0);
    if (Cv.owned.p() != nullptr || where == NPCG_HOST) download(cx, Cv.p, Cv.ld, m, n, c, ldc, where);
    cx.sync();
  });
}

int npcg_gemm_i8(npcg_ctx* ctx, int64_t m, int64_t n, int64_t kp, const int8_t* a8, const int8_t* b8,
                 int32_t* c32) {
  return guard([&] {
    Ctx& cx = C(ctx);
    if (m <= 0 || n <= 0 || kp <= 0 || kp % 128 != 0) invalid("npcg_gemm_i8: bad shape");
    DBuf<int8_t> da(m * kp, cx.stream), db(n * kp, cx.stream);
    DBuf<int32_t> dc(m * n, cx.stream);
    NPCG_CUDA(cudaMemcpyAsync(da.p, a8, m * kp, cudaMemcpyHostToDevice, cx.stream));
    NPCG_CUDA(cudaMemcpyAsync(db.p, b8, n * kp, cudaMemcpyHostToDevice, cx.stream));
    gemm_i8_raw(cx, static_cast<int>(m), static_cast<int>(n), kp, da.p, db.p, dc.p);
    NPCG_CUDA(cudaMemcpyAsync(c32, dc.p, sizeof(int32_t) * m * n, cudaMemcpyDeviceToHost, cx.stream));
    cx.sync();
  });
}

int npcg_thin_svd(npcg_ctx* ctx, int64_t m, int64_t n, const double* b, double* u, double* s, int where) {
  return guard([&] {
    Ctx& c = C(ctx);
    if (m < n) invalid("thin_svd: expected a tall (m >= n) matrix");
    if (n <= 0) return;
    View B = view_in(c, b, m, n, m, where);
    DMat U;
    U.alloc(m, n, c.stream, false);
    DBuf<double> sig(n, c.stream);
    thin_svd(c, B.p, B.ld, m, n, U.p(), U.ld, sig.p);
    download(c, U.p(), U.ld, m, n, u, m, where);
    NPCG_CUDA(cudaMemcpyAsync(s, sig.p, sizeof(double) * n,
                              where == NPCG_HOST ? cudaMemcpyDeviceToHost : cudaMemcpyDeviceToDevice, c.stream));
    c.sync();
  });
}

}  // extern "C"
