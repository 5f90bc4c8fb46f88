// Single-pass ridge Gram matvec (GramRidgeOperator::do_matvec,
// operators.cpp:112-116): out = X^T (X v) / m (+ mu v), reading X once.
//
// X is kept row-major on the device (each data row x_a contiguous), so a CTA
// streams whole rows: for row a it forms s_a = x_a . v (warp shuffles, one
// barrier) and adds s_a x_a into per-thread accumulators while the row is
// still in registers; the next row is already in flight. Every CTA owns a
// contiguous block of rows and emits one n-vector partial; a second kernel
// sums the partials in fixed order and applies /m (+ mu v).
// Algorithmic bytes: 8 m n per matvec (the reference's two GEMVs read X twice).
#include <algorithm>
#include <cstdlib>
#include <vector>

#include "blas.cuh"
#include "gemm.cuh"
#include "ops.cuh"

namespace npcg {
namespace {

constexpr int GT = 256;   // threads per CTA
constexpr int GV = 8;     // double2 column slots per thread -> n <= 2*GT*GV = 4096 per pass

template <int S>
__global__ void __launch_bounds__(GT) gram_pass_kernel(const double* __restrict__ Xr, i64 ldr, i64 m, i64 n,
                                                       i64 col0, const double* __restrict__ V, i64 ldv,
                                                       i64 rows_per_cta, double* __restrict__ partial,
                                                       const int* __restrict__ gate) {
  if (gate && *gate == 0) return;
  __shared__ double red[2][GT / 32][S];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const i64 a0 = static_cast<i64>(blockIdx.x) * rows_per_cta;
  const i64 a1 = min(m, a0 + rows_per_cta);
  // this thread's columns: col0 + 2*(tid + GT*k) + {0,1}
  double2 v[S][GV];
  double2 acc[S][GV];
  bool ok[GV];
#pragma unroll
  for (int k = 0; k < GV; ++k) {
    const i64 j = col0 + 2 * (tid + static_cast<i64>(GT) * k);
    ok[k] = j < n;
#pragma unroll
    for (int s = 0; s < S; ++s) {
      const double* vs = V + s * ldv;
      v[s][k] = make_double2(j < n ? vs[j] : 0.0, j + 1 < n ? vs[j + 1] : 0.0);
      acc[s][k] = make_double2(0.0, 0.0);
    }
  }
  double2 cur[GV], nxt[GV];
  auto load_row = [&](i64 a, double2* dst) {
    const double* row = Xr + a * ldr + col0;
#pragma unroll
    for (int k = 0; k < GV; ++k)
      dst[k] = ok[k] ? __ldcs(reinterpret_cast<const double2*>(row + 2 * (tid + GT * k))) : make_double2(0.0, 0.0);
  };
  if (a0 < a1) load_row(a0, cur);
  int par = 0;
  for (i64 a = a0; a < a1; ++a) {
    if (a + 1 < a1) load_row(a + 1, nxt);
    double part[S];
#pragma unroll
    for (int s = 0; s < S; ++s) {
      double t = 0.0;
#pragma unroll
      for (int k = 0; k < GV; ++k) t += cur[k].x * v[s][k].x + cur[k].y * v[s][k].y;
      part[s] = warp_sum(t);
    }
    if (lane == 0)
#pragma unroll
      for (int s = 0; s < S; ++s) red[par][warp][s] = part[s];
    __syncthreads();
#pragma unroll
    for (int s = 0; s < S; ++s) {
      double sa = 0.0;
#pragma unroll
      for (int w = 0; w < GT / 32; ++w) sa += red[par][w][s];
#pragma unroll
      for (int k = 0; k < GV; ++k) {
        acc[s][k].x += sa * cur[k].x;
        acc[s][k].y += sa * cur[k].y;
      }
    }
    par ^= 1;
#pragma unroll
    for (int k = 0; k < GV; ++k) cur[k] = nxt[k];
  }
  // partial[cta][s][col] (col relative to col0, width 2*GT*GV)
  const i64 width = 2 * GT * GV;
#pragma unroll
  for (int s = 0; s < S; ++s) {
    double* dst = partial + (static_cast<i64>(blockIdx.x) * S + s) * width;
#pragma unroll
    for (int k = 0; k < GV; ++k) reinterpret_cast<double2*>(dst)[tid + GT * k] = acc[s][k];
  }
}

__global__ void gram_finish_kernel(const double* __restrict__ partial, int nparts, int S, i64 n, i64 col0,
                                   double inv_m_div, double mu, const double* __restrict__ P, i64 ldp,
                                   double* __restrict__ out, i64 ldo, const int* __restrict__ gate) {
  if (gate && *gate == 0) return;
  const i64 width = 2 * GT * GV;
  const i64 idx = static_cast<i64>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (idx >= width * S) return;
  const i64 c = idx % width, s = idx / width;
  const i64 j = col0 + c;
  if (j >= n) return;
  double t = 0.0;
  for (int b = 0; b < nparts; ++b) t += partial[(static_cast<i64>(b) * S + s) * width + c];
  double o = t / inv_m_div;  // out /= n_rows (operators.cpp:115: division)
  if (P) o = __dadd_rn(o, __dmul_rn(mu, P[j + s * ldp]));  // out += mu v, unfused
  out[j + s * ldo] = o;
}

template <int S>
void gram_single_pass(Ctx& ctx, const GramOp& op, const double* V, i64 ldv, double mu, const double* P, i64 ldp,
                      double* out, i64 ldo, const int* gate) {
  int per_sm = 0;
  NPCG_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, gram_pass_kernel<S>, GT, 0));
  const i64 nct = std::max<i64>(1, std::min<i64>(op.m, static_cast<i64>(std::max(per_sm, 1)) * ctx.sm_count));
  const i64 rpc = cdiv(op.m, nct);
  const int parts = static_cast<int>(cdiv(op.m, rpc));
  const i64 width = 2 * GT * GV;
  DBuf<double> part(static_cast<i64>(parts) * S * width, ctx.stream);
  for (i64 col0 = 0; col0 < op.n; col0 += width) {
    NPCG_LAUNCH(ctx, gram_pass_kernel<S>, parts, GT, 0, op.xr.p(), op.xr.ld, op.m, op.n, col0, V, ldv, rpc, part.p,
                gate);
    ctx.prof_work(4.0 * op.m * std::min(width, op.n - col0) * S, 8.0 * op.m * std::min(width, op.n - col0));
    NPCG_LAUNCH(ctx, gram_finish_kernel, static_cast<unsigned>(cdiv(width * S, 256)), 256, 0, part.p, parts, S,
                op.n, col0, op.div, mu, P, ldp, out, ldo, gate);
  }
}

}  // namespace

// GramRidgeOperator: out = X^T (X V) / m.
namespace {
// Host design (m x n, ld ldg) -> op.xr through a staging ring of NSLOT row
// blocks: block b crosses PCIe into slot b % NSLOT on the copy stream while
// earlier blocks are transposed (and checked for non-finite entries into
// *bad) on the transpose stream. Device memory: xr plus NSLOT ~80 MB blocks
// (the synchronous constructor; 11.7 ms for cfg 2's 640 MB, the PCIe rate). `ready` receives one
// event per block, recorded on the transpose stream after its transpose.
void upload_blocks(Ctx& c, GramOp& op, const double* g, i64 ldg, int* bad, std::vector<GramOp::Chunk>& ready) {
  const i64 m = op.m, n = op.n;
  cudaStream_t cp = c.aux_stream(), tr = c.aux2_stream();
  cudaEvent_t start;
  NPCG_CUDA(cudaEventCreateWithFlags(&start, cudaEventDisableTiming));
  NPCG_CUDA(cudaEventRecord(start, c.stream));  // xr, its pads and *bad are ready on the context stream
  NPCG_CUDA(cudaStreamWaitEvent(cp, start, 0));
  NPCG_CUDA(cudaStreamWaitEvent(tr, start, 0));
  NPCG_CUDA(cudaEventDestroy(start));
  i64 rows = std::max<i64>(1024, (80ll << 20) / (8 * n) / 128 * 128);
  if (const char* e = std::getenv("NPCG_STREAM_ROWS")) rows = std::max<i64>(16, std::atoll(e) / 16 * 16);  // tests
  rows = std::min(rows, m);
  constexpr int NSLOT = Ctx::kStageSlots;
  const i64 sld = dev_ld(rows), slot_elems = sld * n;
  if (c.stage_slot < slot_elems) {  // (re)allocate the context's ring; earlier uploads must have drained it
    NPCG_CUDA(cudaStreamSynchronize(cp));
    NPCG_CUDA(cudaStreamSynchronize(tr));
    if (c.stage) NPCG_CUDA(cudaFree(c.stage));
    c.stage = nullptr;
    c.stage_slot = 0;
    NPCG_CUDA(cudaMalloc(reinterpret_cast<void**>(&c.stage), sizeof(double) * slot_elems * NSLOT));
    c.stage_slot = slot_elems;
    for (auto& ev : c.stage_free)
      if (ev) {
        cudaEventDestroy(ev);
        ev = nullptr;
      }
  }
  cudaEvent_t copied;
  NPCG_CUDA(cudaEventCreateWithFlags(&copied, cudaEventDisableTiming));
  int blk = 0;
  for (i64 r0 = 0; r0 < m; r0 += rows, ++blk) {
    const i64 r1 = std::min(m, r0 + rows);
    const int q = blk % NSLOT;
    double* slot = c.stage + q * c.stage_slot;
    if (c.stage_free[q]) NPCG_CUDA(cudaStreamWaitEvent(cp, c.stage_free[q], 0));  // the slot's last block is transposed
    else NPCG_CUDA(cudaEventCreateWithFlags(&c.stage_free[q], cudaEventDisableTiming));
    NPCG_CUDA(cudaMemcpy2DAsync(slot, sld * 8, g + r0, ldg * 8, (r1 - r0) * 8, n, cudaMemcpyHostToDevice, cp));
    NPCG_CUDA(cudaEventRecord(copied, cp));
    NPCG_CUDA(cudaStreamWaitEvent(tr, copied, 0));
    transpose_checked(c, tr, slot, sld, r1 - r0, n, op.xr.p() + r0 * op.xr.ld, op.xr.ld, bad);
    NPCG_CUDA(cudaEventRecord(c.stage_free[q], tr));
    GramOp::Chunk ch{r0, r1, nullptr, nullptr};
    NPCG_CUDA(cudaEventCreateWithFlags(&ch.ready, cudaEventDisableTiming));
    NPCG_CUDA(cudaEventRecord(ch.ready, tr));
    ready.push_back(ch);
  }
  NPCG_CUDA(cudaEventDestroy(copied));
}

void alloc_xr(Ctx& c, GramOp& op) {
  op.xr.alloc(op.n, op.m, c.stream, false);
  if (op.xr.ld > op.n)  // pad rows of the row-major copy
    NPCG_CUDA(cudaMemset2DAsync(op.xr.p() + op.n, op.xr.ld * 8, 0, (op.xr.ld - op.n) * 8, op.m, c.stream));
}
}  // namespace

void gram_upload(Ctx& c, GramOp& op, const double* g, i64 ldg, int where) {
  const i64 m = op.m, n = op.n;
  if (ldg < m) invalid("leading dimension smaller than the row count");
  alloc_xr(c, op);
  DBuf<int> flag(1, c.stream);
  flag.zero();
  if (where == NPCG_HOST) {
    std::vector<GramOp::Chunk> blocks;
    upload_blocks(c, op, g, ldg, flag.p, blocks);
    for (auto& ch : blocks) {
      NPCG_CUDA(cudaStreamWaitEvent(c.stream, ch.ready, 0));
      cudaEventDestroy(ch.ready);
    }
  } else {
    transpose_checked(c, c.stream, g, ldg, m, n, op.xr.p(), op.xr.ld, flag.p);
  }
  int h = 0;
  NPCG_CUDA(cudaMemcpyAsync(&h, flag.p, sizeof(int), cudaMemcpyDeviceToHost, c.stream));
  c.sync();
  if (h) invalid("GramRidgeOperator: design matrix has non-finite entries");  // operators.cpp:108-109
}

void gram_upload_streamed(Ctx& c, GramOp& op, const double* g, i64 ldg) {
  // The whole design is staged in the caller's layout; the sketch GEMMs run on
  // each landed block directly (they wait for its copy only), the transposes
  // into xr follow each copy, and only settle() waits for them.
  const i64 m = op.m, n = op.n;
  alloc_xr(c, op);
  op.stage.alloc(m, n, c.stream, false);
  op.bad.alloc(1, c.stream);
  op.bad.zero();
  // transposes on the copy stream itself: measured 20.1 vs 24.6 ms per e2e
  // solve against a separate transpose stream (either priority)
  cudaStream_t cp = c.aux_stream(), tr = cp;
  cudaEvent_t start;
  NPCG_CUDA(cudaEventCreateWithFlags(&start, cudaEventDisableTiming));
  NPCG_CUDA(cudaEventRecord(start, c.stream));
  NPCG_CUDA(cudaStreamWaitEvent(cp, start, 0));
  NPCG_CUDA(cudaStreamWaitEvent(tr, start, 0));
  NPCG_CUDA(cudaEventDestroy(start));
  i64 rows = std::max<i64>(1024, (80ll << 20) / (8 * n) / 128 * 128);
  if (const char* e = std::getenv("NPCG_STREAM_ROWS")) rows = std::max<i64>(16, std::atoll(e) / 16 * 16);  // tests
  for (i64 r0 = 0; r0 < m; r0 += rows) {
    const i64 r1 = std::min(m, r0 + rows);
    GramOp::Chunk ch{r0, r1, nullptr, nullptr};
    NPCG_CUDA(cudaEventCreateWithFlags(&ch.copied, cudaEventDisableTiming));
    NPCG_CUDA(cudaEventCreateWithFlags(&ch.ready, cudaEventDisableTiming));
    NPCG_CUDA(cudaMemcpy2DAsync(op.stage.p() + r0, op.stage.ld * 8, g + r0, ldg * 8, (r1 - r0) * 8, n,
                                cudaMemcpyHostToDevice, cp));
    NPCG_CUDA(cudaEventRecord(ch.copied, cp));
    NPCG_CUDA(cudaStreamWaitEvent(tr, ch.copied, 0));
    transpose_checked(c, tr, op.stage.p() + r0, op.stage.ld, r1 - r0, n, op.xr.p() + r0 * op.xr.ld, op.xr.ld,
                      op.bad.p);
    NPCG_CUDA(cudaEventRecord(ch.ready, tr));
    op.pending.push_back(ch);
  }
}

void GramOp::settle() {
  if (nonfinite) invalid("GramRidgeOperator: design matrix has non-finite entries");
  if (pending.empty()) return;
  for (auto& ch : pending) NPCG_CUDA(cudaStreamWaitEvent(ctx->stream, ch.ready, 0));
  NPCG_CUDA(cudaEventSynchronize(pending.back().ready));
  for (auto& ch : pending) {
    cudaEventDestroy(ch.copied);
    cudaEventDestroy(ch.ready);
  }
  pending.clear();
  stage.buf.release();  // freed on the context stream, which has waited for every transpose
  NPCG_CUDA(cudaMemcpy(&nonfinite, bad.p, sizeof(int), cudaMemcpyDeviceToHost));
  if (nonfinite) invalid("GramRidgeOperator: design matrix has non-finite entries");  // operators.cpp:108-109
}

GramOp::~GramOp() {
  // the side stream may still write xr / read the caller's buffer
  for (auto& ch : pending) {
    cudaStreamWaitEvent(ctx->stream, ch.ready, 0);
    cudaEventSynchronize(ch.ready);
    cudaEventDestroy(ch.copied);
    cudaEventDestroy(ch.ready);
  }
}

void GramOp::apply(const double* V, i64 ldv, i64 k, double* out, i64 ldo, const int* gate) {
  if (!pending.empty() && k > 8) {
    // first product of a streamed operator (the sketch): block by block as
    // the rows land, Z_b = X_b V and out (+)= X_b^T Z_b in fixed block order
    DMat z;
    z.alloc(m, k, ctx->stream, false);
    for (size_t b = 0; b < pending.size(); ++b) {
      const Chunk& ch = pending[b];
      NPCG_CUDA(cudaStreamWaitEvent(ctx->stream, ch.copied, 0));
      const i64 rb = ch.r1 - ch.r0;
      const double* xb = stage.p() + ch.r0;  // the landed block, caller layout (rb x n, ld m)
      gemm(*ctx, rb, k, n, 1.0, Operand{xb, stage.ld, false}, Operand{V, ldv, true}, 0.0, z.p() + ch.r0, z.ld);
      gemm(*ctx, n, k, rb, 1.0, Operand{xb, stage.ld, true}, Operand{z.p() + ch.r0, z.ld, true}, b ? 1.0 : 0.0,
           out, ldo);
    }
    settle();
    divide(*ctx, n, k, out, ldo, div);
    return;
  }
  settle();
  if (k == 1 && n <= 2 * GT * GV) {
    gram_single_pass<1>(*ctx, *this, V, ldv, 0.0, nullptr, 0, out, ldo, gate);
    return;
  }
  if (k == 2 && n <= 2 * GT * GV) {
    gram_single_pass<2>(*ctx, *this, V, ldv, 0.0, nullptr, 0, out, ldo, gate);
    return;
  }
  DMat z;
  z.alloc(m, k, ctx->stream, false);
  if (k <= 8) {  // two-pass skinny GEMVs on the row-major copy
    coldot(*ctx, xr.p(), xr.ld, n, m, V, ldv, static_cast<int>(k), z.p(), z.ld, 0.0, nullptr, 0, gate);
    rowdot(*ctx, xr.p(), xr.ld, n, m, z.p(), z.ld, static_cast<int>(k), nullptr, 0, out, ldo, gate);
  } else {  // sketch-sized blocks: two DMMA GEMMs
    gemm(*ctx, m, k, n, 1.0, Operand{xr.p(), xr.ld, true}, Operand{V, ldv, true}, 0.0, z.p(), z.ld);
    gemm(*ctx, n, k, m, 1.0, Operand{xr.p(), xr.ld, false}, Operand{z.p(), z.ld, true}, 0.0, out, ldo);
  }
  divide(*ctx, n, k, out, ldo, div);
}

void GramOp::apply_shift(const double* P, i64 ldp, int S, double mu, double* out, i64 ldo, const int* gate) {
  settle();
  if (S == 1 && n <= 2 * GT * GV) {
    gram_single_pass<1>(*ctx, *this, P, ldp, mu, P, ldp, out, ldo, gate);
    return;
  }
  if (S == 2 && n <= 2 * GT * GV) {
    gram_single_pass<2>(*ctx, *this, P, ldp, mu, P, ldp, out, ldo, gate);
    return;
  }
  Op::apply_shift(P, ldp, S, mu, out, ldo, gate);
}

}  // namespace npcg
