// Device-resident (P)CG loop — restatement of pcg_loop (solvers.cpp:40-107)
// for S independent right-hand sides.
//
// Per iteration, on one stream, no host round trip:
//   v = A p + mu p                (operator kernel; dense: coldot with fused shift)
//   pv = p.v  -> alpha            (block partials + fixed-order final reduce)
//   x += alpha p; r -= alpha v; ||r||  -> convergence / divergence status
//   z = P^{-1} r                  (U^T r coldot, diag scale, r + U t rowdot)
//   rz' = r.z -> beta; p = z + beta p
// Scalars live in device memory; a converged / failed column freezes. The
// host keeps a few iterations in flight and stops enqueueing when a pinned
// snapshot of the status shows every column finished; iterations enqueued
// after that early-exit on a device flag (the matvec/preconditioner kernels
// read it first), so overshoot costs only empty launches.
#include <chrono>
#include <cmath>
#include <cstring>
#include <sstream>

#include "blas.cuh"
#include "pcg.cuh"

namespace npcg {
namespace {

constexpr int kMaxS = 8;
constexpr int kDepth = 3;  // iterations in flight ahead of the last observed status

struct ColState {
  double rz, pv, alpha, beta, res, eta, bnorm;
  int status;  // 0 running, 1 converged, 2 breakdown, 3 non-finite residual, 4 non-finite initial, 5 max_iter
  int iters;
};
struct State {
  int any_running;
  int pad;
  ColState c[kMaxS];
};

__device__ __forceinline__ double block_reduce_partials(const double* part, int nblk, int stride, int idx,
                                                        double* sh) {
  double v = 0.0;
  for (int b = threadIdx.x; b < nblk; b += blockDim.x) v += part[b * stride + idx];
  return block_sum(v, sh);
}

// r = b - v (v nullable), partials of ||b||^2, ||r||^2
__global__ void resid0_kernel(i64 n, int S, const double* __restrict__ B, i64 ldb, const double* __restrict__ V,
                              i64 ldv, double* __restrict__ R, i64 ldr, double* __restrict__ part) {
  __shared__ double sh[32];
  for (int s = 0; s < S; ++s) {
    double bb = 0.0, rr = 0.0;
    for (i64 i = static_cast<i64>(blockIdx.x) * blockDim.x + threadIdx.x; i < n;
         i += static_cast<i64>(gridDim.x) * blockDim.x) {
      const double b = B[i + s * ldb];
      const double r = V ? b - V[i + s * ldv] : b;
      R[i + s * ldr] = r;
      bb += b * b;
      rr += r * r;
    }
    bb = block_sum(bb, sh);
    rr = block_sum(rr, sh);
    if (threadIdx.x == 0) {
      part[blockIdx.x * 2 * S + 2 * s] = bb;
      part[blockIdx.x * 2 * S + 2 * s + 1] = rr;
    }
  }
}

__global__ void fin0_kernel(State* st, int S, const double* __restrict__ part, int nblk, double eta, int relative,
                            double* __restrict__ hist, i64 hstride) {
  __shared__ double sh[32];
  int running = 0;
  for (int s = 0; s < S; ++s) {
    const double bb = block_reduce_partials(part, nblk, 2 * S, 2 * s, sh);
    const double rr = block_reduce_partials(part, nblk, 2 * S, 2 * s + 1, sh);
    if (threadIdx.x == 0) {
      ColState& c = st->c[s];
      c.bnorm = sqrt(bb);
      c.eta = relative ? eta * c.bnorm : eta;
      c.res = sqrt(rr);
      c.iters = 0;
      hist[s * hstride] = c.res;
      if (!isfinite(c.res)) c.status = 4;
      else if (c.res <= c.eta) c.status = 1;
      else c.status = 0;
      running += c.status == 0;
    }
  }
  if (threadIdx.x == 0) st->any_running = running;
}

// partials of x_s . y_s for running columns; optional copy dst = y (p = z)
__global__ void dot_kernel(i64 n, int S, const double* __restrict__ X, i64 ldx, const double* __restrict__ Y, i64 ldy,
                           double* __restrict__ copy_dst, i64 ldc, const State* __restrict__ st,
                           double* __restrict__ part) {
  if (st->any_running == 0) return;
  __shared__ double sh[32];
  for (int s = 0; s < S; ++s) {
    const bool run = st->c[s].status == 0;
    double acc = 0.0;
    if (run) {
      for (i64 i = static_cast<i64>(blockIdx.x) * blockDim.x + threadIdx.x; i < n;
           i += static_cast<i64>(gridDim.x) * blockDim.x) {
        const double y = Y[i + s * ldy];
        acc += X[i + s * ldx] * y;
        if (copy_dst) copy_dst[i + s * ldc] = y;
      }
    }
    acc = block_sum(acc, sh);
    if (threadIdx.x == 0) part[blockIdx.x * S + s] = acc;
  }
}

// kind 0: rz = sum (init); 1: pv -> alpha (iteration t); 2: rz_next -> beta
__global__ void fin_dot_kernel(State* st, int S, const double* __restrict__ part, int nblk, int kind, int t) {
  if (st->any_running == 0) return;
  __shared__ double sh[32];
  int running = 0;
  for (int s = 0; s < S; ++s) {
    const double v = block_reduce_partials(part, nblk, S, s, sh);
    if (threadIdx.x == 0) {
      ColState& c = st->c[s];
      if (c.status == 0) {
        if (kind == 0) {
          c.rz = v;
        } else if (kind == 1) {
          c.pv = v;
          c.iters = t;
          if (!(v > 0.0) || !isfinite(v)) c.status = 2;  // solvers.cpp:76-81
          else c.alpha = c.rz / v;
        } else {
          c.beta = v / c.rz;
          c.rz = v;
        }
      }
      running += c.status == 0;
    }
  }
  if (threadIdx.x == 0) st->any_running = running;
}

// x += alpha p; r -= alpha v; partial ||r||^2
__global__ void update_kernel(i64 n, int S, double* __restrict__ X, i64 ldx, const double* __restrict__ P, i64 ldp,
                              const double* __restrict__ V, i64 ldv, double* __restrict__ R, i64 ldr,
                              const State* __restrict__ st, double* __restrict__ part) {
  if (st->any_running == 0) return;
  __shared__ double sh[32];
  for (int s = 0; s < S; ++s) {
    const bool run = st->c[s].status == 0;
    const double alpha = st->c[s].alpha;
    double acc = 0.0;
    if (run) {
      for (i64 i = static_cast<i64>(blockIdx.x) * blockDim.x + threadIdx.x; i < n;
           i += static_cast<i64>(gridDim.x) * blockDim.x) {
        X[i + s * ldx] += alpha * P[i + s * ldp];
        const double r = R[i + s * ldr] - alpha * V[i + s * ldv];
        R[i + s * ldr] = r;
        acc += r * r;
      }
    }
    acc = block_sum(acc, sh);
    if (threadIdx.x == 0) part[blockIdx.x * S + s] = acc;
  }
}

__global__ void fin_res_kernel(State* st, int S, const double* __restrict__ part, int nblk, int t, i64 max_iter,
                               double* __restrict__ hist, i64 hstride) {
  if (st->any_running == 0) return;
  __shared__ double sh[32];
  int running = 0;
  for (int s = 0; s < S; ++s) {
    const double v = block_reduce_partials(part, nblk, S, s, sh);
    if (threadIdx.x == 0) {
      ColState& c = st->c[s];
      if (c.status == 0) {
        c.res = sqrt(v);
        hist[s * hstride + t] = c.res;
        if (!isfinite(c.res)) c.status = 3;       // solvers.cpp:88-93
        else if (c.res <= c.eta) c.status = 1;    // :94-97
        else if (t >= max_iter) c.status = 5;
      }
      running += c.status == 0;
    }
  }
  if (threadIdx.x == 0) st->any_running = running;
}

// p = z + beta p
__global__ void pupdate_kernel(i64 n, int S, double* __restrict__ P, i64 ldp, const double* __restrict__ Z, i64 ldz,
                               const State* __restrict__ st) {
  if (st->any_running == 0) return;
  for (int s = 0; s < S; ++s) {
    if (st->c[s].status != 0) continue;
    const double beta = st->c[s].beta;
    for (i64 i = static_cast<i64>(blockIdx.x) * blockDim.x + threadIdx.x; i < n;
         i += static_cast<i64>(gridDim.x) * blockDim.x)
      P[i + s * ldp] = Z[i + s * ldz] + beta * P[i + s * ldp];
  }
}

__global__ void record_kernel(i64 n, int S, const double* __restrict__ X, i64 ldx, double* __restrict__ out,
                              const State* __restrict__ st, const int* __restrict__ running_at_start) {
  // out layout: [t][s][n]. Iteration records mirror solvers.cpp:60/97: every
  // column that entered the iteration, unless it broke down before updating x.
  for (int s = 0; s < S; ++s) {
    if (running_at_start && (!running_at_start[s] || st->c[s].status == 2)) continue;
    for (i64 i = static_cast<i64>(blockIdx.x) * blockDim.x + threadIdx.x; i < n;
         i += static_cast<i64>(gridDim.x) * blockDim.x)
      out[i + s * n] = X[i + s * ldx];
  }
}

__global__ void snapshot_running_kernel(const State* __restrict__ st, int S, int* __restrict__ flags) {
  const int s = threadIdx.x;
  if (s < S) flags[s] = st->c[s].status == 0 ? 1 : 0;
}

}  // namespace

PcgResult pcg_solve(Ctx& ctx, Op& op, Pre* pre, double mu, i64 S, const double* B, i64 ldb, const double* X0,
                    i64 ldx0, const PcgOptions& opt, double* X, i64 ldx, double* iterates, const char* context) {
  using Clock = std::chrono::steady_clock;
  const auto t0 = Clock::now();
  if (S < 1 || S > kMaxS) fail(NPCG_EINVAL, "pcg_solve: 1..8 right-hand sides per batch");
  const i64 n = op.n;
  const int nblk = static_cast<int>(std::max<i64>(1, std::min<i64>(cdiv(n, 2048), 2 * ctx.sm_count)));
  const i64 hstride = opt.max_iter + 1;
  DMat R, Z, P, V;
  R.alloc(n, S, ctx.stream, false);
  P.alloc(n, S, ctx.stream, false);
  V.alloc(n, S, ctx.stream, false);
  const bool identity = pre == nullptr || pre->ell == 0;
  if (!identity) Z.alloc(n, S, ctx.stream, false);
  double* Zp = identity ? R.p() : Z.p();
  const i64 ldz = identity ? R.ld : Z.ld;
  DBuf<State> st(1, ctx.stream);
  st.zero();
  DBuf<double> part(static_cast<i64>(nblk) * 2 * S, ctx.stream);
  DBuf<double> hist(S * hstride, ctx.stream);
  int* gate = &st.p->any_running;

  // x = x0 (or 0); r = b - A_mu x0 (solvers.cpp:52-53; A 0 = 0 is elided, matvec_count keeps the +1)
  if (X0) {
    copy2d(ctx, n, S, X0, ldx0, X, ldx);
    op.apply_shift(X, ldx, static_cast<int>(S), mu, V.p(), V.ld, nullptr);
    NPCG_LAUNCH(ctx, resid0_kernel, nblk, 256, 0, n, static_cast<int>(S), B, ldb, V.p(), V.ld, R.p(), R.ld, part.p);
  } else {
    NPCG_CUDA(cudaMemset2DAsync(X, ldx * 8, 0, n * 8, S, ctx.stream));
    NPCG_LAUNCH(ctx, resid0_kernel, nblk, 256, 0, n, static_cast<int>(S), B, ldb, static_cast<const double*>(nullptr),
                0, R.p(), R.ld, part.p);
  }
  NPCG_LAUNCH(ctx, fin0_kernel, 1, 256, 0, st.p, static_cast<int>(S), part.p, nblk, opt.eta, opt.relative ? 1 : 0,
              hist.p, hstride);
  DBuf<int> run_flags;
  if (iterates) {
    run_flags.alloc(S, ctx.stream);
    NPCG_LAUNCH(ctx, record_kernel, nblk, 256, 0, n, static_cast<int>(S), X, ldx, iterates, st.p,
                static_cast<const int*>(nullptr));
  }
  // z = P^{-1} r; p = z; rz = r.z
  if (!identity) pre_apply_inverse(*pre, R.p(), R.ld, S, Z.p(), Z.ld, gate);
  NPCG_LAUNCH(ctx, dot_kernel, nblk, 256, 0, n, static_cast<int>(S), R.p(), R.ld, Zp, ldz, P.p(), P.ld, st.p, part.p);
  NPCG_LAUNCH(ctx, fin_dot_kernel, 1, 256, 0, st.p, static_cast<int>(S), part.p, nblk, 0, 0);

  // pinned status snapshots, one per in-flight iteration
  State* snap = nullptr;
  NPCG_CUDA(cudaMallocHost(reinterpret_cast<void**>(&snap), sizeof(State) * (kDepth + 1)));
  cudaEvent_t ev[kDepth + 1];
  for (auto& e : ev) NPCG_CUDA(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
  struct Cleanup {
    State* snap;
    cudaEvent_t* ev;
    ~Cleanup() {
      for (int k = 0; k <= kDepth; ++k) cudaEventDestroy(ev[k]);
      cudaFreeHost(snap);
    }
  } cleanup{snap, ev};

  auto enqueue_snapshot = [&](i64 t) {
    const int slot = static_cast<int>(t % (kDepth + 1));
    NPCG_CUDA(cudaMemcpyAsync(&snap[slot], st.p, sizeof(State), cudaMemcpyDeviceToHost, ctx.stream));
    NPCG_CUDA(cudaEventRecord(ev[slot], ctx.stream));
  };
  auto finished = [&](i64 t) {
    const int slot = static_cast<int>(t % (kDepth + 1));
    NPCG_CUDA(cudaEventSynchronize(ev[slot]));
    return snap[slot].any_running == 0;
  };
  enqueue_snapshot(0);
  bool done = false;
  if (opt.max_iter == 0 || finished(0)) done = true;
  for (i64 t = 1; t <= opt.max_iter && !done; ++t) {
    if (iterates) NPCG_LAUNCH(ctx, snapshot_running_kernel, 1, 32, 0, st.p, static_cast<int>(S), run_flags.p);
    op.apply_shift(P.p(), P.ld, static_cast<int>(S), mu, V.p(), V.ld, gate);
    NPCG_LAUNCH(ctx, dot_kernel, nblk, 256, 0, n, static_cast<int>(S), P.p(), P.ld, V.p(), V.ld,
                static_cast<double*>(nullptr), 0, st.p, part.p);
    NPCG_LAUNCH(ctx, fin_dot_kernel, 1, 256, 0, st.p, static_cast<int>(S), part.p, nblk, 1, static_cast<int>(t));
    NPCG_LAUNCH(ctx, update_kernel, nblk, 256, 0, n, static_cast<int>(S), X, ldx, P.p(), P.ld, V.p(), V.ld, R.p(),
                R.ld, st.p, part.p);
    NPCG_LAUNCH(ctx, fin_res_kernel, 1, 256, 0, st.p, static_cast<int>(S), part.p, nblk, static_cast<int>(t),
                opt.max_iter, hist.p, hstride);
    if (iterates)
      NPCG_LAUNCH(ctx, record_kernel, nblk, 256, 0, n, static_cast<int>(S), X, ldx, iterates + t * n * S, st.p,
                  run_flags.p);
    if (!identity) pre_apply_inverse(*pre, R.p(), R.ld, S, Z.p(), Z.ld, gate);
    NPCG_LAUNCH(ctx, dot_kernel, nblk, 256, 0, n, static_cast<int>(S), R.p(), R.ld, Zp, ldz,
                static_cast<double*>(nullptr), 0, st.p, part.p);
    NPCG_LAUNCH(ctx, fin_dot_kernel, 1, 256, 0, st.p, static_cast<int>(S), part.p, nblk, 2, static_cast<int>(t));
    NPCG_LAUNCH(ctx, pupdate_kernel, nblk, 256, 0, n, static_cast<int>(S), P.p(), P.ld, Zp, ldz, st.p);
    enqueue_snapshot(t);
    if (t > kDepth && finished(t - kDepth)) done = true;
  }
  ctx.sync();

  State h;
  NPCG_CUDA(cudaMemcpy(&h, st.p, sizeof(State), cudaMemcpyDeviceToHost));
  std::vector<double> hh(static_cast<size_t>(S * hstride));
  NPCG_CUDA(cudaMemcpy(hh.data(), hist.p, sizeof(double) * hh.size(), cudaMemcpyDeviceToHost));
  PcgResult res;
  res.cols.resize(static_cast<size_t>(S));
  std::ostringstream msg;
  for (i64 s = 0; s < S; ++s) {
    const ColState& c = h.c[s];
    PcgColumnReport& r = res.cols[static_cast<size_t>(s)];
    r.iterations = c.iters;
    r.matvec_count = c.iters + 1;
    r.converged = c.status == 1;
    r.eta_used = c.eta;
    r.status = c.status == 2 ? 1 : c.status == 3 ? 2 : c.status == 4 ? 3 : 0;
    const i64 len = c.status == 4 ? 1 : (c.status == 2 ? c.iters : c.iters + 1);
    r.history.assign(hh.begin() + s * hstride, hh.begin() + s * hstride + len);
    if (r.status != 0) {
      res.diverged = true;
      if (r.status == 1)
        msg << context << ": breakdown at iteration " << c.iters << " (p'Ap = " << c.pv << ")";
      else if (r.status == 2)
        msg << context << ": non-finite residual at iteration " << c.iters;
      else
        msg << context << ": non-finite initial residual";
    }
  }
  res.message = msg.str();
  res.wall_time = std::chrono::duration<double>(Clock::now() - t0).count();
  return res;
}

}  // namespace npcg
