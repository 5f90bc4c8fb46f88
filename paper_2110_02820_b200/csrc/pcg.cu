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
#include <cooperative_groups.h>

#include <algorithm>
#include <chrono>
#include <vector>
#include <cstdio>
#include <cstdlib>
#include <cmath>
#include <cstring>
#include <sstream>
#include <string>

#include "async.cuh"
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

// Row-sharded contexts: this rank's sum of the per-block partials (fixed
// order), all-reduced over the ranks before the fin_* kernel reads it as a
// single block.
__global__ void rank_partials_kernel(const double* __restrict__ part, int nblk, int stride, double* __restrict__ out) {
  const int idx = threadIdx.x;
  if (idx >= stride) return;
  double v = 0.0;
  for (int b = 0; b < nblk; ++b) v += part[b * stride + idx];
  out[idx] = v;
}

__global__ void snapshot_running_kernel(const State* __restrict__ st, int S, int* __restrict__ flags) {
  const int s = threadIdx.x;
  if (s < S) flags[s] = st->c[s].status == 0 ? 1 : 0;
}

// ============================================================================
// Persistent PCG loop: one cooperative launch runs every iteration, one CTA
// per SM, grid-wide barriers between the phases of an iteration. Every CTA
// keeps an identical copy of the column states: the scalars (p.v, ||r||^2,
// r.z) are reduced from per-CTA partials in the same fixed order by every
// CTA, so all CTAs take the same branch (converged / breakdown / max_iter)
// without a broadcast. The loop stops on the device when no column runs.
//
// Iteration t (vector slices: CTA c owns entries [c*slice, (c+1)*slice)):
//   P1  p_t = z + beta p_{t-1} (ping-pong buffers; each CTA recomputes what
//       it needs, the slice owner stores it); v = A p_t:
//         gram:  CTA c streams its rows of X once: partial_c = X_c^T (X_c p)
//         dense: CTA c computes (A p)_j for the columns j of its slice
//   P2  gram: v_j = (sum_c partial_c)_j / m + mu p_j for the slice (fixed
//       order over c); partial p.v of the slice                  | barrier
//   P3  alpha = rz / p.v; x += alpha p, r -= alpha v; partial ||r||^2 | barrier
//   P4  ||r|| -> history / status; identity P: beta = ||r||^2 / rz
//       Nystrom P: t = gain * (U^T r) for CTA c's columns of U   | barrier
//   P5  z = r + U t for the slice; partial r.z                   | barrier
//       beta = r.z / rz (next iteration's P1)
// ============================================================================
constexpr int PT = 512;  // threads per CTA
constexpr int PV = 4;    // double2 slots per thread in the gram row pass: n <= 2*PT*PV
constexpr int PW = 2 * PT * PV;
constexpr int NST = 6;   // shared-memory ring stages of one PW-double segment (a row of X / a column segment of A)
constexpr int RING_BYTES = NST * PW * 8;
// dense path: row-block width per CTA (3-4 right-hand sides use half-width
// blocks: 2 double2 slots per thread keep the accumulators in registers) and
// ring depth (the same bytes in flight)
constexpr int dense_pv(int S) { return S >= 3 ? 1 : PV; }  // 3-4 RHS: 1024-row blocks for the DMMA path
// DMMA symmetric path (3-4 right-hand sides): 24 slots of 1024 rows + a 16-byte pad
constexpr int MDNST = 24, MSLOT = 1024 + 2;
// preconditioner passes of the DMMA path (P4 / P5): 3 chunk slots of 16 column segments of up to 512 rows
constexpr int UCH = 512, USEG = UCH + 2, UNSEG = 16, UNCH = 3;
constexpr int ring_bytes(bool gram, int S) {
  const int chunk = UNCH * UNSEG * USEG * 8;  // P4 / P5 chunk slots (every dense instance)
  const int p1 = (!gram && S >= 3) ? MDNST * MSLOT * 8 : RING_BYTES;
  return gram ? RING_BYTES : (p1 > chunk ? p1 : chunk);
}
constexpr int dense_pw(int S) { return 2 * PT * dense_pv(S); }
constexpr int dense_nst(int S) { return RING_BYTES / (dense_pw(S) * 8); }

__device__ __forceinline__ void pcg_dmma(double& c0, double& c1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
               : "+d"(c0), "+d"(c1)
               : "d"(a), "d"(b));
}

struct PersistArgs {
  i64 n, m;
  const double* A;
  i64 lda;  // gram: X row-major (row a at A + a*lda); dense: n x n col-major
  double mus[8], div;  // the shift of each column (one value repeated unless the batch spans several mu)
  const double* U;
  i64 ldu, ell;
  const double* gain;  // column s uses gain[s*gstride + j] (gstride = 0: one preconditioner for all columns)
  i64 gstride;
  double* X;
  i64 ldx;
  double *R, *Z, *P0, *P1, *V;
  i64 ldw;
  double* T;
  double* part;                       // gram: G x PW; dense: ncb x S x pstride
  i64 nrb, ncb, cpb, pstride;         // dense: row blocks of PW rows, column blocks of cpb columns
  // dense, symmetric use of A (sym != 0): CTA c streams row block unit_rb[c],
  // columns [unit_j0[c], unit_j1[c]) of the block-upper part; row sums go to
  // part[(c*S + s)*DPW + local row], column dots to colpart[(rb*S + s)*pstride + j]
  int sym;
  const i64* unit;                    // segments x 3: rb, j0, j1 (row-major order)
  const int* cseg;                    // G + 1: first segment of each CTA
  const int* ustart;                  // nrb + 1: first segment of each row block
  double* colpart;
  double* pil;                        // dense symmetric: p_t column-interleaved, entry (j, s) at j*SP + s
  double *pv_part, *rr_part, *rz_part;  // G x S
  State* st;
  double* hist;
  i64 hstride, max_iter, rows_per_cta, slice, uslice;
  unsigned* gbar;             // grid barrier counter (zero at launch)
  int pre_dmma;               // dense: P4 / P5 on the DMMA pipe from bulk-copied chunk slots (3+ columns, or large n x ell)
  unsigned long long* trace;  // diagnostics (NPCG_PCG_TRACE): CTA 0 phase timestamps of iterations 2..9
};

template <int S, bool GRAM>
__global__ void __launch_bounds__(PT, 1) pcg_persistent_kernel(const PersistArgs a) {
  // Grid barrier (the launch is cooperative: all CTAs are resident): thread 0
  // counts the CTA in on a monotone global counter and spins until the
  // barrier's generation is complete; the warp reconverges before the closing
  // block barrier, so warp 0 arrives there once, as a whole.
  unsigned grid_gen = 0;
  struct GridBarrier {
    unsigned* counter;
    unsigned& gen;
    unsigned ctas;
    __device__ __forceinline__ void sync() {
      __syncwarp();
      __syncthreads();
      ++gen;
      if (threadIdx.x == 0) {
        __threadfence();
        atomicAdd(counter, 1u);
        const unsigned target = gen * ctas;
        unsigned seen;
        do {
          asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(seen) : "l"(counter) : "memory");
        } while (seen < target);
        __threadfence();
      }
      __syncwarp();
      __syncthreads();
    }
  } grid{a.gbar, grid_gen, gridDim.x};
  __shared__ double sh[32];
  __shared__ double red[2][PT / 32], red2[2][PT / 32];
  // P2/P5 cross-warp staging (S x 16 x 32); the DMMA loop's per-step column dots alias it
  // (P5 stages at most ZS = 4 right-hand sides per round: 5-8 take two rounds, the ring leaves no room for more)
  constexpr int ZS = S < 4 ? S : 4;
  __shared__ double zbuf[(ZS * (PT / 32) * 32) > (!GRAM ? (S >= 3 ? 2 : 1) * (PT / 32) * 64 : 0)
                             ? ZS * (PT / 32) * 32 : (S >= 3 ? 2 : 1) * (PT / 32) * 64];
  constexpr int UQ = S > 4 ? 2 : 4;  // P4: columns of U per pass (4 x 8 accumulators measured slower: 1035 vs 835 us at n = 1e5, ell = 2000)
  __shared__ double wred[UQ * S * (PT / 32)];  // P4: per-warp partials of up to UQ x S dots
  __shared__ ColState cs[S];
  __shared__ int running_sh;
  constexpr int DPV = GRAM ? PV : dense_pv(S), DPW = 2 * PT * DPV, DNST = GRAM ? NST : dense_nst(S);
  __shared__ uint64_t full_bar[DNST > MDNST ? DNST : MDNST];
  __shared__ uint64_t chunk_bar[UNCH];  // P4 / P5 of the DMMA path: one barrier per chunk slot
  // dense symmetric use: p_t entries of the slots' columns, per-step warp
  // partials of the 2S column dots (one set per slot pair), arrival counters
  constexpr int SP = (S + 1) / 2 * 2;  // p entries per column, padded to 16 bytes
  constexpr bool DEC = !GRAM && S == 1;  // the decoupled symmetric loop (one right-hand side)
  constexpr bool MMA = !GRAM && S >= 3;  // the DMMA symmetric loop (3-4 right-hand sides)
  auto mdot = [&](int b, int w, int k) -> double& { return zbuf[(b * (PT / 32) + w) * 64 + k]; };
  __shared__ __align__(16) double pring[DEC ? DNST * SP : 2];
  __shared__ double sdot[DEC ? DNST / 2 : 1][PT / 32][DEC ? 2 * S : 1];
  __shared__ unsigned pair_cnt[DNST / 2];
  extern __shared__ __align__(128) double ring[];  // DNST x DPW doubles, fed by bulk copies (TMA)
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  uint32_t ring_head = 0, ring_tail = 0;  // segments consumed (all threads) / issued (thread 0)
  uint32_t chunk_seq = 0;                  // P4 / P5 chunk slots consumed (all threads)
  if (tid == 0) {
    for (int q = 0; q < (DNST > MDNST ? DNST : MDNST); ++q) mbarrier_init(&full_bar[q], 1);
    for (int q = 0; q < UNCH; ++q) mbarrier_init(&chunk_bar[q], 1);
    mbarrier_fence_init();
  }
  if (tid < DNST / 2) pair_cnt[tid] = 0u;
  auto ring_issue = [&](const double* src, i64 count) {  // thread 0 only
    const int slot = static_cast<int>(ring_tail % DNST);
    const uint32_t bytes = static_cast<uint32_t>(round_up(count, 2) * 8);
    mbarrier_expect_tx(&full_bar[slot], bytes);
    bulk_copy_g2s(ring + static_cast<i64>(slot) * DPW, src, bytes, &full_bar[slot]);
    ++ring_tail;
  };
  auto ring_wait = [&]() -> const double* {  // next segment, in issue order
    const int slot = static_cast<int>(ring_head % DNST);
    mbarrier_wait_parity(&full_bar[slot], (ring_head / DNST) & 1u);
    ++ring_head;
    return ring + static_cast<i64>(slot) * DPW;
  };
  const int G = gridDim.x, c = blockIdx.x;
  const i64 n = a.n;
  const i64 r0 = min(n, static_cast<i64>(c) * a.slice), r1 = min(n, r0 + a.slice);
  auto tick = [&](i64 t, int ph) {
    if (a.trace && c == 0 && tid == 0 && t >= 2 && t < 10) {
      unsigned long long v;
      asm volatile("mov.u64 %0, %globaltimer;" : "=l"(v));
      a.trace[(t - 2) * 12 + ph] = v;
    }
  };
  const bool nys = a.ell > 0;
  const double* zsrc = nys ? a.Z : a.R;

  if (tid < S) cs[tid] = a.st->c[tid];
  // this CTA's columns of U in P4 (shared memory is left to L1: a carve-out for
  // U slows the X stream of P1 more than it saves in P4/P5)
  const i64 u0 = nys ? min(a.ell, static_cast<i64>(c) * a.uslice) : 0, u1 = nys ? min(a.ell, u0 + a.uslice) : 0;
  __syncthreads();
  auto count_running = [&]() {
    int k = 0;
#pragma unroll
    for (int s = 0; s < S; ++s) k += cs[s].status == 0;
    return k;
  };
  // sum over CTAs of part[b*S + s] in fixed order (identical in every CTA)
  auto all_sum = [&](const double* part, int s) {
    double v = 0.0;
    for (int b = tid; b < G; b += PT) v += part[b * S + s];
    return block_sum(v, sh);
  };

  if (count_running() > 0) {
    for (i64 t = 1; t <= a.max_iter; ++t) {
      const double* pold = (t & 1) ? a.P1 : a.P0;  // p_{t-1} (unused at t = 1)
      double* pcur = (t & 1) ? a.P0 : a.P1;         // p_t
      const bool first = t == 1;
      // p_t entry (i, s): z + beta p_{t-1} for running columns, else unchanged
      auto p_at = [&](i64 i, int s) -> double {
        if (first) return pcur[i + s * a.ldw];
        const double po = pold[i + s * a.ldw];
        return cs[s].status == 0 ? zsrc[i + s * a.ldw] + cs[s].beta * po : po;
      };
      // ---- P1
      tick(t, 0);
      if (!first || a.pil)
        for (i64 i = r0 + tid; i < r1; i += PT)
#pragma unroll
          for (int s = 0; s < S; ++s) {
            const double v = p_at(i, s);
            if (!first) pcur[i + s * a.ldw] = v;
            if (a.pil) a.pil[i * SP + s] = v;  // column-interleaved copy: the ring's p entries
          }
      if constexpr (!GRAM) {
        if (!first || a.pil) grid.sync();  // dense streams p_t from pcur / pil
      }
      if constexpr (GRAM) {
        static_assert(S == 1, "gram persistent path is single right-hand side");
        double2 pv[PV], acc[PV], cur[PV], nxt[PV];
        bool ok[PV];
#pragma unroll
        for (int k = 0; k < PV; ++k) {
          const i64 j = 2 * (tid + static_cast<i64>(PT) * k);
          ok[k] = j < n;
          pv[k] = make_double2(j < n ? p_at(j, 0) : 0.0, j + 1 < n ? p_at(j + 1, 0) : 0.0);
          acc[k] = make_double2(0.0, 0.0);
        }
        const i64 a0 = static_cast<i64>(c) * a.rows_per_cta, a1 = min(a.m, a0 + a.rows_per_cta);
        auto load_row = [&](i64 row, double2* dst) {
          const double* x = a.A + row * a.lda;
#pragma unroll
          for (int k = 0; k < PV; ++k)
            dst[k] = (ok[k] && row < a1) ? __ldcs(reinterpret_cast<const double2*>(x + 2 * (tid + PT * k)))
                                         : make_double2(0.0, 0.0);
        };
        // two rows per step (one barrier per pair), the next pair in flight
        double2 cur2[PV], nxt2[PV];
        load_row(a0, cur);
        load_row(a0 + 1, cur2);
        int par = 0;
        for (i64 row = a0; row < a1; row += 2) {
          load_row(row + 2, nxt);
          load_row(row + 3, nxt2);
          double d = 0.0, d2 = 0.0;
#pragma unroll
          for (int k = 0; k < PV; ++k) {
            d += cur[k].x * pv[k].x + cur[k].y * pv[k].y;
            d2 += cur2[k].x * pv[k].x + cur2[k].y * pv[k].y;
          }
#pragma unroll
          for (int o = 16; o > 0; o >>= 1) {
            d += __shfl_xor_sync(0xffffffffu, d, o);
            d2 += __shfl_xor_sync(0xffffffffu, d2, o);
          }
          if (lane == 0) {
            red[par][warp] = d;
            red2[par][warp] = d2;
          }
          __syncthreads();
          double sa0 = 0.0, sa1 = 0.0, sb0 = 0.0, sb1 = 0.0;  // fixed pairing: identical in every thread
#pragma unroll
          for (int w = 0; w < PT / 32; w += 2) {
            sa0 += red[par][w];
            sa1 += red[par][w + 1];
            sb0 += red2[par][w];
            sb1 += red2[par][w + 1];
          }
          const double sa = sa0 + sa1, sb = sb0 + sb1;
#pragma unroll
          for (int k = 0; k < PV; ++k) {
            acc[k].x += sa * cur[k].x;
            acc[k].y += sa * cur[k].y;
            acc[k].x += sb * cur2[k].x;
            acc[k].y += sb * cur2[k].y;
          }
          par ^= 1;
#pragma unroll
          for (int k = 0; k < PV; ++k) {
            cur[k] = nxt[k];
            cur2[k] = nxt2[k];
          }
        }
        double* dst = a.part + static_cast<i64>(c) * PW;
#pragma unroll
        for (int k = 0; k < PV; ++k)
          if (ok[k]) reinterpret_cast<double2*>(dst)[tid + PT * k] = acc[k];
        tick(t, 1);
        grid.sync();
        tick(t, 2);
        // ---- P2: column slice of v, partial p.v. Lanes run over the slice's
        // columns (coalesced rows of the partials), warps over the partials;
        // every load of a lane is independent, so one L2 round trip covers them
        double pvl = 0.0;
        for (i64 jb = r0; jb < r1; jb += 32) {
          const i64 j = jb + lane;
          double s0 = 0.0, s1 = 0.0;
          if (j < r1) {
            int b = warp;
#pragma unroll 4
            for (; b + PT / 32 < G; b += 2 * (PT / 32)) {
              s0 += a.part[static_cast<i64>(b) * PW + j];
              s1 += a.part[static_cast<i64>(b + PT / 32) * PW + j];
            }
            if (b < G) s0 += a.part[static_cast<i64>(b) * PW + j];
          }
          zbuf[warp * 32 + lane] = s0 + s1;
          __syncthreads();
          if (warp == 0 && j < r1) {
            double s = 0.0;
#pragma unroll
            for (int w = 0; w < PT / 32; ++w) s += zbuf[w * 32 + lane];  // fixed order
            const double pj = pcur[j];
            double v = s / a.div;  // operators.cpp:115 (division), then out += mu p
            v = __dadd_rn(v, __dmul_rn(a.mus[0], pj));  // out += mu p, unfused (solvers.cpp:139)
            a.V[j] = v;
            pvl += pj * v;
          }
          __syncthreads();
        }
        pvl = block_sum(pvl, sh);
        if (tid == 0) a.pv_part[c] = pvl;
        tick(t, 3);
      } else {
        // dense: v = A p_t streamed column by column (axpy form, A col-major):
        // CTA (rb, cb) owns rows [rb*DPW, +DPW) x columns [cb*cpb, +cpb); each
        // column segment is one contiguous bulk copy into the shared-memory
        // ring (DNST segments in flight); two columns per step, one block
        // barrier per step frees their slots. partial_cb = A[rows, cols_cb] p_t[cols_cb].
        // Symmetric use (a.sym): CTA c owns row block rb and columns [j0, j1) of
        // the block-upper part (j >= rb*DPW). A column segment beyond the
        // diagonal block is used twice: axpy into the rows of rb (A[R, j] p_j)
        // and a dot with p over those rows, which is (A p)_j's share from the
        // rows of rb (A[j, R] = A[R, j]^T): half of A is read per iteration.
        const int nrb = static_cast<int>(a.nrb), ncb = static_cast<int>(a.ncb);
        // symmetric: CTA c's equal-byte range of the block-upper work list, as
        // segments kseg in [cseg[c], cseg[c+1]) of (row block, column range)
        const int kbeg = a.sym ? a.cseg[c] : c, kend = a.sym ? a.cseg[c + 1] : (c < nrb * ncb ? c + 1 : c);
        if (MMA && a.sym) {
          // Symmetric use, 3-4 right-hand sides, on the FP64 tensor pipe: a step
          // is 8 columns (8 ring slots of the 1024-row block, 3 steps in flight);
          // warp w owns rows 64w..64w+63 of the block and issues per step
          //   16 DMMA  Y[rows, s] += A[rows, cols] P[cols, s]   (8 row tiles x 2 k-halves)
          //   16 DMMA  D[cols, s] += A[rows, cols]^T P[rows, s] (16 row quads, k = rows)
          // so the column dots are reduced inside the tensor core instead of by
          // shuffles; the 16 warp partials of D are summed in fixed order after
          // the step's block barrier. Row permutations inside the fragments
          // (rows {0,1,8,9,16,17,24,25}+o for an 8-row tile, {0,1,16,17}+o for a
          // 4-row quad) with a 16-byte slot pad make every fragment load hit 16
          // distinct bank pairs (2 wavefronts, the minimum for 256 bytes).
          static_assert(!MMA || DPW == 1024, "MMA path: 16 warps x 64 rows");
          constexpr int MS = 8;  // columns per step
          const int q4 = lane & 3, l4 = lane >> 2;
          const int wrow = 64 * warp;
          auto frow_axpy = [&](int t) {  // row (within the warp's 64) of accumulator/A-fragment row l4 of tile t
            return 2 * (t & 3) + 32 * (t >> 2) + (l4 & 1) + 8 * ((l4 >> 1) & 1) + 16 * (l4 >> 2);
          };
          auto frow_dot = [&](int qd) {  // row of the dot's k index q4 in quad qd
            return 2 * (qd & 7) + 32 * (qd >> 3) + (q4 & 1) + 16 * (q4 >> 1);
          };
          for (int kseg = kbeg; kseg < kend; ++kseg) {
            const int rb = static_cast<int>(a.unit[3 * kseg]);
            const i64 rb0 = static_cast<i64>(rb) * DPW, cnt = min(static_cast<i64>(DPW), n - rb0);
            const i64 cb0 = a.unit[3 * kseg + 1], cb1 = a.unit[3 * kseg + 2], offd = rb0 + DPW;
            const i64 ncol = cb1 - cb0, npad = round_up(ncol, MS);
            const uint32_t base = ring_head;  // a multiple of MS: a step's 8 slots are consecutive
            const uint32_t seg_bytes = static_cast<uint32_t>(round_up(cnt, 2) * 8);
            __syncthreads();  // the previous segment's slots and dot buffers are released
            if (cnt < DPW) {  // last row block: zero the slot tails once (TMA fills only cnt rows)
              for (int idx = tid; idx < MDNST * (DPW - static_cast<int>(cnt)); idx += PT) {
                const int sl = idx / (DPW - static_cast<int>(cnt)), r = idx % (DPW - static_cast<int>(cnt));
                ring[static_cast<i64>(sl) * MSLOT + cnt + r] = 0.0;
              }
              asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
              __syncthreads();
            }
            auto mma_issue = [&](i64 q) {  // thread 0: segment column q into its slot
              if (q >= npad) return;
              const int slot = static_cast<int>((base + static_cast<uint32_t>(q)) % MDNST);
              if (q >= ncol) {  // padding column of the last step: complete the slot's phase with no bytes
                mbarrier_arrive(&full_bar[slot]);
                return;
              }
              mbarrier_expect_tx(&full_bar[slot], seg_bytes);
              bulk_copy_g2s(ring + static_cast<i64>(slot) * MSLOT, a.A + (cb0 + q) * a.lda + rb0, seg_bytes,
                            &full_bar[slot]);
            };
            if (tid == 0)
              for (i64 q = 0; q < min(npad, static_cast<i64>(MDNST)); ++q) mma_issue(q);
            // p_t on the warp's rows in the dot's B-fragment layout (k = row, n = rhs)
            double prow[16];
#pragma unroll
            for (int qd = 0; qd < 16; ++qd) {
              const i64 i = rb0 + wrow + frow_dot(qd);
              prow[qd] = (l4 < S && i < n) ? pcur[i + l4 * a.ldw] : 0.0;
            }
            double yacc[8][2];
#pragma unroll
            for (int tt = 0; tt < 8; ++tt) yacc[tt][0] = yacc[tt][1] = 0.0;
            int step = 0;
            for (i64 q = 0; q < npad; q += MS, ++step) {
              const i64 j0 = cb0 + q;
              // the axpy's B fragments: p_t of columns j0 + 4h + q4, rhs l4
              double pc[2];
#pragma unroll
              for (int h = 0; h < 2; ++h) {
                const i64 j = j0 + 4 * h + q4;
                pc[h] = (l4 < S && j < cb1) ? pcur[j + l4 * a.ldw] : 0.0;
              }
              const uint32_t u0 = base + static_cast<uint32_t>(q);
              const int sl0 = static_cast<int>(u0 % MDNST);  // slots sl0 .. sl0+7
              for (int cc = 0; cc < MS && q + cc < ncol; ++cc)
                mbarrier_wait_parity(&full_bar[sl0 + cc], ((u0 + cc) / MDNST) & 1u);
              const double* sb = ring + static_cast<i64>(sl0) * MSLOT + wrow;
#pragma unroll
              for (int h = 0; h < 2; ++h) {
                const bool cok = q + 4 * h + q4 < ncol;
                const double* col = sb + static_cast<i64>(4 * h + q4) * MSLOT;
#pragma unroll
                for (int tt = 0; tt < 8; ++tt) {
                  const double av = cok ? col[frow_axpy(tt)] : 0.0;
                  pcg_dmma(yacc[tt][0], yacc[tt][1], av, pc[h]);
                }
              }
              if (j0 + MS > offd) {
                double d[4][2] = {{0.0, 0.0}, {0.0, 0.0}, {0.0, 0.0}, {0.0, 0.0}};  // four chains over the 16 row quads
                const bool cok = q + l4 < ncol;
                const double* col = sb + static_cast<i64>(l4) * MSLOT;
#pragma unroll
                for (int qd = 0; qd < 16; ++qd) {
                  const double av = cok ? col[frow_dot(qd)] : 0.0;
                  pcg_dmma(d[qd & 3][0], d[qd & 3][1], av, prow[qd]);
                }
                mdot(step & 1, warp, 2 * lane) = (d[0][0] + d[1][0]) + (d[2][0] + d[3][0]);
                mdot(step & 1, warp, 2 * lane + 1) = (d[0][1] + d[1][1]) + (d[2][1] + d[3][1]);
              }
              __syncthreads();  // every warp is done with the step's slots and has posted its dots
              // the step's column dots: one thread per (column, rhs) on the last warps (warp 0 issues the refills)
              if (j0 + MS > offd && tid >= PT - MS * S) {
                const int cc = (tid - (PT - MS * S)) / S, sr = (tid - (PT - MS * S)) % S;
                const i64 j = j0 + cc;
                if (j >= offd && j < cb1) {
                  double sum = 0.0;
#pragma unroll
                  for (int w = 0; w < PT / 32; ++w) sum += mdot(step & 1, w, MS * cc + sr);  // fixed order
                  a.colpart[(static_cast<i64>(rb) * S + sr) * a.pstride + j] = sum;
                }
              }
              if (tid == 0)
                for (int cc = 0; cc < MS; ++cc) mma_issue(q + MDNST + cc);
            }
            ring_head = base + static_cast<uint32_t>(npad);
            // row partials of the segment: Y[row f, rhs 2 q4 + e]
#pragma unroll
            for (int tt = 0; tt < 8; ++tt)
#pragma unroll
              for (int e = 0; e < 2; ++e) {
                const int sr = 2 * q4 + e, row = wrow + frow_axpy(tt);
                if (sr < S && row < cnt) a.part[(static_cast<i64>(kseg) * S + sr) * DPW + row] = yacc[tt][e];
              }
          }
        } else
        for (int kseg = kbeg; kseg < kend; ++kseg) {
          const int rb = a.sym ? static_cast<int>(a.unit[3 * kseg]) : c % nrb, cb = a.sym ? kseg : c / nrb;
          const i64 rb0 = static_cast<i64>(rb) * DPW, cnt = min(static_cast<i64>(DPW), n - rb0);
          const i64 cb0 = a.sym ? a.unit[3 * kseg + 1] : static_cast<i64>(cb) * a.cpb;
          const i64 cb1 = a.sym ? a.unit[3 * kseg + 2] : min(n, cb0 + a.cpb);
          double2 acc[S][DPV];
          bool ok[DPV];
#pragma unroll
          for (int k = 0; k < DPV; ++k) {
            ok[k] = 2 * (tid + static_cast<i64>(PT) * k) < cnt;
#pragma unroll
            for (int s = 0; s < S; ++s) acc[s][k] = make_double2(0.0, 0.0);
          }
          if (DEC && a.sym) {
            // Symmetric use, one right-hand side, warps decoupled: a step is two columns (two ring
            // slots, each the column segment plus its S entries of p_t, one
            // mbarrier). No block barrier per step: every warp takes its slots,
            // does its axpy and its share of the 2S column dots, posts the dots
            // and counts itself in on the step's slot pair; the last warp in
            // sums the 16 warp partials in fixed order, writes the column dots
            // and refills both slots (DNST/2 steps ahead). A fast warp runs at
            // most DNST/2 steps ahead of the slowest.
            const i64 offd = rb0 + DPW;  // first column beyond the diagonal block
            const i64 ncol = cb1 - cb0, npad = round_up(ncol, 2);
            const uint32_t base = ring_head;
            const uint32_t seg_bytes = static_cast<uint32_t>(round_up(cnt, 2) * 8);
            auto sym_issue = [&](i64 q) {  // one thread: segment column q into its slot
              const int slot = static_cast<int>((base + static_cast<uint32_t>(q)) % DNST);
              if (q < ncol) {
                mbarrier_expect_tx(&full_bar[slot], seg_bytes + SP * 8);
                bulk_copy_g2s(ring + static_cast<i64>(slot) * DPW, a.A + (cb0 + q) * a.lda + rb0, seg_bytes,
                              &full_bar[slot]);
                bulk_copy_g2s(pring + slot * SP, a.pil + (cb0 + q) * SP, SP * 8, &full_bar[slot]);
              } else {
                mbarrier_arrive(&full_bar[slot]);  // odd tail: the step's second slot carries nothing
              }
            };
            double2 pr[S][DPV];  // p_t on this thread's rows (column dots)
#pragma unroll
            for (int s = 0; s < S; ++s)
#pragma unroll
              for (int k = 0; k < DPV; ++k) {
                const i64 i = rb0 + 2 * (tid + static_cast<i64>(PT) * k);
                pr[s][k] = make_double2(i < n ? pcur[i + s * a.ldw] : 0.0, i + 1 < n ? pcur[i + 1 + s * a.ldw] : 0.0);
              }
            __syncthreads();  // the previous segment's slots are all released
            if (tid == 0)
              for (i64 q = 0; q < min(npad, static_cast<i64>(DNST)); ++q) sym_issue(q);
            constexpr int NV = 2 * S <= 2 ? 2 : 2 * S <= 4 ? 4 : 8;  // 2S dots padded to a power of two
            constexpr int LG = NV == 2 ? 1 : NV == 4 ? 2 : 3;
            constexpr int LPS = 32 / NV, WPL = (PT / 32) / LPS;      // fixed-order reduction: lanes per dot, warps per lane
            for (i64 q = 0; q < npad; q += 2) {
              const i64 j = cb0 + q;
              const bool two = q + 1 < ncol;
              const uint32_t u0 = base + static_cast<uint32_t>(q);
              const int sl0 = static_cast<int>(u0 % DNST), sl1 = static_cast<int>((u0 + 1) % DNST);
              const int pair = sl0 >> 1;
              mbarrier_wait_parity(&full_bar[sl0], (u0 / DNST) & 1u);
              mbarrier_wait_parity(&full_bar[sl1], ((u0 + 1) / DNST) & 1u);
              const double* s0 = ring + static_cast<i64>(sl0) * DPW;
              const double* s1 = ring + static_cast<i64>(sl1) * DPW;
              double2 c0[DPV], c1[DPV];
              double q0[S], q1[S];
#pragma unroll
              for (int k = 0; k < DPV; ++k) {
                c0[k] = ok[k] ? reinterpret_cast<const double2*>(s0)[tid + PT * k] : make_double2(0.0, 0.0);
                c1[k] = (ok[k] && two) ? reinterpret_cast<const double2*>(s1)[tid + PT * k] : make_double2(0.0, 0.0);
              }
#pragma unroll
              for (int s = 0; s < S; ++s) {
                q0[s] = pring[sl0 * SP + s];
                q1[s] = two ? pring[sl1 * SP + s] : 0.0;
              }
              const bool offdiag = j >= offd;  // both columns beyond the diagonal block (offd and j are even)
              if (offdiag) {
                // the 2S dots (slot e*S + s) reduced over the warp by a transposed
                // butterfly: lane group g ends with slot g
                double d[NV];
#pragma unroll
                for (int v = 0; v < NV; ++v) d[v] = 0.0;
#pragma unroll
                for (int s = 0; s < S; ++s)
#pragma unroll
                  for (int k = 0; k < DPV; ++k) {
                    d[s] += c0[k].x * pr[s][k].x + c0[k].y * pr[s][k].y;
                    d[S + s] += c1[k].x * pr[s][k].x + c1[k].y * pr[s][k].y;
                  }
#pragma unroll
                for (int st = 0; st < LG; ++st) {
                  const int m = 16 >> st, half = NV >> (st + 1);
                  const bool hi = lane & m;
#pragma unroll
                  for (int v = 0; v < half; ++v) {
                    const double send = hi ? d[v] : d[v + half];
                    const double keep = hi ? d[v + half] : d[v];
                    d[v] = keep + __shfl_xor_sync(0xffffffffu, send, m);
                  }
                }
#pragma unroll
                for (int m = 16 >> LG; m >= 1; m >>= 1) d[0] += __shfl_xor_sync(0xffffffffu, d[0], m);
                const int slot = lane >> (5 - LG);
                if ((lane & ((32 >> LG) - 1)) == 0 && slot < 2 * S) sdot[pair][warp][slot] = d[0];
              }
#pragma unroll
              for (int s = 0; s < S; ++s) {
                const double p0 = q0[s], p1 = q1[s];
#pragma unroll
                for (int k = 0; k < DPV; ++k) {
                  acc[s][k].x += c0[k].x * p0;
                  acc[s][k].y += c0[k].y * p0;
                  acc[s][k].x += c1[k].x * p1;
                  acc[s][k].y += c1[k].y * p1;
                }
              }
              // count in on the pair (the slots' values are consumed, the dots posted)
              __syncwarp();  // the warp's reads and dot stores are ordered before lane 0's release
              unsigned last = 0;
              if (lane == 0) last = (atom_add_acq_rel_cta(&pair_cnt[pair], 1u) & (PT / 32 - 1)) == PT / 32 - 1;
              if (__shfl_sync(0xffffffffu, last, 0)) {  // (the shuffle's warp sync orders lane 0's acquire before the reads)
                if (offdiag) {
                  const int slot = lane / LPS, g = lane % LPS;
                  double v = 0.0;
                  if (slot < 2 * S) {
#pragma unroll
                    for (int w = 0; w < WPL; ++w) v += sdot[pair][g * WPL + w][slot];
                  }
#pragma unroll
                  for (int m = LPS / 2; m >= 1; m >>= 1) v += __shfl_xor_sync(0xffffffffu, v, m);
                  const int e = slot / S, s = slot % S;
                  if (g == 0 && slot < 2 * S && j + e < cb1)
                    a.colpart[(static_cast<i64>(rb) * S + s) * a.pstride + j + e] = v;
                }
                if (lane == 0) {
                  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");  // generic reads before the async refill
                  if (q + DNST < npad) {
                    sym_issue(q + DNST);
                    sym_issue(q + DNST + 1);
                  }
                }
              }
            }
            ring_head = base + static_cast<uint32_t>(npad);
          } else {
            // full use (A col-major): CTA (rb, cb) streams rows [rb*DPW, +DPW) of
            // columns [cb*cpb, +cpb); symmetric use with two right-hand sides:
            // the block-upper segments as above, each step's 2S column dots
            // reduced over the warp by a transposed butterfly and across the
            // warps at the next step's block barrier (measured at n = 1e5:
            // decoupled warps 17.7 vs 11.9 ms per iteration at S = 4; the DMMA
            // loop 9.1 vs 7.45 ms at S = 2, 9.3 vs 11.7 ms at S = 4).
            // Each column segment is one contiguous bulk copy into the ring
            // (DNST segments in flight); two columns per step, one block barrier
            // per step frees their slots.
            const i64 offd = rb0 + DPW;  // first column beyond the diagonal block
            // (3+ right-hand sides take the DMMA loop above in symmetric use: SYM2 discards that code here)
            constexpr bool SYM2 = !MMA;
            __shared__ double wdot[2][PT / 32][SYM2 ? 2 * S : 1];
            double2 pr[SYM2 ? S : 1][DPV];  // p_t on this thread's rows (symmetric dots)
            if constexpr (SYM2) if (a.sym) {
#pragma unroll
              for (int s = 0; s < S; ++s)
#pragma unroll
                for (int k = 0; k < DPV; ++k) {
                  const i64 i = rb0 + 2 * (tid + static_cast<i64>(PT) * k);
                  pr[s][k] = make_double2(i < n ? pcur[i + s * a.ldw] : 0.0, i + 1 < n ? pcur[i + 1 + s * a.ldw] : 0.0);
                }
            }
            // column dots of the previous step: the 16 warp partials of each of
            // the 2S dots reduced by a fixed shuffle tree over 16 lanes, on the
            // last four warps (warp 0 issues the ring's bulk copies; a serial sum
            // there made it the laggard at every step's barrier)
            static_assert(PT / 32 == 16 && (!SYM2 || 2 * S * 16 <= 128), "flush layout");
            auto flush_dots = [&](i64 jp, int buf) {
              const int loc = tid - (PT - 128);
              if (loc >= 0) {
                const int slot = loc >> 4, w = loc & 15;
                double v = (SYM2 && slot < 2 * S) ? wdot[buf][w][SYM2 ? slot : 0] : 0.0;
#pragma unroll
                for (int m = 8; m >= 1; m >>= 1) v += __shfl_xor_sync(0xffffffffu, v, m);
                const int e = slot / S, s = slot % S;
                if (w == 0 && slot < 2 * S && jp + e < cb1)
                  a.colpart[(static_cast<i64>(rb) * S + s) * a.pstride + jp + e] = v;
              }
            };
            i64 jprev = -1;
            int step = 0;
            if (tid == 0)
              for (i64 j = cb0; j < min(cb1, cb0 + DNST); ++j) ring_issue(a.A + j * a.lda + rb0, cnt);
            // p_t of the whole vector is in pcur (slice owners wrote it before the barrier)
            auto load_p = [&](i64 j, double* dst) {
#pragma unroll
              for (int s = 0; s < S; ++s) dst[s] = j < cb1 ? pcur[j + s * a.ldw] : 0.0;
            };
            double q0[S], q1[S];
            for (i64 j = cb0; j < cb1; j += 2) {
              const bool two = j + 1 < cb1;
              load_p(j, q0);
              load_p(j + 1, q1);
              const double* s0 = ring_wait();
              const double* s1 = two ? ring_wait() : nullptr;
              double2 c0[DPV], c1[DPV];
#pragma unroll
              for (int k = 0; k < DPV; ++k) {
                c0[k] = ok[k] ? reinterpret_cast<const double2*>(s0)[tid + PT * k] : make_double2(0.0, 0.0);
                c1[k] = (ok[k] && two) ? reinterpret_cast<const double2*>(s1)[tid + PT * k] : make_double2(0.0, 0.0);
              }
              __syncthreads();  // every thread holds its values: the two slots may be refilled
              if (tid == 0) {
                if (j + DNST < cb1) ring_issue(a.A + (j + DNST) * a.lda + rb0, cnt);
                if (j + DNST + 1 < cb1) ring_issue(a.A + (j + DNST + 1) * a.lda + rb0, cnt);
              }
              if constexpr (SYM2) if (a.sym) {
                if (jprev >= 0) flush_dots(jprev, (step - 1) & 1);
                jprev = -1;
                if (j >= offd) {  // both columns are beyond the diagonal block (offd is even)
                  // the 2S dots (slot e*S + s), padded to a power of two, reduced over
                  // the warp by a transposed butterfly: lane group g ends with slot g
                  constexpr int NV = 2 * S <= 2 ? 2 : 2 * S <= 4 ? 4 : 8;
                  constexpr int LG = NV == 2 ? 1 : NV == 4 ? 2 : 3;
                  double d[NV];
#pragma unroll
                  for (int v = 0; v < NV; ++v) d[v] = 0.0;
#pragma unroll
                  for (int s = 0; s < S; ++s)
#pragma unroll
                    for (int k = 0; k < DPV; ++k) {
                      d[s] += c0[k].x * pr[s][k].x + c0[k].y * pr[s][k].y;
                      d[S + s] += c1[k].x * pr[s][k].x + c1[k].y * pr[s][k].y;
                    }
#pragma unroll
                  for (int st = 0; st < LG; ++st) {
                    const int m = 16 >> st, half = NV >> (st + 1);
                    const bool hi = lane & m;
#pragma unroll
                    for (int v = 0; v < half; ++v) {
                      const double send = hi ? d[v] : d[v + half];
                      const double keep = hi ? d[v + half] : d[v];
                      d[v] = keep + __shfl_xor_sync(0xffffffffu, send, m);
                    }
                  }
#pragma unroll
                  for (int m = 16 >> LG; m >= 1; m >>= 1) d[0] += __shfl_xor_sync(0xffffffffu, d[0], m);
                  const int slot = lane >> (5 - LG);
                  if ((lane & ((32 >> LG) - 1)) == 0 && slot < 2 * S) wdot[step & 1][warp][slot] = d[0];
                  jprev = j;
                }
                ++step;
              }
#pragma unroll
              for (int s = 0; s < S; ++s) {
                const double p0 = q0[s], p1 = q1[s];
#pragma unroll
                for (int k = 0; k < DPV; ++k) {
                  acc[s][k].x += c0[k].x * p0;
                  acc[s][k].y += c0[k].y * p0;
                  acc[s][k].x += c1[k].x * p1;
                  acc[s][k].y += c1[k].y * p1;
                }
              }
            }
            if (a.sym) {
              __syncthreads();
              if (jprev >= 0) flush_dots(jprev, (step - 1) & 1);
            }
          }
#pragma unroll
          for (int s = 0; s < S; ++s) {
            double* dst = a.sym ? a.part + (static_cast<i64>(kseg) * S + s) * DPW
                                : a.part + (static_cast<i64>(cb) * S + s) * a.pstride + rb0;
#pragma unroll
            for (int k = 0; k < DPV; ++k) {
              const i64 i = 2 * (tid + static_cast<i64>(PT) * k);
              if (i + 1 < cnt) {
                reinterpret_cast<double2*>(dst)[tid + PT * k] = acc[s][k];
              } else if (i < cnt) {
                dst[i] = acc[s][k].x;
              }
            }
          }
        }
        tick(t, 1);
        grid.sync();
        tick(t, 2);
        // ---- P2 (dense): v = (sum_cb partial_cb) + mu p for the slice, partial p.v
        double pvl[S];
#pragma unroll
        for (int s = 0; s < S; ++s) pvl[s] = 0.0;
        if (a.sym) {
          // symmetric: thread per row (coalesced over the warp); row sums of the
          // units of j's row block, then the column dots of the row blocks above,
          // in that fixed order
          for (i64 j = r0 + tid; j < r1; j += PT) {
            const int rbj = static_cast<int>(j / DPW);
            const int us = a.ustart[rbj], nu = a.ustart[rbj + 1] - us;
            const i64 loc = j - static_cast<i64>(rbj) * DPW;
            // (partials outermost: the S sums' loads of several partials are in flight together;
            // each sum keeps its order)
            double sum[S];
#pragma unroll
            for (int s = 0; s < S; ++s) sum[s] = 0.0;
            for (int b = 0; b < nu; ++b)
#pragma unroll
              for (int s = 0; s < S; ++s) sum[s] += a.part[(static_cast<i64>(us + b) * S + s) * DPW + loc];
#pragma unroll 4
            for (int b = 0; b < rbj; ++b)
#pragma unroll
              for (int s = 0; s < S; ++s) sum[s] += a.colpart[(static_cast<i64>(b) * S + s) * a.pstride + j];
#pragma unroll
            for (int s = 0; s < S; ++s) {
              const double pj = pcur[j + s * a.ldw];
              double v = sum[s];  // operators.cpp:72-78 then solvers.cpp:137-141: out = A p; out += mu p
              v = __dadd_rn(v, __dmul_rn(a.mus[s], pj));  // out += mu p, unfused (solvers.cpp:139)
              a.V[j + s * a.ldw] = v;
              pvl[s] += pj * v;
            }
          }
        }
        for (i64 j = r0 + warp; j < r1 && !a.sym; j += PT / 32) {
#pragma unroll
          for (int s = 0; s < S; ++s) {
            double sum = 0.0;
            for (int b = lane; b < ncb; b += 32) sum += a.part[(static_cast<i64>(b) * S + s) * a.pstride + j];
            sum = warp_sum(sum);
            const double pj = pcur[j + s * a.ldw];
            double v = sum;  // operators.cpp:72-78 then solvers.cpp:137-141: out = A p; out += mu p
            v = __dadd_rn(v, __dmul_rn(a.mus[s], pj));  // out += mu p, unfused (solvers.cpp:139)
            if (lane == 0) {
              a.V[j + s * a.ldw] = v;
              pvl[s] += pj * v;
            }
          }
        }
#pragma unroll
        for (int s = 0; s < S; ++s) {
          const double tot = block_sum(pvl[s], sh);
          if (tid == 0) a.pv_part[c * S + s] = tot;
        }
        tick(t, 3);
      }
      grid.sync();
      tick(t, 4);
      // ---- P3: alpha (fin_dot kind 1), x and r updates, partial ||r||^2
#pragma unroll
      for (int s = 0; s < S; ++s) {
        const double pv = all_sum(a.pv_part, s);
        if (tid == 0 && cs[s].status == 0) {
          cs[s].pv = pv;
          cs[s].iters = static_cast<int>(t);
          if (!(pv > 0.0) || !isfinite(pv)) cs[s].status = 2;  // solvers.cpp:76-81
          else cs[s].alpha = cs[s].rz / pv;
        }
      }
      __syncthreads();
#pragma unroll
      for (int s = 0; s < S; ++s) {
        double rr = 0.0;
        if (cs[s].status == 0) {
          const double al = cs[s].alpha;
          for (i64 i = r0 + tid; i < r1; i += PT) {
            const i64 o = i + s * a.ldw;
            a.X[i + s * a.ldx] += al * pcur[o];
            const double r = a.R[o] - al * a.V[o];
            a.R[o] = r;
            rr += r * r;
          }
        }
        rr = block_sum(rr, sh);
        if (tid == 0) a.rr_part[c * S + s] = rr;
      }
      if constexpr (!GRAM) asm volatile("fence.proxy.async.global;" ::: "memory");  // P4 bulk-copies r
      tick(t, 5);
      grid.sync();
      tick(t, 6);
      // ---- P4: the preconditioner's U^T r first (independent of the convergence
      // test, so its loads overlap the residual reduction), then ||r|| and status
      double rr_pre[S];  // this thread's entry of the residual partials, loaded ahead of the U pass
#pragma unroll
      for (int s = 0; s < S; ++s) rr_pre[s] = tid < G ? a.rr_part[tid * S + s] : 0.0;
      if (!GRAM && nys && a.pre_dmma) {
        // DMMA path: T[cols, s] = U[:, cols]^T R[:, s] for this CTA's columns of U, 8 at a
        // time. A chunk slot holds 512 rows of r (S segments) and of the 8 columns
        // (bulk copies, 3 chunks in flight); warp w owns rows 32w..32w+31 of the
        // chunk and accumulates 8 DMMA.8x8x4 per chunk (m = column, n = rhs, k =
        // row) in four chains; the 16 warp partials are summed in fixed order.
        const int q4 = lane & 3, l4 = lane >> 2;
        const i64 nch = cdiv(n, static_cast<i64>(UCH));
        for (i64 jt = u0; jt < u1; jt += 8) {
          const int ncols = static_cast<int>(min(static_cast<i64>(8), u1 - jt));
          const uint32_t seq0 = chunk_seq;
          auto issue = [&](i64 k) {  // thread 0: chunk k of this column tile
            if (k >= nch) return;
            const int slot = static_cast<int>((seq0 + static_cast<uint32_t>(k)) % UNCH);
            const i64 rb0 = k * UCH;
            const uint32_t bytes = static_cast<uint32_t>(round_up(min(static_cast<i64>(UCH), n - rb0), 2) * 8);
            double* dst = ring + static_cast<i64>(slot) * UNSEG * USEG;
            mbarrier_expect_tx(&chunk_bar[slot], bytes * static_cast<uint32_t>(S + ncols));
            for (int sr = 0; sr < S; ++sr) bulk_copy_g2s(dst + sr * USEG, a.R + sr * a.ldw + rb0, bytes, &chunk_bar[slot]);
            for (int cc = 0; cc < ncols; ++cc)
              bulk_copy_g2s(dst + (8 + cc) * USEG, a.U + (jt + cc) * a.ldu + rb0, bytes, &chunk_bar[slot]);
          };
          if (tid == 0) {
            asm volatile("fence.proxy.async.global;" ::: "memory");
            for (i64 k = 0; k < UNCH; ++k) issue(k);
          }
          __syncwarp();  // warp 0 reconverges before its lanes spin on the first chunk's barrier
          double d[4][2] = {{0.0, 0.0}, {0.0, 0.0}, {0.0, 0.0}, {0.0, 0.0}};
          for (i64 k = 0; k < nch; ++k) {
            const uint32_t sq = seq0 + static_cast<uint32_t>(k);
            const int slot = static_cast<int>(sq % UNCH);
            const int cnt = static_cast<int>(min(static_cast<i64>(UCH), n - k * UCH));
            mbarrier_wait_parity(&chunk_bar[slot], (sq / UNCH) & 1u);
            const double* rs = ring + (static_cast<i64>(slot) * UNSEG + l4) * USEG + 32 * warp;
            const double* us = rs + 8 * USEG;
            const bool rok = l4 < S, cok = l4 < ncols;
#pragma unroll
            for (int qd = 0; qd < 8; ++qd) {
              const int row = 2 * qd + (q4 & 1) + 16 * (q4 >> 1);  // bank-conflict-free quad permutation
              const bool in = 32 * warp + row < cnt;
              const double av = (cok && in) ? us[row] : 0.0;
              const double bv = (rok && in) ? rs[row] : 0.0;
              pcg_dmma(d[qd & 3][0], d[qd & 3][1], av, bv);
            }
            __syncthreads();  // every warp is done with the chunk slot
            if (tid == 0) issue(k + UNCH);
          }
          chunk_seq = seq0 + static_cast<uint32_t>(nch);
          mdot(0, warp, 2 * lane) = (d[0][0] + d[1][0]) + (d[2][0] + d[3][0]);      // (column l4, rhs 2 q4)
          mdot(0, warp, 2 * lane + 1) = (d[0][1] + d[1][1]) + (d[2][1] + d[3][1]);  // (column l4, rhs 2 q4 + 1)
          __syncthreads();
          if (tid < 64) {
            const int cc = tid >> 3, sr = tid & 7;
            if (cc < ncols && sr < S) {
              double tot = 0.0;
#pragma unroll
              for (int w = 0; w < PT / 32; ++w) tot += mdot(0, w, 8 * cc + sr);  // fixed order
              a.T[(jt + cc) + sr * a.ell] = tot * a.gain[jt + cc + sr * a.gstride];
            }
          }
          __syncthreads();
        }
      } else if (nys) {
        // this CTA's columns of U, up to UQ at a time: r is read once per row for all of them
        // and the UQ x S dots are reduced together (one barrier)
        for (i64 j0 = u0; j0 < u1; j0 += UQ) {
          double w[UQ][S];
#pragma unroll
          for (int q = 0; q < UQ; ++q)
#pragma unroll
            for (int s = 0; s < S; ++s) w[q][s] = 0.0;
#pragma unroll 4
          for (i64 i = tid; i < n; i += PT) {  // unrolled: the rows' loads are in flight together
            double ri[S];
#pragma unroll
            for (int s = 0; s < S; ++s) ri[s] = a.R[i + s * a.ldw];
#pragma unroll
            for (int q = 0; q < UQ; ++q) {
              if (j0 + q < u1) {
                const double uiq = a.U[i + (j0 + q) * a.ldu];
#pragma unroll
                for (int s = 0; s < S; ++s) w[q][s] += uiq * ri[s];
              }
            }
          }
#pragma unroll
          for (int q = 0; q < UQ; ++q)
#pragma unroll
            for (int s = 0; s < S; ++s) {
              const double tot = warp_sum(w[q][s]);
              if (lane == 0) wred[(q * S + s) * (PT / 32) + warp] = tot;
            }
          __syncthreads();
          if (tid < UQ * S) {
            const int q = tid / S, s = tid % S;
            if (j0 + q < u1) {
              double tot = 0.0;
              for (int ww = 0; ww < PT / 32; ++ww) tot += wred[tid * (PT / 32) + ww];  // fixed order
              a.T[(j0 + q) + s * a.ell] = tot * a.gain[j0 + q + s * a.gstride];
            }
          }
          __syncthreads();
        }
      }
      // residual norm, status (fin_res)
#pragma unroll
      for (int s = 0; s < S; ++s) {
        const double rr = G <= PT ? block_sum(rr_pre[s], sh) : all_sum(a.rr_part, s);  // same order as all_sum
        if (tid == 0 && cs[s].status == 0) {
          const double res = sqrt(rr);
          cs[s].res = res;
          if (c == 0) a.hist[s * a.hstride + t] = res;
          if (!isfinite(res)) cs[s].status = 3;      // solvers.cpp:88-93
          else if (res <= cs[s].eta) cs[s].status = 1;  // :94-97
          else if (t >= a.max_iter) cs[s].status = 5;
          if (!nys && cs[s].status == 0) {  // z = r: r.z = ||r||^2 (fin_dot kind 2)
            cs[s].beta = rr / cs[s].rz;
            cs[s].rz = rr;
          }
        }
      }
      __syncthreads();
      if (tid == 0) running_sh = count_running();
      __syncthreads();
      if (running_sh == 0) break;
      if (!nys) continue;
      tick(t, 7);
      grid.sync();
      tick(t, 8);
      // ---- P5: z = r + U t on the slice (32 rows x 16 column groups; U read once
      // for all S right-hand sides), partial r.z
      auto uat = [&](i64 i, i64 j) { return a.U[i + j * a.ldu]; };
      if (!GRAM && a.pre_dmma) {
        // DMMA path: Z[rows, s] = R + U[rows, :] T[:, s] on the slice, in row chunks of
        // up to 512 rows; a chunk slot holds 16 columns of U on those rows (bulk
        // copies, 3 slots in flight); warp w owns rows 32w..32w+31: 4 row tiles x
        // 4 k-steps of DMMA.8x8x4 per slot (m = row, n = rhs, k = column).
        const int q4 = lane & 3, l4 = lane >> 2;
        const i64 cnt_s = r1 - r0;
        const i64 nrc = cdiv(cnt_s, static_cast<i64>(UCH));
        const i64 crows = nrc > 0 ? round_up(cdiv(cnt_s, nrc), 32) : 0;  // rows per chunk (<= 512)
        const i64 ngr = cdiv(a.ell, static_cast<i64>(UNSEG));
        double rzl[2] = {0.0, 0.0};  // r.z of right-hand sides 2 q4, 2 q4 + 1 on this lane's rows
        for (i64 rc = 0; rc < nrc; ++rc) {
          const i64 rb0 = r0 + rc * crows;
          const int cnt = static_cast<int>(min(crows, r1 - rb0));
          const uint32_t bytes = static_cast<uint32_t>(round_up(static_cast<i64>(cnt), 2) * 8);
          const uint32_t seq0 = chunk_seq;
          auto issue = [&](i64 g) {  // thread 0: columns 16 g .. 16 g + 15 of U on the chunk's rows
            if (g >= ngr) return;
            const int slot = static_cast<int>((seq0 + static_cast<uint32_t>(g)) % UNCH);
            const int nc = static_cast<int>(min(static_cast<i64>(UNSEG), a.ell - g * UNSEG));
            double* dst = ring + static_cast<i64>(slot) * UNSEG * USEG;
            mbarrier_expect_tx(&chunk_bar[slot], bytes * static_cast<uint32_t>(nc));
            for (int cc = 0; cc < nc; ++cc)
              bulk_copy_g2s(dst + cc * USEG, a.U + (g * UNSEG + cc) * a.ldu + rb0, bytes, &chunk_bar[slot]);
          };
          if (tid == 0)
            for (i64 g = 0; g < UNCH; ++g) issue(g);
          __syncwarp();  // warp 0 reconverges before its lanes spin on the first slot's barrier
          double yacc[4][2];
#pragma unroll
          for (int tt = 0; tt < 4; ++tt) yacc[tt][0] = yacc[tt][1] = 0.0;
          auto frow = [&](int tt) { return 2 * tt + (l4 & 1) + 8 * ((l4 >> 1) & 1) + 16 * (l4 >> 2); };
          for (i64 g = 0; g < ngr; ++g) {
            const uint32_t sq = seq0 + static_cast<uint32_t>(g);
            const int slot = static_cast<int>(sq % UNCH);
            double tb[4];  // T[16 g + 4 h + q4, rhs l4]
#pragma unroll
            for (int h = 0; h < 4; ++h) {
              const i64 j = g * UNSEG + 4 * h + q4;
              tb[h] = (l4 < S && j < a.ell) ? a.T[j + l4 * a.ell] : 0.0;
            }
            mbarrier_wait_parity(&chunk_bar[slot], (sq / UNCH) & 1u);
            const double* sb = ring + static_cast<i64>(slot) * UNSEG * USEG + 32 * warp;
            if (32 * warp < cnt) {
#pragma unroll
              for (int h = 0; h < 4; ++h) {
                const bool cok = g * UNSEG + 4 * h + q4 < a.ell;
                const double* col = sb + static_cast<i64>(4 * h + q4) * USEG;
#pragma unroll
                for (int tt = 0; tt < 4; ++tt) {
                  const int row = frow(tt);
                  const double av = (cok && 32 * warp + row < cnt) ? col[row] : 0.0;
                  pcg_dmma(yacc[tt][0], yacc[tt][1], av, tb[h]);
                }
              }
            }
            __syncthreads();  // every warp is done with the slot
            if (tid == 0) issue(g + UNCH);
          }
          chunk_seq = seq0 + static_cast<uint32_t>(ngr);
#pragma unroll
          for (int tt = 0; tt < 4; ++tt)
#pragma unroll
            for (int e = 0; e < 2; ++e) {
              const int sr = 2 * q4 + e, row = 32 * warp + frow(tt);
              if (sr < S && row < cnt) {
                const i64 o = rb0 + row + sr * a.ldw;
                const double r = a.R[o];
                const double z = r + yacc[tt][e];
                a.Z[o] = z;
                rzl[e] += r * z;
              }
            }
        }
#pragma unroll
        for (int s = 0; s < S; ++s) {
          const double tot = block_sum((s >> 1) == q4 ? rzl[s & 1] : 0.0, sh);
          if (tid == 0) a.rz_part[c * S + s] = tot;
        }
      } else {
        double rz = 0.0;  // warp s < S accumulates r.z of right-hand side s
        for (i64 i0 = r0; i0 < r1; i0 += 32) {
          const i64 i = i0 + lane;
          double acc[S];
#pragma unroll
          for (int s = 0; s < S; ++s) acc[s] = 0.0;
          if (i < r1) {
            double acc1[S];  // two chains, loads several columns ahead
#pragma unroll
            for (int s = 0; s < S; ++s) acc1[s] = 0.0;
            i64 j = warp;
#pragma unroll 2
            for (; j + PT / 32 < a.ell; j += 2 * (PT / 32)) {
              const double u0 = uat(i, j), u1 = uat(i, j + PT / 32);
#pragma unroll
              for (int s = 0; s < S; ++s) {
                acc[s] += u0 * a.T[j + s * a.ell];
                acc1[s] += u1 * a.T[j + PT / 32 + s * a.ell];
              }
            }
            if (j < a.ell) {
              const double u0 = uat(i, j);
#pragma unroll
              for (int s = 0; s < S; ++s) acc[s] += u0 * a.T[j + s * a.ell];
            }
#pragma unroll
            for (int s = 0; s < S; ++s) acc[s] += acc1[s];
          }
#pragma unroll
          for (int h = 0; h < S; h += ZS) {  // ZS right-hand sides per round
#pragma unroll
            for (int s = h; s < h + ZS && s < S; ++s) zbuf[((s - h) * (PT / 32) + warp) * 32 + lane] = acc[s];
            __syncthreads();
            if (warp >= h && warp < h + ZS && warp < S && i < r1) {
              double u = 0.0;
#pragma unroll
              for (int w = 0; w < PT / 32; ++w) u += zbuf[((warp - h) * (PT / 32) + w) * 32 + lane];
              const double r = a.R[i + warp * a.ldw];
              const double z = r + u;
              a.Z[i + warp * a.ldw] = z;
              rz += r * z;
            }
            __syncthreads();
          }
        }
#pragma unroll
        for (int s = 0; s < S; ++s) {
          const double tot = block_sum(warp == s ? rz : 0.0, sh);
          if (tid == 0) a.rz_part[c * S + s] = tot;
        }
      }
      tick(t, 9);
      grid.sync();
      tick(t, 10);
#pragma unroll
      for (int s = 0; s < S; ++s) {
        const double rz = all_sum(a.rz_part, s);
        if (tid == 0 && cs[s].status == 0) {  // fin_dot kind 2
          cs[s].beta = rz / cs[s].rz;
          cs[s].rz = rz;
        }
      }
      __syncthreads();
    }
  }
  if (c == 0 && tid < S) a.st->c[tid] = cs[tid];
  if (c == 0 && tid == 0) a.st->any_running = 0;
}

bool persistent_eligible(const Ctx& ctx, Op& op, i64 S) {
  (void)ctx;
  if (auto* g = dynamic_cast<GramOp*>(&op)) return S == 1 && g->n <= PW && g->m >= 1;
  if (dynamic_cast<DenseOp*>(&op))  // 1-4 or 8 columns (5-7 are not instantiated)
    return (S <= 4 || S == 8) && cdiv(op.n, dense_pw(static_cast<int>(S))) <= ctx.sm_count;
  return false;
}

template <int S, bool GRAM>
void launch_persistent(Ctx& ctx, PersistArgs& pa, int G, int smem) {
  void* args[] = {&pa};
  ctx.prof_begin(GRAM ? "pcg_persistent_kernel<gram>" : "pcg_persistent_kernel<dense>");
  // dynamic shared memory: the ring that streams A (dense), U's resident blocks (gram)
  NPCG_CUDA(cudaLaunchCooperativeKernel(reinterpret_cast<void*>(pcg_persistent_kernel<S, GRAM>), G, PT, args,
                                        smem, ctx.stream));
  ctx.check_launch("pcg_persistent_kernel");
  ctx.prof_end();
}

template <int S, bool GRAM>
int persistent_grid(const Ctx& ctx) {
  NPCG_CUDA(cudaFuncSetAttribute(pcg_persistent_kernel<S, GRAM>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                 ring_bytes(GRAM, S)));
  int per_sm = 0;
  NPCG_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, pcg_persistent_kernel<S, GRAM>, PT,
                                                          GRAM ? 0 : ring_bytes(GRAM, S)));
  if (per_sm < 1) fail(NPCG_ECUDA, "pcg_persistent_kernel does not fit on an SM");
  return ctx.sm_count;  // one CTA per SM: cheapest grid barrier, enough bytes in flight
}

void run_persistent(Ctx& ctx, Op& op, Pre* pre, double mu, const PcgMuCols* cols, i64 S, double* X, i64 ldx, DMat& R,
                    DMat& Z, DMat& P, DMat& V, State* st, double* hist, i64 hstride, i64 max_iter) {
  auto* gram = dynamic_cast<GramOp*>(&op);
  auto* dense = dynamic_cast<DenseOp*>(&op);
  if (gram) gram->settle();
  const i64 n = op.n;
  const bool nys = pre != nullptr && pre->ell > 0;
  const int G = gram ? persistent_grid<1, true>(ctx)
                     : S == 1 ? persistent_grid<1, false>(ctx)
                     : S == 2 ? persistent_grid<2, false>(ctx)
                     : S == 3 ? persistent_grid<3, false>(ctx)
                     : S == 4 ? persistent_grid<4, false>(ctx) : persistent_grid<8, false>(ctx);
  DMat P1;
  P1.alloc(n, S, ctx.stream, false);
  DBuf<double> part, T, scal(3 * static_cast<i64>(G) * S, ctx.stream);
  if (gram) part.alloc(static_cast<i64>(G) * PW, ctx.stream);
  i64 nrb = 0, ncb = 0, cpb = 0, pstride = 0;
  DBuf<i64> units;
  DBuf<int> cseg, ustart;
  double sym_entries = 0.0;  // entries of A streamed per iteration in symmetric use
  DBuf<double> colpart, pil;
  int sym = 0;
  if (dense) {
    const i64 dpw = dense_pw(static_cast<int>(S));
    nrb = cdiv(n, dpw);
    pstride = round_up(n, 2);
    static const bool full = std::getenv("NPCG_DENSE_FULL") != nullptr;  // diagnostics: read all of A
    sym = (!full && nrb > 1 && nrb <= G) ? 1 : 0;
    if (sym) {
      // block-upper part: row block rb streams columns [rb*dpw, n) of cnt_rb
      // rows; CTA c takes the byte range [c W / G, (c+1) W / G) of that work
      // list in row-major order (one segment per row block it touches;
      // boundaries on even columns so a step's two columns share a side of the
      // diagonal block)
      std::vector<double> cum(static_cast<size_t>(nrb + 1), 0.0);
      for (i64 rb = 0; rb < nrb; ++rb) {
        const i64 cnt = std::min(dpw, n - rb * dpw);
        cum[static_cast<size_t>(rb + 1)] = cum[static_cast<size_t>(rb)] + static_cast<double>(n - rb * dpw) * cnt;
      }
      const double W = cum[static_cast<size_t>(nrb)];
      sym_entries = W;
      auto pos = [&](i64 c) -> std::pair<i64, i64> {  // (row block, column) where CTA c starts
        if (c >= G) return {nrb - 1, n};
        const double wc = W * static_cast<double>(c) / static_cast<double>(G);
        i64 rb = std::upper_bound(cum.begin(), cum.end(), wc) - cum.begin() - 1;
        rb = std::min<i64>(std::max<i64>(rb, 0), nrb - 1);
        const i64 cnt = std::min(dpw, n - rb * dpw);
        const i64 off = static_cast<i64>(std::ceil((wc - cum[static_cast<size_t>(rb)]) / static_cast<double>(cnt)));
        return {rb, std::min(n, rb * dpw + round_up(off, 2))};
      };
      std::vector<i64> hu;
      std::vector<int> hc(static_cast<size_t>(G + 1)), hs(static_cast<size_t>(nrb + 1), -1);
      for (i64 c = 0; c < G; ++c) {
        hc[static_cast<size_t>(c)] = static_cast<int>(hu.size() / 3);
        const auto [ra, ja] = pos(c);
        const auto [rz, jz] = pos(c + 1);
        for (i64 rb = ra; rb <= rz; ++rb) {
          const i64 j0 = rb == ra ? ja : rb * dpw, j1 = rb == rz ? jz : n;
          if (j0 >= j1) continue;
          if (hs[static_cast<size_t>(rb)] < 0) hs[static_cast<size_t>(rb)] = static_cast<int>(hu.size() / 3);
          hu.insert(hu.end(), {rb, j0, j1});
        }
      }
      const int nseg = static_cast<int>(hu.size() / 3);
      hc[static_cast<size_t>(G)] = nseg;
      hs[static_cast<size_t>(nrb)] = nseg;
      for (i64 rb = nrb - 1; rb >= 0; --rb)
        if (hs[static_cast<size_t>(rb)] < 0) hs[static_cast<size_t>(rb)] = hs[static_cast<size_t>(rb + 1)];
      units.alloc(3 * static_cast<i64>(nseg), ctx.stream);
      cseg.alloc(G + 1, ctx.stream);
      ustart.alloc(nrb + 1, ctx.stream);
      NPCG_CUDA(cudaMemcpyAsync(units.p, hu.data(), sizeof(i64) * hu.size(), cudaMemcpyHostToDevice, ctx.stream));
      NPCG_CUDA(cudaMemcpyAsync(cseg.p, hc.data(), sizeof(int) * hc.size(), cudaMemcpyHostToDevice, ctx.stream));
      NPCG_CUDA(cudaMemcpyAsync(ustart.p, hs.data(), sizeof(int) * hs.size(), cudaMemcpyHostToDevice, ctx.stream));
      part.alloc(static_cast<i64>(nseg) * S * dpw, ctx.stream);
      colpart.alloc(nrb * S * pstride, ctx.stream);
      if (S == 1) pil.alloc(2 * n, ctx.stream);
      ctx.sync();  // host staging vectors go out of scope
    } else {
      ncb = std::max<i64>(1, G / nrb);
      cpb = cdiv(n, ncb);
      ncb = cdiv(n, cpb);
      part.alloc(ncb * S * pstride, ctx.stream);
    }
  }
  if (nys) T.alloc(pre->ell * S, ctx.stream);
  PersistArgs pa{};
  pa.n = n;
  for (i64 s = 0; s < kMaxS; ++s) pa.mus[s] = cols && s < S ? cols->mu[static_cast<size_t>(s)] : mu;
  DBuf<double> gains;  // several preconditioners in one batch: their gains side by side (ell x S)
  if (gram) {
    pa.m = gram->m;
    pa.A = gram->xr.p();
    pa.lda = gram->xr.ld;
    pa.div = gram->div;
    pa.rows_per_cta = cdiv(gram->m, G);
  } else {
    pa.A = dense->a.p();
    pa.lda = dense->a.ld;
    pa.div = 1.0;
  }
  if (nys) {
    pa.U = pre->fac->u.p();
    pa.ldu = pre->fac->u.ld;
    pa.ell = pre->ell;
    pa.gain = pre->gain_inv.p;
    if (cols) {
      gains.alloc(pre->ell * S, ctx.stream);
      for (i64 s = 0; s < S; ++s)
        NPCG_CUDA(cudaMemcpyAsync(gains.p + s * pre->ell, cols->pre[static_cast<size_t>(s)]->gain_inv.p,
                                  sizeof(double) * pre->ell, cudaMemcpyDeviceToDevice, ctx.stream));
      pa.gain = gains.p;
      pa.gstride = pre->ell;
    }
    pa.T = T.p;
    pa.uslice = cdiv(pre->ell, G);
  }
  pa.X = X;
  pa.ldx = ldx;
  pa.R = R.p();
  pa.Z = nys ? Z.p() : nullptr;
  pa.P0 = P.p();
  pa.P1 = P1.p();
  pa.V = V.p();
  pa.ldw = R.ld;
  pa.part = part.p;
  pa.nrb = nrb;
  pa.ncb = ncb;
  pa.cpb = cpb;
  pa.pstride = pstride;
  pa.sym = sym;
  pa.unit = units.p;
  pa.cseg = cseg.p;
  pa.ustart = ustart.p;
  pa.colpart = colpart.p;
  pa.pil = sym && S == 1 ? pil.p : nullptr;
  pa.pv_part = scal.p;
  pa.rr_part = scal.p + G * S;
  pa.rz_part = scal.p + 2 * G * S;
  pa.st = st;
  pa.hist = hist;
  pa.hstride = hstride;
  pa.max_iter = max_iter;
  pa.slice = cdiv(n, G);
  // 1-2 columns: the scalar passes win while U is small (latency); the bulk-copied DMMA passes once it streams from HBM
  pa.pre_dmma = dense && nys && (S >= 3 || static_cast<double>(n) * static_cast<double>(pre->ell) >= 8e6) ? 1 : 0;
  if (const char* f = std::getenv("NPCG_PCG_PRE")) pa.pre_dmma = dense && nys && (S >= 3 || f[0] == 'd') ? 1 : 0;  // diagnostics
  if (dense && pa.pre_dmma) pa.slice = round_up(pa.slice, 8);  // the DMMA path bulk-copies U on the slice's rows (16-byte aligned)
  if (P.ld != R.ld || V.ld != R.ld || P1.ld != R.ld || (nys && Z.ld != R.ld)) fail(NPCG_ERUNTIME, "pcg: work layout");
  DBuf<unsigned> gbar(1, ctx.stream);
  gbar.zero();
  pa.gbar = gbar.p;
  static const bool tracing = std::getenv("NPCG_PCG_TRACE") != nullptr;  // diagnostics
  DBuf<unsigned long long> tr;
  if (tracing) {
    tr.alloc(8 * 12, ctx.stream);
    tr.zero();
    pa.trace = tr.p;
  }
  const int smem = gram ? 0 : ring_bytes(false, static_cast<int>(S));
  if (gram) launch_persistent<1, true>(ctx, pa, G, smem);
  else if (S == 1) launch_persistent<1, false>(ctx, pa, G, smem);
  else if (S == 2) launch_persistent<2, false>(ctx, pa, G, smem);
  else if (S == 3) launch_persistent<3, false>(ctx, pa, G, smem);
  else if (S == 4) launch_persistent<4, false>(ctx, pa, G, smem);
  else launch_persistent<8, false>(ctx, pa, G, smem);
  ctx.sync();  // work buffers are released on return
  if (tracing) {
    unsigned long long h[8 * 12];
    NPCG_CUDA(cudaMemcpy(h, tr.p, sizeof(h), cudaMemcpyDeviceToHost));
    for (int t = 0; t < 8; ++t) {
      const unsigned long long* q = h + t * 12;
      if (!q[0] || !q[4]) continue;
      std::fprintf(stderr, "[pcg it %d] P1 %.2f s1 %.2f P2 %.2f s2 %.2f P3 %.2f s3 %.2f P4 %.2f s4 %.2f P5 %.2f s5 %.2f "
                   "total %.2f us\n", t + 2, (q[1] - q[0]) * 1e-3, (q[2] - q[1]) * 1e-3, (q[3] - q[2]) * 1e-3,
                   (q[4] - q[3]) * 1e-3, (q[5] - q[4]) * 1e-3, (q[6] - q[5]) * 1e-3, (q[7] - q[6]) * 1e-3,
                   (q[8] - q[7]) * 1e-3, (q[9] - q[8]) * 1e-3, (q[10] - q[9]) * 1e-3, (q[10] - q[0]) * 1e-3);
    }
  }
  if (ctx.prof) {  // algorithmic traffic of the launch: per iteration A once, U twice, ~10 n-vectors
    State h;
    NPCG_CUDA(cudaMemcpy(&h, st, sizeof(State), cudaMemcpyDeviceToHost));
    i64 iters = 0;
    for (i64 s = 0; s < S; ++s) iters = std::max<i64>(iters, h.c[s].iters);
    // bytes the kernel's algorithm streams: X, all of A, or A's block-upper part
    const double a_bytes = gram ? 8.0 * gram->m * n : sym ? 8.0 * sym_entries : 8.0 * n * n;
    const double a_flops = gram ? 4.0 * gram->m * n * S : 2.0 * n * n * S;
    const double u_bytes = nys ? 2.0 * 8.0 * n * pre->ell : 0.0;
    const double u_flops = nys ? 4.0 * n * pre->ell * S : 0.0;
    ctx.prof_work(iters * (a_flops + u_flops + 10.0 * n * S), iters * (a_bytes + u_bytes + 80.0 * n * S));
  }
}

}  // namespace

bool pcg_mu_batch_eligible(Ctx& ctx, Op& op, i64 S) {
  if (ctx.sharded()) return false;
  if (std::getenv("NPCG_PCG") && std::string(std::getenv("NPCG_PCG")) == "classic") return false;
  if (auto* reg = dynamic_cast<RegOp*>(&op)) return false;
  return S == kMaxS && persistent_eligible(ctx, op, S);
}

PcgResult pcg_solve(Ctx& ctx, Op& op, Pre* pre, double mu, i64 S, const double* B, i64 ldb, const double* X0,
                    i64 ldx0, const PcgOptions& opt, double* X, i64 ldx, IterateRec* iterates, const char* context,
                    const PcgMuCols* cols) {
  if (cols) {  // columns with their own shift and preconditioner: the persistent loop only, cold start
    if (X0 || iterates || !pcg_mu_batch_eligible(ctx, op, S) || static_cast<i64>(cols->mu.size()) != S ||
        static_cast<i64>(cols->pre.size()) != S)
      fail(NPCG_ERUNTIME, "pcg_solve: per-column shifts need the persistent loop (8 columns, x0 = 0)");
    pre = cols->pre[0];
    mu = cols->mu[0];
    for (i64 s = 0; s < S; ++s) {
      const Pre* q = cols->pre[static_cast<size_t>(s)];
      if (!q || q->fac.get() != pre->fac.get() || q->ell != pre->ell || q->mu != cols->mu[static_cast<size_t>(s)])
        fail(NPCG_ERUNTIME, "pcg_solve: per-column preconditioners must share one factorisation");
    }
  }
  // cg on RegularizedOperator(base, a) (solvers.cpp:111-120 + operators.cpp:95-98)
  // is nystrom_pcg's loop on base with shift a: the same products, the same
  // rounding (out = base p; out += a p), so the fused kernels apply.
  if (auto* reg = dynamic_cast<RegOp*>(&op); reg && mu == 0.0)
    return pcg_solve(ctx, *reg->base, pre, reg->mu, S, B, ldb, X0, ldx0, opt, X, ldx, iterates, context);
  using Clock = std::chrono::steady_clock;
  const auto t0 = Clock::now();
  if (S < 1 || S > kMaxS) fail(NPCG_EINVAL, "pcg_solve: 1..8 right-hand sides per batch");
  const i64 n = op.nloc;  // this rank's rows of every vector (all of them unsharded)
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
  // Sharded: every dot / norm is this rank's partial; combine() sums the
  // block partials per rank and all-reduces them (bitwise-identical scalars on
  // every rank, so all ranks take the same convergence branch).
  DBuf<double> rsum(2 * S, ctx.stream);
  auto combine = [&](int stride) -> std::pair<const double*, int> {
    if (!ctx.sharded()) return {part.p, nblk};
    NPCG_LAUNCH(ctx, rank_partials_kernel, 1, 32, 0, part.p, nblk, stride, rsum.p);
    rows_allreduce(ctx, rsum.p, stride);
    return {rsum.p, 1};
  };

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
  {
    const auto [pp, nb] = combine(2 * static_cast<int>(S));
    NPCG_LAUNCH(ctx, fin0_kernel, 1, 256, 0, st.p, static_cast<int>(S), pp, nb, opt.eta, opt.relative ? 1 : 0,
                hist.p, hstride);
  }
  DBuf<int> run_flags;
  // iterate record: room for iteration t (doubling growth, zero-filled)
  auto reserve_iterate = [&](i64 t) -> double* {
    if (t >= iterates->cap) {
      const i64 cap = std::min<i64>(opt.max_iter + 1, std::max<i64>({t + 1, 2 * iterates->cap, 16}));
      DBuf<double> nb(cap * n * S, ctx.stream);
      nb.zero();
      if (iterates->cap > 0)
        NPCG_CUDA(cudaMemcpyAsync(nb.p, iterates->buf.p, sizeof(double) * iterates->cap * n * S,
                                  cudaMemcpyDeviceToDevice, ctx.stream));
      iterates->buf = std::move(nb);
      iterates->cap = cap;
    }
    return iterates->buf.p + t * n * S;
  };
  if (iterates) {
    run_flags.alloc(S, ctx.stream);
    NPCG_LAUNCH(ctx, record_kernel, nblk, 256, 0, n, static_cast<int>(S), X, ldx, reserve_iterate(0), st.p,
                static_cast<const int*>(nullptr));
  }
  // z = P^{-1} r; p = z; rz = r.z
  if (!identity && cols) {  // runs of columns with the same preconditioner
    for (i64 s0 = 0; s0 < S;) {
      i64 s1 = s0 + 1;
      while (s1 < S && cols->pre[static_cast<size_t>(s1)] == cols->pre[static_cast<size_t>(s0)]) ++s1;
      pre_apply_inverse(*cols->pre[static_cast<size_t>(s0)], R.p() + s0 * R.ld, R.ld, s1 - s0, Z.p() + s0 * Z.ld, Z.ld,
                        gate);
      s0 = s1;
    }
  } else if (!identity) {
    pre_apply_inverse(*pre, R.p(), R.ld, S, Z.p(), Z.ld, gate);
  }
  NPCG_LAUNCH(ctx, dot_kernel, nblk, 256, 0, n, static_cast<int>(S), R.p(), R.ld, Zp, ldz, P.p(), P.ld, st.p, part.p);
  {
    const auto [pp, nb] = combine(static_cast<int>(S));
    NPCG_LAUNCH(ctx, fin_dot_kernel, 1, 256, 0, st.p, static_cast<int>(S), pp, nb, 0, 0);
  }

  if (!iterates && persistent_eligible(ctx, op, S) && !(std::getenv("NPCG_PCG") && std::string(std::getenv("NPCG_PCG")) == "classic")) {
    run_persistent(ctx, op, pre, mu, cols, S, X, ldx, R, Z, P, V, st.p, hist.p, hstride, opt.max_iter);
  } else {
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
      {
        const auto [pp, nb] = combine(static_cast<int>(S));
        NPCG_LAUNCH(ctx, fin_dot_kernel, 1, 256, 0, st.p, static_cast<int>(S), pp, nb, 1, static_cast<int>(t));
      }
      NPCG_LAUNCH(ctx, update_kernel, nblk, 256, 0, n, static_cast<int>(S), X, ldx, P.p(), P.ld, V.p(), V.ld, R.p(),
                  R.ld, st.p, part.p);
      {
        const auto [pp, nb] = combine(static_cast<int>(S));
        NPCG_LAUNCH(ctx, fin_res_kernel, 1, 256, 0, st.p, static_cast<int>(S), pp, nb, static_cast<int>(t),
                    opt.max_iter, hist.p, hstride);
      }
      if (iterates)
        NPCG_LAUNCH(ctx, record_kernel, nblk, 256, 0, n, static_cast<int>(S), X, ldx, reserve_iterate(t), st.p,
                    run_flags.p);
      if (!identity) pre_apply_inverse(*pre, R.p(), R.ld, S, Z.p(), Z.ld, gate);
      NPCG_LAUNCH(ctx, dot_kernel, nblk, 256, 0, n, static_cast<int>(S), R.p(), R.ld, Zp, ldz,
                  static_cast<double*>(nullptr), 0, st.p, part.p);
      {
        const auto [pp, nb] = combine(static_cast<int>(S));
        NPCG_LAUNCH(ctx, fin_dot_kernel, 1, 256, 0, st.p, static_cast<int>(S), pp, nb, 2, static_cast<int>(t));
      }
      NPCG_LAUNCH(ctx, pupdate_kernel, nblk, 256, 0, n, static_cast<int>(S), P.p(), P.ld, Zp, ldz, st.p);
      enqueue_snapshot(t);
      const i64 depth = op.costly() ? 1 : kDepth;  // no overshoot products when one product is expensive
      if (t > depth && finished(t - depth)) done = true;
    }
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
