// FP64 GEMM on the B200 tensor pipe (DMMA) fed by TMA — see gemm.cuh.
//
// CTA tiles 128x128 (8 consumer warps, 64x32 each) or 128x80 (10 warps,
// 64x16 each; N = 400 = 5 x 80 runs without padding), BK = 16, 5-stage smem
// ring, warp-specialised: the last warp (one elected lane) issues
// cp.async.bulk.tensor loads with 128-byte swizzle and arms the stage's
// mbarrier with expect_tx; the consumer warps issue mma.sync.m8n8k4.f64.
// Fragment reads are 16-byte LDS that hit all 32 banks once per 128 B (the
// swizzle + a k-pair / m-pair register mapping makes every fragment load
// conflict-free for both K-major and M-major operands, so all four transpose
// combinations run at the same speed). A wave model picks the tile and the
// split-K count per shape; split partials are summed in fixed order.
#include <cuda.h>

#include <algorithm>
#include <cstdlib>
#include <mutex>

#include "gemm.cuh"

namespace npcg {
namespace {

constexpr int BK = 16;

// CTA tile BM x BN with WM x WN consumer warps (warp tile TM x TN of m8n8
// fragments) plus one TMA producer warp.
template <int BM_, int BN_, int WM_, int WN_, int STAGES_>
struct Tile {
  static constexpr int BM = BM_, BN = BN_, WM = WM_, WN = WN_, STAGES = STAGES_;
  static constexpr int NCW = WM * WN;
  // Whole consumer warpgroups: the producer gets its own warpgroup and hands
  // its registers to the consumers (setmaxnreg); otherwise a single producer warp.
  static constexpr bool WG = NCW % 4 == 0;
  static constexpr int THREADS = (NCW + (WG ? 4 : 1)) * 32;
  static constexpr int TM = BM / WM, TN = BN / WN, FM = TM / 8, FN = TN / 8;
  static constexpr int A_BYTES = BM * BK * 8, B_BYTES = BN * BK * 8, STAGE_BYTES = A_BYTES + B_BYTES;
  static constexpr int SMEM_BYTES = STAGES * STAGE_BYTES + 1024 + 2 * STAGES * 8;
  static_assert(TM % 16 == 0 && TN % 8 == 0, "warp tile must hold m pairs / whole n fragments");
  static_assert(STAGE_BYTES % 1024 == 0 && A_BYTES % 1024 == 0, "128B-swizzle atoms need 1 KB alignment");
};
using TileWide = Tile<128, 128, 2, 4, 6>;    // 64 x 32 warp tiles, 6 x 32 KB stages
using TileNarrow = Tile<128, 80, 2, 5, 8>;   // 64 x 16 warp tiles, 8 x 26 KB stages; N = 80 k without padding
using TileTall = Tile<256, 80, 4, 2, 5>;     // 64 x 40 warp tiles (odd n-fragment count: K-major B only)

__device__ __forceinline__ uint32_t su32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(su32(bar)), "r"(count));
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(su32(bar)), "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(su32(bar)) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  asm volatile(
      "{\n\t.reg .pred P1;\n\t"
      "LAB_WAIT:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n\t"
      "@P1 bra DONE;\n\t"
      "bra LAB_WAIT;\n\t"
      "DONE:\n\t}" ::"r"(su32(bar)),
      "r"(parity)
      : "memory");
}
__device__ __forceinline__ void tma2d(void* dst, const CUtensorMap* map, uint64_t* bar, int c0, int c1) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes"
      " [%0], [%1, {%3, %4}], [%2];" ::"r"(su32(dst)),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(su32(bar)), "r"(c0), "r"(c1)
      : "memory");
}
__device__ __forceinline__ void dmma(double& c0, double& c1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
               : "+d"(c0), "+d"(c1)
               : "d"(a), "d"(b));
}
__device__ __forceinline__ double2 lds128(const uint8_t* p) {
  return *reinterpret_cast<const double2*>(p);
}

template <class T, bool AK, bool BKM>
__global__ void __launch_bounds__(T::THREADS, 1)
    gemm_dmma_kernel(const __grid_constant__ CUtensorMap mapA, const __grid_constant__ CUtensorMap mapB,
                     int M, int N, int ktiles, int ktiles_per_split, double alpha, double beta,
                     double* __restrict__ C, i64 ldc, double* __restrict__ partial, const GemmEpi epi) {
  constexpr int BM = T::BM, BN = T::BN, NCW = T::NCW, TM = T::TM, TN = T::TN, FM = T::FM, FN = T::FN;
  constexpr int A_BYTES = T::A_BYTES, STAGE_BYTES = T::STAGE_BYTES, STAGES = T::STAGES;
  static_assert(BKM || T::TN % 16 == 0, "N-major B reads n fragments in pairs");
  extern __shared__ uint8_t smem_raw[];
  // 1 KB-aligned ring; offsetting smem_raw (not casting through an integer)
  // keeps the pointer in the shared window, so fragment reads compile to LDS
  // (generic loads are not ordered before the mbarrier arrive that frees a stage).
  uint8_t* smem = smem_raw + ((1024u - (su32(smem_raw) & 1023u)) & 1023u);
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + STAGES * STAGE_BYTES);
  uint64_t* empty = full + STAGES;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int m0 = blockIdx.y * BM, n0 = blockIdx.x * BN, split = blockIdx.z;
  const int kt0 = split * ktiles_per_split;
  const int klim = epi.tri ? min(ktiles, (n0 + BN + BK - 1) / BK) : ktiles;  // triangular B: rows k <= last column
  const int nk = max(0, min(kt0 + ktiles_per_split, klim) - kt0);
  if (epi.sym && n0 + BN <= m0) return;  // Gram product: a tile strictly below the diagonal is mirrored later

  if (threadIdx.x == 0) {
    for (int s = 0; s < STAGES; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], NCW);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();

  if (warp >= NCW) {  // ---- TMA producer
    if constexpr (T::WG) asm volatile("setmaxnreg.dec.sync.aligned.u32 40;");
    if (warp == NCW && lane == 0) {
      for (int i = 0; i < nk; ++i) {
        const int s = i % STAGES, r = i / STAGES;
        if (r > 0) mbar_wait(&empty[s], (r - 1) & 1);
        mbar_expect_tx(&full[s], STAGE_BYTES);
        const int k0 = (kt0 + i) * BK;
        uint8_t* a_dst = smem + s * STAGE_BYTES;
        uint8_t* b_dst = a_dst + A_BYTES;
        if (AK) {
          tma2d(a_dst, &mapA, &full[s], k0, m0);
        } else {
#pragma unroll
          for (int p = 0; p < BM / 16; ++p) tma2d(a_dst + p * 2048, &mapA, &full[s], m0 + p * 16, k0);
        }
        if (BKM) {
          tma2d(b_dst, &mapB, &full[s], k0, n0);
        } else {
#pragma unroll
          for (int p = 0; p < BN / 16; ++p) tma2d(b_dst + p * 2048, &mapB, &full[s], n0 + p * 16, k0);
        }
      }
    }
    return;
  }

  // ---- DMMA consumers: warp (wm, wn) owns rows wm*TM.., cols wn*TN..
  if constexpr (T::WG) asm volatile("setmaxnreg.inc.sync.aligned.u32 232;");
  const int wm = warp / T::WN, wn = warp % T::WN;
  const int g = lane >> 2, t = lane & 3;
  double acc[FM][FN][2];
#pragma unroll
  for (int i = 0; i < FM; ++i)
#pragma unroll
    for (int j = 0; j < FN; ++j) acc[i][j][0] = acc[i][j][1] = 0.0;

  for (int i = 0; i < nk; ++i) {
    const int s = i % STAGES, r = i / STAGES;
    mbar_wait(&full[s], r & 1);
    const uint8_t* As = smem + s * STAGE_BYTES;
    const uint8_t* Bs = As + A_BYTES;
#pragma unroll
    for (int kc = 0; kc < 2; ++kc) {
      double a[FM][2], b[FN][2];
      if (AK) {  // [m][16 k] rows of 128 B; k-pair (2t, 2t+1) -> steps 0/1
#pragma unroll
        for (int f = 0; f < FM; ++f) {
          const int m = wm * TM + f * 8 + g;
          const double2 v = lds128(As + m * 128 + (((kc * 4 + t) ^ g) << 4));
          a[f][0] = v.x;
          a[f][1] = v.y;
        }
      } else {  // slabs of [16 k][16 m]; m-pair (2g, 2g+1) -> fragments 2p / 2p+1, k = 8kc + 2t + ss
#pragma unroll
        for (int ss = 0; ss < 2; ++ss) {
          const int k = kc * 8 + 2 * t + ss;  // same k <-> (lane, step) map as the K-major path
#pragma unroll
          for (int p = 0; p < FM / 2; ++p) {
            const double2 v = lds128(As + (wm * (TM / 16) + p) * 2048 + k * 128 + ((g ^ (k & 7)) << 4));
            a[2 * p][ss] = v.x;
            a[2 * p + 1][ss] = v.y;
          }
        }
      }
      if (BKM) {
#pragma unroll
        for (int f = 0; f < FN; ++f) {
          const int n = wn * TN + f * 8 + g;
          const double2 v = lds128(Bs + n * 128 + (((kc * 4 + t) ^ g) << 4));
          b[f][0] = v.x;
          b[f][1] = v.y;
        }
      } else {
#pragma unroll
        for (int ss = 0; ss < 2; ++ss) {
          const int k = kc * 8 + 2 * t + ss;
#pragma unroll
          for (int p = 0; p < FN / 2; ++p) {
            const double2 v = lds128(Bs + (wn * (TN / 16) + p) * 2048 + k * 128 + ((g ^ (k & 7)) << 4));
            b[2 * p][ss] = v.x;
            b[2 * p + 1][ss] = v.y;
          }
        }
      }
#pragma unroll
      for (int ss = 0; ss < 2; ++ss)
#pragma unroll
        for (int f = 0; f < FM; ++f)
#pragma unroll
          for (int j = 0; j < FN; ++j) dmma(acc[f][j][0], acc[f][j][1], a[f][ss], b[j][ss]);
    }
    __syncwarp();
    if (lane == 0) mbar_arrive(&empty[s]);
  }

  // ---- epilogue
#pragma unroll
  for (int f = 0; f < FM; ++f) {
    const int row = AK ? wm * TM + f * 8 + g : wm * TM + (f >> 1) * 16 + 2 * g + (f & 1);
    const int gm = m0 + row;
    if (gm >= M) continue;
#pragma unroll
    for (int j = 0; j < FN; ++j)
#pragma unroll
      for (int e = 0; e < 2; ++e) {
        const int x = 2 * t + e;
        const int col = BKM ? wn * TN + j * 8 + x : wn * TN + (j >> 1) * 16 + 2 * x + (j & 1);
        const int gn = n0 + col;
        if (gn >= N) continue;
        if (partial) {
          partial[(static_cast<i64>(split) * N + gn) * M + gm] = acc[f][j][e];
        } else if (epi.norms) {  // Gaussian kernel entry from -2 x_i.x_j: (-2 x.x + n_i) + n_j, the reference's order
          double v = alpha * acc[f][j][e];
          v = v + epi.norms[gm];
          v = v + epi.norms[gn];
          C[gm + static_cast<i64>(gn) * ldc] = gm == gn ? 1.0 : exp(fmax(v, 0.0) * epi.c);
        } else {
          double* cp = C + gm + static_cast<i64>(gn) * ldc;
          *cp = beta == 0.0 ? alpha * acc[f][j][e] : alpha * acc[f][j][e] + beta * *cp;
        }
      }
  }
}

__global__ void splitk_reduce_kernel(const double* __restrict__ partial, int splits, int M, int N,
                                     double alpha, double beta, double* __restrict__ C, i64 ldc) {
  const i64 idx = static_cast<i64>(blockIdx.x) * blockDim.x + threadIdx.x;
  const i64 total = static_cast<i64>(M) * N;
  if (idx >= total) return;
  const int m = static_cast<int>(idx % M), n = static_cast<int>(idx / M);
  double s = 0.0;
  for (int k = 0; k < splits; ++k) s += partial[static_cast<i64>(k) * total + idx];
  double* cp = C + m + static_cast<i64>(n) * ldc;
  *cp = beta == 0.0 ? alpha * s : alpha * s + beta * *cp;
}

// Gram product: strict lower triangle from the upper one
__global__ void mirror_upper_kernel(double* __restrict__ C, int n, i64 ldc) {
  const i64 idx = static_cast<i64>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (idx >= static_cast<i64>(n) * n) return;
  const int i = static_cast<int>(idx % n), j = static_cast<int>(idx / n);
  if (i > j) C[i + static_cast<i64>(j) * ldc] = C[j + static_cast<i64>(i) * ldc];
}

// 2D FP64 tensor map: inner dimension `inner` (contiguous), outer `outer`,
// row pitch ld doubles, box (16 x box_outer), 128-byte swizzle, OOB -> 0.
CUtensorMap make_map(Ctx& ctx, const double* p, i64 inner, i64 outer, i64 ld, int box_outer) {
  CUtensorMap m;
  cuuint64_t dims[2] = {static_cast<cuuint64_t>(std::max<i64>(inner, 1)),
                        static_cast<cuuint64_t>(std::max<i64>(outer, 1))};
  cuuint64_t strides[1] = {static_cast<cuuint64_t>(ld) * 8};
  cuuint32_t box[2] = {16, static_cast<cuuint32_t>(box_outer)};
  cuuint32_t estr[2] = {1, 1};
  CUresult r = ctx.encode_tiled(&m, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 2, const_cast<double*>(p), dims,
                                strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
                                CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                                CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS)
    fail(NPCG_ECUDA, "cuTensorMapEncodeTiled failed (" + std::to_string(static_cast<int>(r)) + ")");
  return m;
}

template <class T, bool AK, bool BKM>
void launch(Ctx& ctx, const CUtensorMap& ma, const CUtensorMap& mb, int M, int N, int ktiles, int kps,
            int splits, double alpha, double beta, double* C, i64 ldc, double* partial, GemmEpi epi) {
  static std::once_flag once;
  std::call_once(once, [] {
    NPCG_CUDA(cudaFuncSetAttribute(gemm_dmma_kernel<T, AK, BKM>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                   T::SMEM_BYTES));
  });
  // n-tiles fastest: the CTAs that share an A row block run together (A is read once from HBM)
  dim3 grid(static_cast<unsigned>(cdiv(N, T::BN)), static_cast<unsigned>(cdiv(M, T::BM)),
            static_cast<unsigned>(splits));
  NPCG_LAUNCH(ctx, (gemm_dmma_kernel<T, AK, BKM>), grid, T::THREADS, T::SMEM_BYTES, ma, mb, M, N, ktiles, kps,
              alpha, beta, C, ldc, partial, epi);
}

// Tile shape + split-K count minimising a wave model of the launch: every CTA
// of a wave runs kps k-tiles at the per-SM DMMA rate (narrow tiles a little
// slower: less fragment reuse), plus a fixed pipeline fill / epilogue cost and,
// when split, the fixed-order reduction of the partials through HBM.
enum TileKind { kWide = 0, kNarrow = 1, kTall = 2 };
struct Plan {
  TileKind tile;
  int splits, kps;
};
Plan plan_gemm(const Ctx& ctx, i64 M, i64 N, i64 K, bool b_kmajor, bool sym) {
  const int ktiles = static_cast<int>(cdiv(K, BK));
  const double sm_rate = 36e12 / 148.0;  // measured DMMA flop/s per SM (wide tile, 8192^3)
  Plan best{kWide, 1, ktiles};
  double best_us = 1e300;
  for (int tk = 0; tk < 3; ++tk) {
    if (tk == kTall && !b_kmajor) continue;
    const int bm = tk == kWide ? TileWide::BM : tk == kNarrow ? TileNarrow::BM : TileTall::BM;
    const int bn = tk == kWide ? TileWide::BN : tk == kNarrow ? TileNarrow::BN : TileTall::BN;
    const double eff = tk == kNarrow ? 0.83 : 1.0;  // measured at 8192^3: 30.1 vs 36.1 TF/s
    i64 tiles = cdiv(M, bm) * cdiv(N, bn);
    if (sym) {  // tiles that reach the diagonal or lie above it
      tiles = 0;
      for (i64 tm = 0; tm < cdiv(M, bm); ++tm)
        for (i64 tn = 0; tn < cdiv(N, bn); ++tn) tiles += (tn + 1) * bn > tm * bm;
    }
    const int max_split = std::max(1, std::min(64, ktiles / 4));
    for (int s = 1; s <= max_split; ++s) {
      const int kps = static_cast<int>(cdiv(ktiles, s));
      const int se = static_cast<int>(cdiv(ktiles, kps));
      if (se != s) continue;
      const i64 waves = cdiv(tiles * se, ctx.sm_count);
      double us = waves * (kps * 2.0 * bm * bn * BK / (sm_rate * eff) * 1e6 + 4.0);
      if (se > 1) us += (se + 2.0) * M * N * 8.0 / 6e12 * 1e6 + 3.0;
      if (us < best_us * 0.999) {
        best_us = us;
        best = Plan{static_cast<TileKind>(tk), se, kps};
      }
    }
  }
  if (const char* f = std::getenv("NPCG_GEMM_FORCE")) {  // diagnostics: "<w|n|t>:<splits>"
    const int s = std::max(1, std::min(ktiles, std::atoi(f + 2)));
    best.tile = f[0] == 'n' ? kNarrow : (f[0] == 't' && b_kmajor) ? kTall : kWide;
    best.kps = static_cast<int>(cdiv(ktiles, s));
    best.splits = static_cast<int>(cdiv(ktiles, best.kps));
  }
  return best;
}

template <class T>
void dispatch(Ctx& ctx, Operand A, Operand B, int m, int n, i64 K, int ktiles, int kps, int splits, double alpha,
              double beta, double* C, i64 ldc, double* pp, GemmEpi epi) {
  const CUtensorMap ma = A.kmajor ? make_map(ctx, A.p, K, m, A.ld, T::BM) : make_map(ctx, A.p, m, K, A.ld, 16);
  const CUtensorMap mb = B.kmajor ? make_map(ctx, B.p, K, n, B.ld, T::BN) : make_map(ctx, B.p, n, K, B.ld, 16);
  if constexpr (T::TN % 16 == 0) {
    if (A.kmajor && B.kmajor) launch<T, true, true>(ctx, ma, mb, m, n, ktiles, kps, splits, alpha, beta, C, ldc, pp, epi);
    else if (A.kmajor) launch<T, true, false>(ctx, ma, mb, m, n, ktiles, kps, splits, alpha, beta, C, ldc, pp, epi);
    else if (B.kmajor) launch<T, false, true>(ctx, ma, mb, m, n, ktiles, kps, splits, alpha, beta, C, ldc, pp, epi);
    else launch<T, false, false>(ctx, ma, mb, m, n, ktiles, kps, splits, alpha, beta, C, ldc, pp, epi);
  } else {
    if (!B.kmajor) fail(NPCG_ERUNTIME, "gemm: tile needs a K-major B operand");
    if (A.kmajor) launch<T, true, true>(ctx, ma, mb, m, n, ktiles, kps, splits, alpha, beta, C, ldc, pp, epi);
    else launch<T, false, true>(ctx, ma, mb, m, n, ktiles, kps, splits, alpha, beta, C, ldc, pp, epi);
  }
}

}  // namespace

void gemm(Ctx& ctx, i64 M, i64 N, i64 K, double alpha, Operand A, Operand B, double beta, double* C,
          i64 ldc, GemmEpi epi) {
  if (epi.norms && (beta != 0.0 || K <= 0)) invalid("gemm: the kernel epilogue needs beta = 0 and K > 0");
  if (M <= 0 || N <= 0) return;
  if (M > INT32_MAX || N > INT32_MAX) invalid("gemm: dimension too large");
  if (K <= 0) {  // C = beta C
    if (beta == 1.0) return;
    // reuse the reduce kernel with zero splits: C = beta*C (or 0)
    const i64 total = M * N;
    NPCG_LAUNCH(ctx, splitk_reduce_kernel, static_cast<unsigned>(cdiv(total, 256)), 256, 0,
                static_cast<const double*>(nullptr), 0, static_cast<int>(M), static_cast<int>(N), alpha,
                beta, C, ldc);
    return;
  }
  const int ktiles = static_cast<int>(cdiv(K, BK));
  if (epi.sym && (M != N || beta != 0.0 || epi.norms)) invalid("gemm: the Gram form needs M = N, beta = 0 and no kernel epilogue");
  Plan plan = plan_gemm(ctx, M, N, K, B.kmajor, epi.sym);
  if (epi.norms || epi.tri) {  // the kernel epilogue runs on whole dot products, the triangular K range is per tile: no split-K
    plan.splits = 1;
    plan.kps = ktiles;
  }
  const int splits = plan.splits, kps = plan.kps;
  DBuf<double> part;
  double* pp = nullptr;
  if (splits > 1) {
    part.alloc(static_cast<i64>(splits) * M * N, ctx.stream);
    pp = part.p;
  }
  const int m = static_cast<int>(M), n = static_cast<int>(N);
  if (plan.tile == kNarrow) dispatch<TileNarrow>(ctx, A, B, m, n, K, ktiles, kps, splits, alpha, beta, C, ldc, pp, epi);
  else if (plan.tile == kTall) dispatch<TileTall>(ctx, A, B, m, n, K, ktiles, kps, splits, alpha, beta, C, ldc, pp, epi);
  else dispatch<TileWide>(ctx, A, B, m, n, K, ktiles, kps, splits, alpha, beta, C, ldc, pp, epi);
  ctx.prof_work(2.0 * static_cast<double>(M) * N * K, 8.0 * (static_cast<double>(M) * K + static_cast<double>(K) * N +
                                                              static_cast<double>(M) * N));
  if (ctx.prof) {
    const double fl = 2.0 * static_cast<double>(M) * N * K;
    ctx.prof_label(fl >= 1e10 ? "gemm_dmma_kernel[" + std::to_string(M) + "x" + std::to_string(N) + "x" +
                                    std::to_string(K) + "]"
                              : fl >= 1e8 ? "gemm_dmma_kernel[medium]" : "gemm_dmma_kernel[small]");
  }
  if (splits > 1) {
    const i64 total = M * N;
    NPCG_LAUNCH(ctx, splitk_reduce_kernel, static_cast<unsigned>(cdiv(total, 256)), 256, 0, pp, splits, m, n,
                alpha, beta, C, ldc);
  }
  if (epi.sym)
    NPCG_LAUNCH(ctx, mirror_upper_kernel, static_cast<unsigned>(cdiv(M * N, 256)), 256, 0, C, m, ldc);
}

}  // namespace npcg
