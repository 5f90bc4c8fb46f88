// FP64 GEMM on the B200 tensor pipe (DMMA) fed by TMA — see gemm.cuh.
//
// CTA tile 128x128x16, 5-stage smem ring (32 KB/stage), warp-specialised:
// warp 8 (one elected lane) issues cp.async.bulk.tensor loads with
// 128-byte swizzle and arms the stage's mbarrier with expect_tx; warps 0-7
// each own a 64x32 accumulator block (8x4 m8n8 fragments, 64 FP64 regs) and
// issue mma.sync.m8n8k4.f64. Fragment reads are 16-byte LDS that hit all 32
// banks once per 128 B (the swizzle + a k-pair / m-pair register mapping
// makes every fragment load conflict-free for both K-major and M-major
// operands, so all four transpose combinations run at the same speed).
// Small output grids split K across CTAs; partials are summed in fixed order.
#include <cuda.h>

#include <algorithm>
#include <mutex>

#include "gemm.cuh"

namespace npcg {
namespace {

constexpr int BM = 128, BN = 128, BK = 16, STAGES = 5, NCW = 8;
constexpr int THREADS = (NCW + 1) * 32;
constexpr int A_BYTES = BM * BK * 8;
constexpr int B_BYTES = BN * BK * 8;
constexpr int STAGE_BYTES = A_BYTES + B_BYTES;
constexpr int SMEM_BYTES = STAGES * STAGE_BYTES + 1024 + 2 * STAGES * 8;

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

template <bool AK, bool BKM>
__global__ void __launch_bounds__(THREADS, 1)
    gemm_dmma_kernel(const __grid_constant__ CUtensorMap mapA, const __grid_constant__ CUtensorMap mapB,
                     int M, int N, int ktiles, int ktiles_per_split, double alpha, double beta,
                     double* __restrict__ C, i64 ldc, double* __restrict__ partial) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + STAGES * STAGE_BYTES);
  uint64_t* empty = full + STAGES;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int m0 = blockIdx.x * BM, n0 = blockIdx.y * BN, split = blockIdx.z;
  const int kt0 = split * ktiles_per_split;
  const int nk = max(0, min(kt0 + ktiles_per_split, ktiles) - kt0);

  if (threadIdx.x == 0) {
    for (int s = 0; s < STAGES; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], NCW);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();

  if (warp == NCW) {  // ---- TMA producer
    if (lane == 0) {
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

  // ---- DMMA consumers: warp (wm, wn) owns rows wm*64.., cols wn*32..
  const int wm = warp >> 2, wn = warp & 3;
  const int g = lane >> 2, t = lane & 3;
  double acc[8][4][2];
#pragma unroll
  for (int i = 0; i < 8; ++i)
#pragma unroll
    for (int j = 0; j < 4; ++j) acc[i][j][0] = acc[i][j][1] = 0.0;

  for (int i = 0; i < nk; ++i) {
    const int s = i % STAGES, r = i / STAGES;
    mbar_wait(&full[s], r & 1);
    const uint8_t* As = smem + s * STAGE_BYTES;
    const uint8_t* Bs = As + A_BYTES;
#pragma unroll
    for (int kc = 0; kc < 2; ++kc) {
      double a[8][2], b[4][2];
      if (AK) {  // [m][16 k] rows of 128 B; k-pair (2t, 2t+1) -> steps 0/1
#pragma unroll
        for (int f = 0; f < 8; ++f) {
          const int m = wm * 64 + f * 8 + g;
          const double2 v = lds128(As + m * 128 + (((kc * 4 + t) ^ g) << 4));
          a[f][0] = v.x;
          a[f][1] = v.y;
        }
      } else {  // slabs of [16 k][16 m]; m-pair (2g, 2g+1) -> fragments 2p / 2p+1, k = 8kc + 2t + ss
#pragma unroll
        for (int ss = 0; ss < 2; ++ss) {
          const int k = kc * 8 + 2 * t + ss;  // same k <-> (lane, step) map as the K-major path
#pragma unroll
          for (int p = 0; p < 4; ++p) {
            const double2 v = lds128(As + (wm * 4 + p) * 2048 + k * 128 + ((g ^ (k & 7)) << 4));
            a[2 * p][ss] = v.x;
            a[2 * p + 1][ss] = v.y;
          }
        }
      }
      if (BKM) {
#pragma unroll
        for (int f = 0; f < 4; ++f) {
          const int n = wn * 32 + f * 8 + g;
          const double2 v = lds128(Bs + n * 128 + (((kc * 4 + t) ^ g) << 4));
          b[f][0] = v.x;
          b[f][1] = v.y;
        }
      } else {
#pragma unroll
        for (int ss = 0; ss < 2; ++ss) {
          const int k = kc * 8 + 2 * t + ss;
#pragma unroll
          for (int p = 0; p < 2; ++p) {
            const double2 v = lds128(Bs + (wn * 2 + p) * 2048 + k * 128 + ((g ^ (k & 7)) << 4));
            b[2 * p][ss] = v.x;
            b[2 * p + 1][ss] = v.y;
          }
        }
      }
#pragma unroll
      for (int ss = 0; ss < 2; ++ss)
#pragma unroll
        for (int f = 0; f < 8; ++f)
#pragma unroll
          for (int j = 0; j < 4; ++j) dmma(acc[f][j][0], acc[f][j][1], a[f][ss], b[j][ss]);
    }
    __syncwarp();
    if (lane == 0) mbar_arrive(&empty[s]);
  }

  // ---- epilogue
#pragma unroll
  for (int f = 0; f < 8; ++f) {
    const int row = AK ? wm * 64 + f * 8 + g : wm * 64 + (f >> 1) * 16 + 2 * g + (f & 1);
    const int gm = m0 + row;
    if (gm >= M) continue;
#pragma unroll
    for (int j = 0; j < 4; ++j)
#pragma unroll
      for (int e = 0; e < 2; ++e) {
        const int x = 2 * t + e;
        const int col = BKM ? wn * 32 + j * 8 + x : wn * 32 + (j >> 1) * 16 + 2 * x + (j & 1);
        const int gn = n0 + col;
        if (gn >= N) continue;
        if (partial) {
          partial[(static_cast<i64>(split) * N + gn) * M + gm] = acc[f][j][e];
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

template <bool AK, bool BKM>
void launch(Ctx& ctx, const CUtensorMap& ma, const CUtensorMap& mb, int M, int N, int ktiles, int kps,
            int splits, double alpha, double beta, double* C, i64 ldc, double* partial) {
  static std::once_flag once;
  std::call_once(once, [] {
    NPCG_CUDA(cudaFuncSetAttribute(gemm_dmma_kernel<AK, BKM>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                   SMEM_BYTES));
  });
  dim3 grid(static_cast<unsigned>(cdiv(M, BM)), static_cast<unsigned>(cdiv(N, BN)), static_cast<unsigned>(splits));
  NPCG_LAUNCH(ctx, (gemm_dmma_kernel<AK, BKM>), grid, THREADS, SMEM_BYTES, ma, mb, M, N, ktiles, kps,
              alpha, beta, C, ldc, partial);
}

}  // namespace

void gemm(Ctx& ctx, i64 M, i64 N, i64 K, double alpha, Operand A, Operand B, double beta, double* C,
          i64 ldc) {
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
  const CUtensorMap ma = A.kmajor ? make_map(ctx, A.p, K, M, A.ld, BM) : make_map(ctx, A.p, M, K, A.ld, 16);
  const CUtensorMap mb = B.kmajor ? make_map(ctx, B.p, K, N, B.ld, BN) : make_map(ctx, B.p, N, K, B.ld, 16);
  const int ktiles = static_cast<int>(cdiv(K, BK));
  const i64 tiles = cdiv(M, BM) * cdiv(N, BN);
  int splits = 1;
  if (tiles < ctx.sm_count && ktiles >= 16) {
    splits = static_cast<int>(std::max<i64>(1, std::min<i64>(ctx.sm_count / tiles, ktiles / 8)));
  }
  const int kps = static_cast<int>(cdiv(ktiles, splits));
  splits = static_cast<int>(cdiv(ktiles, kps));
  DBuf<double> part;
  double* pp = nullptr;
  if (splits > 1) {
    part.alloc(static_cast<i64>(splits) * M * N, ctx.stream);
    pp = part.p;
  }
  const int m = static_cast<int>(M), n = static_cast<int>(N);
  if (A.kmajor && B.kmajor) launch<true, true>(ctx, ma, mb, m, n, ktiles, kps, splits, alpha, beta, C, ldc, pp);
  else if (A.kmajor) launch<true, false>(ctx, ma, mb, m, n, ktiles, kps, splits, alpha, beta, C, ldc, pp);
  else if (B.kmajor) launch<false, true>(ctx, ma, mb, m, n, ktiles, kps, splits, alpha, beta, C, ldc, pp);
  else launch<false, false>(ctx, ma, mb, m, n, ktiles, kps, splits, alpha, beta, C, ldc, pp);
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
}

}  // namespace npcg
