// FP64 GEMM on the INT8 tensor cores by digit-plane splitting — see ozaki.cuh.
//
// ozaki_split_kernel: one CTA per operand row (K contiguous): the row maximum,
//   then the NS digit planes as bit fields of one rounded 64-bit fixed-point
//   integer per entry (signed digits by a constant offset),
//   four digits packed per 32-bit store, K padded to a multiple of 128 with 0.
// i8_gemm_kernel: persistent, warp-specialised tcgen05 GEMM. Warp 0 (one
//   lane) streams 128x128 A and 256x128 B int8 tiles into a 4-stage ring by
//   3D TMA (128-byte swizzle) and arms the stage's mbarrier; warp 1 allocates
//   TMEM (2 x 256 columns: the accumulator of the next tile fills while the
//   epilogue drains the last) and one lane issues tcgen05.mma.kind::i8
//   (M = 128, N = 256, K = 32) with shared-memory descriptors, committing each
//   stage back to the producer and each finished tile to the epilogue; warps
//   2-5 move the int32 accumulator out with tcgen05.ld (warp w reads TMEM
//   lanes 32(w%4)..+31 = its 32 rows), scale it by 2^(E_i+F_j-12-7(g-2)) and
//   add it into the FP64 C (coalesced: a warp writes 32 consecutive rows of a
//   column). One launch per digit plane g: its K loop runs over the (A plane t,
//   B plane g-t) pairs back to back.
#include <cuda.h>

#include <algorithm>
#include <cstdlib>
#include <mutex>
#include <string>

#include "async.cuh"
#include "gemm.cuh"
#include "ozaki.cuh"

namespace npcg {
namespace {

constexpr int NS = 8;                 // digit planes per operand
constexpr int BM = 128, BN = 256, BKB = 128;  // tile rows (A), tile rows (B), K bytes per stage
constexpr int STAGES = 4;
constexpr int A_TILE = BM * BKB, B_TILE = BN * BKB, STAGE_BYTES = A_TILE + B_TILE;
constexpr int GEMM_THREADS = 192;     // producer, MMA, 4 epilogue warps
constexpr int GEMM_SMEM = STAGES * STAGE_BYTES + 1024 + 256;
constexpr i64 KCHUNK = 511 * BKB;     // |P_g| <= 8 * 65408 * 64^2 < 2^31

// ---------------------------------------------------------------- splitting
__device__ __forceinline__ double block_max(double v, double* sh) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v = fmax(v, __shfl_xor_sync(0xffffffffu, v, o));
  const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
  if (l == 0) sh[w] = v;
  __syncthreads();
  if (w == 0) {
    v = l < static_cast<int>(blockDim.x >> 5) ? sh[l] : 0.0;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v = fmax(v, __shfl_xor_sync(0xffffffffu, v, o));
    if (l == 0) sh[32] = v;
  }
  __syncthreads();
  return sh[32];
}

// rows of a K-major operand (entry k of row r at p[k + r*ld], 16-byte aligned
// rows) -> planes D[t][r][0..Kp), exponents E[r]. Persistent: one row per CTA
// at a time, one CTA per SM, so the second pass over a row (<= ~0.5 MB) hits L2
// and A crosses HBM once.
constexpr int SPLIT_THREADS = 1024;
__global__ void __launch_bounds__(SPLIT_THREADS, 1)
    ozaki_split_kernel(const double* __restrict__ p, i64 ld, i64 R, i64 K, i64 Kp, i64 plane,
                       int8_t* __restrict__ D, int* __restrict__ E) {
  __shared__ double sh[33];
  const i64 pw = plane / 4;                     // plane stride in 32-bit words
  for (i64 r = blockIdx.x; r < R; r += gridDim.x) {
    const double* row = p + r * ld;
    double m0 = 0.0, m1 = 0.0;
    const i64 K2 = K / 2;
#pragma unroll 4
    for (i64 k = threadIdx.x; k < K2; k += SPLIT_THREADS) {
      const double2 v = reinterpret_cast<const double2*>(row)[k];
      m0 = fmax(m0, fabs(v.x));
      m1 = fmax(m1, fabs(v.y));
    }
    if ((K & 1) && threadIdx.x == 0) m0 = fmax(m0, fabs(row[K - 1]));
    const double m = block_max(fmax(m0, m1), sh);
    int e = 0;
    if (m > 0.0) frexp(m, &e);  // m < 2^e
    if (threadIdx.x == 0) E[r] = e;
    // X = round(a 2^(55-e)) (|X| <= 2^55; two factors keep the scale representable
    // for any e); X + OFF = sum_t u_t 128^(7-t) with 7-bit fields u_t (u_0 the
    // top, 8 bits), so the signed digits d_t = u_t - 64 are plain bit fields
    const int s1 = (55 - e) / 2, s2 = (55 - e) - s1;
    const double f1 = ldexp(1.0, s1), f2 = ldexp(1.0, s2);
    constexpr unsigned long long OFF = 0x0102040810204080ull >> 1;  // 64 * sum_{t<8} 128^t
    uint32_t* out = reinterpret_cast<uint32_t*>(D + r * Kp);
    for (i64 k0 = 4 * static_cast<i64>(threadIdx.x); k0 < Kp; k0 += 4 * SPLIT_THREADS) {
      double v[4];
      if (k0 + 3 < K) {
        const double2 u0 = reinterpret_cast<const double2*>(row + k0)[0], u1 = reinterpret_cast<const double2*>(row + k0)[1];
        v[0] = u0.x; v[1] = u0.y; v[2] = u1.x; v[3] = u1.y;
      } else {
#pragma unroll
        for (int q = 0; q < 4; ++q) v[q] = k0 + q < K ? row[k0 + q] : 0.0;
      }
      uint32_t w[NS];
#pragma unroll
      for (int t = 0; t < NS; ++t) w[t] = 0u;
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        const unsigned long long X = static_cast<unsigned long long>(__double2ll_rn((v[q] * f1) * f2)) + OFF;
#pragma unroll
        for (int t = 0; t < NS; ++t) {
          const uint32_t u = static_cast<uint32_t>(X >> (7 * (NS - 1 - t))) & (t == 0 ? 0xffu : 0x7fu);
          w[t] |= ((u - 64u) & 0xffu) << (8 * q);
        }
      }
#pragma unroll
      for (int t = 0; t < NS; ++t) out[t * pw + k0 / 4] = w[t];
    }
    __syncthreads();  // sh is reused by the next row's maximum
  }
}

// ---------------------------------------------------------------- tcgen05 helpers
__device__ __forceinline__ void tma3d(void* dst, const CUtensorMap* map, uint64_t* bar, int c0, int c1, int c2) {
  asm volatile(
      "cp.async.bulk.tensor.3d.shared::cluster.global.tile.mbarrier::complete_tx::bytes"
      " [%0], [%1, {%3, %4, %5}], [%2];" ::"r"(smem_u32(dst)),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(smem_u32(bar)), "r"(c0), "r"(c1), "r"(c2)
      : "memory");
}
// K-major operand tile, rows of 128 bytes, 128-byte swizzle (8-row atoms 1024 B apart)
__device__ __forceinline__ uint64_t smem_desc(uint32_t saddr) {
  uint64_t d = 0;
  d |= static_cast<uint64_t>((saddr & 0x3FFFFu) >> 4);
  d |= static_cast<uint64_t>(1) << 16;                 // leading byte offset (unused for swizzled K-major)
  d |= static_cast<uint64_t>(1024 >> 4) << 32;         // stride byte offset: next 8-row atom
  d |= static_cast<uint64_t>(1) << 46;                 // descriptor version (sm_100)
  d |= static_cast<uint64_t>(2) << 61;                 // SWIZZLE_128B
  return d;
}
// instruction descriptor: D s32, A/B signed 8-bit, both K-major, N = 256, M = 128
constexpr uint32_t IDESC = (2u << 4) | (1u << 7) | (1u << 10) | (static_cast<uint32_t>(BN >> 3) << 17) |
                           (static_cast<uint32_t>(BM >> 4) << 24);
__device__ __forceinline__ void mma_i8(uint32_t tmem_d, uint64_t ad, uint64_t bd, uint32_t accum) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %3, p;\n\t}" ::"r"(tmem_d),
      "l"(ad), "l"(bd), "r"(IDESC), "r"(accum));
}
__device__ __forceinline__ void mma_commit(uint64_t* bar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_u32(bar))
               : "memory");
}
__device__ __forceinline__ void tc_fence_before() { asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory"); }
__device__ __forceinline__ void tc_fence_after() { asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory"); }
__device__ __forceinline__ void tmem_ld32(uint32_t taddr, uint32_t (&r)[32]) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,"
      "%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
        "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15]),
        "=r"(r[16]), "=r"(r[17]), "=r"(r[18]), "=r"(r[19]), "=r"(r[20]), "=r"(r[21]), "=r"(r[22]), "=r"(r[23]),
        "=r"(r[24]), "=r"(r[25]), "=r"(r[26]), "=r"(r[27]), "=r"(r[28]), "=r"(r[29]), "=r"(r[30]), "=r"(r[31])
      : "r"(taddr));
  asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
}

struct I8Args {
  int M, N;
  int kb0, nkb;     // K blocks [kb0, kb0 + nkb) of every plane pair
  int t_lo, t_hi;   // A planes t_lo..t_hi (0-based), B plane g - 2 - t
  int g2;           // g - 2 (0-based plane sum)
  const int *EA, *EB;
  double* C;        // FP64 out (mode 0/1) or int32 out (mode 2)
  i64 ldc;
  int mode;         // 0: C = v, 1: C += v, 2: raw int32
};

__global__ void __launch_bounds__(GEMM_THREADS, 1)
    i8_gemm_kernel(const __grid_constant__ CUtensorMap mapA, const __grid_constant__ CUtensorMap mapB,
                   const I8Args a) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + STAGES * STAGE_BYTES);
  uint64_t* empty = full + STAGES;
  uint64_t* tfull = empty + STAGES;   // 2 accumulator buffers
  uint64_t* tempty = tfull + 2;
  uint32_t* tmem_base_sh = reinterpret_cast<uint32_t*>(tempty + 2);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int tiles_n = (a.N + BN - 1) / BN, tiles = ((a.M + BM - 1) / BM) * tiles_n;
  const int npairs = a.t_hi - a.t_lo + 1, kiters = npairs * a.nkb;

  if (threadIdx.x == 0) {
    for (int s = 0; s < STAGES; ++s) {
      mbarrier_init(&full[s], 1);
      mbarrier_init(&empty[s], 1);
    }
    for (int b = 0; b < 2; ++b) {
      mbarrier_init(&tfull[b], 1);
      mbarrier_init(&tempty[b], 4);
    }
    mbarrier_fence_init();
  }
  if (warp == 1) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(smem_u32(tmem_base_sh)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_base_sh;

  if (warp == 0) {  // ---- TMA producer (the warp waits, one lane issues)
    uint32_t it = 0;
    for (int tile = blockIdx.x; tile < tiles; tile += gridDim.x) {
      const int m0 = (tile / tiles_n) * BM, n0 = (tile % tiles_n) * BN;
      for (int i = 0; i < kiters; ++i, ++it) {
        const int s = static_cast<int>(it % STAGES);
        if (it >= STAGES) mbarrier_wait_parity(&empty[s], ((it / STAGES) - 1) & 1u);
        if (lane == 0) {
          const int t = a.t_lo + i / a.nkb, u = a.g2 - t, kb = a.kb0 + i % a.nkb;
          uint8_t* sa = smem + s * STAGE_BYTES;
          mbarrier_expect_tx(&full[s], STAGE_BYTES);
          tma3d(sa, &mapA, &full[s], kb * BKB, m0, t);
          tma3d(sa + A_TILE, &mapB, &full[s], kb * BKB, n0, u);
        }
        __syncwarp();
      }
    }
  } else if (warp == 1) {  // ---- MMA issuer (the warp waits, one lane issues)
    uint32_t it = 0, lt = 0;
    for (int tile = blockIdx.x; tile < tiles; tile += gridDim.x, ++lt) {
      const int buf = static_cast<int>(lt & 1u);
      if (lt >= 2) mbarrier_wait_parity(&tempty[buf], ((lt >> 1) - 1) & 1u);
      tc_fence_after();
      const uint32_t d = tmem + static_cast<uint32_t>(buf * BN);
      for (int i = 0; i < kiters; ++i, ++it) {
        const int s = static_cast<int>(it % STAGES);
        mbarrier_wait_parity(&full[s], (it / STAGES) & 1u);
        tc_fence_after();
        if (lane == 0) {
          const uint32_t sa = smem_u32(smem + s * STAGE_BYTES);
          const uint64_t ad = smem_desc(sa), bd = smem_desc(sa + A_TILE);
#pragma unroll
          for (int k = 0; k < BKB / 32; ++k)  // K = 32 bytes per instruction: +2 in the descriptor's address field
            mma_i8(d, ad + 2 * k, bd + 2 * k, (i > 0 || k > 0) ? 1u : 0u);
          mma_commit(&empty[s]);  // the stage is free once these MMAs have read it
        }
        __syncwarp();
      }
      if (lane == 0) mma_commit(&tfull[buf]);  // the accumulator is complete
      __syncwarp();
    }
  } else {  // ---- epilogue: warps 2..5, TMEM lanes 32*(warp%4)..+31
    const int q = warp & 3;
    uint32_t lt = 0;
    for (int tile = blockIdx.x; tile < tiles; tile += gridDim.x, ++lt) {
      const int buf = static_cast<int>(lt & 1u);
      const int m0 = (tile / tiles_n) * BM, n0 = (tile % tiles_n) * BN;
      mbarrier_wait_parity(&tfull[buf], (lt >> 1) & 1u);
      tc_fence_after();
      const int row = m0 + 32 * q + lane;
      const bool rok = row < a.M;
      const int ea = (a.mode != 2 && rok) ? a.EA[row] : 0;
      for (int c = 0; c < BN / 32; ++c) {
        uint32_t r[32];
        tmem_ld32(tmem + (static_cast<uint32_t>(32 * q) << 16) + static_cast<uint32_t>(buf * BN + 32 * c), r);
        if (!rok) continue;
#pragma unroll
        for (int j = 0; j < 32; ++j) {
          const int col = n0 + 32 * c + j;
          if (col >= a.N) continue;
          if (a.mode == 2) {
            reinterpret_cast<int32_t*>(a.C)[row + static_cast<i64>(col) * a.ldc] = static_cast<int32_t>(r[j]);
          } else {
            const double v = ldexp(static_cast<double>(static_cast<int32_t>(r[j])), ea + a.EB[col] - 12 - 7 * a.g2);
            double* cp = a.C + row + static_cast<i64>(col) * a.ldc;
            *cp = a.mode == 0 ? v : *cp + v;
          }
        }
      }
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbarrier_arrive(&tempty[buf]);
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 1) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tmem));
}

// 3D int8 tensor map over planes [planes][rows][Kp], box (128 bytes, box_rows, 1), 128-byte swizzle
CUtensorMap plane_map(Ctx& ctx, const int8_t* p, i64 Kp, i64 rows, int planes, int box_rows) {
  CUtensorMap m;
  cuuint64_t dims[3] = {static_cast<cuuint64_t>(Kp), static_cast<cuuint64_t>(rows), static_cast<cuuint64_t>(planes)};
  cuuint64_t strides[2] = {static_cast<cuuint64_t>(Kp), static_cast<cuuint64_t>(Kp * rows)};
  cuuint32_t box[3] = {static_cast<cuuint32_t>(BKB), static_cast<cuuint32_t>(box_rows), 1};
  cuuint32_t estr[3] = {1, 1, 1};
  CUresult r = ctx.encode_tiled(&m, CU_TENSOR_MAP_DATA_TYPE_UINT8, 3, const_cast<int8_t*>(p), dims, strides, box,
                                estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                                CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS)
    fail(NPCG_ECUDA, "cuTensorMapEncodeTiled (int8 planes) failed (" + std::to_string(static_cast<int>(r)) + ")");
  return m;
}

void launch_i8(Ctx& ctx, const CUtensorMap& ma, const CUtensorMap& mb, const I8Args& args) {
  static std::once_flag once;
  std::call_once(once, [] {
    NPCG_CUDA(cudaFuncSetAttribute(i8_gemm_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, GEMM_SMEM));
  });
  const int tiles = static_cast<int>(cdiv(args.M, BM) * cdiv(args.N, BN));
  const int grid = std::min(tiles, ctx.sm_count);
  NPCG_LAUNCH(ctx, i8_gemm_kernel, grid, GEMM_THREADS, GEMM_SMEM, ma, mb, args);
}

}  // namespace

void gemm_i8_raw(Ctx& ctx, int M, int N, i64 Kp, const int8_t* A8, const int8_t* B8, int32_t* C32) {
  if (Kp % BKB != 0) invalid("gemm_i8_raw: K must be a multiple of 128");
  const CUtensorMap ma = plane_map(ctx, A8, Kp, M, 1, BM), mb = plane_map(ctx, B8, Kp, N, 1, BN);
  I8Args args{};
  args.M = M;
  args.N = N;
  args.kb0 = 0;
  args.nkb = static_cast<int>(Kp / BKB);
  args.t_lo = 0;
  args.t_hi = 0;
  args.g2 = 0;
  args.C = reinterpret_cast<double*>(C32);
  args.ldc = M;
  args.mode = 2;
  launch_i8(ctx, ma, mb, args);
}

void gemm_ozaki(Ctx& ctx, i64 M, i64 N, i64 K, const double* A, i64 lda, const double* B, i64 ldb, double* C,
                i64 ldc) {
  if (M <= 0 || N <= 0) return;
  if (M > INT32_MAX || N > INT32_MAX) invalid("gemm_ozaki: dimension too large");
  if (K <= 0) {
    NPCG_CUDA(cudaMemset2DAsync(C, ldc * 8, 0, M * 8, N, ctx.stream));
    return;
  }
  if (((lda | ldb) & 1) || (reinterpret_cast<uintptr_t>(A) & 15) || (reinterpret_cast<uintptr_t>(B) & 15)) {
    // the splitter reads rows as 16-byte pairs: unaligned operands stay on the FP64 DMMA GEMM
    gemm(ctx, M, N, K, 1.0, Operand{A, lda, true}, Operand{B, ldb, true}, 0.0, C, ldc);
    return;
  }
  const i64 Kp = round_up(K, BKB);
  // A in row panels: the planes of one panel (NS bytes per entry) stay within a workspace budget
  size_t free_b = 0, total_b = 0;
  NPCG_CUDA(cudaMemGetInfo(&free_b, &total_b));
  const i64 budget = std::max<i64>(i64(1) << 30, std::min<i64>(i64(24) << 30, static_cast<i64>(free_b / 4)));
  i64 prow = std::max<i64>(BM, budget / (NS * Kp) / BM * BM);
  prow = std::min(prow, round_up(M, BM));
  DBuf<int8_t> a8(NS * prow * Kp, ctx.stream), b8(NS * N * Kp, ctx.stream);
  DBuf<int> ea(prow, ctx.stream), eb(N, ctx.stream);
  const unsigned sgrid = static_cast<unsigned>(ctx.sm_count);
  NPCG_LAUNCH(ctx, ozaki_split_kernel, sgrid, SPLIT_THREADS, 0, B, ldb, N, K, Kp, N * Kp, b8.p, eb.p);
  const CUtensorMap mb = plane_map(ctx, b8.p, Kp, N, NS, BN);
  const int nkb_all = static_cast<int>(Kp / BKB);
  for (i64 r0 = 0; r0 < M; r0 += prow) {
    const i64 rows = std::min(prow, M - r0);
    NPCG_LAUNCH(ctx, ozaki_split_kernel, sgrid, SPLIT_THREADS, 0, A + r0 * lda, lda, rows, K, Kp, rows * Kp, a8.p,
                ea.p);
    const CUtensorMap ma = plane_map(ctx, a8.p, Kp, rows, NS, BM);
    bool first = true;
    for (int kb0 = 0; kb0 < nkb_all; kb0 += static_cast<int>(KCHUNK / BKB)) {
      const int nkb = std::min(nkb_all - kb0, static_cast<int>(KCHUNK / BKB));
      // smallest planes first: g = NS + 1 .. 2 (0-based plane sum g2 = NS - 1 .. 0)
      for (int g2 = NS - 1; g2 >= 0; --g2) {
        I8Args args{};
        args.M = static_cast<int>(rows);
        args.N = static_cast<int>(N);
        args.kb0 = kb0;
        args.nkb = nkb;
        args.t_lo = 0;
        args.t_hi = g2;
        args.g2 = g2;
        args.EA = ea.p;
        args.EB = eb.p;
        args.C = C + r0;
        args.ldc = ldc;
        args.mode = first ? 0 : 1;
        first = false;
        launch_i8(ctx, ma, mb, args);
      }
    }
  }
  ctx.prof_work(2.0 * static_cast<double>(M) * N * K, 8.0 * (static_cast<double>(M) * K + static_cast<double>(K) * N +
                                                              static_cast<double>(M) * N));
}

}  // namespace npcg
