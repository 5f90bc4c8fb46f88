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
                       int8_t* __restrict__ D, int* __restrict__ E, double* __restrict__ S) {
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
    if (threadIdx.x == 0) {
      E[r] = e;
      S[r] = ldexp(1.0, e);
    }
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
      for (int t = 0; t < NS; ++t) __stcs(out + t * pw + k0 / 4, w[t]);  // streaming: keep the row in L2 for the digit pass
    }
    __syncthreads();  // sh is reused by the next row's maximum
  }
}

// rows of an M-major operand (entry (m, k) at p[m + k*ld]) -> the same K-major
// planes: 32 rows per CTA, lanes run over m (coalesced), warps over k; digits
// are transposed through shared memory in 32 x 128 tiles (one 128-byte plane
// row per store).
constexpr int SPM_THREADS = 256;
__global__ void __launch_bounds__(SPM_THREADS)
    ozaki_split_mmajor_kernel(const double* __restrict__ p, i64 ld, i64 R, i64 K, i64 Kp, i64 plane,
                              int8_t* __restrict__ D, int* __restrict__ E, double* __restrict__ S) {
  __shared__ double wmax[SPM_THREADS / 32][32];
  __shared__ double fsh[2][32];
  __shared__ uint32_t tile[NS][32][33];  // [plane][row][word of 4 digits] (+1: conflict-free rows)
  constexpr int NW = SPM_THREADS / 32;
  constexpr unsigned long long OFF = 0x0102040810204080ull >> 1;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const i64 m = static_cast<i64>(blockIdx.x) * 32 + lane;
  const bool ok = m < R;
  double mx = 0.0;
  if (ok)
    for (i64 k = warp; k < K; k += NW) mx = fmax(mx, fabs(p[m + k * ld]));
  wmax[warp][lane] = mx;
  __syncthreads();
  if (warp == 0) {
    double v = 0.0;
#pragma unroll
    for (int w = 0; w < NW; ++w) v = fmax(v, wmax[w][lane]);
    int e = 0;
    if (v > 0.0) frexp(v, &e);
    if (ok) {
      E[m] = e;
      S[m] = ldexp(1.0, e);
    }
    const int s1 = (55 - e) / 2, s2 = (55 - e) - s1;
    fsh[0][lane] = ldexp(1.0, s1);
    fsh[1][lane] = ldexp(1.0, s2);
  }
  __syncthreads();
  const double f1 = fsh[0][lane], f2 = fsh[1][lane];
  for (i64 k0 = 0; k0 < Kp; k0 += 128) {
    // warp w: k0 + 16w .. +15 (4 words of 4 digits) for row m = lane
#pragma unroll
    for (int wq = 0; wq < 4; ++wq) {
      uint32_t w[NS];
#pragma unroll
      for (int t = 0; t < NS; ++t) w[t] = 0u;
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        const i64 k = k0 + 16 * warp + 4 * wq + q;
        const double v = (ok && k < K) ? p[m + k * ld] : 0.0;
        const unsigned long long X = static_cast<unsigned long long>(__double2ll_rn((v * f1) * f2)) + OFF;
#pragma unroll
        for (int t = 0; t < NS; ++t) {
          const uint32_t u = static_cast<uint32_t>(X >> (7 * (NS - 1 - t))) & (t == 0 ? 0xffu : 0x7fu);
          w[t] |= ((u - 64u) & 0xffu) << (8 * q);
        }
      }
#pragma unroll
      for (int t = 0; t < NS; ++t) tile[t][lane][4 * warp + wq] = w[t];
    }
    __syncthreads();
    // plane t, row r: 32 words (128 bytes) at D + t*plane + (m0 + r)*Kp + k0
    for (int idx = threadIdx.x; idx < NS * 32 * 32; idx += SPM_THREADS) {
      const int wd = idx & 31, r = (idx >> 5) & 31, t = idx >> 10;
      const i64 mr = static_cast<i64>(blockIdx.x) * 32 + r;
      if (mr < R) reinterpret_cast<uint32_t*>(D + t * plane + mr * Kp + k0)[wd] = tile[t][r][wd];
    }
    __syncthreads();
  }
}

// C = beta C + sum_c part[c] in fixed order (chunked K)
__global__ void chunk_sum_kernel(const double* __restrict__ part, int nchunk, i64 M, i64 N, double beta,
                                 double* __restrict__ C, i64 ldc) {
  const i64 total = M * N;
  for (i64 idx = static_cast<i64>(blockIdx.x) * blockDim.x + threadIdx.x; idx < total;
       idx += static_cast<i64>(gridDim.x) * blockDim.x) {
    double s = 0.0;
    for (int c = 0; c < nchunk; ++c) s += part[c * total + idx];
    const i64 i = idx % M, j = idx / M;
    double* cp = C + i + j * ldc;
    *cp = beta == 0.0 ? s : *cp + s;
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
  int nkb, ckb;     // K blocks of every plane pair; blocks per K chunk (a work unit is (chunk, tile))
  int nchunk;       // > 1: chunk c writes the partial C + c * cstride (combined afterwards in fixed order)
  i64 cstride;
  int kb_off_b;     // B's K block = A's K block + kb_off_b (B planes split once over a longer K)
  int g2_hi, g2_lo; // plane sums g2 = g2_hi .. g2_lo (g - 2, 0-based) per unit; A plane t in [0, g2], B plane g2 - t
  const int* EA;    // row exponents of A
  const double* SB; // column factors 2^F_j of B
  double* C;        // FP64 out (mode 0/1) or int32 out (mode 2)
  i64 ldc;
  int mode;         // the unit's first plane sum: 0 C = v, 1 C += v, 2 raw int32; later ones add
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
  const int units = tiles * a.nchunk, NG = a.g2_hi - a.g2_lo + 1;  // sub-tiles (unit, plane sum)
  // unit u: chunk u / tiles (K blocks [c*ckb, min(nkb, (c+1)*ckb))), tile u % tiles (n fastest)
  auto chunk_kb = [&](int u, int& kb0) {
    kb0 = (u / tiles) * a.ckb;
    return min(a.ckb, a.nkb - kb0);
  };

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
    for (int un = blockIdx.x; un < units; un += gridDim.x) {
      const int tile = un % tiles, m0 = (tile / tiles_n) * BM, n0 = (tile % tiles_n) * BN;
      int kb0;
      const int ck = chunk_kb(un, kb0);
      for (int g2 = a.g2_hi; g2 >= a.g2_lo; --g2) {
        const int kiters = (g2 + 1) * ck;
        for (int i = 0; i < kiters; ++i, ++it) {
          const int s = static_cast<int>(it % STAGES);
          if (it >= STAGES) mbarrier_wait_parity(&empty[s], ((it / STAGES) - 1) & 1u);
          if (lane == 0) {
            const int t = i / ck, u = g2 - t, kb = kb0 + i % ck;
            uint8_t* sa = smem + s * STAGE_BYTES;
            mbarrier_expect_tx(&full[s], STAGE_BYTES);
            tma3d(sa, &mapA, &full[s], kb * BKB, m0, t);
            tma3d(sa + A_TILE, &mapB, &full[s], (kb + a.kb_off_b) * BKB, n0, u);
          }
          __syncwarp();
        }
      }
    }
  } else if (warp == 1) {  // ---- MMA issuer (the warp waits, one lane issues)
    uint32_t it = 0, lt = 0;
    for (int sub = blockIdx.x * NG; sub < units * NG; sub += (sub % NG == NG - 1) ? (gridDim.x - 1) * NG + 1 : 1, ++lt) {
      const int un = sub / NG, g2 = a.g2_hi - sub % NG;
      int kb0;
      const int kiters = (g2 + 1) * chunk_kb(un, kb0);
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
    for (int sub = blockIdx.x * NG; sub < units * NG; sub += (sub % NG == NG - 1) ? (gridDim.x - 1) * NG + 1 : 1, ++lt) {
      const int un = sub / NG, g2 = a.g2_hi - sub % NG;
      const int mode = g2 == a.g2_hi ? a.mode : 1;
      const int buf = static_cast<int>(lt & 1u);
      const int tile = un % tiles, m0 = (tile / tiles_n) * BM, n0 = (tile % tiles_n) * BN;
      double* Cu = a.C + static_cast<i64>(un / tiles) * a.cstride;
      mbarrier_wait_parity(&tfull[buf], (lt >> 1) & 1u);
      tc_fence_after();
      const int row = m0 + 32 * q + lane;
      const bool rok = row < a.M;
      // v = P 2^(E_i + F_j - 12 - 7 g2): row factor once per sub-tile, column factor 2^F_j from the split
      const double sr = (mode != 2 && rok) ? ldexp(1.0, a.EA[row] - 12 - 7 * g2) : 0.0;
      for (int c = 0; c < BN / 32; ++c) {
        uint32_t r[32];
        tmem_ld32(tmem + (static_cast<uint32_t>(32 * q) << 16) + static_cast<uint32_t>(buf * BN + 32 * c), r);
        if (!rok) continue;
        const int cb = n0 + 32 * c;
        if (mode == 2) {
#pragma unroll
          for (int j = 0; j < 32; ++j)
            if (cb + j < a.N) reinterpret_cast<int32_t*>(Cu)[row + static_cast<i64>(cb + j) * a.ldc] = static_cast<int32_t>(r[j]);
          continue;
        }
        double* cp = Cu + row + static_cast<i64>(cb) * a.ldc;  // (L2-resident across a fused unit's plane sums)
        double o[32];
        if (mode == 1) {  // all 32 loads in flight before any store (no load-after-store chain)
#pragma unroll
          for (int j = 0; j < 32; ++j) o[j] = cb + j < a.N ? cp[static_cast<i64>(j) * a.ldc] : 0.0;
        }
#pragma unroll
        for (int j = 0; j < 32; ++j) {
          if (cb + j >= a.N) continue;
          const double v = (static_cast<double>(static_cast<int32_t>(r[j])) * a.SB[cb + j]) * sr;
          cp[static_cast<i64>(j) * a.ldc] = mode == 0 ? v : o[j] + v;
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
  const int units = static_cast<int>(cdiv(args.M, BM) * cdiv(args.N, BN)) * args.nchunk;
  const int grid = std::min(units, ctx.sm_count);
  NPCG_LAUNCH(ctx, i8_gemm_kernel, grid, GEMM_THREADS, GEMM_SMEM, ma, mb, args);
}

}  // namespace

void gemm_i8_raw(Ctx& ctx, int M, int N, i64 Kp, const int8_t* A8, const int8_t* B8, int32_t* C32) {
  if (Kp % BKB != 0) invalid("gemm_i8_raw: K must be a multiple of 128");
  const CUtensorMap ma = plane_map(ctx, A8, Kp, M, 1, BM), mb = plane_map(ctx, B8, Kp, N, 1, BN);
  I8Args args{};
  args.M = M;
  args.N = N;
  args.nkb = static_cast<int>(Kp / BKB);
  args.ckb = args.nkb;
  args.nchunk = 1;
  args.g2_hi = 0;
  args.g2_lo = 0;
  args.C = reinterpret_cast<double*>(C32);
  args.ldc = M;
  args.mode = 2;
  launch_i8(ctx, ma, mb, args);
}

void ozaki_split(Ctx& ctx, const double* P, i64 ld, bool kmajor, i64 rows, i64 K, OzakiPlanes& out) {
  out.rows = rows;
  out.K = K;
  out.Kp = round_up(std::max<i64>(K, 1), BKB);
  out.d.alloc(NS * rows * out.Kp, ctx.stream);
  out.e.alloc(rows, ctx.stream);
  out.s.alloc(rows, ctx.stream);
  if (kmajor)
    NPCG_LAUNCH(ctx, ozaki_split_kernel, static_cast<unsigned>(ctx.sm_count), SPLIT_THREADS, 0, P, ld, rows, K, out.Kp,
                rows * out.Kp, out.d.p, out.e.p, out.s.p);
  else
    NPCG_LAUNCH(ctx, ozaki_split_mmajor_kernel, static_cast<unsigned>(cdiv(rows, 32)), SPM_THREADS, 0, P, ld, rows, K,
                out.Kp, rows * out.Kp, out.d.p, out.e.p, out.s.p);
}

bool ozaki_splittable(const double* P, i64 ld, bool kmajor) {
  // the K-major splitter reads rows as 16-byte pairs
  return !kmajor || ((ld & 1) == 0 && (reinterpret_cast<uintptr_t>(P) & 15) == 0);
}

void gemm_ozaki_planes(Ctx& ctx, const OzakiPlanes& A, const OzakiPlanes& B, i64 k_off_b, double beta, double* C,
                       i64 ldc) {
  const i64 M = A.rows, N = B.rows, K = A.K;
  if (M <= 0 || N <= 0) return;
  if (M > INT32_MAX || N > INT32_MAX) invalid("gemm_ozaki: dimension too large");
  if (beta != 0.0 && beta != 1.0) invalid("gemm_ozaki: beta must be 0 or 1");
  if (k_off_b % BKB != 0 || k_off_b + K > B.K) invalid("gemm_ozaki: B planes do not cover the K range");
  // K chunks: int32-safe (<= 511 blocks) and, for few output tiles, enough
  // (chunk, tile) units to fill the SMs in whole waves
  const int nkb = static_cast<int>(A.Kp / BKB);
  const i64 tiles = cdiv(M, BM) * cdiv(N, BN);
  int nchunk = static_cast<int>(cdiv(nkb, KCHUNK / BKB));
  if (tiles < 2 * ctx.sm_count) {
    double best = -1.0;
    for (int nc = nchunk; nc <= 32 && nc <= std::max(1, nkb / 16); ++nc) {
      const i64 units = tiles * nc, waves = cdiv(units, ctx.sm_count);
      const double eff = static_cast<double>(units) / static_cast<double>(waves * ctx.sm_count);
      if (eff > best + 0.02) {
        best = eff;
        nchunk = nc;
      }
    }
  }
  const int ckb = static_cast<int>(cdiv(nkb, nchunk));
  nchunk = static_cast<int>(cdiv(nkb, ckb));
  // K split into int32-safe chunks: each chunk's partial is assembled on its own, then summed in fixed order
  DBuf<double> part;
  if (nchunk > 1) part.alloc(static_cast<i64>(nchunk) * M * N, ctx.stream);
  const CUtensorMap ma = plane_map(ctx, A.d.p, A.Kp, M, NS, BM), mb = plane_map(ctx, B.d.p, B.Kp, N, NS, BN);
  // Plane sums g = NS + 1 .. 2, smallest first. When B's planes fit in L2 each
  // unit runs all of them back to back in one launch (its C tile stays in L2
  // across the additions); otherwise one launch per plane sum, so all CTAs
  // stream the same B planes at the same time (B tiles are shared through L2).
  const bool fused = static_cast<double>(NS) * N * B.Kp < 48.0 * (1 << 20) || static_cast<double>(NS) * N * K < 48.0 * (1 << 20);
  for (int g2 = NS - 1; g2 >= 0; g2 = fused ? -1 : g2 - 1) {
    I8Args args{};
    args.M = static_cast<int>(M);
    args.N = static_cast<int>(N);
    args.nkb = nkb;
    args.ckb = ckb;
    args.nchunk = nchunk;
    args.kb_off_b = static_cast<int>(k_off_b / BKB);
    args.g2_hi = g2;
    args.g2_lo = fused ? 0 : g2;
    args.EA = A.e.p;
    args.SB = B.s.p;
    const bool first = g2 == NS - 1;
    if (nchunk > 1) {
      args.C = part.p;
      args.ldc = M;
      args.cstride = M * N;
      args.mode = first ? 0 : 1;
    } else {
      args.C = C;
      args.ldc = ldc;
      args.mode = (first && beta == 0.0) ? 0 : 1;
    }
    launch_i8(ctx, ma, mb, args);
    if (ctx.prof) ctx.prof_label(fused ? "i8_gemm_kernel[fused]" : "i8_gemm_kernel[per-plane]");
  }
  if (nchunk > 1)
    NPCG_LAUNCH(ctx, chunk_sum_kernel, static_cast<unsigned>(std::min<i64>(cdiv(M * N, 256), 8 * ctx.sm_count)), 256, 0,
                part.p, nchunk, M, N, beta, C, ldc);
  ctx.prof_work(2.0 * static_cast<double>(M) * N * K, 8.0 * (static_cast<double>(M) * K + static_cast<double>(K) * N +
                                                              static_cast<double>(M) * N));
}

void gemm_ozaki(Ctx& ctx, i64 M, i64 N, i64 K, const double* A, i64 lda, bool a_kmajor, const double* B, i64 ldb,
                double beta, double* C, i64 ldc, bool b_kmajor) {
  if (M <= 0 || N <= 0) return;
  if (beta != 0.0 && beta != 1.0) invalid("gemm_ozaki: beta must be 0 or 1");
  if (K <= 0) {
    if (beta == 0.0) NPCG_CUDA(cudaMemset2DAsync(C, ldc * 8, 0, M * 8, N, ctx.stream));
    return;
  }
  if (!ozaki_splittable(A, lda, a_kmajor) || !ozaki_splittable(B, ldb, b_kmajor)) {
    gemm(ctx, M, N, K, 1.0, Operand{A, lda, a_kmajor}, Operand{B, ldb, b_kmajor}, beta, C, ldc);
    return;
  }
  // A in row panels: the planes of one panel (NS bytes per entry) stay within a workspace budget
  const i64 Kp = round_up(K, BKB);
  size_t free_b = 0, total_b = 0;
  NPCG_CUDA(cudaMemGetInfo(&free_b, &total_b));
  const i64 budget = std::max<i64>(i64(1) << 30, std::min<i64>(i64(24) << 30, static_cast<i64>(free_b / 4)));
  i64 prow = std::max<i64>(BM, budget / (NS * Kp) / BM * BM);
  prow = std::min(prow, round_up(M, BM));
  OzakiPlanes bp;
  ozaki_split(ctx, B, ldb, b_kmajor, N, K, bp);
  for (i64 r0 = 0; r0 < M; r0 += prow) {
    const i64 rows = std::min(prow, M - r0);
    OzakiPlanes ap;
    ozaki_split(ctx, a_kmajor ? A + r0 * lda : A + r0, lda, a_kmajor, rows, K, ap);
    gemm_ozaki_planes(ctx, ap, bp, 0, beta, C + r0, ldc);
  }
}

}  // namespace npcg
