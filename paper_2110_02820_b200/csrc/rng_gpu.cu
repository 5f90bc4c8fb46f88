// The reference generator on the GPU: the mt19937_64
// word stream continued from a host engine's state (rng.hpp Mt64), bit for bit,
// and the reference's Box-Muller transform (random.cpp:11-18: two words per
// deviate, u1 = (w1 + 1) 2^-64, u2 = w2 2^-64, sqrt(-2 ln u1) cos(2 pi u2),
// column-major fills as gaussian_matrix, random.cpp:27-32).
//
// The engine recurrence is serial across twists, so one CTA owns the stream:
// each twist of the 312-word block runs in two dependent half-phases on 312
// threads (x[k] for k < 156 from the old block, then k >= 156 from the new
// words k - 156), the block is tempered and stored. A second, grid-wide
// kernel turns word pairs into deviates and scatters this rank's rows of each
// column. Words stream through a bounded device buffer in chunks; the engine
// state round-trips through device memory between chunks and is handed back
// to the host engine at the end, so the caller's Rng stands exactly where the
// reference's would after the same draw.
//
// log / cos are CUDA's (max 1 / 2 ulp); the host transform uses libm. Engine
// words are identical; deviates agree to a few ulp.
#include <algorithm>
#include <cmath>
#include <vector>

#include "blas.cuh"
#include "rng.hpp"

namespace npcg {
namespace {

using u64 = unsigned long long;
constexpr int kN = 312, kM = 156;

__device__ __forceinline__ u64 mt_temper(u64 z) {
  z ^= (z >> 29) & 0x5555555555555555ull;
  z ^= (z << 17) & 0x71D67FFFEDA60000ull;
  z ^= (z << 37) & 0xFFF7EEE000000000ull;
  z ^= z >> 43;
  return z;
}
__device__ __forceinline__ u64 mt_mix(u64 a, u64 b, u64 c) {  // c ^ twist(a, b)
  const u64 y = (a & (~0ull << 31)) | (b & ((1ull << 31) - 1));
  return c ^ (y >> 1) ^ ((y & 1ull) ? 0xB5026F5AA96619E9ull : 0ull);
}

// state[0..311] = block, state[312] = p. Writes `count` tempered words to out.
__global__ void __launch_bounds__(320, 1) mt64_stream_kernel(u64* __restrict__ state, i64 count, u64* __restrict__ out) {
  __shared__ u64 blk[2][kN];
  __shared__ int sp;
  const int tid = threadIdx.x;
  int cur = 0;
  for (int k = tid; k < kN; k += blockDim.x) blk[0][k] = state[k];
  if (tid == 0) sp = static_cast<int>(state[kN]);
  __syncthreads();
  int p = sp;
  i64 done = 0;
  while (done < count) {
    if (p >= kN) {  // twist: new block from the old one
      const u64* xo = blk[cur];
      u64* xn = blk[cur ^ 1];
      if (tid < kN - kM) xn[tid] = mt_mix(xo[tid], xo[tid + 1], xo[tid + kM]);
      __syncthreads();
      if (tid >= kN - kM && tid < kN) {
        const u64 b = tid + 1 < kN ? xo[tid + 1] : xn[0];
        xn[tid] = mt_mix(xo[tid], b, xn[tid - (kN - kM)]);
      }
      __syncthreads();
      cur ^= 1;
      p = 0;
    }
    const i64 cnt = std::min<i64>(kN - p, count - done);
    for (int i = tid; i < cnt; i += blockDim.x) out[done + i] = mt_temper(blk[cur][p + i]);
    done += cnt;
    p += static_cast<int>(cnt);
  }
  __syncthreads();
  for (int k = tid; k < kN; k += blockDim.x) state[k] = blk[cur][k];
  if (tid == 0) state[kN] = static_cast<u64>(p);
}

// Deviates d = first .. first + npairs - 1 of the draw from word pairs
// (words[2(d - first)], words[2(d - first) + 1]); deviate d is entry
// (d % rows, d / rows) of the rows x cols block; rows [r0, r0 + rcnt) land in
// dst (ld), row r0 at dst[0].
__global__ void box_muller_kernel(const u64* __restrict__ words, i64 first, i64 npairs, i64 rows, i64 r0, i64 rcnt,
                                  double* __restrict__ dst, i64 ld) {
  for (i64 t = static_cast<i64>(blockIdx.x) * blockDim.x + threadIdx.x; t < npairs;
       t += static_cast<i64>(gridDim.x) * blockDim.x) {
    const i64 d = first + t;
    const i64 i = d % rows, j = d / rows;
    if (i < r0 || i >= r0 + rcnt) continue;
    const double u1 = __dmul_rn(__dadd_rn(__ull2double_rn(words[2 * t]), 1.0), 0x1.0p-64);
    const double u2 = __dmul_rn(__ull2double_rn(words[2 * t + 1]), 0x1.0p-64);
    const double two_pi = 6.283185307179586;  // 2.0 * std::numbers::pi (exact doubling)
    dst[(i - r0) + j * ld] = __dmul_rn(sqrt(__dmul_rn(-2.0, log(u1))), cos(__dmul_rn(two_pi, u2)));
  }
}

// Hand the (block, p) state to / from the device.
void state_to_device(Ctx& ctx, const Mt64& e, u64* dstate) {
  u64 h[kN + 1];
  for (int k = 0; k < kN; ++k) h[k] = e.x[k];
  h[kN] = static_cast<u64>(e.p);
  NPCG_CUDA(cudaMemcpyAsync(dstate, h, sizeof(h), cudaMemcpyHostToDevice, ctx.stream));
  ctx.sync();
}
void state_from_device(Ctx& ctx, Mt64& e, const u64* dstate, i64 words) {
  u64 h[kN + 1];
  NPCG_CUDA(cudaMemcpyAsync(h, dstate, sizeof(h), cudaMemcpyDeviceToHost, ctx.stream));
  ctx.sync();
  for (int k = 0; k < kN; ++k) e.x[k] = h[k];
  e.p = static_cast<int>(h[kN]);
  e.words += static_cast<std::uint64_t>(words);
}

}  // namespace

void device_words(Ctx& ctx, Mt64& e, i64 count, unsigned long long* out) {
  if (count <= 0) return;
  DBuf<u64> st(kN + 1, ctx.stream);
  state_to_device(ctx, e, st.p);
  NPCG_LAUNCH(ctx, mt64_stream_kernel, 1, 320, 0, st.p, count, out);
  state_from_device(ctx, e, st.p, count);
}

void device_gaussian(Ctx& ctx, Mt64& e, i64 rows, i64 cols, i64 r0, i64 rcnt, double* dst, i64 ld) {
  const i64 total = rows * cols;
  if (total <= 0) return;
  constexpr i64 kChunkPairs = i64{1} << 25;  // 2^26 words (512 MB) in flight
  const i64 chunk = std::min(kChunkPairs, total);
  DBuf<u64> st(kN + 1, ctx.stream), words(2 * chunk, ctx.stream);
  state_to_device(ctx, e, st.p);
  for (i64 first = 0; first < total; first += chunk) {
    const i64 np = std::min(chunk, total - first);
    NPCG_LAUNCH(ctx, mt64_stream_kernel, 1, 320, 0, st.p, 2 * np, words.p);
    NPCG_LAUNCH(ctx, box_muller_kernel, static_cast<unsigned>(std::min<i64>(cdiv(np, 256), ctx.sm_count * 8)), 256, 0,
                words.p, first, np, rows, r0, rcnt, dst, ld);
  }
  state_from_device(ctx, e, st.p, 2 * total);
}

}  // namespace npcg
