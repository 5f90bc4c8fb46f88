// Microbenchmark: latency of the 32x32 diagonal-tile Cholesky + inverse used
// by chol.cu -- one warp (current) vs the whole CTA (diagnostic, standalone).
#include <cstdio>
#include <cmath>
#include <vector>
constexpr int CB = 32, TS = 33, CT = 256;
using Tile = double[CB][TS];

__device__ __noinline__ bool diag_warp(Tile& T, Tile& Xs, int nr) {
  const int lane = threadIdx.x & 31;
  double row[CB];
#pragma unroll
  for (int k = 0; k < CB; ++k) row[k] = lane < nr ? (k < nr ? T[lane][k] : 0.0) : (k == lane ? 1.0 : 0.0);
  __shared__ double rs[CB];
  __shared__ double lv[2][CB];
  bool ok = true;
#pragma unroll
  for (int j = 0; j < CB; ++j) {
    double d = __shfl_sync(0xffffffffu, row[j], j);
    if (!(d > 0.0) || !isfinite(d)) { ok = false; d = 1.0; }
    const double r = rsqrt(d);
    if (lane == 0) rs[j] = r;
    const double l = lane == j ? d * r : row[j] * r;
    if (lane >= j) row[j] = l;
    lv[j & 1][lane] = l;
    __syncwarp();
#pragma unroll
    for (int c = j + 1; c < CB; ++c) {
      const double lc = lv[j & 1][c];
      if (lane >= c) row[c] -= l * lc;
    }
  }
  if (!ok) return false;
  __syncwarp();
#pragma unroll
  for (int k = 0; k < CB; ++k) T[lane][k] = k <= lane ? row[k] : 0.0;
  __syncwarp();
  double x[CB];
#pragma unroll
  for (int i = 0; i < CB; ++i) x[i] = i == lane ? 1.0 : 0.0;
#pragma unroll
  for (int k = 0; k < CB; ++k) {
    x[k] *= rs[k];
#pragma unroll
    for (int i = k + 1; i < CB; ++i) x[i] -= T[i][k] * x[k];
  }
#pragma unroll
  for (int i = 0; i < CB; ++i) Xs[i][lane] = x[i];
  return true;
}

// whole CTA: thread t owns rows i = t & 31 of columns c = (t >> 5) + 8u, u < 4
__device__ bool diag_cta(Tile& T, Tile& Xs, int nr) {
  const int t = threadIdx.x, i = t & 31, cb = t >> 5;
  __shared__ double rs[CB];
  __shared__ int bad;
  double a[4];
#pragma unroll
  for (int u = 0; u < 4; ++u) {
    const int c = cb + 8 * u;
    a[u] = i < nr ? (c < nr ? T[i][c] : 0.0) : (c == i ? 1.0 : 0.0);
  }
  if (t == 0) bad = 0;
  __syncthreads();
#pragma unroll
  for (int u = 0; u < 4; ++u) T[i][cb + 8 * u] = a[u];  // padded copy
  __syncthreads();
  for (int j = 0; j < CB; ++j) {
    double d = T[j][j];
    if (!(d > 0.0) || !isfinite(d)) { bad = 1; d = 1.0; }
    const double r = rsqrt(d);
    const double li = T[i][j] * r;
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      const int c = cb + 8 * u;
      if (c > j && i >= c) a[u] -= li * (T[c][j] * r);
    }
    if (t == 0) rs[j] = r;
    __syncthreads();  // every thread has read column j
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      const int c = cb + 8 * u;
      if (c > j && i >= c) T[i][c] = a[u];
    }
    __syncthreads();
  }
  if (bad) return false;
  // L: scale the columns; X = L^{-1} right-looking, thread (i, c) owns X[i][c]
  double lrow[4];
#pragma unroll
  for (int u = 0; u < 4; ++u) {
    const int c = cb + 8 * u;
    lrow[u] = i > c ? T[i][c] * rs[c] : (i == c ? T[i][c] * rs[c] : 0.0);
  }
  __syncthreads();
#pragma unroll
  for (int u = 0; u < 4; ++u) T[i][cb + 8 * u] = lrow[u];
  __syncthreads();
  double x[4];
#pragma unroll
  for (int u = 0; u < 4; ++u) x[u] = i == cb + 8 * u ? 1.0 : 0.0;
  for (int k = 0; k < CB; ++k) {
    if (i == k) {
#pragma unroll
      for (int u = 0; u < 4; ++u) { x[u] *= rs[k]; Xs[k][cb + 8 * u] = x[u]; }
    }
    __syncthreads();
    if (i > k) {
      const double lik = T[i][k];
#pragma unroll
      for (int u = 0; u < 4; ++u) x[u] -= lik * Xs[k][cb + 8 * u];
    }
  }
  __syncthreads();
  return true;
}


// one warp, column j broadcast by shuffles (no shared memory on the chain)
template <bool INV>
__device__ __noinline__ bool diag_shfl(Tile& T, Tile& Xs, int nr) {
  const int lane = threadIdx.x & 31;
  double row[CB];
#pragma unroll
  for (int k = 0; k < CB; ++k) row[k] = lane < nr ? (k < nr ? T[lane][k] : 0.0) : (k == lane ? 1.0 : 0.0);
  double rsl = 0.0;  // lane j keeps 1 / L_jj
  bool ok = true;
#pragma unroll
  for (int j = 0; j < CB; ++j) {
    double d = __shfl_sync(0xffffffffu, row[j], j);
    if (!(d > 0.0) || !isfinite(d)) { ok = false; d = 1.0; }
    const double r = rsqrt(d);
    if (lane == j) rsl = r;
    const double l = lane == j ? d * r : row[j] * r;
    if (lane >= j) row[j] = l;
#pragma unroll
    for (int c = j + 1; c < CB; ++c) {
      const double lc = __shfl_sync(0xffffffffu, l, c);
      if (lane >= c) row[c] -= l * lc;
    }
  }
  if (!ok) return false;
#pragma unroll
  for (int k = 0; k < CB; ++k) T[lane][k] = k <= lane ? row[k] : 0.0;
  __syncwarp();
  if (!INV) return true;
  double x[CB];
#pragma unroll
  for (int i = 0; i < CB; ++i) x[i] = i == lane ? 1.0 : 0.0;
#pragma unroll
  for (int k = 0; k < CB; ++k) {
    x[k] *= __shfl_sync(0xffffffffu, rsl, k);
#pragma unroll
    for (int i = k + 1; i < CB; ++i) x[i] -= T[i][k] * x[k];
  }
#pragma unroll
  for (int i = 0; i < CB; ++i) Xs[i][lane] = x[i];
  return true;
}

template <int V>
__global__ void bench(const double* in, double* outL, double* outX, int reps, long long* cyc) {
  __shared__ Tile T, Xs;
  long long t0 = 0;
  for (int rep = 0; rep < reps; ++rep) {
    for (int idx = threadIdx.x; idx < CB * CB; idx += blockDim.x) T[idx & 31][idx >> 5] = in[idx];
    __syncthreads();
    if (rep == 1) t0 = clock64();
    if (V == 0) { if (threadIdx.x < 32) diag_warp(T, Xs, CB); }
    else if (V == 2) { if (threadIdx.x < 32) diag_shfl<true>(T, Xs, CB); }
    else if (V == 3) { if (threadIdx.x < 32) diag_shfl<false>(T, Xs, CB); }
    else diag_cta(T, Xs, CB);
    __syncthreads();
  }
  if (threadIdx.x == 0) cyc[0] = (clock64() - t0) / (reps - 1);
  for (int idx = threadIdx.x; idx < CB * CB; idx += blockDim.x) {
    outL[idx] = T[idx & 31][idx >> 5];
    outX[idx] = Xs[idx & 31][idx >> 5];
  }
}

int main() {
  std::vector<double> h(CB * CB);
  for (int i = 0; i < CB; ++i)
    for (int j = 0; j < CB; ++j) h[i + j * CB] = (i == j ? CB : 0.0) + 1.0 / (1.0 + i + j);
  double *in, *L, *X; long long* cyc;
  cudaMalloc(&in, 8 * CB * CB); cudaMalloc(&L, 8 * CB * CB); cudaMalloc(&X, 8 * CB * CB); cudaMalloc(&cyc, 8);
  cudaMemcpy(in, h.data(), 8 * CB * CB, cudaMemcpyHostToDevice);
  std::vector<double> l0(CB * CB), x0(CB * CB), l1(CB * CB), x1(CB * CB);
  long long c0, c1;
  bench<0><<<1, CT>>>(in, L, X, 50, cyc); cudaMemcpy(&c0, cyc, 8, cudaMemcpyDeviceToHost);
  cudaMemcpy(l0.data(), L, 8 * CB * CB, cudaMemcpyDeviceToHost); cudaMemcpy(x0.data(), X, 8 * CB * CB, cudaMemcpyDeviceToHost);
  bench<1><<<1, CT>>>(in, L, X, 50, cyc); cudaMemcpy(&c1, cyc, 8, cudaMemcpyDeviceToHost);
  cudaMemcpy(l1.data(), L, 8 * CB * CB, cudaMemcpyDeviceToHost); cudaMemcpy(x1.data(), X, 8 * CB * CB, cudaMemcpyDeviceToHost);
  long long c2;
  std::vector<double> l2(CB * CB), x2(CB * CB);
  bench<2><<<1, CT>>>(in, L, X, 50, cyc); cudaMemcpy(&c2, cyc, 8, cudaMemcpyDeviceToHost);
  cudaMemcpy(l2.data(), L, 8 * CB * CB, cudaMemcpyDeviceToHost); cudaMemcpy(x2.data(), X, 8 * CB * CB, cudaMemcpyDeviceToHost);
  double dl2 = 0, dx2 = 0;
  for (int i = 0; i < CB * CB; ++i) { dl2 = fmax(dl2, fabs(l0[i] - l2[i])); dx2 = fmax(dx2, fabs(x0[i] - x2[i])); }
  printf("shfl: %lld cycles/call, max |dL| %.2e |dX| %.2e\n", c2, dl2, dx2);
  long long c3;
  bench<3><<<1, CT>>>(in, L, X, 50, cyc); cudaMemcpy(&c3, cyc, 8, cudaMemcpyDeviceToHost);
  printf("shfl factor only: %lld cycles/call\n", c3);
  double dl = 0, dx = 0;
  for (int i = 0; i < CB * CB; ++i) { dl = fmax(dl, fabs(l0[i] - l1[i])); dx = fmax(dx, fabs(x0[i] - x1[i])); }
  printf("warp: %lld cycles/call, cta: %lld cycles/call, max |dL| %.2e |dX| %.2e (err %s)\n", c0, c1, dl, dx,
         cudaGetErrorString(cudaGetLastError()));
  return 0;
}
