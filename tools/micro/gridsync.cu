// Microbenchmark: cost of cooperative grid.sync and of a warp-level 32x32
// Cholesky-like shuffle chain (diagnostic, standalone).
#include <cooperative_groups.h>
#include <cstdio>
namespace cg = cooperative_groups;
__global__ void gs_kernel(int iters, int* out) {
  cg::grid_group g = cg::this_grid();
  for (int i = 0; i < iters; ++i) g.sync();
  if (blockIdx.x == 0 && threadIdx.x == 0) out[0] = iters;
}
__global__ void cluster_kernel(int iters, int* out) {
  cg::cluster_group c = cg::this_cluster();
  for (int i = 0; i < iters; ++i) c.sync();
  if (blockIdx.x == 0 && threadIdx.x == 0) out[0] = iters;
}
int main() {
  int* out;
  cudaMalloc(&out, 4);
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  for (int G : {1, 16, 48, 90, 148}) {
    int iters = 2000;
    void* args[] = {&iters, &out};
    cudaLaunchCooperativeKernel((void*)gs_kernel, G, 256, args, 0, 0);
    cudaEventRecord(a);
    cudaLaunchCooperativeKernel((void*)gs_kernel, G, 256, args, 0, 0);
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    float ms;
    cudaEventElapsedTime(&ms, a, b);
    printf("grid.sync G=%d: %.3f us per sync (%s)\n", G, ms * 1e3 / iters, cudaGetErrorString(cudaGetLastError()));
  }
  for (int C : {8, 16}) {
    cudaFuncSetAttribute(cluster_kernel, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(C);
    cfg.blockDim = dim3(256);
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeClusterDimension;
    at[0].val.clusterDim.x = C;
    at[0].val.clusterDim.y = 1;
    at[0].val.clusterDim.z = 1;
    cfg.attrs = at;
    cfg.numAttrs = 1;
    int iters = 2000;
    cudaLaunchKernelEx(&cfg, cluster_kernel, iters, out);
    cudaEventRecord(a);
    cudaLaunchKernelEx(&cfg, cluster_kernel, iters, out);
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    float ms;
    cudaEventElapsedTime(&ms, a, b);
    printf("cluster.sync C=%d: %.3f us per sync (%s)\n", C, ms * 1e3 / iters, cudaGetErrorString(cudaGetLastError()));
  }
  return 0;
}
