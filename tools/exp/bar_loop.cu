// Developer experiment: CTA barrier loop cost in a plain CTA vs in an 8-CTA
// cluster whose other CTAs wait at the cluster barrier (does not ship).
#include <cooperative_groups.h>
#include <cstdio>
namespace cg = cooperative_groups;
__device__ __forceinline__ unsigned long long gt() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}
template <bool CL, int WAITMODE>
__global__ void __launch_bounds__(1024, 1) k(unsigned long long* out, int iters) {
  __shared__ unsigned nom[2][32];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  if (CL) cg::this_cluster().sync(); else __syncthreads();
  unsigned word = tid * 2654435761u, acc = 0;
  if (blockIdx.x == 0) {
    unsigned long long t0 = gt();
    for (int c = 0; c < iters; ++c) {
      const int par = c & 1;
      const unsigned bal = __ballot_sync(0xffffffffu, (word >> (c & 31)) & 1u);
      if (lane == 0) nom[par][warp] = bal ? 32 * warp + __ffs(bal) : 0xFFFFFFFFu;
      __syncthreads();
      const unsigned m = __reduce_min_sync(0xffffffffu, nom[par][lane]);
      word ^= m;
      acc += m;
    }
    unsigned long long t1 = gt();
    if (tid == 0) out[0] = t1 - t0;
  } else if (WAITMODE == 1) {
    // nothing: go straight to the cluster barrier
  }
  if (tid == 1023) out[1] = acc;
  if (CL) cg::this_cluster().sync(); else __syncthreads();
}
int main() {
  unsigned long long* d;
  cudaMalloc(&d, 64);
  unsigned long long h[2];
  for (int rep = 0; rep < 3; ++rep) {
    k<false, 0><<<1, 1024>>>(d, 32);
    cudaMemcpy(h, d, 16, cudaMemcpyDeviceToHost);
    printf("plain CTA 32 iters: %llu ns\n", h[0]);
    k<false, 0><<<8, 1024>>>(d, 32);
    cudaMemcpy(h, d, 16, cudaMemcpyDeviceToHost);
    printf("8 plain CTAs 32 iters: %llu ns\n", h[0]);
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(8);
    cfg.blockDim = dim3(1024);
    cudaLaunchAttribute a[1];
    a[0].id = cudaLaunchAttributeClusterDimension;
    a[0].val.clusterDim.x = 8;
    a[0].val.clusterDim.y = 1;
    a[0].val.clusterDim.z = 1;
    cfg.attrs = a;
    cfg.numAttrs = 1;
    cudaLaunchKernelEx(&cfg, k<true, 1>, d, 32);
    cudaMemcpy(h, d, 16, cudaMemcpyDeviceToHost);
    printf("cluster (others wait) 32 iters: %llu ns (%s)\n", h[0], cudaGetErrorString(cudaGetLastError()));
  }
  return 0;
}
