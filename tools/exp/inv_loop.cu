// Developer experiment: cost of a warp ballot/shuffle loop in a 1024-thread
// CTA vs an 8-CTA cluster (does not ship).
#include <cooperative_groups.h>
#include <cstdio>
namespace cg = cooperative_groups;

__device__ __forceinline__ unsigned long long gt() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}

template <bool CL>
__global__ void __launch_bounds__(1024, 1) k(unsigned long long* out, int r2) {
  __shared__ int pc[32], pr[32];
  __shared__ unsigned orig[1024];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  for (int i = tid; i < 1024; i += 1024) orig[i] = 0x9E3779B9u * (i + 1);
  if (tid < 32) {
    pc[tid] = tid;
    pr[tid] = tid;
  }
  if (CL) cg::this_cluster().sync(); else __syncthreads();
  if (blockIdx.x == 0 && warp == 0) {
    unsigned long long t0 = gt();
    long long c0 = clock64();
    unsigned x = 0, inv = 0, used = 0;
    if (lane < r2) {
      const unsigned ow = (1u << lane) | (orig[pr[lane]] & ((1u << lane) - 1u));  // unit lower triangular
      for (int t = 0; t < r2; ++t) x |= ((ow >> pc[t]) & 1u) << t;
      inv = 1u << lane;
    }
    int myq = 0;
    for (int q = 0; q < r2; ++q) {
      const unsigned bal = __ballot_sync(0xffffffffu, lane < r2 && !((used >> lane) & 1u) && ((x >> q) & 1u));
      const int pv = __ffs(bal) - 1;
      used |= 1u << pv;
      const unsigned px = __shfl_sync(0xffffffffu, x, pv), pi = __shfl_sync(0xffffffffu, inv, pv);
      if (lane != pv && ((x >> q) & 1u)) {
        x ^= px;
        inv ^= pi;
      }
      if (lane == pv) myq = q;
    }
    long long c1 = clock64();
    unsigned long long t1 = gt();
    if (lane == 0) {
      out[0] = t1 - t0;
      out[1] = c1 - c0;
      out[2] = myq + inv;
    }
  }
  if (CL) cg::this_cluster().sync(); else __syncthreads();
}

int main() {
  unsigned long long* d;
  cudaMalloc(&d, 64);
  unsigned long long h[3];
  for (int rep = 0; rep < 3; ++rep) {
    k<false><<<1, 1024>>>(d, 32);
    cudaMemcpy(h, d, 24, cudaMemcpyDeviceToHost);
    printf("plain CTA: %llu ns %llu cycles\n", h[0], h[1]);
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
    cudaLaunchKernelEx(&cfg, k<true>, d, 32);
    cudaMemcpy(h, d, 24, cudaMemcpyDeviceToHost);
    printf("cluster  : %llu ns %llu cycles (%s)\n", h[0], h[1], cudaGetErrorString(cudaGetLastError()));
  }
  return 0;
}
