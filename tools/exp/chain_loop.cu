// Developer experiment: the GF(2) panel chain (8 warps x 4 rows per lane,
// ballot nomination, shared atomicMin, 256-thread named barrier), timed on
// its own in block 0 of an 8-CTA cluster (does not ship).
#include <cooperative_groups.h>
#include <cstdio>
#include <cstdint>
namespace cg = cooperative_groups;
__device__ __forceinline__ unsigned long long gt() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}
template <int V>
__global__ void __launch_bounds__(1024, 1) k(unsigned long long* out, int wc) {
  __shared__ unsigned nomr[3][32];
  __shared__ std::uint32_t orig[1024];
  __shared__ std::uint8_t fl[1024];
  __shared__ std::uint32_t nomw[2][32], nomc[2][32];
  __shared__ unsigned best[3];
  __shared__ int pc[32], pr[32];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  for (int i = tid; i < 1024; i += 1024) {
    orig[i] = (i * 2654435761u) ^ (i >> 3) * 40503u;
    fl[i] = i < 7 ? 1 : 0;
  }
  cg::this_cluster().sync();
  if (blockIdx.x == 0) {
    constexpr int kChainWarps = 8, kRowsPerLane = 4;
    unsigned long long t0 = gt();
    if (warp < kChainWarps) {
      std::uint32_t word[kRowsPerLane], coef[kRowsPerLane];
      std::uint32_t pivm = 0;
#pragma unroll
      for (int s2 = 0; s2 < kRowsPerLane; ++s2) {
        word[s2] = orig[256 * s2 + tid];
        coef[s2] = 0u;
        pivm |= std::uint32_t(fl[256 * s2 + tid] != 0) << s2;
      }
      int r2 = 0;
      if (tid < 3) best[tid] = 0xFFFFFFFFu;
      asm volatile("bar.sync 1, 256;" ::: "memory");
#pragma unroll 1
      for (int c = 0; c < wc; ++c) {
        const int par = c & 1, b3 = c % 3;
        int ws = -1, wl = 0;
#pragma unroll
        for (int s2 = 0; s2 < kRowsPerLane; ++s2) {
          const unsigned b = __ballot_sync(0xffffffffu, ((word[s2] >> c) & 1u) && !((pivm >> s2) & 1u));
          if (ws < 0 && b) {
            ws = s2;
            wl = __ffs(b) - 1;
          }
        }
        if (ws >= 0 && lane == wl) {
          std::uint32_t wv = 0, cv = 0;
#pragma unroll
          for (int t = 0; t < kRowsPerLane; ++t)
            if (t == ws) {
              wv = word[t];
              cv = coef[t];
            }
          nomw[par][warp] = wv;
          nomc[par][warp] = cv;
          if (V == 1) atomicMin(&best[b3], unsigned(256 * ws + 32 * warp + wl));
          else nomr[b3][warp] = unsigned(256 * ws + 32 * warp + wl);
        } else if (V != 1 && lane == 0 && ws < 0) {
          nomr[b3][warp] = 0xFFFFFFFFu;
        }
        asm volatile("bar.sync 1, 256;" ::: "memory");
        unsigned m;
        if (V == 1) {
          m = best[b3];
          if (tid == 0) best[(c + 2) % 3] = 0xFFFFFFFFu;
        } else {
          m = __reduce_min_sync(0xffffffffu, lane < kChainWarps ? nomr[b3][lane] : 0xFFFFFFFFu);
        }
        if (m == 0xFFFFFFFFu) continue;
        const unsigned owner = (m & 255u) >> 5;
        const std::uint32_t pw = nomw[par][owner], pcf = nomc[par][owner] ^ (1u << r2);
#pragma unroll
        for (int s2 = 0; s2 < kRowsPerLane; ++s2) {
          const unsigned row = unsigned(256 * s2 + tid);
          if (row == m) pivm |= 1u << s2;
          else if ((word[s2] >> c) & 1u) {
            word[s2] ^= pw;
            if (V != 3) coef[s2] ^= pcf;
          }
        }
        if (tid == 0) {
          pc[r2] = c;
          pr[r2] = int(m);
        }
        ++r2;
      }
      if (tid == 0) out[2] = r2;
    }
    __syncthreads();
    unsigned long long t1 = gt();
    if (tid == 0) {
      out[0] = t1 - t0;
      out[1] = pr[0] + pc[1];
    }
  }
  cg::this_cluster().sync();
}
int main() {
  unsigned long long* d;
  cudaMalloc(&d, 64);
  unsigned long long h[3];
  for (int rep = 0; rep < 3; ++rep) {
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
    cudaLaunchKernelEx(&cfg, k<1>, d, 32);
    cudaMemcpy(h, d, 24, cudaMemcpyDeviceToHost);
    printf("V1 atomicMin: %llu ns, r2 %llu (%s)\n", h[0], h[2], cudaGetErrorString(cudaGetLastError()));
    cudaLaunchKernelEx(&cfg, k<2>, d, 32);
    cudaMemcpy(h, d, 24, cudaMemcpyDeviceToHost);
    printf("V2 redux: %llu ns, r2 %llu\n", h[0], h[2]);
    cudaLaunchKernelEx(&cfg, k<3>, d, 32);
    cudaMemcpy(h, d, 24, cudaMemcpyDeviceToHost);
    printf("V3 redux, no coef: %llu ns, r2 %llu\n", h[0], h[2]);
  }
  return 0;
}
