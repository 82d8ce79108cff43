// Developer experiment: the column-layout GF(2) window chain alone (does not ship).
#include <cstdio>
#include <cstdint>
__device__ __forceinline__ unsigned long long gt() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}
__global__ void __launch_bounds__(1024, 1) k(unsigned long long* out, int wc, int nthreads_busy) {
  __shared__ int pc[32], pr[32];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  __syncthreads();
  if (warp == 0) {
    const std::uint32_t w0 = (lane + 1) * 2654435761u, w1 = (lane + 77) * 40503u * 2654435761u;
    unsigned long long t0 = gt();
    long long c0 = clock64();
    std::uint64_t cmask = 0, kmask = 0;
#pragma unroll
    for (int q = 0; q < 32; ++q) {
      const unsigned lo32 = __ballot_sync(0xffffffffu, (w0 >> q) & 1u);
      const unsigned hi32 = __ballot_sync(0xffffffffu, (w1 >> q) & 1u);
      if (lane == q) cmask = std::uint64_t(lo32) | (std::uint64_t(hi32) << 32);
    }
    long long c1 = clock64();
    std::uint64_t piv = 0;
    int r2 = 0;
    for (int c = 0; c < wc; ++c) {
      const std::uint64_t col = __shfl_sync(0xffffffffu, cmask, c);
      const std::uint64_t cand = col & ~piv;
      if (!cand) break;
      const int p = __ffsll(static_cast<long long>(cand)) - 1;
      const std::uint64_t sset = col & ~(std::uint64_t(1) << p);
      if ((cmask >> p) & 1u) cmask ^= sset;
      if (lane < r2 && ((kmask >> p) & 1u)) kmask ^= sset;
      if (lane == r2) kmask = sset;
      piv |= std::uint64_t(1) << p;
      if (lane == 0) {
        pc[r2] = c;
        pr[r2] = p;
      }
      ++r2;
    }
    long long c2 = clock64();
    unsigned long long t1 = gt();
    if (lane == 0) {
      out[0] = t1 - t0;
      out[1] = c1 - c0;
      out[2] = c2 - c1;
      out[3] = r2 + pc[3] + pr[5] + (kmask & 1);
    }
  }
  __syncthreads();
}
int main() {
  unsigned long long* d;
  cudaMalloc(&d, 64);
  unsigned long long h[4];
  for (int rep = 0; rep < 3; ++rep) {
    k<<<1, 1024>>>(d, 32, 0);
    cudaMemcpy(h, d, 32, cudaMemcpyDeviceToHost);
    printf("total %llu ns, transpose %llu cyc, chain %llu cyc, r2 %llu\n", h[0], h[1], h[2], h[3]);
  }
  return 0;
}
