// Developer experiment: the kernel's window_chain alone (does not ship).
#include <cstdio>
#include <cstdint>
__device__ __forceinline__ unsigned long long gt() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}
__global__ void __launch_bounds__(1024, 1) k(unsigned long long* out, int rows, int cols) {
  __shared__ std::uint32_t orig[1024];
  __shared__ std::uint8_t fl[1024];
  __shared__ int pc[32], pr[32], r2_sh, ok_sh, lo_sh;
  __shared__ std::uint32_t pcoef[32];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  orig[tid] = (tid * 2654435761u) ^ ((tid >> 3) * 40503u);
  fl[tid] = tid < 13 ? 1 : 0;
  if (tid == 0) lo_sh = 0;
  __syncthreads();
  auto window_chain = [&](int k) {
    const int wc = cols - 32 * k < 32 ? cols - 32 * k : 32;
    int lo = lo_sh;
    for (;;) {
      const int idx = lo + lane;
      const unsigned b = __ballot_sync(0xffffffffu, idx < rows && fl[idx] == 0);
      if (b || lo >= rows) {
        if (b) lo += __ffs(b) - 1;
        break;
      }
      lo += 32;
    }
    if (lo > rows) lo = rows;
    const int i0 = lo + lane, i1 = lo + 32 + lane;
    const std::uint32_t w0 = i0 < 1024 ? orig[i0] : 0u, w1 = i1 < 1024 ? orig[i1] : 0u;
    const bool p0 = i0 >= rows || fl[i0] != 0, p1 = i1 >= rows || fl[i1] != 0;
    std::uint64_t cmask = 0, kmask = 0;
#pragma unroll
    for (int q = 0; q < 32; ++q) {
      const unsigned lo32 = __ballot_sync(0xffffffffu, (w0 >> q) & 1u);
      const unsigned hi32 = __ballot_sync(0xffffffffu, (w1 >> q) & 1u);
      if (lane == q) cmask = std::uint64_t(lo32) | (std::uint64_t(hi32) << 32);
    }
    std::uint64_t piv = std::uint64_t(__ballot_sync(0xffffffffu, p0)) |
                        (std::uint64_t(__ballot_sync(0xffffffffu, p1)) << 32);
    // Four columns per round: their current masks are broadcast together,
    // every lane derives the four pivots from them in registers (each
    // pivot's elimination applied to the later columns of the round), then
    // applies the four eliminations to its own column and coefficient mask.
    int r2 = 0, ok = 1;
    for (int c0 = 0; c0 < wc && ok; c0 += 4) {
      const int nt = wc - c0 < 4 ? wc - c0 : 4;
      std::uint64_t bc[4], ss[4];
      int pv[4];
#pragma unroll
      for (int t = 0; t < 4; ++t) bc[t] = __shfl_sync(0xffffffffu, cmask, (c0 + t) & 31);
      int np = 0;
#pragma unroll
      for (int t = 0; t < 4; ++t) {
        pv[t] = -1;
        ss[t] = 0;
        if (t < nt && ok) {
          const std::uint64_t cand = bc[t] & ~piv;
          if (!cand) {
            ok = 0;  // a column without a window candidate: uniform
          } else {
            const int p = __ffsll(static_cast<long long>(cand)) - 1;
            pv[t] = p;
            ss[t] = bc[t] & ~(std::uint64_t(1) << p);
            piv |= std::uint64_t(1) << p;
#pragma unroll
            for (int u = t + 1; u < 4; ++u)
              if ((bc[u] >> p) & 1u) bc[u] ^= ss[t];
            ++np;
          }
        }
      }
#pragma unroll
      for (int t = 0; t < 4; ++t) {
        if (pv[t] < 0) continue;
        const int p = pv[t], q = r2 + t;
        if ((cmask >> p) & 1u) cmask ^= ss[t];
        if (lane < q && ((kmask >> p) & 1u)) kmask ^= ss[t];
        if (lane == q) kmask = ss[t];
        if (lane == 0) {
          pc[q] = c0 + t;
          pr[q] = lo + p;
        }
      }
      r2 += np;
    }
    __syncwarp();
    if (ok)
      for (int t = 0; t < r2; ++t) {
        const unsigned cf = __ballot_sync(0xffffffffu, (kmask >> (pr[t] - lo)) & 1u);
        if (lane == t) pcoef[t] = cf ^ (1u << t);
      }
    if (lane == 0) {
      ok_sh = ok;
      r2_sh = r2;
      lo_sh = lo;
    }
  };

  if (warp == 0) {
    unsigned long long t0 = gt();
    long long c0 = clock64();
    window_chain(0);
    long long c1 = clock64();
    unsigned long long t1 = gt();
    if (lane == 0) { out[0] = t1 - t0; out[1] = c1 - c0; out[2] = r2_sh * 100 + ok_sh; }
  }
}
int main() {
  unsigned long long* d;
  cudaMalloc(&d, 64);
  unsigned long long h[3];
  for (int rep = 0; rep < 3; ++rep) {
    k<<<1, 1024>>>(d, 1024, 1024);
    cudaMemcpy(h, d, 24, cudaMemcpyDeviceToHost);
    printf("window_chain %llu ns %llu cycles r2*100+ok %llu (%s)\n", h[0], h[1], h[2], cudaGetErrorString(cudaGetLastError()));
  }
}
