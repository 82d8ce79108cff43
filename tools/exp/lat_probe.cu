// Developer experiment: single-warp dependent-chain latencies (SHFL, VOTE,
// the GF(2) row-layout pivot step) on one SM (does not ship).
#include <cstdio>
#include <cstdint>
__shared__ volatile int g_stop;
template <int NT, int MODE>
__global__ void __launch_bounds__(NT, 1) k(long long* out, unsigned seed, int iters) {
  const int lane = threadIdx.x & 31;
  __shared__ unsigned buf[4096];
  if (threadIdx.x == 0) g_stop = 0;
  for (int i = threadIdx.x; i < 4096; i += NT) buf[i] = i * 2654435761u;
  __syncthreads();
  if (threadIdx.x >= 32) {
    if (MODE == 1) {  // smem traffic like the stripe update
      unsigned acc = threadIdx.x;
      while (!g_stop) {
#pragma unroll 8
        for (int q = 0; q < 64; ++q) acc ^= buf[(acc + q * 33) & 4095];
      }
      if (acc == 12345) out[7] = acc;
    } else if (MODE == 2) {  // spin on a shared flag
      while (!g_stop) {}
    }
    __syncthreads();
    return;
  }
  unsigned v = seed * (lane + 1);
  long long t0 = clock64();
  for (int i = 0; i < iters; ++i) v = __shfl_sync(0xffffffffu, v, (v + i) & 31) + 1;
  long long t1 = clock64();
  unsigned b = v;
  for (int i = 0; i < iters; ++i) b = __ballot_sync(0xffffffffu, (b >> (lane & 7)) & 1) * 2654435761u + i;
  long long t2 = clock64();
  // row-layout GF(2) pivot step, 32 columns per round
  unsigned w0 = v * 2654435761u ^ b, w1 = w0 * 2246822519u + lane, k0 = 0, k1 = 0;
  bool p0 = false, p1 = false;
  int r2 = 0;
  for (int i = 0; i < iters; ++i) {
    const int c = i & 31;
    const unsigned b0 = __ballot_sync(0xffffffffu, !p0 && ((w0 >> c) & 1u));
    const unsigned b1 = __ballot_sync(0xffffffffu, !p1 && ((w1 >> c) & 1u));
    if (!(b0 | b1)) { w0 = w0 * 3 + 1; continue; }
    const bool hi = b0 == 0;
    const int sl = __ffs(hi ? b1 : b0) - 1;
    const unsigned pw = __shfl_sync(0xffffffffu, hi ? w1 : w0, sl);
    const unsigned pk = __shfl_sync(0xffffffffu, hi ? k1 : k0, sl) ^ (1u << (r2 & 31));
    const bool me0 = !hi && lane == sl, me1 = hi && lane == sl;
    if (!me0 && ((w0 >> c) & 1u)) { w0 ^= pw; k0 ^= pk; }
    if (!me1 && ((w1 >> c) & 1u)) { w1 ^= pw; k1 ^= pk; }
    if (c == 31) { p0 = p1 = false; w0 = w0 * 2654435761u + 7; w1 = w1 * 2246822519u + 3; }
    ++r2;
  }
  long long t3 = clock64();
  // exact in-kernel loop shape (row layout + register bookkeeping), 32-col panels
  int mpc = 0, mpr = 0, q0 = -1, q1 = -1, tot = 0;
  for (int it = 0; it < iters / 32; ++it) {
    unsigned x0 = w0 * 2654435761u + it, x1 = w1 * 2246822519u + it, kk0 = 0, kk1 = 0;
    bool pp0 = false, pp1 = false;
    int rr = 0, ok = 1;
    const bool covers_all = (it & 1);
#pragma unroll 1
    for (int c = 0; c < 32; ++c) {
      const unsigned b0 = __ballot_sync(0xffffffffu, !pp0 && ((x0 >> c) & 1u));
      const unsigned b1 = __ballot_sync(0xffffffffu, !pp1 && ((x1 >> c) & 1u));
      if (!(b0 | b1)) {
        if (covers_all) continue;
        ok = 0;
        break;
      }
      const bool hi = b0 == 0;
      const int sl = __ffs(hi ? b1 : b0) - 1;
      const unsigned pw = __shfl_sync(0xffffffffu, hi ? x1 : x0, sl);
      const unsigned pk = __shfl_sync(0xffffffffu, hi ? kk1 : kk0, sl) ^ (1u << rr);
      const bool me0 = !hi && lane == sl, me1 = hi && lane == sl;
      if (!me0 && ((x0 >> c) & 1u)) { x0 ^= pw; kk0 ^= pk; }
      if (!me1 && ((x1 >> c) & 1u)) { x1 ^= pw; kk1 ^= pk; }
      if (me0) { pp0 = true; q0 = rr; }
      if (me1) { pp1 = true; q1 = rr; }
      if (lane == rr) { mpc = c; mpr = (hi ? 32 : 0) + sl; }
      ++rr;
    }
    tot += rr + ok + mpc + mpr + q0 + q1 + int(kk0 ^ kk1);
  }
  long long t4 = clock64();
  if (lane == 0) {
    out[0] = t1 - t0; out[1] = t2 - t1; out[2] = t3 - t2; out[3] = w0 ^ w1 ^ k0 ^ k1 ^ v ^ b ^ tot;
    out[4] = t4 - t3;
    g_stop = 1;
  }
  __syncthreads();
}
int main() {
  long long* d; cudaMalloc(&d, 64);
  long long h[5];
  const int iters = 4096;
  for (int rep = 0; rep < 4; ++rep) {
    const char* names[4] = {"32 thr", "1024 idle", "1024 smem-busy", "1024 spin"};
    printf("%-16s ", names[rep]);
    if (rep == 0) k<32, 0><<<1, 32>>>(d, 12345 + rep, iters);
    else if (rep == 1) k<1024, 0><<<1, 1024>>>(d, 12345 + rep, iters);
    else if (rep == 2) k<1024, 1><<<1, 1024>>>(d, 12345 + rep, iters);
    else k<1024, 2><<<1, 1024>>>(d, 12345 + rep, iters);
    cudaMemcpy(h, d, sizeof h, cudaMemcpyDeviceToHost);
    printf("per iter cycles: shfl chain %.1f  vote chain %.1f  gf2 row step %.1f  kernel-shape %.1f\n", double(h[0]) / iters,
           double(h[1]) / iters, double(h[2]) / iters, double(h[4]) / iters);
  }
  return 0;
}
