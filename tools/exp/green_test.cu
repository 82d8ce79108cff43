// Developer experiment: can the runtime launch into a green-context stream,
// which SMs does the partition's work use, and does an 8-CTA cluster kernel
// on a primary high-priority stream start promptly while a persistent
// kernel fills the green partition?
//   nvcc -gencode arch=compute_100a,code=sm_100a -O2 green_test.cu -o green_test -lcuda
#include <cuda.h>
#include <cuda_runtime.h>

#include <cstdio>
#include <cstdlib>
#include <set>
#include <vector>

#define CK(x) do { auto e_ = (x); if (e_ != 0) { std::printf("FAIL %s:%d %s -> %d\n", __FILE__, __LINE__, #x, int(e_)); std::exit(1); } } while (0)

__device__ __forceinline__ unsigned smid() { unsigned r; asm volatile("mov.u32 %0, %%smid;" : "=r"(r)); return r; }
__device__ __forceinline__ unsigned long long gt() { unsigned long long t; asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t)); return t; }

// persistent: each CTA spins for `ns` and records its SM
__global__ void __launch_bounds__(128) spin(unsigned* sms, unsigned long long ns) {
  extern __shared__ char big[];
  if (threadIdx.x == 0) {
    sms[blockIdx.x] = smid();
    big[0] = 1;
    const unsigned long long t0 = gt();
    while (gt() - t0 < ns) {}
  }
}
__global__ void __cluster_dims__(8, 1, 1) __launch_bounds__(128) cl8(unsigned long long* t, unsigned* sms) {
  extern __shared__ char big2[];
  if (threadIdx.x == 0) {
    big2[0] = 1;
    sms[blockIdx.x] = smid();
    if (blockIdx.x == 0) t[0] = gt();
  }
}
__global__ void stamp(unsigned long long* t) { t[0] = gt(); }

int main(int argc, char** argv) {
  const int reserve = argc > 1 ? std::atoi(argv[1]) : 16;
  CK(cudaSetDevice(0));
  CK(cudaFree(0));
  CUdevice dev;
  CK(cuDeviceGet(&dev, 0));
  CUdevResource all;
  CK(cuDeviceGetDevResource(dev, &all, CU_DEV_RESOURCE_TYPE_SM));
  std::printf("device SMs %u\n", all.sm.smCount);
  for (unsigned flags = 0; flags < 3; flags += 2)
    for (unsigned mc : {8u, 16u, 18u, 20u, 24u, 32u}) {
      CUdevResource gr[32], rem;
      unsigned n = 32;
      if (cuDevSmResourceSplitByCount(gr, &n, &all, &rem, flags, mc) != CUDA_SUCCESS) {
        std::printf("split flags %u min %u: error\n", flags, mc);
        continue;
      }
      std::printf("split flags %u min %u: %u groups:", flags, mc, n);
      for (unsigned q = 0; q < n; ++q) std::printf(" %u", gr[q].sm.smCount);
      std::printf(" remaining %u\n", rem.sm.smCount);
    }
  // bulk = every group of `reserve` SMs but the first, plus the remainder
  CUdevResource gr[32], rest;
  unsigned ng = 32;
  CK(cuDevSmResourceSplitByCount(gr, &ng, &all, &rest, 2, reserve));
  std::vector<CUdevResource> bulk_res(gr + 1, gr + ng);
  if (rest.sm.smCount) bulk_res.push_back(rest);
  unsigned bulk_sms = 0;
  for (auto& r : bulk_res) bulk_sms += r.sm.smCount;
  std::printf("bulk partition: %zu resources, %u SMs; critical group %u SMs\n", bulk_res.size(), bulk_sms,
              gr[0].sm.smCount);
  CUdevResourceDesc desc;
  CK(cuDevResourceGenerateDesc(&desc, bulk_res.data(), unsigned(bulk_res.size())));
  CUgreenCtx g;
  CK(cuGreenCtxCreate(&g, desc, dev, CU_GREEN_CTX_DEFAULT_STREAM));
  CUstream gs;
  CK(cuGreenCtxStreamCreate(&gs, g, CU_STREAM_NON_BLOCKING, 0));
  int lo, hi;
  CK(cudaDeviceGetStreamPriorityRange(&lo, &hi));
  cudaStream_t ps;
  CK(cudaStreamCreateWithPriority(&ps, cudaStreamNonBlocking, hi));
  cudaStream_t ns;
  CK(cudaStreamCreateWithPriority(&ns, cudaStreamNonBlocking, lo));

  unsigned *d_sms, *d_cl;
  unsigned long long* d_t;
  CK(cudaMalloc(&d_sms, 4096 * 4));
  CK(cudaMalloc(&d_cl, 64 * 4));
  CK(cudaMalloc(&d_t, 64 * 8));
  CK(cudaFuncSetAttribute(spin, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024));
  CK(cudaFuncSetAttribute(cl8, cudaFuncAttributeMaxDynamicSharedMemorySize, 100 * 1024));

  for (int mode = 0; mode < 2; ++mode) {
    // mode 0: persistent spin (grid = all SMs, 1 CTA/SM via 200 KB smem) on a
    //         normal primary stream; mode 1: the same on the green stream
    cudaStream_t bulk = mode == 0 ? ns : reinterpret_cast<cudaStream_t>(gs);
    CK(cudaMemset(d_sms, 0xFF, 4096 * 4));
    spin<<<all.sm.smCount, 128, 200 * 1024, bulk>>>(d_sms, 200000000ull);  // 200 ms
    CK(cudaGetLastError());
    { const unsigned long long h0 = 0; (void)h0; }
    for (int w = 0; w < 200 && cudaStreamQuery(bulk) == cudaErrorNotReady; ++w) {}
    { volatile double x = 0; for (int w = 0; w < 3000000; ++w) x = x + 1.0; }
    // give the spin kernel time to occupy its SMs, then time the cluster launch
    stamp<<<1, 1, 0, ps>>>(d_t + 1);
    cl8<<<8, 128, 100 * 1024, ps>>>(d_t, d_cl);
    CK(cudaGetLastError());
    CK(cudaDeviceSynchronize());
    unsigned long long t[2];
    CK(cudaMemcpy(t, d_t, 16, cudaMemcpyDeviceToHost));
    std::vector<unsigned> sm(all.sm.smCount), cl(8);
    CK(cudaMemcpy(sm.data(), d_sms, sm.size() * 4, cudaMemcpyDeviceToHost));
    CK(cudaMemcpy(cl.data(), d_cl, 32, cudaMemcpyDeviceToHost));
    std::set<unsigned> used(sm.begin(), sm.end());
    std::printf("mode %s: spin used %zu distinct SMs; cluster started %.3f ms after the stamp; cluster SMs:",
                mode == 0 ? "primary" : "green", used.size(), double(t[0] - t[1]) / 1e6);
    for (unsigned c : cl) std::printf(" %u", c);
    std::printf("\n");
  }
  std::printf("OK\n");
  return 0;
}
