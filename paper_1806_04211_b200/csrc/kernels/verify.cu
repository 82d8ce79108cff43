// verify.cu -- device checks behind gfrref::verify (reference
// src/chief.cpp:531-590): an entry-wise comparison with a mismatch count and
// the first mismatching position, and the echelon-shape test of the
// remnant R (a pivot row has no nonzero entry left of its pivot).
// Both are HBM-streaming reductions (a thread per 16-byte row segment or
// entry, one pair of atomics per warp).
#include "../common.hpp"
#include "kernels.hpp"

namespace gfq::dev {
namespace {

__device__ __forceinline__ void note_mismatch(bool bad, std::uint64_t pos,
                                              unsigned long long* count,
                                              unsigned long long* first) {
  const unsigned mask = __ballot_sync(0xffffffffu, bad);
  if (!mask) return;
  std::uint64_t lo = bad ? pos : ~0ull;
#pragma unroll
  for (int o = 16; o; o >>= 1) {
    const std::uint64_t other = __shfl_xor_sync(0xffffffffu, lo, o);
    lo = other < lo ? other : lo;
  }
  if ((threadIdx.x & 31) == 0) {
    atomicAdd(count, static_cast<unsigned long long>(__popc(mask)));
    atomicMin(first, static_cast<unsigned long long>(lo));
  }
}

// Each thread compares 16 consecutive columns of one row (a 16 B segment).
__global__ void compare_kernel(std::int64_t rows, std::int64_t cols, const std::uint8_t* A,
                               std::int64_t lda, const std::uint8_t* B, std::int64_t ldb,
                               int mode, std::uint8_t value, unsigned long long* count,
                               unsigned long long* first) {
  const std::int64_t segs = (cols + 15) / 16;
  const std::int64_t total = rows * segs;
  for (std::int64_t t = blockIdx.x * std::int64_t(blockDim.x) + threadIdx.x;
       t - threadIdx.x < total; t += std::int64_t(gridDim.x) * blockDim.x) {
    bool bad = false;
    std::uint64_t pos = ~0ull;
    if (t < total) {
      const std::int64_t r = t / segs, c0 = (t % segs) * 16;
      const int nc = int(cols - c0 < 16 ? cols - c0 : 16);
      const std::uint8_t* a = A + r * lda + c0;
      const std::uint8_t* b = B ? B + r * ldb + c0 : nullptr;
      for (int c = 0; c < nc; ++c) {
        std::uint8_t want = 0;
        if (mode == 0) want = b[c];
        else if (mode == 2) want = (r == c0 + c) ? value : 0;
        if (a[c] != want) {
          bad = true;
          pos = std::uint64_t(r) * std::uint64_t(cols) + std::uint64_t(c0 + c);
          break;
        }
      }
    }
    note_mismatch(bad, pos, count, first);
  }
}

__global__ void echelon_check_kernel(std::int64_t rows, std::int64_t cols, const std::uint8_t* R,
                                     std::int64_t ldr, const std::int32_t* pivcol,
                                     const std::int32_t* restcol, unsigned long long* count,
                                     unsigned long long* first) {
  const std::int64_t total = rows * cols;
  for (std::int64_t t = blockIdx.x * std::int64_t(blockDim.x) + threadIdx.x;
       t - threadIdx.x < total; t += std::int64_t(gridDim.x) * blockDim.x) {
    bool bad = false;
    std::uint64_t pos = ~0ull;
    if (t < total) {
      const std::int64_t r = t / cols, c = t % cols;
      if (restcol[c] < pivcol[r] && R[r * ldr + c] != 0) {
        bad = true;
        pos = std::uint64_t(t);
      }
    }
    note_mismatch(bad, pos, count, first);
  }
}

int grid_for(std::int64_t work, int threads) {
  const std::int64_t want = (work + threads - 1) / threads;
  const std::int64_t cap = std::int64_t(sm_count()) * 16;
  return int(want < 1 ? 1 : (want < cap ? want : cap));
}

}  // namespace

void compare(std::int64_t rows, std::int64_t cols, const std::uint8_t* A, std::int64_t lda,
             const std::uint8_t* B, std::int64_t ldb, int mode, std::uint8_t value,
             unsigned long long* count_first, cudaStream_t s) {
  if (rows <= 0 || cols <= 0) return;
  const std::int64_t segs = rows * ((cols + 15) / 16);
  compare_kernel<<<grid_for(segs, 256), 256, 0, s>>>(rows, cols, A, lda, B, ldb, mode, value,
                                                      count_first, count_first + 1);
  GFQ_CUDA(cudaGetLastError());
  count_launch();
}

void echelon_check(std::int64_t rows, std::int64_t cols, const std::uint8_t* R, std::int64_t ldr,
                   const std::int32_t* pivcol, const std::int32_t* restcol,
                   unsigned long long* count_first, cudaStream_t s) {
  if (rows <= 0 || cols <= 0) return;
  echelon_check_kernel<<<grid_for(rows * cols, 256), 256, 0, s>>>(
      rows, cols, R, ldr, pivcol, restcol, count_first, count_first + 1);
  GFQ_CUDA(cudaGetLastError());
  count_launch();
}

}  // namespace gfq::dev
