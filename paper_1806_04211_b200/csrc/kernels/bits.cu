// bits.cu -- GF(2) byte matrices <-> packed bit rows, for the host-buffer
// entry point's transfers: a GF(2) element is one bit of information in a
// byte, so the input crosses PCIe packed 8:1 (the host packs, pack_bits'
// inverse unpacks in HBM) and the outputs leave packed (pack_bits here, the
// host unpacks).  Row r of a rows x cols block packs to ceil(cols / 8)
// bytes, element c at bit c % 8 of byte c / 8 (LSB first).  HBM-bound:
// 1 + 1/8 bytes moved per element.
#include "../common.hpp"
#include "kernels.hpp"

namespace gfq::dev {
namespace {

// one thread: 64 elements (8 packed bytes) of one row
__global__ void __launch_bounds__(256) pack_bits_kernel(const std::uint8_t* __restrict__ src, std::int64_t ld,
                                                        std::int64_t rows, std::int64_t cols,
                                                        std::uint8_t* __restrict__ dst, std::int64_t ldb) {
  pdl_wait_and_release();
  const std::int64_t nb = (cols + 7) / 8, per_row = (nb + 7) / 8;
  const bool al = ((reinterpret_cast<std::uintptr_t>(src) | std::uintptr_t(ld)) & 15) == 0 &&
                  ((reinterpret_cast<std::uintptr_t>(dst) | std::uintptr_t(ldb)) & 7) == 0;
  for (std::int64_t t = std::int64_t(blockIdx.x) * blockDim.x + threadIdx.x; t < rows * per_row;
       t += std::int64_t(gridDim.x) * blockDim.x) {
    const std::int64_t r = t / per_row, q = t - r * per_row;
    const std::int64_t c0 = q * 64;
    const std::uint8_t* s = src + r * ld + c0;
    std::uint8_t* d = dst + r * ldb + q * 8;
    if (al && c0 + 64 <= cols) {
      std::uint64_t out = 0;
#pragma unroll
      for (int v = 0; v < 4; ++v) {
        const uint4 x = reinterpret_cast<const uint4*>(s)[v];
        const std::uint32_t w[4] = {x.x, x.y, x.z, x.w};
#pragma unroll
        for (int k = 0; k < 4; ++k) {
          // bit 0 of each byte -> 4 consecutive bits
          const std::uint32_t b = w[k] & 0x01010101u;
          const std::uint32_t nib = (b | (b >> 7) | (b >> 14) | (b >> 21)) & 0xFu;
          out |= std::uint64_t(nib) << (16 * v + 4 * k);
        }
      }
      *reinterpret_cast<std::uint64_t*>(d) = out;
    } else {
      for (std::int64_t j = 0; j < 8 && q * 8 + j < nb; ++j) {
        std::uint32_t byte = 0;
        for (int k = 0; k < 8; ++k) {
          const std::int64_t c = c0 + 8 * j + k;
          if (c < cols) byte |= std::uint32_t(s[8 * j + k] & 1u) << k;
        }
        d[j] = static_cast<std::uint8_t>(byte);
      }
    }
  }
}

// one thread: 8 packed bytes -> 64 elements of one row
__global__ void __launch_bounds__(256) unpack_bits_kernel(const std::uint8_t* __restrict__ src, std::int64_t ldb,
                                                          std::int64_t rows, std::int64_t cols,
                                                          std::uint8_t* __restrict__ dst, std::int64_t ld) {
  pdl_wait_and_release();
  const std::int64_t nb = (cols + 7) / 8, per_row = (nb + 7) / 8;
  const bool al = ((reinterpret_cast<std::uintptr_t>(dst) | std::uintptr_t(ld)) & 15) == 0 &&
                  ((reinterpret_cast<std::uintptr_t>(src) | std::uintptr_t(ldb)) & 7) == 0;
  for (std::int64_t t = std::int64_t(blockIdx.x) * blockDim.x + threadIdx.x; t < rows * per_row;
       t += std::int64_t(gridDim.x) * blockDim.x) {
    const std::int64_t r = t / per_row, q = t - r * per_row;
    const std::int64_t c0 = q * 64;
    const std::uint8_t* s = src + r * ldb + q * 8;
    std::uint8_t* d = dst + r * ld + c0;
    if (al && c0 + 64 <= cols) {
      const std::uint64_t x = *reinterpret_cast<const std::uint64_t*>(s);
#pragma unroll
      for (int v = 0; v < 4; ++v) {
        std::uint32_t w[4];
#pragma unroll
        for (int k = 0; k < 4; ++k) {
          const std::uint32_t nib = std::uint32_t(x >> (16 * v + 4 * k)) & 0xFu;
          w[k] = (nib & 1u) | ((nib & 2u) << 7) | ((nib & 4u) << 14) | ((nib & 8u) << 21);
        }
        reinterpret_cast<uint4*>(d)[v] = make_uint4(w[0], w[1], w[2], w[3]);
      }
    } else {
      for (std::int64_t j = 0; j < 8 && q * 8 + j < nb; ++j) {
        const std::uint32_t byte = s[j];
        for (int k = 0; k < 8; ++k) {
          const std::int64_t c = c0 + 8 * j + k;
          if (c < cols) d[8 * j + k] = static_cast<std::uint8_t>((byte >> k) & 1u);
        }
      }
    }
  }
}

unsigned bits_grid(std::int64_t rows, std::int64_t cols) {
  const std::int64_t work = rows * (((cols + 7) / 8 + 7) / 8);
  const std::int64_t cap = std::int64_t(sm_count()) * 16;
  const std::int64_t g = (work + 255) / 256;
  return unsigned(g < 1 ? 1 : (g > cap ? cap : g));
}

}  // namespace

void pack_bits(const std::uint8_t* src, std::int64_t ld, std::int64_t rows, std::int64_t cols, std::uint8_t* dst,
               std::int64_t ldb, cudaStream_t s) {
  if (rows <= 0 || cols <= 0) return;
  GFQ_CUDA(launch_pdl(pack_bits_kernel, dim3(bits_grid(rows, cols)), dim3(256), 0, s, src, ld, rows, cols, dst, ldb));
  count_launch();
}

void unpack_bits(const std::uint8_t* src, std::int64_t ldb, std::int64_t rows, std::int64_t cols, std::uint8_t* dst,
                 std::int64_t ld, cudaStream_t s) {
  if (rows <= 0 || cols <= 0) return;
  GFQ_CUDA(launch_pdl(unpack_bits_kernel, dim3(bits_grid(rows, cols)), dim3(256), 0, s, src, ldb, rows, cols, dst,
                      ld));
  count_launch();
}

}  // namespace gfq::dev
