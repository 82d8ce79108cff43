// wide.cu -- the kernels of the "wide" fields: GF(p) with 251 < p < 2^16
// and GF(p^k) with 256 < p^k < 2^20 (the rest of the reference's field
// range, src/field.cpp:143-149), whose elements are stored as u32.
//
// Arithmetic: prime fields by 64-bit integer remainders; extension fields by
// the log / antilog / Zech tables of FieldSpec::wide_dev (the reference's
// own representation, src/field.cpp:180-212):
//   a.b   = g^(log a + log b)
//   a + b = g^(log a + zech[log b - log a]),  zech[n] = log(1 + g^n)
// on elements encoded like the reference (sum_i c_i p^i).
//
// Kernels: the contraction D = Cin + A.B (K1w, a shared-memory tiled SIMT
// kernel: these fields have no exact tensor-core encoding at u8 / E2M1
// width), the one-CTA base case of the split/combine ECH (K2w, the same
// column-wise Gauss-Jordan with -1 pivots as ech_base), identity planting
// and the SplitMix64 generator (K6w).
#include <algorithm>

#include "../common.hpp"
#include "kernels.hpp"

namespace gfq::dev {
namespace {

__device__ __forceinline__ std::uint32_t wmul(const WideField& f, std::uint32_t a, std::uint32_t b) {
  if (f.k == 1) return std::uint32_t(std::uint64_t(a) * b % f.p);
  if (a == 0 || b == 0) return 0;
  std::uint32_t e = f.log[a] + f.log[b];
  if (e >= f.q - 1) e -= f.q - 1;
  return f.exp[e];
}
__device__ __forceinline__ std::uint32_t wadd(const WideField& f, std::uint32_t a, std::uint32_t b) {
  if (f.k == 1) {
    const std::uint32_t s = a + b;
    return s >= f.p ? s - f.p : s;
  }
  if (a == 0) return b;
  if (b == 0) return a;
  const std::uint32_t la = f.log[a], lb = f.log[b];
  const std::uint32_t d = lb >= la ? lb - la : lb + (f.q - 1) - la;
  const std::int32_t z = f.zech[d];
  if (z < 0) return 0;
  std::uint32_t e = la + std::uint32_t(z);
  if (e >= f.q - 1) e -= f.q - 1;
  return f.exp[e];
}
__device__ __forceinline__ std::uint32_t wneg(const WideField& f, std::uint32_t a) {
  if (f.k == 1) return a == 0 ? 0 : f.p - a;
  if (a == 0 || f.p == 2) return a;
  std::uint32_t e = f.log[a] + (f.q - 1) / 2;  // -1 = g^((q-1)/2)
  if (e >= f.q - 1) e -= f.q - 1;
  return f.exp[e];
}
__device__ __forceinline__ std::uint32_t winv(const WideField& f, std::uint32_t a) {
  if (f.k == 1) {
    std::uint64_t r = 1, b = a;
    for (std::uint32_t e = f.p - 2; e; e >>= 1) {
      if (e & 1) r = r * b % f.p;
      b = b * b % f.p;
    }
    return std::uint32_t(r);
  }
  const std::uint32_t l = f.log[a];
  return f.exp[l == 0 ? 0 : f.q - 1 - l];
}

// ---- K1w: D = Cin + A.B, 32 x 32 output tiles, K staged 32 at a time
constexpr int kWT = 32;
__global__ void __launch_bounds__(256) mad_wide_kernel(WideField f, int m, int n, int k, const std::uint32_t* A,
                                                       std::int64_t lda, const std::uint32_t* B, std::int64_t ldb,
                                                       const std::uint32_t* Cin, std::int64_t ldc, std::uint32_t* D,
                                                       std::int64_t ldd) {
  pdl_wait_and_release();
  __shared__ std::uint32_t sa[kWT][kWT + 1], sb[kWT][kWT + 1];
  const int tx = threadIdx.x & 31, ty = threadIdx.x >> 5;  // 32 x 8 threads, 4 rows each
  const int row0 = blockIdx.y * kWT, col = blockIdx.x * kWT + tx;
  std::uint64_t accp[4] = {0, 0, 0, 0};  // prime fields: exact sums, reduced every 2^31 / p^2 steps
  std::uint32_t acce[4] = {0, 0, 0, 0};  // extension fields
  const bool prime = f.k == 1;
  for (int k0 = 0; k0 < k; k0 += kWT) {
    for (int r = ty; r < kWT; r += 8) {
      const int ar = row0 + r, ac = k0 + tx;
      sa[r][tx] = (ar < m && ac < k) ? A[std::int64_t(ar) * (lda / 4) + ac] : 0u;
      const int br = k0 + r, bc = blockIdx.x * kWT + tx;
      sb[r][tx] = (br < k && bc < n) ? B[std::int64_t(br) * (ldb / 4) + bc] : 0u;
    }
    __syncthreads();
    const int kk = k - k0 < kWT ? k - k0 : kWT;
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      const int r = ty + 8 * q;
      if (prime) {
        std::uint64_t s = 0;
        for (int t = 0; t < kk; ++t) s += std::uint64_t(sa[r][t]) * sb[t][tx];  // < 32 p^2 < 2^37
        accp[q] = (accp[q] + s) % f.p;
      } else {
        std::uint32_t s = acce[q];
        for (int t = 0; t < kk; ++t) s = wadd(f, s, wmul(f, sa[r][t], sb[t][tx]));
        acce[q] = s;
      }
    }
    __syncthreads();
  }
  if (col >= n) return;
#pragma unroll
  for (int q = 0; q < 4; ++q) {
    const int row = row0 + ty + 8 * q;
    if (row >= m) continue;
    std::uint32_t v = prime ? std::uint32_t(accp[q]) : acce[q];
    if (Cin) v = wadd(f, v, Cin[std::int64_t(row) * (ldc / 4) + col]);
    D[std::int64_t(row) * (ldd / 4) + col] = v;
  }
}

// ---- K2w: one CTA, rows x cols <= kEchBaseWideMax^2, the contract of ech_base
__global__ void __launch_bounds__(1024) ech_base_wide_kernel(WideField f, int rows, int cols,
                                                             const std::uint32_t* __restrict__ H, std::int64_t ldh,
                                                             std::uint32_t* W, std::int64_t ldw, std::uint32_t* Tc,
                                                             std::int64_t ldt, std::int32_t* info) {
  extern __shared__ __align__(16) std::uint32_t wsm[];
  const int rmax = rows < cols ? rows : cols;
  std::uint32_t* w = wsm;
  std::uint32_t* t = w + rows * cols;
  std::uint32_t* coef = t + rows * (rmax > 0 ? rmax : 1);
  std::uint32_t* piv = coef + rows;
  __shared__ int sel_s;
  __shared__ int pcol[kEchBaseWideMax], prow[kEchBaseWideMax];
  const int tid = threadIdx.x, nt = blockDim.x;
  for (int e = tid; e < rows * cols; e += nt) w[e] = H[std::int64_t(e / cols) * (ldh / 4) + (e % cols)];
  for (int e = tid; e < rows * rmax; e += nt) t[e] = 0;
  for (int e = tid; e < rows; e += nt) piv[e] = 0;
  __syncthreads();
  const std::uint32_t minus1 = wneg(f, 1);
  int r = 0;
  for (int col = 0; col < cols && r < rmax; ++col) {
    if (tid == 0) sel_s = rows;
    __syncthreads();
    for (int i = tid; i < rows; i += nt)
      if (!piv[i] && w[i * cols + col]) atomicMin(&sel_s, i);
    __syncthreads();
    const int s = sel_s;
    if (s == rows) continue;  // block-uniform
    const std::uint32_t scale = wneg(f, winv(f, w[s * cols + col]));  // pivot entry -> -1
    for (int i = tid; i < rows; i += nt) coef[i] = (i == s) ? 0u : w[i * cols + col];
    __syncthreads();
    const int wcols = cols - col;
    for (int c = tid; c < wcols; c += nt) w[s * cols + col + c] = wmul(f, scale, w[s * cols + col + c]);
    for (int q = tid; q <= r; q += nt) t[s * rmax + q] = q == r ? scale : wmul(f, scale, t[s * rmax + q]);
    __syncthreads();
    // row i += coef_i . (pivot row): the pivot entry is -1, so column col clears
    const int width = wcols + r + 1;
    for (int e = tid; e < rows * width; e += nt) {
      const int i = e / width, c = e - i * width;
      const std::uint32_t cf = coef[i];
      if (!cf) continue;
      if (c < wcols) {
        const int idx = i * cols + col + c;
        w[idx] = wadd(f, w[idx], wmul(f, cf, w[s * cols + col + c]));
      } else {
        const int q = c - wcols;
        t[i * rmax + q] = wadd(f, t[i * rmax + q], wmul(f, cf, t[s * rmax + q]));
      }
    }
    if (tid == 0) {
      piv[s] = 1;
      pcol[r] = col;
      prow[r] = s;
    }
    ++r;
    __syncthreads();
  }
  (void)minus1;
  for (int e = tid; e < rows * cols; e += nt) W[std::int64_t(e / cols) * (ldw / 4) + (e % cols)] = w[e];
  if (r > 0)
    for (int e = tid; e < rows * r; e += nt) Tc[std::int64_t(e / r) * (ldt / 4) + (e % r)] = t[(e / r) * rmax + (e % r)];
  if (tid == 0) info[0] = r;
  for (int q = tid; q < r; q += nt) {
    info[1 + q] = pcol[q];
    info[1 + rmax + q] = prow[q];
  }
}

__global__ void set_entries_u32_kernel(std::uint8_t* dst, std::int64_t ldd, const std::int32_t* pos, std::int64_t n,
                                       std::uint32_t value) {
  pdl_wait_and_release();
  for (std::int64_t q = blockIdx.x * blockDim.x + threadIdx.x; q < n; q += std::int64_t(gridDim.x) * blockDim.x)
    *reinterpret_cast<std::uint32_t*>(dst + std::int64_t(pos[2 * q]) * ldd + 4 * std::int64_t(pos[2 * q + 1])) =
        value;
}

// ---- K6w: counter-form SplitMix64 draws below q (src/generate.cpp:5-24)
__device__ __forceinline__ std::uint64_t mix64(std::uint64_t z) {
  z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ull;
  z = (z ^ (z >> 27)) * 0x94d049bb133111ebull;
  return z ^ (z >> 31);
}
__global__ void random_fill_wide_kernel(std::uint32_t q, std::int64_t rows, std::int64_t cols, std::uint64_t seed,
                                        std::uint64_t draw0, std::int64_t draw_ld, std::uint8_t* dst,
                                        std::int64_t ldd, std::uint32_t* rejects) {
  const std::uint64_t lim = ~0ull - (~0ull % q);
  const std::int64_t total = rows * cols;
  for (std::int64_t e = std::int64_t(blockIdx.x) * blockDim.x + threadIdx.x; e < total;
       e += std::int64_t(gridDim.x) * blockDim.x) {
    const std::int64_t r = e / cols, c = e - r * cols;
    const std::uint64_t t = draw0 + std::uint64_t(r) * std::uint64_t(draw_ld) + std::uint64_t(c);
    const std::uint64_t v = mix64(seed + (t + 1) * 0x9e3779b97f4a7c15ull);
    if (v >= lim) atomicAdd(rejects, 1u);
    *reinterpret_cast<std::uint32_t*>(dst + r * ldd + 4 * c) = std::uint32_t(v % q);
  }
}

__global__ void nonzero_mask_u32_kernel(std::int64_t rows, std::int64_t cols, const std::uint8_t* src,
                                        std::int64_t lds, std::uint8_t* dst, std::int64_t ldd) {
  for (std::int64_t i = blockIdx.y; i < rows; i += gridDim.y)
    for (std::int64_t j = std::int64_t(blockIdx.x) * blockDim.x + threadIdx.x; j < cols;
         j += std::int64_t(gridDim.x) * blockDim.x)
      dst[i * ldd + j] = reinterpret_cast<const std::uint32_t*>(src + i * lds)[j] != 0u;
}

}  // namespace

void nonzero_mask_u32(std::int64_t rows, std::int64_t cols, const std::uint8_t* src, std::int64_t lds,
                      std::uint8_t* dst, std::int64_t ldd, cudaStream_t s) {
  if (rows <= 0 || cols <= 0) return;
  const dim3 grid(unsigned(std::min<std::int64_t>((cols + 255) / 256, 64)), unsigned(std::min<std::int64_t>(rows, 65535)));
  nonzero_mask_u32_kernel<<<grid, 256, 0, s>>>(rows, cols, src, lds, dst, ldd);
  GFQ_CUDA(cudaGetLastError());
  count_launch();
}

void mad_wide(const WideField& f, std::int64_t m, std::int64_t n, std::int64_t k, const std::uint8_t* A,
              std::int64_t lda, const std::uint8_t* B, std::int64_t ldb, const std::uint8_t* Cin, std::int64_t ldc,
              std::uint8_t* D, std::int64_t ldd, cudaStream_t s) {
  if (m <= 0 || n <= 0) return;
  if (k == 0) {
    // D = Cin or 0
    if (Cin == D && ldc == ldd) return;
    if (Cin)
      select2d(D, ldd, m, 4 * n, Cin, ldc, nullptr, 0, nullptr, nullptr, s);
    else
      fill2d(D, ldd, m, 4 * n, 0, s);
    return;
  }
  ProfScope ps(kProfSimt, 2.0 * double(m) * double(n) * double(k), s);
  const dim3 grid(unsigned((n + kWT - 1) / kWT), unsigned((m + kWT - 1) / kWT));
  GFQ_CUDA(launch_pdl(mad_wide_kernel, grid, dim3(256), 0, s, f, int(m), int(n), int(k),
                      reinterpret_cast<const std::uint32_t*>(A), lda, reinterpret_cast<const std::uint32_t*>(B), ldb,
                      reinterpret_cast<const std::uint32_t*>(Cin), ldc, reinterpret_cast<std::uint32_t*>(D), ldd));
  count_launch();
}

void ech_base_wide(const WideField& f, std::int64_t rows, std::int64_t cols, const std::uint8_t* H, std::int64_t ldh,
                   std::uint8_t* W, std::int64_t ldw, std::uint8_t* Tc, std::int64_t ldt, std::int32_t* info,
                   cudaStream_t s) {
  if (rows > kEchBaseWideMax || cols > kEchBaseWideMax) throw std::invalid_argument("ech_base_wide: block too large");
  const int rmax = int(std::min(rows, cols));
  const std::size_t smem = std::size_t(rows * cols + rows * std::max(rmax, 1) + 2 * rows) * 4;
  static bool attr = false;
  if (!attr) {
    GFQ_CUDA(cudaFuncSetAttribute(ech_base_wide_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 96 * 1024));
    attr = true;
  }
  ech_base_wide_kernel<<<1, 1024, smem, s>>>(f, int(rows), int(cols), reinterpret_cast<const std::uint32_t*>(H), ldh,
                                             reinterpret_cast<std::uint32_t*>(W), ldw,
                                             reinterpret_cast<std::uint32_t*>(Tc), ldt, info);
  GFQ_CUDA(cudaGetLastError());
  count_launch();
}

void set_entries_u32(std::uint8_t* dst, std::int64_t ldd, const std::int32_t* pos, std::int64_t n,
                     std::uint32_t value, cudaStream_t s) {
  if (n == 0) return;
  GFQ_CUDA(launch_pdl(set_entries_u32_kernel, dim3(unsigned((n + 255) / 256)), dim3(256), 0, s, dst, ldd, pos, n,
                      value));
  count_launch();
}

void random_fill_wide(std::uint32_t q, std::int64_t rows, std::int64_t cols, std::uint64_t seed, std::uint64_t draw0,
                      std::int64_t draw_ld, std::uint8_t* dst, std::int64_t ldd, std::uint32_t* rejects,
                      cudaStream_t s) {
  if (rows <= 0 || cols <= 0) return;
  const std::int64_t total = rows * cols;
  const unsigned grid = unsigned(std::min<std::int64_t>((total + 255) / 256, std::int64_t(sm_count()) * 8));
  random_fill_wide_kernel<<<grid, 256, 0, s>>>(q, rows, cols, seed, draw0, draw_ld, dst, ldd, rejects);
  GFQ_CUDA(cudaGetLastError());
  count_launch();
}

}  // namespace gfq::dev
