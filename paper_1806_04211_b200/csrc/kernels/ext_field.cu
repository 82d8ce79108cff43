// ext_field.cu -- GF(p^k) (q = p^k <= 256) on the B200 path.
//
// Elements are stored encoded, one byte each (reference include/gfrref/
// field.hpp:12-14: sum_i c_i p^i), so every gather / riffle / view of the
// prime-field path applies unchanged.  Arithmetic:
//   * the block product (reference src/matrix.cpp:116-131, table-driven
//     there) becomes ONE tcgen05 contraction over GF(p): in the polynomial
//     basis, a.b has digit u = sum_{i,j} a_i b_j red[i+j][u] (red = digits
//     of x^s mod the modulus), so with A's digits interleaved (m x kK) and B
//     expanded to the k x k multiplication-by-element blocks (kK x kn), the
//     GF(p) product A'.B' holds the digits of A.B (m x kn), added digit-wise
//     to the addend's digits and re-encoded;
//   * the base-case ECH uses q x q mul / add tables in shared memory.
#include <cstdint>
#include <stdexcept>

#include "../common.hpp"
#include "kernels.hpp"

namespace gfq::dev {
namespace {

// dst[i][k.j + d] = digit d of src[i][j]
__global__ void ext_split_kernel(std::uint32_t k, const std::uint8_t* __restrict__ dig,
                                 std::int64_t rows, std::int64_t cols,
                                 const std::uint8_t* __restrict__ src, std::int64_t lds,
                                 std::uint8_t* __restrict__ dst, std::int64_t ldd) {
  for (std::int64_t i = blockIdx.y; i < rows; i += gridDim.y)
    for (std::int64_t j = blockIdx.x * std::int64_t(blockDim.x) + threadIdx.x; j < cols;
         j += std::int64_t(gridDim.x) * blockDim.x) {
      const std::uint8_t* d = dig + std::uint32_t(src[i * lds + j]) * k;
      std::uint8_t* o = dst + i * ldd + j * k;
      for (std::uint32_t t = 0; t < k; ++t) o[t] = d[t];
    }
}

// Bexp[k.t + i][k.j + u] = sum_{j'} red[i + j'][u] . digit j' of B[t][j]  (mod p).
// One thread writes 16 consecutive bytes of one Bexp row (a 16-byte store);
// the k x k x k coefficients red[i + j'][u] sit in shared memory.
__global__ void ext_expand_kernel(std::uint32_t p, std::uint32_t k,
                                  const std::uint8_t* __restrict__ dig,
                                  const std::uint8_t* __restrict__ red, std::int64_t K,
                                  std::int64_t n, const std::uint8_t* __restrict__ B,
                                  std::int64_t ldb, std::uint8_t* __restrict__ E,
                                  std::int64_t lde) {
  __shared__ std::uint8_t cf[8][8][8];  // cf[i][u][j'] = red[i + j'][u]
  for (std::uint32_t e = threadIdx.x; e < k * k * k; e += blockDim.x) {
    const std::uint32_t i = e / (k * k), u = (e / k) % k, jj = e % k;
    cf[i][u][jj] = red[(i + jj) * k + u];
  }
  __syncthreads();
  const std::int64_t width = std::int64_t(k) * n, nch = (width + 15) / 16;
  for (std::int64_t row = blockIdx.y; row < K * k; row += gridDim.y) {
    const std::int64_t t = row / k;
    const std::uint32_t i = std::uint32_t(row % k);
    const std::uint8_t* brow = B + t * ldb;
    for (std::int64_t ch = blockIdx.x * std::int64_t(blockDim.x) + threadIdx.x; ch < nch;
         ch += std::int64_t(gridDim.x) * blockDim.x) {
      std::uint32_t w[4] = {0, 0, 0, 0};
      const std::int64_t c0 = 16 * ch;
      std::int64_t j = c0 / k;
      std::uint32_t u = std::uint32_t(c0 % k);
      const std::uint8_t* bd = dig + std::uint32_t(j < n ? brow[j] : 0) * k;
      for (int q = 0; q < 16; ++q) {
        if (c0 + q >= width) break;
        std::uint32_t acc = 0;
        for (std::uint32_t jj = 0; jj < k; ++jj) acc += std::uint32_t(cf[i][u][jj]) * bd[jj];
        w[q >> 2] |= (acc % p) << (8 * (q & 3));
        if (++u == k) {
          u = 0;
          ++j;
          bd = dig + std::uint32_t(j < n ? brow[j] : 0) * k;
        }
      }
      *reinterpret_cast<uint4*>(E + row * lde + c0) = make_uint4(w[0], w[1], w[2], w[3]);
    }
  }
}

// dst[i][j] = sum_d src[i][k.j + d] p^d
__global__ void ext_merge_kernel(std::uint32_t p, std::uint32_t k, std::int64_t rows,
                                 std::int64_t cols, const std::uint8_t* __restrict__ src,
                                 std::int64_t lds, std::uint8_t* __restrict__ dst,
                                 std::int64_t ldd) {
  for (std::int64_t i = blockIdx.y; i < rows; i += gridDim.y)
    for (std::int64_t j = blockIdx.x * std::int64_t(blockDim.x) + threadIdx.x; j < cols;
         j += std::int64_t(gridDim.x) * blockDim.x) {
      const std::uint8_t* s = src + i * lds + j * k;
      std::uint32_t v = 0;
      for (std::uint32_t t = k; t-- > 0;) v = v * p + s[t];
      dst[i * ldd + j] = std::uint8_t(v);
    }
}

inline std::int64_t pad16(std::int64_t x) { return (x + 15) / 16 * 16; }

dim3 grid2(std::int64_t rows, std::int64_t cols) {
  const std::int64_t gx = (cols + 127) / 128;
  return dim3(unsigned(gx < 64 ? gx : 64), unsigned(rows < 65535 ? rows : 65535));
}

// Base-case ECH over GF(p^k) (same schedule and conventions as
// ech_base_kernel in kernels.cu: column-wise pivot rule, -1 pivots, compact
// transform in discovery order).
__global__ void __launch_bounds__(1024)
ech_base_ext_kernel(ExtTables f, int rows, int cols, const std::uint8_t* __restrict__ H,
                    std::int64_t ldh, std::uint8_t* W, std::int64_t ldw, std::uint8_t* Tc,
                    std::int64_t ldt, std::int32_t* info) {
  extern __shared__ __align__(16) std::uint8_t sm[];
  const int q = int(f.q);
  const int rmax = rows < cols ? rows : cols;
  std::uint8_t* mulT = sm;              // q x q
  std::uint8_t* addT = mulT + q * q;    // q x q
  std::uint8_t* w = addT + q * q;       // rows x cols
  std::uint8_t* t = w + rows * cols;    // rows x rmax
  std::uint8_t* coef = t + rows * (rmax > 0 ? rmax : 1);
  std::uint8_t* piv = coef + rows;
  __shared__ int sel_s;
  __shared__ int pcol[kEchBaseMax], prow[kEchBaseMax];
  const int tid = threadIdx.x, nt = blockDim.x;
  const int warp = tid >> 5, lane = tid & 31, nw = nt >> 5;

  for (int e = tid; e < q * q; e += nt) {
    mulT[e] = f.mul[e];
    addT[e] = f.add[e];
  }
  for (int e = tid; e < rows * cols; e += nt) w[e] = H[std::int64_t(e / cols) * ldh + (e % cols)];
  for (int e = tid; e < rows * rmax; e += nt) t[e] = 0;
  for (int e = tid; e < rows; e += nt) piv[e] = 0;
  __syncthreads();

  int r = 0;
  for (int col = 0; col < cols && r < rmax; ++col) {
    if (tid == 0) sel_s = rows;
    __syncthreads();
    for (int i = tid; i < rows; i += nt)
      if (!piv[i] && w[i * cols + col]) atomicMin(&sel_s, i);
    __syncthreads();
    const int s = sel_s;
    if (s == rows) continue;  // block-uniform
    const int scale = f.neg[f.inv[w[s * cols + col]]];  // -1/pivot
    for (int i = tid; i < rows; i += nt) coef[i] = (i == s) ? 0 : w[i * cols + col];
    __syncthreads();
    const int wcols = cols - col;
    for (int c = tid; c < wcols; c += nt)
      w[s * cols + col + c] = mulT[scale * q + w[s * cols + col + c]];
    for (int u = tid; u <= r; u += nt)
      t[s * rmax + u] = u == r ? std::uint8_t(scale) : mulT[scale * q + t[s * rmax + u]];
    __syncthreads();
    // x_i += coef_i . (normalised pivot row), whose pivot entry is -1
    const int width = wcols + r + 1;
    for (int i = warp; i < rows; i += nw) {
      const int cf = coef[i];
      if (!cf) continue;
      for (int e = lane; e < width; e += 32) {
        std::uint8_t* x;
        std::uint8_t b;
        if (e < wcols) {
          x = w + i * cols + col + e;
          b = w[s * cols + col + e];
        } else {
          x = t + i * rmax + (e - wcols);
          b = t[s * rmax + (e - wcols)];
        }
        *x = addT[*x * q + mulT[cf * q + b]];
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
  for (int e = tid; e < rows * cols; e += nt) W[std::int64_t(e / cols) * ldw + (e % cols)] = w[e];
  if (r > 0)
    for (int e = tid; e < rows * r; e += nt)
      Tc[std::int64_t(e / r) * ldt + (e % r)] = t[(e / r) * rmax + (e % r)];
  if (tid == 0) info[0] = r;
  for (int u = tid; u < r; u += nt) {
    info[1 + u] = pcol[u];
    info[1 + rmax + u] = prow[u];
  }
}

}  // namespace

std::int64_t mad_ext_scratch_bytes(std::uint32_t k, std::int64_t m, std::int64_t n, std::int64_t K) {
  return m * pad16(k * K) + K * k * pad16(k * n) + 2 * m * pad16(k * n) + 64;
}

void mad_ext(const ExtTables& f, std::int64_t m, std::int64_t n, std::int64_t K,
             const std::uint8_t* A, std::int64_t lda, const std::uint8_t* B, std::int64_t ldb,
             const std::uint8_t* Cin, std::int64_t ldc, std::uint8_t* D, std::int64_t ldd,
             std::uint8_t* scratch, cudaStream_t s) {
  if (m == 0 || n == 0) return;
  const std::uint32_t k = f.k;
  const std::int64_t lda2 = pad16(k * K), lde = pad16(k * n), ldc2 = pad16(k * n);
  std::uint8_t* A2 = scratch;
  std::uint8_t* E = A2 + m * lda2;
  std::uint8_t* C2 = E + K * k * lde;
  std::uint8_t* D2 = C2 + m * ldc2;
  const std::uint8_t* cin2 = nullptr;
  if (Cin) {
    ext_split_kernel<<<grid2(m, n), 128, 0, s>>>(k, f.dig, m, n, Cin, ldc, C2, ldc2);
    GFQ_CUDA(cudaGetLastError());
    count_launch();
    cin2 = C2;
  }
  if (K > 0) {
    ext_split_kernel<<<grid2(m, K), 128, 0, s>>>(k, f.dig, m, K, A, lda, A2, lda2);
    GFQ_CUDA(cudaGetLastError());
    {
      const std::int64_t nch = (std::int64_t(k) * n + 15) / 16, rows = K * k;
      const dim3 g(unsigned((nch + 127) / 128 < 64 ? (nch + 127) / 128 : 64),
                   unsigned(rows < 65535 ? rows : 65535));
      ext_expand_kernel<<<g, 128, 0, s>>>(f.p, k, f.dig, f.red, K, n, B, ldb, E, lde);
    }
    GFQ_CUDA(cudaGetLastError());
    count_launch(2);
  }
  // the digits of Cin + A.B over GF(p): one K1 contraction (k K deep)
  mad(f.p, m, k * n, k * K, A2, lda2, E, lde, cin2, ldc2, D2, ldc2, s);
  ext_merge_kernel<<<grid2(m, n), 128, 0, s>>>(f.p, k, m, n, D2, ldc2, D, ldd);
  GFQ_CUDA(cudaGetLastError());
  count_launch();
}

void ech_base_ext(const ExtTables& f, std::int64_t rows, std::int64_t cols, const std::uint8_t* H,
                  std::int64_t ldh, std::uint8_t* W, std::int64_t ldw, std::uint8_t* Tc,
                  std::int64_t ldt, std::int32_t* info, cudaStream_t s) {
  if (rows > kEchBaseMax || cols > kEchBaseMax)
    throw std::invalid_argument("ech_base_ext: block exceeds the base-case size");
  const std::int64_t rmax = rows < cols ? rows : cols;
  const std::size_t smem = std::size_t(2 * f.q * f.q + rows * cols + rows * (rmax > 0 ? rmax : 1) +
                                       2 * rows);
  static bool attr_set = false;
  if (!attr_set) {
    GFQ_CUDA(cudaFuncSetAttribute(ech_base_ext_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                  200 * 1024));
    attr_set = true;
  }
  int threads = int(rows * 32);
  threads = threads < 64 ? 64 : (threads > 1024 ? 1024 : threads);
  ech_base_ext_kernel<<<1, threads, smem, s>>>(f, int(rows), int(cols), H, ldh, W, ldw, Tc, ldt,
                                               info);
  GFQ_CUDA(cudaGetLastError());
  count_launch();
}

}  // namespace gfq::dev
