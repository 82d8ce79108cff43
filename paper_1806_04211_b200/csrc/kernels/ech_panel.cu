// ech_panel.cu -- K2: the panel step of the device ECH.
//
// The block H (rows x cols) is eliminated in place inside the augmented
// matrix Aug = [W | T] (T = I at the start) by right-looking Gauss-Jordan
// over panels of w <= 32 columns.  This kernel is the latency-critical part
// of a panel: one CTA holds the panel columns of every row in shared memory
// and runs the reference's column-wise pivot rule on the rows that are not
// yet pivotal (first non-pivotal row with a nonzero entry, reference
// src/chief.cpp:436-460; the same canonical rho/gamma as direct_gauss,
// SURVEY 8c): warp min-reduction + one shared atomic per warp for the pivot
// search, the pivot row broadcast through shared memory, a packed rank-1
// elimination of the panel (XOR words for p = 2).  It then inverts the
// r2 x r2 pivot block with the whole CTA and emits the panel multipliers
//   G = Ap.N2, Ap = Aug[:, c0 + gamma2] (+ I on the new pivot rows),
//   N2 = -inv(Aug[rho2, c0 + gamma2]),
// so that Aug[:, c0:] += G.Aug[rho2, c0:] finishes the panel (K1).  Nothing
// returns to the host until the last panel: the ECH is a fixed launch
// sequence.
#include <algorithm>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <stdexcept>
#include <unordered_map>
#include <mutex>

#include "../common.hpp"
#include "kernels.hpp"

namespace gfq::dev {
namespace {

__device__ __forceinline__ std::uint32_t modp(std::uint32_t x, std::uint32_t p,
                                              std::uint32_t magic) {
  const std::uint32_t q = __umulhi(x, magic);
  const std::int32_t r = static_cast<std::int32_t>(x - q * p);
  return static_cast<std::uint32_t>(r < 0 ? r + static_cast<std::int32_t>(p) : r);
}

__device__ __forceinline__ std::uint32_t powmod(std::uint32_t a, std::uint32_t e,
                                                std::uint32_t p) {
  std::uint32_t r = 1, b = a % p;
  while (e) {
    if (e & 1) r = (r * b) % p;
    b = (b * b) % p;
    e >>= 1;
  }
  return r;
}

constexpr int kW = 32;  // max panel width (bytes per panel row in smem)

// Load the 32-byte panel segment of row i (bytes >= wc zeroed).
__device__ __forceinline__ void load_seg(const std::uint8_t* src, int wc, uint4& a, uint4& b) {
  // (L2 loads: the overlapped step chain reads rows another grid is still
  // updating -- see ech_step)
  if (wc == kW && (reinterpret_cast<std::uintptr_t>(src) & 15) == 0) {
    a = __ldcg(reinterpret_cast<const uint4*>(src));
    b = __ldcg(reinterpret_cast<const uint4*>(src) + 1);
    return;
  }
  std::uint32_t w[8] = {0, 0, 0, 0, 0, 0, 0, 0};
#pragma unroll
  for (int c = 0; c < kW; ++c)
    if (c < wc) w[c >> 2] |= std::uint32_t(__ldcg(src + c)) << (8 * (c & 3));
  a = make_uint4(w[0], w[1], w[2], w[3]);
  b = make_uint4(w[4], w[5], w[6], w[7]);
}

// byte k (0..31) of a row held as 8 packed words
// (a select tree in PTX: a plain select chain is turned back into a
// dynamically indexed local-memory array by the compiler)
__device__ __forceinline__ std::uint32_t sel(bool c, std::uint32_t a, std::uint32_t b) {
  std::uint32_t r;
  asm("{ .reg .pred q; setp.ne.u32 q, %1, 0; selp.b32 %0, %2, %3, q; }"
      : "=r"(r) : "r"(std::uint32_t(c)), "r"(a), "r"(b));
  return r;
}
__device__ __forceinline__ std::uint32_t byte_of(const std::uint32_t (&w)[8], int k) {
  const bool b2 = k & 4, b3 = k & 8, b4 = k & 16;
  const std::uint32_t x01 = sel(b2, w[1], w[0]), x23 = sel(b2, w[3], w[2]);
  const std::uint32_t x45 = sel(b2, w[5], w[4]), x67 = sel(b2, w[7], w[6]);
  const std::uint32_t x = sel(b4, sel(b3, x67, x45), sel(b3, x23, x01));
  return (x >> (8 * (k & 3))) & 0xFFu;
}
// Step outputs of the two-level ECH (ech_step_chain_kernel): instead of G
// for every row, the 32 x 32 map NT (NT[t][c] = multiplier of panel column
// c's ORIGINAL value in G[i][t], zero for non-pivot columns, so G[i] =
// seg_i . NT^T for every row that is not a new pivot) and Gpiv (G rows of
// the r2 new pivot rows, in pivot order); ech_step_update_kernel applies them.
struct StepOut {
  std::uint8_t* NT;
  std::uint8_t* Gpiv;
};

__device__ __forceinline__ void panel_full(std::uint32_t p, std::uint32_t magic, int rows, int c0,
                                           int wc, const std::uint8_t* __restrict__ Aug,
                                           std::int64_t ld, std::uint8_t* flags, std::int32_t* info,
                                           int cap, std::uint8_t* G, std::int64_t ldg,
                                           std::int32_t* rho2, StepOut so = StepOut{nullptr, nullptr}) {
  extern __shared__ __align__(16) std::uint8_t sm[];
  std::uint8_t* P = sm;                   // rows x kW
  std::uint8_t* fl = sm + rows * kW;      // rows (pivot flags)
  __shared__ std::uint8_t invt[256];
  __shared__ __align__(16) std::uint8_t prow[kW];
  __shared__ unsigned sel_s;
  __shared__ int pc[kW], pr[kW];
  __shared__ std::uint8_t X[kW][2 * kW];  // [pivot block | I] -> [I | inverse]
  __shared__ std::uint32_t N2[kW][kW];    // -inverse, zero padded
  __shared__ int r_old, piv_s;
  const int tid = threadIdx.x, nt = blockDim.x, lane = tid & 31;

  for (int a = tid; a < 256; a += nt)
    invt[a] = (a > 0 && std::uint32_t(a) < p) ? std::uint8_t(powmod(a, p - 2, p)) : 0;
  for (int i = tid; i < rows; i += nt) {
    const std::uint8_t f = __ldcg(flags + i);
    fl[i] = f;
    if (!f) {
      uint4 a, b;
      load_seg(Aug + std::int64_t(i) * ld + c0, wc, a, b);
      reinterpret_cast<uint4*>(P + i * kW)[0] = a;
      reinterpret_cast<uint4*>(P + i * kW)[1] = b;
    }
  }
  if (tid == 0) r_old = __ldcg(info);
  __syncthreads();

  // ---- column-wise Gauss-Jordan on the non-pivotal rows of the panel
  int r2 = 0;
  for (int c = 0; c < wc; ++c) {
    if (tid == 0) sel_s = 0xFFFFFFFFu;
    __syncthreads();
    unsigned cand = 0xFFFFFFFFu;
    for (int i = tid; i < rows; i += nt)
      if (!fl[i] && P[i * kW + c] && unsigned(i) < cand) cand = unsigned(i);
    cand = __reduce_min_sync(0xffffffffu, cand);
    if (lane == 0 && cand != 0xFFFFFFFFu) atomicMin(&sel_s, cand);
    __syncthreads();
    const unsigned s = sel_s;
    if (s != 0xFFFFFFFFu) {
      const std::uint32_t scale = p - invt[P[s * kW + c]];
      if (tid < kW)
        prow[tid] = tid < c ? 0 : std::uint8_t(modp(scale * P[s * kW + tid], p, magic));
      if (tid == 0) {
        fl[s] = 1;
        pc[r2] = c;
        pr[r2] = int(s);
      }
      __syncthreads();
      const std::uint32_t* pw = reinterpret_cast<const std::uint32_t*>(prow);
      const int w0 = c >> 2;
      for (int i = tid; i < rows; i += nt) {
        if (fl[i]) continue;
        const std::uint32_t cf = P[i * kW + c];
        if (!cf) continue;
        std::uint32_t* rw = reinterpret_cast<std::uint32_t*>(P + i * kW);
        if (p == 2) {
#pragma unroll
          for (int q = 0; q < kW / 4; ++q)
            if (q >= w0) rw[q] ^= pw[q];
        } else {
#pragma unroll
          for (int q = 0; q < kW / 4; ++q) {
            if (q < w0) continue;
            const std::uint32_t a = rw[q], b = pw[q];
            // two 16-bit lanes per multiply: (p-1)^2 + (p-1) < 2^16
            const std::uint32_t lo = (a & 0x00FF00FFu) + cf * (b & 0x00FF00FFu);
            const std::uint32_t hi = ((a >> 8) & 0x00FF00FFu) + cf * ((b >> 8) & 0x00FF00FFu);
            rw[q] = modp(lo & 0xFFFF, p, magic) | (modp(hi & 0xFFFF, p, magic) << 8) |
                    (modp(lo >> 16, p, magic) << 16) | (modp(hi >> 16, p, magic) << 24);
          }
        }
      }
      ++r2;
    }
    __syncthreads();
  }

  // ---- N2 = -inv(Aug[rho2, c0 + gamma2]) with the whole CTA
  for (int e = tid; e < kW * 2 * kW; e += nt) {
    const int q = e / (2 * kW), t = e % (2 * kW);
    std::uint8_t v = 0;
    if (q < r2 && t < r2) v = __ldcg(Aug + std::int64_t(pr[q]) * ld + c0 + pc[t]);
    else if (q < r2 && t >= kW && t - kW == q) v = 1;
    X[q][t] = v;
  }
  __syncthreads();
  for (int q = 0; q < r2; ++q) {
    if (tid < 32) {
      const unsigned bal = __ballot_sync(0xffffffffu, tid >= q && tid < r2 && X[tid][q] != 0);
      if (tid == 0) piv_s = __ffs(bal) - 1;
    }
    __syncthreads();
    const int pv = piv_s;
    if (pv != q && tid < 2 * kW) {
      const std::uint8_t t0 = X[q][tid];
      X[q][tid] = X[pv][tid];
      X[pv][tid] = t0;
    }
    __syncthreads();
    const std::uint32_t iv = invt[X[q][q]];
    __syncthreads();
    if (tid < 2 * kW) X[q][tid] = std::uint8_t(modp(iv * X[q][tid], p, magic));
    __syncthreads();
    // eliminate column q from the other rows: element (row, col) per thread
    for (int e = tid; e < kW * 2 * kW; e += nt) {
      const int row = e / (2 * kW), col = e % (2 * kW);
      if (row >= r2 || row == q) continue;
      const std::uint32_t f = X[row][q];
      if (!f || col == q) continue;
      X[row][col] = std::uint8_t(modp(X[row][col] + (p - f) * X[q][col], p, magic));
    }
    __syncthreads();
    if (tid < kW && tid < r2 && tid != q) X[tid][q] = 0;
    __syncthreads();
  }
  for (int e = tid; e < kW * kW; e += nt) {
    const int q = e / kW, t = e % kW;
    std::uint32_t v = 0;
    if (q < r2 && t < r2) {
      const std::uint32_t x = X[q][kW + t];
      v = x ? p - x : 0;
    }
    N2[q][t] = v;
  }
  if (tid < kW) rho2[tid] = tid < r2 ? pr[tid] : -1;
  if (tid < r2) {
    info[1 + r_old + tid] = c0 + pc[tid];
    info[1 + cap + r_old + tid] = pr[tid];
    flags[pr[tid]] = 1;
  }
  if (tid == 0) info[0] = r_old + r2;
  __syncthreads();

  if (so.NT) {
    // NT[t][pc[q]] = N2[q][t]; Gpiv[q] = Ap[pr[q]].N2 (Ap row with its +1)
    for (int e = tid; e < kW * kW; e += nt) {
      const int t = e / kW, c = e % kW;
      std::uint32_t v = 0;
      for (int q = 0; q < r2; ++q)
        if (pc[q] == c) v = N2[q][t];
      so.NT[e] = std::uint8_t(v);
    }
    for (int e = tid; e < kW * kW; e += nt) {
      const int q = e / kW, t = e % kW;
      std::uint32_t acc = 0;
      if (q < r2) {
        const std::uint8_t* src = Aug + std::int64_t(pr[q]) * ld + c0;
        acc = N2[q][t];
        for (int u = 0; u < r2; ++u) acc += std::uint32_t(__ldcg(src + pc[u])) * N2[u][t];
      }
      so.Gpiv[e] = std::uint8_t(modp(acc, p, magic));
    }
    return;
  }

  // ---- G[i] = Ap[i].N2, Ap[i][q] = Aug[i][c0 + pc[q]] (+1 on pivot row of q)
  for (int i = tid; i < rows; i += nt) {
    uint4 a, b;
    load_seg(Aug + std::int64_t(i) * ld + c0, wc, a, b);
    const std::uint32_t seg[8] = {a.x, a.y, a.z, a.w, b.x, b.y, b.z, b.w};
    std::uint32_t acc[kW];
#pragma unroll
    for (int t = 0; t < kW; ++t) acc[t] = 0;
    for (int q = 0; q < r2; ++q) {
      const int cq = pc[q];
      std::uint32_t v = byte_of(seg, cq);
      if (pr[q] == i) v += 1;
      if (!v) continue;
#pragma unroll
      for (int t = 0; t < kW; ++t) acc[t] += v * N2[q][t];
    }
    std::uint32_t outw[kW / 4];
#pragma unroll
    for (int t4 = 0; t4 < kW / 4; ++t4) {
      std::uint32_t word = 0;
#pragma unroll
      for (int by = 0; by < 4; ++by) word |= modp(acc[4 * t4 + by], p, magic) << (8 * by);
      outw[t4] = word;
    }
    uint4* dst = reinterpret_cast<uint4*>(G + std::int64_t(i) * ldg);
    dst[0] = make_uint4(outw[0], outw[1], outw[2], outw[3]);
    dst[1] = make_uint4(outw[4], outw[5], outw[6], outw[7]);
  }
}

__global__ void __launch_bounds__(1024)
ech_panel_kernel(std::uint32_t p, std::uint32_t magic, int rows, int c0, int wc, int w,
                 const std::uint8_t* __restrict__ Aug, std::int64_t ld, std::uint8_t* flags,
                 std::int32_t* info, int cap, std::uint8_t* G, std::int64_t ldg,
                 std::int32_t* rho2) {
  (void)w;
  panel_full(p, magic, rows, c0, wc, Aug, ld, flags, info, cap, G, ldg, rho2);
}

// a + v * b, bytewise mod p (two 16-bit lanes per product)
__device__ __forceinline__ std::uint32_t axpy4(std::uint32_t a, std::uint32_t v, std::uint32_t b,
                                               std::uint32_t p, std::uint32_t magic) {
  const std::uint32_t lo = (a & 0x00FF00FFu) + v * (b & 0x00FF00FFu);
  const std::uint32_t hi = ((a >> 8) & 0x00FF00FFu) + v * ((b >> 8) & 0x00FF00FFu);
  return modp(lo & 0xFFFF, p, magic) | (modp(hi & 0xFFFF, p, magic) << 8) |
         (modp(lo >> 16, p, magic) << 16) | (modp(hi >> 16, p, magic) << 24);
}

// General p, windowed: the panel's pivots all lie in the 64 rows from the
// first non-pivotal one when the panel has full rank (the chosen row is the
// FIRST non-pivotal row with a nonzero), so warp 0 runs the chain on that
// window alone (2 rows per lane, no barriers), tracking for each row the
// coefficients of the pivot rows' ORIGINAL values added to it (Gauss-Jordan,
// so pivot rows are reduced too; a pivot row is scaled by -1/pivot).  Then
//   G[pivot row q] = its coefficients ĉ_q,
//   G[other row i] = a_i . (I + Ĉ), a_i = orig_i at the pivot columns,
// the same multipliers ech_panel_kernel produces through -inv(pivot block).
// A column without a window candidate while rows outside the window are
// still open sends the panel to the full CTA algorithm.
__device__ __forceinline__ void win_body(std::uint32_t p, std::uint32_t magic, int rows, int c0, int wc,
                                         const std::uint8_t* __restrict__ Aug, std::int64_t ld,
                                         std::uint8_t* flags, std::int32_t* info, int cap,
                                         std::uint8_t* G, std::int64_t ldg, std::int32_t* rho2,
                                         std::int32_t* lo_state, StepOut so) {
  __shared__ std::uint8_t invw[256];
  __shared__ int wpc[kW], wpr[kW], wr2, wok, wrold;
  __shared__ __align__(16) std::uint32_t chat[kW][kW / 4];  // pivot q's coefficients (packed)
  __shared__ std::uint32_t Nm[kW][kW];                       // I + Ĉ
  __shared__ std::uint32_t sP[8], sCP[8];                    // current pivot row / coefficients
  const int tid = threadIdx.x, nt = blockDim.x, lane = tid & 31;
  for (int a = tid; a < 256; a += nt)
    invw[a] = (a > 0 && std::uint32_t(a) < p) ? std::uint8_t(powmod(a, p - 2, p)) : 0;
  if (tid == 0) wrold = info[0];
  __syncthreads();
  if (tid < 32) {
    const int r_old = wrold;
    int lo = *lo_state;
    for (;;) {
      const int idx = lo + lane;
      const unsigned b = __ballot_sync(0xffffffffu, idx < rows && flags[idx] == 0);
      if (b || lo >= rows) {
        if (b) lo += __ffs(b) - 1;
        break;
      }
      lo += 32;
    }
    if (lo > rows) lo = rows;
    const int i0 = lo + lane, i1 = lo + 32 + lane;
    std::uint32_t w0[8], w1[8], k0[8], k1[8];
    {
      uint4 a, b;
      if (i0 < rows) load_seg(Aug + std::int64_t(i0) * ld + c0, wc, a, b);
      else a = b = make_uint4(0, 0, 0, 0);
      w0[0] = a.x; w0[1] = a.y; w0[2] = a.z; w0[3] = a.w; w0[4] = b.x; w0[5] = b.y; w0[6] = b.z; w0[7] = b.w;
      if (i1 < rows) load_seg(Aug + std::int64_t(i1) * ld + c0, wc, a, b);
      else a = b = make_uint4(0, 0, 0, 0);
      w1[0] = a.x; w1[1] = a.y; w1[2] = a.z; w1[3] = a.w; w1[4] = b.x; w1[5] = b.y; w1[6] = b.z; w1[7] = b.w;
    }
#pragma unroll
    for (int q = 0; q < 8; ++q) k0[q] = k1[q] = 0;
    bool p0 = i0 >= rows || flags[i0] != 0, p1 = i1 >= rows || flags[i1] != 0;
    const int open_in = __popc(__ballot_sync(0xffffffffu, !p0)) + __popc(__ballot_sync(0xffffffffu, !p1));
    const bool covers_all = open_in == rows - r_old;
    int q0 = -1, q1 = -1;  // pivot index of my rows, if any
    int r2 = 0, ok = 1;
    // one column per iteration, NOT unrolled: the unrolled 32-column chain
    // is ~300 KB of SASS run once by one warp, i.e. instruction-fetch bound
#pragma unroll 1
    for (int c = 0; c < wc; ++c) {
      const int cw = c >> 2;
      const std::uint32_t v0 = byte_of(w0, c), v1 = byte_of(w1, c);
      const unsigned b0 = __ballot_sync(0xffffffffu, v0 != 0 && !p0);
      const unsigned b1 = __ballot_sync(0xffffffffu, v1 != 0 && !p1);
      if (!(b0 | b1)) {
        if (covers_all) continue;  // a free column
        ok = 0;
        goto chain_done;
      }
      const int hi = b0 ? 0 : 1;
      const int sl = __ffs(hi ? b1 : b0) - 1;
      // the pivot lane scales its row by s = -1/v and forms the coefficients
      if (lane == sl) {
        std::uint32_t P[8], CP[8];
        const std::uint32_t v = hi ? v1 : v0;
        const std::uint32_t sc = p - invw[v];
#pragma unroll
        for (int q = 0; q < 8; ++q) {
          P[q] = axpy4(0, sc, hi ? w1[q] : w0[q], p, magic);
          CP[q] = axpy4(0, sc, hi ? k1[q] : k0[q], p, magic);
        }
        // + (s - 1) on its own pivot index r2
        const int wq = r2 >> 2, sh = 8 * (r2 & 3);
#pragma unroll
        for (int q = 0; q < 8; ++q) {
          const std::uint32_t m = sel(q == wq, 0xFFu << sh, 0u);
          const std::uint32_t nv = modp(((CP[q] >> sh) & 0xFFu) + sc + p - 1, p, magic);
          CP[q] = (CP[q] & ~m) | ((nv << sh) & m);
        }
#pragma unroll
        for (int q = 0; q < 8; ++q) {
          sP[q] = P[q];
          sCP[q] = CP[q];
        }
      }
      __syncwarp();
      const std::uint32_t* P = sP;
      const std::uint32_t* CP = sCP;
      const bool me0 = !hi && lane == sl, me1 = hi && lane == sl;
      // the pivot's own index bit: coefficient v on pivot r2 (the "+e_q")
      const int wq = r2 >> 2, sh = 8 * (r2 & 3);
      if (me0) {
#pragma unroll
        for (int q = 0; q < 8; ++q) { w0[q] = P[q]; k0[q] = CP[q]; }
        p0 = true;
        q0 = r2;
      } else if (v0) {
#pragma unroll
        for (int q = 0; q < 8; ++q) {
          if (q >= cw) w0[q] = axpy4(w0[q], v0, P[q], p, magic);
          const std::uint32_t e = sel(q == wq, 1u << sh, 0u);
          k0[q] = axpy4(k0[q], v0, CP[q] + e, p, magic);
        }
      }
      if (me1) {
#pragma unroll
        for (int q = 0; q < 8; ++q) { w1[q] = P[q]; k1[q] = CP[q]; }
        p1 = true;
        q1 = r2;
      } else if (v1) {
#pragma unroll
        for (int q = 0; q < 8; ++q) {
          if (q >= cw) w1[q] = axpy4(w1[q], v1, P[q], p, magic);
          const std::uint32_t e = sel(q == wq, 1u << sh, 0u);
          k1[q] = axpy4(k1[q], v1, CP[q] + e, p, magic);
        }
      }
      __syncwarp();  // sP/sCP are rewritten by the next pivot
      if (lane == 0) {
        wpc[r2] = c;
        wpr[r2] = lo + 32 * hi + sl;
      }
      ++r2;
    }
  chain_done:
    if (ok) {
      if (q0 >= 0) {
#pragma unroll
        for (int q = 0; q < 8; ++q) chat[q0][q] = k0[q];
      }
      if (q1 >= 0) {
#pragma unroll
        for (int q = 0; q < 8; ++q) chat[q1][q] = k1[q];
      }
    }
    if (lane == 0) {
      wok = ok;
      wr2 = r2;
      *lo_state = lo;
    }
  }
  __syncthreads();
  if (!wok) {
    panel_full(p, magic, rows, c0, wc, Aug, ld, flags, info, cap, G, ldg, rho2, so);
    return;
  }
  const int r2 = wr2, r_old = wrold;
  // N = I + Ĉ (u32 entries < p)
  for (int e = tid; e < kW * kW; e += nt) {
    const int q = e / kW, t = e % kW;
    std::uint32_t v = 0;
    if (q < r2 && t < r2) {
      v = (chat[q][t >> 2] >> (8 * (t & 3))) & 0xFFu;
      if (t == q) v = v + 1 == p ? 0 : v + 1;
    }
    Nm[q][t] = v;
  }
  if (tid < kW) rho2[tid] = tid < r2 ? wpr[tid] : -1;
  if (tid < r2) {
    info[1 + r_old + tid] = c0 + wpc[tid];
    info[1 + cap + r_old + tid] = wpr[tid];
  }
  __syncthreads();
  if (so.NT) {
    // NT[t][wpc[q]] = Nm[q][t]; Gpiv[q] = ĉ_q
    for (int e = tid; e < kW * kW; e += nt) {
      const int t = e / kW, c = e % kW;
      std::uint32_t v = 0;
      for (int q = 0; q < r2; ++q)
        if (wpc[q] == c) v = Nm[q][t];
      so.NT[e] = std::uint8_t(v);
      const int q = e / kW, tt = e % kW;
      so.Gpiv[e] = q < r2 ? std::uint8_t((chat[q][tt >> 2] >> (8 * (tt & 3))) & 0xFFu) : 0;
    }
    if (tid < r2) flags[wpr[tid]] = 1;
    if (tid == 0) info[0] = r_old + r2;
    return;
  }
  for (int i = tid; i < rows; i += nt) {
    int qi = -1;
    for (int q = 0; q < r2; ++q)
      if (wpr[q] == i) qi = q;
    std::uint32_t outw[kW / 4];
    if (qi >= 0) {
#pragma unroll
      for (int t4 = 0; t4 < kW / 4; ++t4) outw[t4] = chat[qi][t4];
    } else {
      uint4 a, b;
      load_seg(Aug + std::int64_t(i) * ld + c0, wc, a, b);
      const std::uint32_t seg[8] = {a.x, a.y, a.z, a.w, b.x, b.y, b.z, b.w};
      std::uint32_t acc[kW];
#pragma unroll
      for (int t = 0; t < kW; ++t) acc[t] = 0;
      for (int q = 0; q < r2; ++q) {
        const int cq = wpc[q];
        const std::uint32_t v = byte_of(seg, cq);
        if (!v) continue;
#pragma unroll
        for (int t = 0; t < kW; ++t) acc[t] += v * Nm[q][t];
      }
#pragma unroll
      for (int t4 = 0; t4 < kW / 4; ++t4) {
        std::uint32_t word = 0;
#pragma unroll
        for (int by = 0; by < 4; ++by) word |= modp(acc[4 * t4 + by], p, magic) << (8 * by);
        outw[t4] = word;
      }
    }
    uint4* dst = reinterpret_cast<uint4*>(G + std::int64_t(i) * ldg);
    dst[0] = make_uint4(outw[0], outw[1], outw[2], outw[3]);
    dst[1] = make_uint4(outw[4], outw[5], outw[6], outw[7]);
  }
  __syncthreads();
  if (tid < r2) flags[wpr[tid]] = 1;
  if (tid == 0) info[0] = r_old + r2;
}

__global__ void __launch_bounds__(1024)
ech_panel_win_kernel(std::uint32_t p, std::uint32_t magic, int rows, int c0, int wc,
                     const std::uint8_t* __restrict__ Aug, std::int64_t ld, std::uint8_t* flags,
                     std::int32_t* info, int cap, std::uint8_t* G, std::int64_t ldg,
                     std::int32_t* rho2, std::int32_t* lo_state) {
  pdl_wait_and_release();
  win_body(p, magic, rows, c0, wc, Aug, ld, flags, info, cap, G, ldg, rho2, lo_state,
           StepOut{nullptr, nullptr});
}

// Two-level ECH, step part 1 (one CTA of kChainThreads): the pivot chain of
// the 32-wide step at scratch column c0 on the 64-row window from the first
// open row (the pivots all lie there when the step's panel has full rank --
// the chosen row is the FIRST open row with a nonzero).  Warp 0 runs the
// chain alone, barrier-free (see the loop below); a column with no window
// candidate while open rows lie outside the window sends the step to the
// full CTA algorithm (panel_full, all threads).
// Then
//   * NT / Gpiv (StepOut) instead of G: G[new pivot q] = ĉ_q, G[other i] =
//     seg_i[pc] . (I + Ĉ)  (the multipliers of ech_panel_kernel),
//   * Y[rho2[q], r_old + q - *base] = 1 (the outer panel's tracking units),
//   * BpT[j][q] = Z[rho2[q]][c0 + j] for j < n (q >= r2: 0), the step's
//     pivot rows transposed so ech_step_update_kernel contracts over q with
//     dp4a (n x 32 bytes).
constexpr int kStepThreads = 256;
// The step kernels chain with programmatic dependent launch (launch_pdl,
// kernels.hpp): the chain releases its dependents only after the chain loop,
// so the update's CTAs do not sit on SMs other streams' K1 tiles could use.
// developer timing (GFQ_STEP_DEBUG): globaltimer stamps of the chain phases
__device__ unsigned long long g_step_stamps[16];
// developer timeline (GFQ_STEP_TL=N): per step, globaltimer at the chain's
// entry / counter wait / loop end / exit and the update's CTA-0 entry /
// first-pass signal / exit and the last update CTA's exit
constexpr int kTlSteps = 512;
__device__ unsigned long long g_tl[kTlSteps][8];
__device__ __forceinline__ unsigned long long gtime() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}
__device__ __forceinline__ void stamp(int k) {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  if (threadIdx.x == 0) {
    g_step_stamps[k] = t;
    g_step_stamps[8 + k] = clock64();
  }
}
// warp 0 runs the chain; the other warps join the fallback and the outputs
constexpr int kChainThreads = 128;
constexpr int kStepRows = 32, kStepMaxN = 512;
// Overlapped steps (ech_step, `chained`): the chain of step s+1 runs while
// the update of step s is still writing, synchronised through two counters
// instead of the grid boundary: every update CTA bumps ctr[0] once its
// rows' first 128 columns (the next step's panel columns among them) are
// final and ctr[1] once all its columns are; the chain waits for ctr[0] to
// read the panel and for ctr[1] before it reads whole rows or writes
// anything the update reads (rho2 / NT / Gpiv / BpT, the Y units).  The
// counters only grow (a reset would race: the chain of step s+1 may start
// while that of step s is still writing its outputs).
__device__ __forceinline__ void spin_until(const std::int32_t* p, int target) {
  for (;;) {
    int v;
    asm volatile("ld.acquire.gpu.global.b32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
    if (v >= target) break;
    __nanosleep(20);
  }
}
// MODE 1 (TW): the chain in two warps (warp w holds window rows lo + 32w +
// lane), exchanging votes and the pivot row through shared memory at named
// barriers: half the per-lane update work on each of two SMSPs.
// MODE 0: one warp does both (GFQ_CHAIN_MODE=0; A/B).  (A split variant --
// warp 0 the panel part and the pivot choice, warp 1 replaying the
// coefficient updates from a shared-memory queue -- measured slower: the
// per-column cost is latency, not FMA issue.)
template <int MODE>
__global__ void __launch_bounds__(kChainThreads, 1)
ech_step_chain_kernel(std::uint32_t p, std::uint32_t magic, int rows, int c0, int wc, int n,
                      std::uint8_t* __restrict__ Z, std::int64_t ld, std::uint8_t* flags,
                      std::int32_t* info, int cap, std::int32_t* rho2, std::int32_t* lo_state,
                      std::uint8_t* NT, std::uint8_t* Gpiv, std::uint8_t* Y, const std::int32_t* base,
                      std::uint8_t* BpT, const std::uint8_t* __restrict__ invtab, std::int32_t* ctr,
                      int wait_prev, int seq, int tl) {
  // wait_prev > 0: ctr[0] / ctr[1] must reach wait_prev (they only grow:
  // the previous chain may still be running when this one starts)
  extern __shared__ __align__(16) std::uint8_t dsm[];
  __shared__ std::uint8_t invw[256];
  __shared__ int s_lo, s_rold;
  __shared__ __align__(16) float wrow[64];  // the column's pivot row (raw, then reduced)
  __shared__ int s_ok, s_r2;
  __shared__ int colq[kW];
  __shared__ std::uint8_t chatb[kW][kW];
  __shared__ int wpc[kW], wpr[kW], s_pr[kW];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  if (tl >= 0 && tid == 0) g_tl[tl][0] = gtime();
  if (wait_prev) {
    if (tid == 0) spin_until(ctr, wait_prev);
    __syncthreads();
  } else {
    pdl_wait();  // released after the chain (below): the update's CTAs
                 // should not sit on SMs other streams' K1 tiles could use
  }
  stamp(0);
  for (int a = tid; a < 256; a += kChainThreads) invw[a] = invtab[a];  // inverses mod p (cached)
  if (warp == 0) {
    int lo = __ldcg(lo_state);
    for (;;) {
      const int idx = lo + lane;
      const unsigned b = __ballot_sync(0xffffffffu, idx < rows && __ldcg(flags + idx) == 0);
      if (b || lo >= rows) {
        if (b) lo += __ffs(b) - 1;
        break;
      }
      lo += 32;
    }
    if (lo > rows) lo = rows;
    if (lane == 0) {
      s_lo = lo;
      s_rold = __ldcg(info);
      *lo_state = lo;
    }
  }
  __syncthreads();
  const int lo = s_lo, r_old = s_rold;
  if (tl >= 0 && tid == 0) g_tl[tl][1] = gtime();
  // warps 1.. stage the window rows' step columns [c0, c0 + n) in shared
  // memory while warp 0 runs the chain: the step's pivot rows are window
  // rows, so BpT is built from here (the region doubles as panel_full's
  // fallback storage, after which the tail reads Z instead)
  std::uint8_t* Ws = dsm;  // 64 x n
  constexpr int kChainW = MODE == 0 ? 1 : 2;  // warps running the chain
  if (warp >= kChainW) {
    if (wait_prev) {
      if (lane == 0) spin_until(ctr + 1, wait_prev);
      __syncwarp();
    }
    const int nv = n / 16;
    for (int e = tid - 32 * kChainW; e < 64 * nv; e += kChainThreads - 32 * kChainW) {
      const int r = e / nv, ch = e % nv;
      uint4 v = make_uint4(0, 0, 0, 0);
      if (lo + r < rows) v = __ldcg(reinterpret_cast<const uint4*>(Z + std::int64_t(lo + r) * ld + c0 + 16 * ch));
      reinterpret_cast<uint4*>(Ws + r * n)[ch] = v;
    }
  }
  // ---- the window chain, in warp 0 alone (no CTA barriers): lane l holds
  // window rows lo + l and lo + 32 + l, each as 32 panel elements (kept
  // SHIFTED so the current column is element 0: no dynamic register
  // indexing) and 32 coefficients (of the pivot rows' ORIGINAL values),
  // all fp32 integers.  Updates are LAZY: x += f.y with f and the
  // published pivot row y reduced (< p), so after <= 32 columns
  // x < p + 32 (p-1)^2 < 2^24 stays exact.  Per column: two ballots pick
  // the first open row with a nonzero; its lane stores the raw row to
  // shared memory, the warp reduces it (two elements a lane) and plants the
  // unit at coefficient r2; every lane applies x_i += f_i.(x_s + e_r2) with
  // f_i = v_i.sc (f_s = sc - 1 on the pivot row), sc = -1/v_s -- normalising
  // the pivot row and eliminating with it in one update.
  const float fp = float(p), invp = 1.0f / fp, roff = 0.5f * invp - 0.5f;
  // x mod p for 0 <= x < 2^24: (x + 0.5) / p lies 0.5/p away from an integer
  // boundary and the fp32 error of x.invp is below 0.25/p, so rounding
  // x.invp + (0.5/p - 0.5) to nearest (the 1.5 . 2^23 trick) gives floor(x/p)
  const auto red = [&](float v) {
    const float q = (fmaf(v, invp, roff) + 12582912.0f) - 12582912.0f;
    return fmaf(-fp, q, v);
  };
  if (MODE == 1 && warp < 2) {
    __shared__ unsigned s_ball[2][2];
    __shared__ int s_cnt[2];
    __shared__ std::uint32_t s_iv;
    const auto bar = [] { asm volatile("bar.sync 1, 64;" ::: "memory"); };
    float w[32], k[32];
    const int row = lo + 32 * warp + lane;
    bool open = row < rows && __ldcg(flags + row) == 0;
#pragma unroll
    for (int e = 0; e < 32; ++e) w[e] = k[e] = 0.0f;
    if (row < rows) {
      const std::uint8_t* src = Z + std::int64_t(row) * ld + c0;
      if (wc == kW) {
        const uint4 a = __ldcg(reinterpret_cast<const uint4*>(src)), b = __ldcg(reinterpret_cast<const uint4*>(src) + 1);
        const std::uint32_t ww[8] = {a.x, a.y, a.z, a.w, b.x, b.y, b.z, b.w};
#pragma unroll
        for (int e = 0; e < 32; ++e) w[e] = float((ww[e >> 2] >> (8 * (e & 3))) & 0xFFu);
      } else {
#pragma unroll
        for (int e = 0; e < 32; ++e)
          if (e < wc) w[e] = float(__ldcg(src + e));
      }
    }
    {
      const unsigned ob = __ballot_sync(0xffffffffu, open);
      if (lane == 0) s_cnt[warp] = __popc(ob);
    }
    bar();
    const bool covers_all = s_cnt[0] + s_cnt[1] == rows - r_old;
    stamp(1);
    int r2 = 0, ok = 1, q = -1, mpc = 0, mpr = 0;
    float v = red(w[0]);
    std::uint32_t iv = invw[int(v)];
    unsigned b = __ballot_sync(0xffffffffu, open && v != 0.0f);
#pragma unroll 1
    for (int c = 0; c < wc; ++c) {
      if (lane == 0) s_ball[c & 1][warp] = b;
      bar();
      const unsigned ball0 = s_ball[c & 1][0], ball1 = s_ball[c & 1][1];
      if (!(ball0 | ball1)) {
        if (!covers_all) {
          ok = 0;
          break;
        }
#pragma unroll
        for (int e = 0; e < 31; ++e) w[e] = w[e + 1];
        w[31] = 0.0f;
        v = red(w[0]);
        iv = invw[int(v)];
        b = __ballot_sync(0xffffffffu, open && v != 0.0f);
        continue;  // a free column
      }
      const int pw = ball0 ? 0 : 1;
      const unsigned bb = pw ? ball1 : ball0;
      const int pl = __ffs(bb) - 1;
      const bool mine = warp == pw && lane == pl;
      if (mine) {
        float4* dst = reinterpret_cast<float4*>(wrow);
#pragma unroll
        for (int e = 0; e < 8; ++e) {
          dst[e] = make_float4(w[4 * e], w[4 * e + 1], w[4 * e + 2], w[4 * e + 3]);
          dst[8 + e] = make_float4(k[4 * e], k[4 * e + 1], k[4 * e + 2], k[4 * e + 3]);
        }
        s_iv = iv;
      }
      bar();
      // reduce the published row, one element a thread; plant e_r2 (that
      // coefficient is still 0 in every row)
      {
        const int t = 32 * warp + lane;
        wrow[t] = t == 32 + r2 ? 1.0f : red(wrow[t]);
      }
      bar();
      const float sc = float(p - s_iv);
      float y[64];
      {
        const float4* src = reinterpret_cast<const float4*>(wrow);
#pragma unroll
        for (int e = 0; e < 16; ++e) {
          const float4 t = src[e];
          y[4 * e] = t.x; y[4 * e + 1] = t.y; y[4 * e + 2] = t.z; y[4 * e + 3] = t.w;
        }
      }
      const float f = mine ? sc - 1.0f : red(v * sc);
      if (mine) {
        open = false;
        q = r2;
      }
      if (warp == 0 && lane == r2) {
        mpc = c;
        mpr = lo + 32 * pw + pl;
      }
      ++r2;
      const float h = fmaf(f, y[1], w[1]);
      v = red(h);
      iv = invw[int(v)];
#pragma unroll
      for (int e = 1; e < 31; ++e) w[e] = fmaf(f, y[e + 1], w[e + 1]);
      w[0] = h;
      w[31] = 0.0f;
#pragma unroll
      for (int e = 0; e < 32; ++e) k[e] = fmaf(f, y[32 + e], k[e]);
      b = __ballot_sync(0xffffffffu, open && v != 0.0f);
    }
    if (warp == 0 && lane < r2) {
      wpc[lane] = mpc;
      wpr[lane] = mpr;
    }
    if (ok && q >= 0) {
#pragma unroll
      for (int e = 0; e < 32; ++e) chatb[q][e] = std::uint8_t(int(red(k[e])));
    }
    if (warp == 0 && lane == 0) {
      s_ok = ok;
      s_r2 = r2;
    }
  }
  if (MODE == 0 && warp == 0) {
    float w0[32], w1[32], k0[32], k1[32];
    const int i0 = lo + lane, i1 = lo + 32 + lane;
    bool open0 = i0 < rows && __ldcg(flags + i0) == 0, open1 = i1 < rows && __ldcg(flags + i1) == 0;
#pragma unroll
    for (int e = 0; e < 32; ++e) w0[e] = w1[e] = k0[e] = k1[e] = 0.0f;
    const auto load = [&](int gi, float (&w)[32]) {
      if (gi >= rows) return;
      const std::uint8_t* src = Z + std::int64_t(gi) * ld + c0;
      if (wc == kW) {
        const uint4 a = __ldcg(reinterpret_cast<const uint4*>(src)), b = __ldcg(reinterpret_cast<const uint4*>(src) + 1);
        const std::uint32_t ww[8] = {a.x, a.y, a.z, a.w, b.x, b.y, b.z, b.w};
#pragma unroll
        for (int e = 0; e < 32; ++e) w[e] = float((ww[e >> 2] >> (8 * (e & 3))) & 0xFFu);
      } else {
#pragma unroll
        for (int e = 0; e < 32; ++e)
          if (e < wc) w[e] = float(__ldcg(src + e));
      }
    };
    load(i0, w0);
    load(i1, w1);
    const int open_in = __popc(__ballot_sync(0xffffffffu, open0)) + __popc(__ballot_sync(0xffffffffu, open1));
    const bool covers_all = open_in == rows - r_old;
    stamp(1);
    int r2 = 0, ok = 1, q0 = -1, q1 = -1, mpc = 0, mpr = 0;
    const unsigned lanebit = 1u << lane;
    // Rotated loop: the next column's head (its elements after this
    // column's update, their residues, inverse lookups and the two votes)
    // is computed right after f0 / f1 are known and BEFORE the bulk of the
    // update, so the bulk's independent FMAs fill the latency of the head's
    // shared-memory lookups and votes instead of sitting in front of them
    // (in-order issue in one warp).
    float v0 = red(w0[0]), v1 = red(w1[0]);
    std::uint32_t iv0 = invw[int(v0)], iv1 = invw[int(v1)];
    unsigned b0 = __ballot_sync(0xffffffffu, open0 && v0 != 0.0f);
    unsigned b1 = __ballot_sync(0xffffffffu, open1 && v1 != 0.0f);
#pragma unroll 1
    for (int c = 0; c < wc; ++c) {
      // the shifted panel moves on whether or not the column has a pivot
      if (!(b0 | b1)) {
        if (!covers_all) {
          ok = 0;
          break;
        }
#pragma unroll
        for (int e = 0; e < 31; ++e) {
          w0[e] = w0[e + 1];
          w1[e] = w1[e + 1];
        }
        w0[31] = w1[31] = 0.0f;
        v0 = red(w0[0]);
        v1 = red(w1[0]);
        iv0 = invw[int(v0)];
        iv1 = invw[int(v1)];
        b0 = __ballot_sync(0xffffffffu, open0 && v0 != 0.0f);
        b1 = __ballot_sync(0xffffffffu, open1 && v1 != 0.0f);
        continue;  // a free column
      }
      const bool hi = b0 == 0;
      const unsigned bb = hi ? b1 : b0;
      const bool mine = (bb & (0u - bb) & lanebit) != 0;
      // the pivot lane publishes its raw row: 32 panel + 32 coefficient values
      // (two predicated store runs, no per-element selects)
      float4* dst = reinterpret_cast<float4*>(wrow);
      if (mine && !hi) {
#pragma unroll
        for (int e = 0; e < 8; ++e) {
          dst[e] = make_float4(w0[4 * e], w0[4 * e + 1], w0[4 * e + 2], w0[4 * e + 3]);
          dst[8 + e] = make_float4(k0[4 * e], k0[4 * e + 1], k0[4 * e + 2], k0[4 * e + 3]);
        }
      }
      if (mine && hi) {
#pragma unroll
        for (int e = 0; e < 8; ++e) {
          dst[e] = make_float4(w1[4 * e], w1[4 * e + 1], w1[4 * e + 2], w1[4 * e + 3]);
          dst[8 + e] = make_float4(k1[4 * e], k1[4 * e + 1], k1[4 * e + 2], k1[4 * e + 3]);
        }
      }
      const std::uint32_t ivp = __shfl_sync(0xffffffffu, hi ? iv1 : iv0, __ffs(bb) - 1);
      __syncwarp();
      // reduce the published row, two elements a lane; plant e_r2 (that
      // coefficient is still 0 in every row)
      wrow[lane] = red(wrow[lane]);
      wrow[32 + lane] = lane == r2 ? 1.0f : red(wrow[32 + lane]);
      __syncwarp();
      const float sc = float(p - ivp);
      float y[64];
      {
        const float4* src = reinterpret_cast<const float4*>(wrow);
#pragma unroll
        for (int e = 0; e < 16; ++e) {
          const float4 t = src[e];
          y[4 * e] = t.x; y[4 * e + 1] = t.y; y[4 * e + 2] = t.z; y[4 * e + 3] = t.w;
        }
      }
      const bool me0 = !hi && mine, me1 = hi && mine;
      const float f0 = me0 ? sc - 1.0f : red(v0 * sc);
      const float f1 = me1 ? sc - 1.0f : red(v1 * sc);
      if (me0) {
        open0 = false;
        q0 = r2;
      }
      if (me1) {
        open1 = false;
        q1 = r2;
      }
      if ((lanebit >> r2) & 1u) {
        mpc = c;
        mpr = lo + (hi ? 32 : 0) + (__ffs(bb) - 1);
      }
      ++r2;
      // the next column's head first
      const float h0 = fmaf(f0, y[1], w0[1]), h1 = fmaf(f1, y[1], w1[1]);
      v0 = red(h0);
      v1 = red(h1);
      iv0 = invw[int(v0)];
      iv1 = invw[int(v1)];
      // then the bulk: shift the panel part while updating; coefficients in place
#pragma unroll
      for (int e = 1; e < 31; ++e) {
        w0[e] = fmaf(f0, y[e + 1], w0[e + 1]);
        w1[e] = fmaf(f1, y[e + 1], w1[e + 1]);
      }
      w0[0] = h0;
      w1[0] = h1;
      w0[31] = w1[31] = 0.0f;
#pragma unroll
      for (int e = 0; e < 32; ++e) {
        k0[e] = fmaf(f0, y[32 + e], k0[e]);
        k1[e] = fmaf(f1, y[32 + e], k1[e]);
      }
      b0 = __ballot_sync(0xffffffffu, open0 && v0 != 0.0f);
      b1 = __ballot_sync(0xffffffffu, open1 && v1 != 0.0f);
      __syncwarp();  // wrow is rewritten by the next column's pivot lane
    }
    if (lane < r2) {
      wpc[lane] = mpc;
      wpr[lane] = mpr;
    }
    if (ok) {
      if (q0 >= 0) {
#pragma unroll
        for (int e = 0; e < 32; ++e) chatb[q0][e] = std::uint8_t(int(red(k0[e])));
      }
      if (q1 >= 0) {
#pragma unroll
        for (int e = 0; e < 32; ++e) chatb[q1][e] = std::uint8_t(int(red(k1[e])));
      }
    }
    if (lane == 0) {
      s_ok = ok;
      s_r2 = r2;
    }
  }
  __syncthreads();
  stamp(2);
  if (tl >= 0 && tid == 0) g_tl[tl][2] = gtime();
  pdl_release();
  const int ok = s_ok, r2 = s_r2;
  if (!ok) {
    panel_full(p, magic, rows, c0, wc, Z, ld, flags, info, cap, nullptr, 0, rho2,
               StepOut{NT, Gpiv});
  } else {
    if (tid < kW) colq[tid] = -1;
    __syncthreads();
    if (tid < r2) colq[wpc[tid]] = tid;
    __syncthreads();
    // NT[t][wpc[q]] = (I + Ĉ)[q][t]; Gpiv[q] = ĉ_q
    for (int e = tid; e < kW * kW; e += kChainThreads) {
      const int t = e / kW, c = e % kW;
      const int q = colq[c];
      std::uint32_t v = 0;
      if (q >= 0) {
        v = chatb[q][t];
        if (t == q) v = v + 1 == p ? 0 : v + 1;
      }
      NT[e] = std::uint8_t(v);
      const int qq = e / kW;
      Gpiv[e] = qq < r2 ? chatb[qq][e % kW] : 0;
    }
    if (tid < kW) rho2[tid] = tid < r2 ? wpr[tid] : -1;
    if (tid < r2) {
      info[1 + r_old + tid] = c0 + wpc[tid];
      info[1 + cap + r_old + tid] = wpr[tid];
      flags[wpr[tid]] = 1;
    }
    if (tid == 0) info[0] = r_old + r2;
  }
  __syncthreads();
  stamp(3);
  if (tid < kW) {
    const int r = rho2[tid];
    s_pr[tid] = r;
    if (r >= 0) Y[std::int64_t(r) * ld + (r_old + tid - *base)] = 1;
  }
  __syncthreads();
  // the pivot rows (32 x n) in shared memory -- from the window staging
  // (plus the Y unit just planted) or, after a fallback, from Z -- then
  // written transposed
  std::uint8_t* Bs = dsm + 64 * n;  // 32 x n, after the staged window
  const int y_col = int(Y - Z) - c0;  // Y's first column relative to c0
  for (int e = tid; e < kW * (n / 16); e += kChainThreads) {
    const int q = e / (n / 16), ch = e % (n / 16);
    const int r = s_pr[q];
    uint4 v = make_uint4(0, 0, 0, 0);
    if (r >= 0)
      v = ok ? reinterpret_cast<const uint4*>(Ws + (r - lo) * n)[ch]
             : __ldcg(reinterpret_cast<const uint4*>(Z + std::int64_t(r) * ld + c0 + 16 * ch));
    reinterpret_cast<uint4*>(Bs + q * n)[ch] = v;
  }
  __syncthreads();
  if (ok && tid < kW && s_pr[tid] >= 0) Bs[tid * n + y_col + (r_old + tid - *base)] = 1;
  __syncthreads();
  for (int j = tid; j < n; j += kChainThreads) {
    std::uint32_t o[8] = {0, 0, 0, 0, 0, 0, 0, 0};
#pragma unroll
    for (int q = 0; q < kW; ++q) o[q >> 2] |= std::uint32_t(Bs[q * n + j]) << (8 * (q & 3));
    uint4* dst = reinterpret_cast<uint4*>(BpT + std::int64_t(j) * kW);
    dst[0] = make_uint4(o[0], o[1], o[2], o[3]);
    dst[1] = make_uint4(o[4], o[5], o[6], o[7]);
  }
  __syncthreads();
  stamp(4);
  if (tid == 0) {
    // the update of this step may start (its CTAs wait for ctr[2] >= seq
    // instead of the grid boundary)
    __threadfence();
    asm volatile("st.release.gpu.global.b32 [%0], %1;" ::"l"(ctr + 2), "r"(seq) : "memory");
    if (tl >= 0) g_tl[tl][3] = gtime();
  }
}

// Two-level ECH, step part 2: Z[i][c0 + j] += G[i] . Bp[:, j] for every row
// i and j < n (n a multiple of 16), with G[i] = seg_i . NT^T (mod p) or the
// pivot row's Gpiv.  One CTA per 32 rows: warp 0 forms the 32 rows' G
// (lane = row, 8 x 32 dp4a against NT) into shared memory while the CTA
// stages BpT; then the 8 warps split the 16-column chunks, lane = row:
// 16 x 8 dp4a per chunk against BpT rows broadcast from shared memory, the
// Barrett reduction with the old values, one 16-byte load and store per lane.
// A row's columns must stay in ONE CTA: G is formed from the row's panel
// segment, which the same update overwrites in place (splitting the columns
// over CTAs races -- measured 3% faster and wrong on cfg3).
__global__ void __launch_bounds__(kStepThreads)
ech_step_update_kernel(std::uint32_t p, std::uint32_t magic, int rows, int c0, int n,
                       std::uint8_t* Z, std::int64_t ld, const std::uint8_t* NT, const std::uint8_t* Gpiv,
                       const std::int32_t* rho2, const std::uint8_t* BpT, std::int32_t* ctr, int signal,
                       int seq, int tl) {
  __shared__ __align__(16) std::uint32_t sB[kStepMaxN * 8];
  __shared__ __align__(16) std::uint32_t sNT[kW * 8];
  __shared__ std::uint32_t sG[kStepRows][9];
  // The chain's outputs are published by its ready flag (ctr[2] = seq), so
  // the CTAs wait for that rather than for the chain grid to retire; all
  // reads of data another grid writes go to L2 (__ldcg: an SM's L1 may
  // still hold the previous step's lines).
  pdl_release();
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  if (tid == 0) spin_until(ctr + 2, seq);
  __syncthreads();
  const int i0 = blockIdx.x * kStepRows;
  for (int e = tid; e < n * 2; e += kStepThreads)
    reinterpret_cast<uint4*>(sB)[e] = __ldcg(reinterpret_cast<const uint4*>(BpT) + e);
  if (tid < kW * 2) reinterpret_cast<uint4*>(sNT)[tid] = __ldcg(reinterpret_cast<const uint4*>(NT) + tid);
  __syncthreads();
  {
    // warp w forms G[i][4w .. 4w+3] of the CTA's 32 rows (lane = row)
    const int i = i0 + lane;
    const int r = __ldcg(rho2 + lane);
    int myq = -1;
#pragma unroll
    for (int u = 0; u < kW; ++u)
      if (__shfl_sync(0xffffffffu, r, u) == i) myq = u;
    std::uint32_t gw = 0;
    if (i < rows && myq >= 0) {
      gw = __ldcg(reinterpret_cast<const std::uint32_t*>(Gpiv + myq * kW) + warp);
    } else if (i < rows) {
      const uint4* src = reinterpret_cast<const uint4*>(Z + std::int64_t(i) * ld + c0);
      const uint4 a = __ldcg(src), b = __ldcg(src + 1);
#pragma unroll
      for (int tt = 0; tt < 4; ++tt) {
        const uint4* nt4 = reinterpret_cast<const uint4*>(sNT + (4 * warp + tt) * 8);
        const uint4 x = nt4[0], y = nt4[1];
        std::uint32_t acc = 0;
        acc = __dp4a(a.x, x.x, acc); acc = __dp4a(a.y, x.y, acc);
        acc = __dp4a(a.z, x.z, acc); acc = __dp4a(a.w, x.w, acc);
        acc = __dp4a(b.x, y.x, acc); acc = __dp4a(b.y, y.y, acc);
        acc = __dp4a(b.z, y.z, acc); acc = __dp4a(b.w, y.w, acc);
        gw |= modp(acc, p, magic) << (8 * tt);
      }
    }
    sG[lane][warp] = gw;
  }
  __syncthreads();
  const int i = i0 + lane;
  const bool live = i < rows;
  std::uint32_t g[8];
#pragma unroll
  for (int w = 0; w < 8; ++w) g[w] = sG[lane][w];
  std::uint8_t* zrow = Z + std::int64_t(i) * ld + c0;
  const auto chunk = [&](int ch) {
    std::uint32_t out[4];
    const uint4 old = __ldcg(reinterpret_cast<const uint4*>(zrow + 16 * ch));
    const std::uint32_t ow[4] = {old.x, old.y, old.z, old.w};
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      std::uint32_t word = 0;
#pragma unroll
      for (int by = 0; by < 4; ++by) {
        const uint4* b4 = reinterpret_cast<const uint4*>(sB + (16 * ch + 4 * q + by) * 8);
        const uint4 x = b4[0], y = b4[1];
        std::uint32_t acc = (ow[q] >> (8 * by)) & 0xFFu;
        acc = __dp4a(g[0], x.x, acc); acc = __dp4a(g[1], x.y, acc);
        acc = __dp4a(g[2], x.z, acc); acc = __dp4a(g[3], x.w, acc);
        acc = __dp4a(g[4], y.x, acc); acc = __dp4a(g[5], y.y, acc);
        acc = __dp4a(g[6], y.z, acc); acc = __dp4a(g[7], y.w, acc);
        word |= modp(acc, p, magic) << (8 * by);
      }
      out[q] = word;
    }
    *reinterpret_cast<uint4*>(zrow + 16 * ch) = make_uint4(out[0], out[1], out[2], out[3]);
  };
  constexpr int kWarps = kStepThreads / 32;
  // the first chunk a warp: columns [c0, c0 + 128), the next step's panel
  // among them (the overlapped chain waits for these, see spin_until)
  if (tl >= 0 && tid == 0 && blockIdx.x == 0) g_tl[tl][4] = gtime();
  if (live && warp < n / 16) chunk(warp);
  if (signal) {
    __threadfence();
    __syncthreads();
    if (tid == 0) atomicAdd(ctr, 1);
  }
  if (tl >= 0 && tid == 0 && blockIdx.x == 0) g_tl[tl][5] = gtime();
  if (live)
    for (int ch = warp + kWarps; ch < n / 16; ch += kWarps) chunk(ch);
  if (signal) {
    __threadfence();
    __syncthreads();
    if (tid == 0) atomicAdd(ctr + 1, 1);
  }
  if (tl >= 0 && tid == 0) {
    if (blockIdx.x == 0) g_tl[tl][6] = gtime();
    atomicMax(&g_tl[tl][7], gtime());
  }
}

// GF(2): the 32 panel columns of a row are one 32-bit word, a row
// operation is one XOR, the pivot block inversion is a 32 x 32 bit-matrix
// Gauss-Jordan in one warp's registers and G = Ap.N2 is a masked XOR of
// N2's row words.  Same outputs as ech_panel_kernel for p = 2.
__global__ void __launch_bounds__(1024)
ech_panel_gf2_kernel(int rows, int c0, int wc, const std::uint8_t* __restrict__ Aug, std::int64_t ld,
                     std::uint8_t* flags, std::int32_t* info, int cap, std::uint8_t* G,
                     std::int64_t ldg, std::int32_t* rho2) {
  pdl_wait_and_release();
  extern __shared__ __align__(16) std::uint8_t sm[];
  std::uint32_t* bits = reinterpret_cast<std::uint32_t*>(sm);  // rows words
  std::uint8_t* fl = sm + 4 * rows;                             // rows flags
  __shared__ unsigned sel_s[2];
  __shared__ int pc[kW], pr[kW];
  __shared__ std::uint32_t n2[kW];  // N2 rows as bit words (column t = bit t)
  __shared__ int r_old;
  const int tid = threadIdx.x, nt = blockDim.x, lane = tid & 31;

  for (int i = tid; i < rows; i += nt) {
    const std::uint8_t f = __ldcg(flags + i);
    fl[i] = f;
    std::uint32_t word = 0;
    if (!f) {
      uint4 a, b;
      load_seg(Aug + std::int64_t(i) * ld + c0, wc, a, b);
      const std::uint32_t wds[8] = {a.x, a.y, a.z, a.w, b.x, b.y, b.z, b.w};
#pragma unroll
      for (int q = 0; q < 8; ++q) {
        const std::uint32_t v = wds[q] & 0x01010101u;  // one bit per byte
        word |= ((v & 1u) | ((v >> 7) & 2u) | ((v >> 14) & 4u) | ((v >> 21) & 8u)) << (4 * q);
      }
    }
    bits[i] = word;
  }
  if (tid == 0) {
    r_old = info[0];
    sel_s[0] = 0xFFFFFFFFu;
  }
  __syncthreads();

  int r2 = 0;
  for (int c = 0; c < wc; ++c) {
    unsigned cand = 0xFFFFFFFFu;
    for (int i = tid; i < rows; i += nt)
      if (!fl[i] && ((bits[i] >> c) & 1u) && unsigned(i) < cand) cand = unsigned(i);
    cand = __reduce_min_sync(0xffffffffu, cand);
    if (lane == 0 && cand != 0xFFFFFFFFu) atomicMin(&sel_s[c & 1], cand);
    __syncthreads();
    const unsigned s = sel_s[c & 1];
    if (tid == 0) sel_s[(c + 1) & 1] = 0xFFFFFFFFu;
    if (s != 0xFFFFFFFFu) {
      const std::uint32_t ps = bits[s];
      for (int i = tid; i < rows; i += nt)
        if (i != int(s) && !fl[i] && ((bits[i] >> c) & 1u)) bits[i] ^= ps;
      if (tid == 0) {
        fl[s] = 1;
        pc[r2] = c;
        pr[r2] = int(s);
      }
      ++r2;
    }
    __syncthreads();
  }

  // N2 = inv(X) (= -inv over GF(2)), X[q][t] = Aug[pr[q]][c0 + pc[t]]
  if (tid < 32) {
    std::uint32_t x = 0, inv = 0;  // row `lane` of [X | I] as two bit words
    if (lane < r2) {
      const std::uint8_t* src = Aug + std::int64_t(pr[lane]) * ld + c0;
      for (int t = 0; t < r2; ++t) x |= std::uint32_t(src[pc[t]] & 1u) << t;
      inv = 1u << lane;
    }
    for (int q = 0; q < r2; ++q) {
      const unsigned bal = __ballot_sync(0xffffffffu, lane >= q && lane < r2 && ((x >> q) & 1u));
      const int pv = __ffs(bal) - 1;
      // swap rows q and pv
      const std::uint32_t xq = __shfl_sync(0xffffffffu, x, q), iq = __shfl_sync(0xffffffffu, inv, q);
      const std::uint32_t xp = __shfl_sync(0xffffffffu, x, pv), ip = __shfl_sync(0xffffffffu, inv, pv);
      if (lane == q) {
        x = xp;
        inv = ip;
      } else if (lane == pv) {
        x = xq;
        inv = iq;
      }
      const std::uint32_t px = __shfl_sync(0xffffffffu, x, q), pi = __shfl_sync(0xffffffffu, inv, q);
      if (lane != q && ((x >> q) & 1u)) {
        x ^= px;
        inv ^= pi;
      }
    }
    n2[lane] = lane < r2 ? inv : 0u;
    if (lane < kW) rho2[lane] = lane < r2 ? pr[lane] : -1;
    if (lane < r2) {
      info[1 + r_old + lane] = c0 + pc[lane];
      info[1 + cap + r_old + lane] = pr[lane];
      flags[pr[lane]] = 1;
    }
    if (lane == 0) info[0] = r_old + r2;
  }
  __syncthreads();

  // G[i] = (Aug[i, c0 + gamma2] + e_{pivot of i}) . N2 over GF(2)
  for (int i = tid; i < rows; i += nt) {
    uint4 a, b;
    load_seg(Aug + std::int64_t(i) * ld + c0, wc, a, b);
    const std::uint32_t seg[8] = {a.x, a.y, a.z, a.w, b.x, b.y, b.z, b.w};
    std::uint32_t g = 0;
    for (int q = 0; q < r2; ++q) {
      const int cq = pc[q];
      std::uint32_t v = (seg[cq >> 2] >> (8 * (cq & 3))) & 1u;
      if (pr[q] == i) v ^= 1u;
      if (v) g ^= n2[q];
    }
    std::uint32_t outw[8];
#pragma unroll
    for (int q = 0; q < 8; ++q) {
      const std::uint32_t nib = (g >> (4 * q)) & 0xFu;
      outw[q] = (nib & 1u) | ((nib & 2u) << 7) | ((nib & 4u) << 14) | ((nib & 8u) << 21);
    }
    uint4* dst = reinterpret_cast<uint4*>(G + std::int64_t(i) * ldg);
    dst[0] = make_uint4(outw[0], outw[1], outw[2], outw[3]);
    dst[1] = make_uint4(outw[4], outw[5], outw[6], outw[7]);
  }
}

// GF(2), rows <= 1024: the pivot chain of the panel runs in ONE warp with
// no block barriers.  Lane l owns rows 32r + l (r < 32) as 32-bit panel
// words in registers; per column: a ballot-style mask of candidate rows,
// a warp min-reduction (first non-pivotal row with the bit set), the pivot
// word broadcast by shuffle and a masked XOR of the lane's rows.  The rest
// of the CTA then writes G in parallel.
__global__ void __launch_bounds__(1024)
ech_panel_gf2w_kernel(int rows, int c0, int wc, const std::uint8_t* __restrict__ Aug,
                      std::int64_t ld, std::uint8_t* flags, std::int32_t* info, int cap,
                      std::uint8_t* G, std::int64_t ldg, std::int32_t* rho2) {
  pdl_wait_and_release();
  __shared__ std::uint32_t orig[1024];
  __shared__ int pc[kW], pr[kW];
  __shared__ std::uint32_t n2[kW];
  __shared__ int r2_s;
  const int tid = threadIdx.x, nt = blockDim.x, lane = tid & 31;

  for (int i = tid; i < 1024; i += nt) {
    std::uint32_t word = 0;
    if (i < rows) {  // every row: G needs the panel bits of old pivot rows too
      uint4 a, b;
      load_seg(Aug + std::int64_t(i) * ld + c0, wc, a, b);
      const std::uint32_t wds[8] = {a.x, a.y, a.z, a.w, b.x, b.y, b.z, b.w};
#pragma unroll
      for (int q = 0; q < 8; ++q) {
        const std::uint32_t v = wds[q] & 0x01010101u;
        word |= ((v & 1u) | ((v >> 7) & 2u) | ((v >> 14) & 4u) | ((v >> 21) & 8u)) << (4 * q);
      }
    }
    orig[i] = word;
  }
  __syncthreads();

  if (tid < 32) {
    std::uint32_t row[32];
    std::uint32_t fm = 0;  // bit r: row 32r + lane is pivotal (or absent)
#pragma unroll
    for (int r = 0; r < 32; ++r) {
      const int i = 32 * r + lane;
      row[r] = orig[i];
      if (i >= rows || flags[i]) fm |= 1u << r;
    }
    int r2 = 0;
    for (int c = 0; c < wc; ++c) {
      std::uint32_t cm = 0;
#pragma unroll
      for (int r = 0; r < 32; ++r) cm |= ((row[r] >> c) & 1u) << r;
      cm &= ~fm;
      unsigned cand = cm ? unsigned(32 * (__ffs(cm) - 1) + lane) : 0xFFFFFFFFu;
      cand = __reduce_min_sync(0xffffffffu, cand);
      if (cand == 0xFFFFFFFFu) continue;
      const int sl = int(cand & 31), sr = int(cand >> 5);
      std::uint32_t mine = 0;
#pragma unroll
      for (int r = 0; r < 32; ++r) mine = (r == sr) ? row[r] : mine;
      const std::uint32_t ps = __shfl_sync(0xffffffffu, mine, sl);
      if (lane == sl) {
        cm &= ~(1u << sr);
        fm |= 1u << sr;
      }
#pragma unroll
      for (int r = 0; r < 32; ++r) row[r] ^= ps & (0u - ((cm >> r) & 1u));
      if (lane == 0) {
        pc[r2] = c;
        pr[r2] = int(cand);
      }
      ++r2;
    }
    __syncwarp();
    // N2 = inv(X), X[q][t] = bit pc[t] of the original word of row pr[q]
    std::uint32_t x = 0, inv = 0;
    if (lane < r2) {
      const std::uint32_t ow = orig[pr[lane]];
      for (int t = 0; t < r2; ++t) x |= ((ow >> pc[t]) & 1u) << t;
      inv = 1u << lane;
    }
    for (int q = 0; q < r2; ++q) {
      const unsigned bal = __ballot_sync(0xffffffffu, lane >= q && lane < r2 && ((x >> q) & 1u));
      const int pv = __ffs(bal) - 1;
      const std::uint32_t xq = __shfl_sync(0xffffffffu, x, q), iq = __shfl_sync(0xffffffffu, inv, q);
      const std::uint32_t xp = __shfl_sync(0xffffffffu, x, pv), ip = __shfl_sync(0xffffffffu, inv, pv);
      if (lane == q) {
        x = xp;
        inv = ip;
      } else if (lane == pv) {
        x = xq;
        inv = iq;
      }
      const std::uint32_t px = __shfl_sync(0xffffffffu, x, q), pi = __shfl_sync(0xffffffffu, inv, q);
      if (lane != q && ((x >> q) & 1u)) {
        x ^= px;
        inv ^= pi;
      }
    }
    n2[lane] = lane < r2 ? inv : 0u;
    rho2[lane] = lane < r2 ? pr[lane] : -1;
    const int r_old = info[0];
    if (lane < r2) {
      info[1 + r_old + lane] = c0 + pc[lane];
      info[1 + cap + r_old + lane] = pr[lane];
      flags[pr[lane]] = 1;
    }
    __syncwarp();
    if (lane == 0) {
      info[0] = r_old + r2;
      r2_s = r2;
    }
  }
  __syncthreads();
  // G[i] = (orig bits of row i at gamma2, + e on its own pivot) . N2
  const int r2 = r2_s;
  for (int i = tid; i < rows; i += nt) {
    const std::uint32_t ow = orig[i];
    std::uint32_t g = 0;
    for (int q = 0; q < r2; ++q)
      if (((ow >> pc[q]) & 1u) ^ (pr[q] == i ? 1u : 0u)) g ^= n2[q];
    std::uint32_t outw[8];
#pragma unroll
    for (int q = 0; q < 8; ++q) {
      const std::uint32_t nib = (g >> (4 * q)) & 0xFu;
      outw[q] = (nib & 1u) | ((nib & 2u) << 7) | ((nib & 4u) << 14) | ((nib & 8u) << 21);
    }
    uint4* dst = reinterpret_cast<uint4*>(G + std::int64_t(i) * ldg);
    dst[0] = make_uint4(outw[0], outw[1], outw[2], outw[3]);
    dst[1] = make_uint4(outw[4], outw[5], outw[6], outw[7]);
  }
}

// Blocked ECH bookkeeping (see ech_panel_plant / ech_outer_finish below).
__global__ void ech_plant_kernel(std::uint8_t* Y, std::int64_t ldy, const std::int32_t* rho2,
                                 const std::int32_t* info, const std::int32_t* base) {
  pdl_wait_and_release();
  const int lane = threadIdx.x;
  const int r = rho2[lane];
  const unsigned valid = __ballot_sync(0xffffffffu, r >= 0);
  if (r >= 0) {
    const int slot = info[0] - __popc(valid) + lane - *base;
    Y[std::int64_t(r) * ldy + slot] = 1;
  }
}

__global__ void ech_outer_finish_kernel(std::uint32_t p, std::uint8_t* Y, std::int64_t ldy, int kcols,
                                        std::int32_t* info, int cap, std::int32_t* base,
                                        std::int32_t* rmap, int col0) {
  pdl_wait_and_release();
  const int r_now = info[0], b0 = *base;
  for (int t = threadIdx.x; t < kcols; t += blockDim.x) {
    const int g = b0 + t;
    int row = -1;
    if (g < r_now) {
      info[1 + g] += col0;  // the steps recorded scratch-local pivot columns
      row = info[1 + cap + g];
      std::uint8_t* y = Y + std::int64_t(row) * ldy + t;
      *y = std::uint8_t((*y + p - 1) % p);
    }
    rmap[t] = row;
  }
  __syncthreads();
  if (threadIdx.x == 0) *base = r_now;
}

__global__ void scatter_rows_kernel(std::uint8_t* dst, std::int64_t ldd, std::int64_t rows,
                                    std::int64_t cols, const std::uint8_t* src,
                                    std::int64_t lds, const std::int32_t* rmap) {
  for (std::int64_t i = blockIdx.y; i < rows; i += gridDim.y) {
    const std::int32_t t = rmap[i];
    if (t < 0) continue;
    for (std::int64_t j = blockIdx.x * blockDim.x + threadIdx.x; j < cols;
         j += std::int64_t(gridDim.x) * blockDim.x)
      dst[std::int64_t(t) * ldd + j] = src[i * lds + j];
  }
}

}  // namespace

void ech_panel(std::uint32_t p, std::int64_t rows, std::int64_t c0, std::int64_t wc,
               std::int64_t w, const std::uint8_t* Aug, std::int64_t ld, std::uint8_t* flags,
               std::int32_t* info, std::int64_t cap, std::uint8_t* G, std::int64_t ldg,
               std::int32_t* rho2, cudaStream_t s) {
  if (w != kW || wc > w) throw std::invalid_argument("ech_panel: panel width must be 32");
  if ((ldg & 15) || (reinterpret_cast<std::uintptr_t>(G) & 15))
    throw std::invalid_argument("ech_panel: G must be 16-byte aligned");
  static bool attr = false;
  if (!attr) {
    GFQ_CUDA(cudaFuncSetAttribute(ech_panel_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                  kPanelSmem));
    GFQ_CUDA(cudaFuncSetAttribute(ech_panel_gf2_kernel,
                                  cudaFuncAttributeMaxDynamicSharedMemorySize, kPanelSmem));
    attr = true;
  }
  // Threads per panel CTA: each thread owns rows/threads rows; fewer warps
  // make the per-column barriers cheaper (GFQ_PANEL_THREADS overrides).
  static const int max_threads = [] {
    const char* e = std::getenv("GFQ_PANEL_THREADS");
    const int v = e ? std::atoi(e) : 0;
    return v >= 64 && v <= 1024 ? v : 1024;
  }();
  const std::int64_t r32 = (rows + 31) / 32 * 32;
  const int threads = r32 >= max_threads ? max_threads : int(r32 < 64 ? 64 : r32);
  // algorithmic bytes: the rows x 32 panel read, G (rows x 32) written
  ProfScope ps(kProfEchPanel, 2.0 * double(rows) * double(kW), s);
  if (p == 2 && rows <= 1024) {
    GFQ_CUDA(launch_pdl(ech_panel_gf2w_kernel, dim3(1), dim3(1024), 0, s, int(rows), int(c0), int(wc), Aug, ld, flags, info,
                                             int(cap), G, ldg, rho2));
    GFQ_CUDA(cudaGetLastError());
    count_launch();
    return;
  }
  if (p == 2) {
    const std::size_t smem2 = std::size_t(rows) * 5;
    if (smem2 > std::size_t(kPanelSmem)) throw std::invalid_argument("ech_panel: block too tall");
    GFQ_CUDA(launch_pdl(ech_panel_gf2_kernel, dim3(1), dim3(threads), smem2, s, int(rows), int(c0), int(wc), Aug, ld, flags,
                                                   info, int(cap), G, ldg, rho2));
    GFQ_CUDA(cudaGetLastError());
    count_launch();
    return;
  }
  const std::size_t smem = std::size_t(rows) * (kW + 1);
  if (smem > std::size_t(kPanelSmem)) throw std::invalid_argument("ech_panel: block too tall");
  const std::uint32_t magic = static_cast<std::uint32_t>((0x100000000ULL / p) + 1);
  static bool attr_w = false;
  if (!attr_w) {
    GFQ_CUDA(cudaFuncSetAttribute(ech_panel_win_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                  kPanelSmem));
    attr_w = true;
  }
  // the window start persists after the flags (the caller allocates
  // ech_panel_flag_bytes(rows) and zeroes them before the first panel)
  auto* lo_state = reinterpret_cast<std::int32_t*>(flags + ((rows + 15) / 16) * 16);
  GFQ_CUDA(launch_pdl(ech_panel_win_kernel, dim3(1), dim3(threads), smem, s, p, magic, int(rows), int(c0), int(wc), Aug, ld, flags,
                                                info, int(cap), G, ldg, rho2, lo_state));
  GFQ_CUDA(cudaGetLastError());
  count_launch();
}

// inverses mod p (0 -> 0), one 256-byte device table per prime, built once
const std::uint8_t* inv_table(std::uint32_t p) {
  static std::mutex mtx;
  static std::unordered_map<std::uint32_t, std::uint8_t*>* tabs =
      new std::unordered_map<std::uint32_t, std::uint8_t*>();  // process lifetime
  std::lock_guard<std::mutex> lk(mtx);
  auto it = tabs->find(p);
  if (it != tabs->end()) return it->second;
  std::uint8_t host[256] = {0};
  for (std::uint32_t a = 1; a < p && a < 256; ++a) {
    std::uint64_t r = 1, b = a;
    for (std::uint32_t e = p - 2; e; e >>= 1) {
      if (e & 1) r = r * b % p;
      b = b * b % p;
    }
    host[a] = std::uint8_t(r);
  }
  std::uint8_t* d = nullptr;
  GFQ_CUDA(cudaMalloc(&d, 256));
  GFQ_CUDA(cudaMemcpy(d, host, 256, cudaMemcpyHostToDevice));
  (*tabs)[p] = d;
  return d;
}

void ech_step(std::uint32_t p, std::int64_t rows, std::int64_t c0, std::int64_t wc, std::int64_t n,
              std::uint8_t* Z, std::int64_t ld, std::uint8_t* flags, std::int32_t* info,
              std::int64_t cap, std::int32_t* rho2, std::uint8_t* step_scratch, std::uint8_t* Y,
              const std::int32_t* base, bool chained_prev, bool chained_next, int seq, int signalled,
              cudaStream_t s) {
  if (wc > kW || c0 % kW || n % 16 || n > kStepMaxN || (ld & 15) ||
      (reinterpret_cast<std::uintptr_t>(Z) & 15))
    throw std::invalid_argument("ech_step: bad step geometry");
  const std::size_t smem = std::max<std::size_t>(std::size_t(rows) * (kW + 1), std::size_t(64 + kW) * n);
  if (smem > std::size_t(kPanelSmem)) throw std::invalid_argument("ech_step: block too tall");
  static bool attr = false;
  if (!attr) {
    for (auto fn : {ech_step_chain_kernel<0>, ech_step_chain_kernel<1>})
      GFQ_CUDA(cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, kPanelSmem));
    // both step kernels ask for the largest shared-memory carveout so the SM
    // does not reconfigure L1 / shared memory between them
    if (!std::getenv("GFQ_NO_CARVEOUT")) {
      for (auto fn : {ech_step_chain_kernel<0>, ech_step_chain_kernel<1>})
        GFQ_CUDA(cudaFuncSetAttribute(fn, cudaFuncAttributePreferredSharedMemoryCarveout, 100));
      GFQ_CUDA(cudaFuncSetAttribute(ech_step_update_kernel,
                                    cudaFuncAttributePreferredSharedMemoryCarveout, 100));
    }
    attr = true;
  }
  const std::uint32_t magic = static_cast<std::uint32_t>((0x100000000ULL / p) + 1);
  // algorithmic bytes: the step's rows x n slice of Z read and written
  ProfScope ps(kProfEchPanel, 2.0 * double(rows) * double(n), s);
  auto* lo_state = reinterpret_cast<std::int32_t*>(flags + ((rows + 15) / 16) * 16);
  std::uint8_t* NT = step_scratch;
  std::uint8_t* Gpiv = step_scratch + kW * kW;
  std::uint8_t* BpT = step_scratch + 2 * kW * kW;
  auto* ctr = reinterpret_cast<std::int32_t*>(step_scratch + 2 * kW * kW + kStepMaxN * kW);
  static const bool overlap = [] {
    const char* e = std::getenv("GFQ_STEP_OVERLAP");
    return !(e && e[0] == '0');
  }();
  // the chain waits until every CTA of the updates signalled so far
  // (`signalled`, the previous one included) has bumped the counters
  const int n_upd = int((rows + kStepRows - 1) / kStepRows);
  const int wait_prev = overlap && chained_prev && pdl_enabled() ? n_upd * signalled : 0;
  const int signal = overlap && chained_next && pdl_enabled() ? 1 : 0;
  const std::uint8_t* invt = inv_table(p);
  static int tl_n = std::getenv("GFQ_STEP_TL") ? std::atoi(std::getenv("GFQ_STEP_TL")) : 0;
  static int tl_i = 0;
  const int tl = tl_i < std::min(tl_n, kTlSteps) ? tl_i : -1;
  if (tl == 0) {
    static const unsigned long long zero[kTlSteps][8] = {};
    GFQ_CUDA(cudaMemcpyToSymbol(g_tl, zero, sizeof zero));
  }
  static const int mode = [] {  // A/B: GFQ_CHAIN_MODE = 0 one warp, 1 two row halves (default)
    const char* e = std::getenv("GFQ_CHAIN_MODE");
    return e && std::atoi(e) == 0 ? 0 : 1;
  }();
  GFQ_CUDA(launch_pdl(mode == 0 ? ech_step_chain_kernel<0> : ech_step_chain_kernel<1>, dim3(1),
                      dim3(kChainThreads), smem, s, p, magic, int(rows),
                      int(c0), int(wc), int(n), Z, ld, flags, info, int(cap), rho2, lo_state, NT, Gpiv,
                      Y, base, BpT, invt, ctr, wait_prev, seq, tl));
  GFQ_CUDA(launch_pdl(ech_step_update_kernel, dim3(unsigned((rows + kStepRows - 1) / kStepRows)),
                      dim3(kStepThreads), 0, s, p, magic, int(rows), int(c0), int(n), Z, ld, NT, Gpiv,
                      rho2, BpT, ctr, signal, seq, tl));
  if (tl >= 0 && ++tl_i == std::min(tl_n, kTlSteps)) {
    GFQ_CUDA(cudaStreamSynchronize(s));
    static unsigned long long h[kTlSteps][8];
    GFQ_CUDA(cudaMemcpyFromSymbol(h, g_tl, sizeof h));
    const unsigned long long t0 = h[0][0];

    for (int k = 0; k < tl_i; ++k) {
      std::fprintf(stderr, "TL %d", k);
      for (int j = 0; j < 8; ++j) std::fprintf(stderr, " %.2f", h[k][j] ? (double(h[k][j]) - double(t0)) * 1e-3 : -1.0);
      std::fprintf(stderr, "\n");
    }
  }
  static int dbg = std::getenv("GFQ_STEP_DEBUG") ? std::atoi(std::getenv("GFQ_STEP_DEBUG")) : 0;
  if (dbg > 0) {
    --dbg;
    unsigned long long st[16];
    GFQ_CUDA(cudaStreamSynchronize(s));
    GFQ_CUDA(cudaMemcpyFromSymbol(st, g_step_stamps, sizeof st));
    std::fprintf(stderr,
                 "ech_step rows %lld c0 %lld: setup %.2f chain %.2f outputs %.2f bpt %.2f us; "
                 "chain %llu cycles (%.2f GHz)\n",
                 (long long)rows, (long long)c0, (st[1] - st[0]) * 1e-3, (st[2] - st[1]) * 1e-3,
                 (st[3] - st[2]) * 1e-3, (st[4] - st[3]) * 1e-3, st[10] - st[9],
                 double(st[10] - st[9]) / double(st[2] - st[1]));
  }
  count_launch(2);
}

void ech_panel_plant(std::uint8_t* Y, std::int64_t ldy, const std::int32_t* rho2,
                     const std::int32_t* info, const std::int32_t* base, cudaStream_t s) {
  GFQ_CUDA(launch_pdl(ech_plant_kernel, dim3(1), dim3(32), 0, s, Y, ldy, rho2, info, base));
  GFQ_CUDA(cudaGetLastError());
  count_launch();
}

void ech_outer_finish(std::uint32_t p, std::uint8_t* Y, std::int64_t ldy, std::int64_t kcols,
                      std::int32_t* info, std::int64_t cap, std::int32_t* base,
                      std::int32_t* rmap, std::int64_t col0, cudaStream_t s) {
  GFQ_CUDA(launch_pdl(ech_outer_finish_kernel, dim3(1), dim3(256), 0, s, p, Y, ldy, int(kcols), info,
                      int(cap), base, rmap, int(col0)));
  count_launch();
}

// dst[i][0:wd] = src[i][0:wd], dst[i][wd:width] = 0 (16-byte aligned rows,
// width a multiple of 16): the two-level ECH's scratch load and write-back
// as one kernel in the step kernels' PDL chain (a cudaMemcpy2D / memset
// would break it)
__global__ void copy_cols_kernel(std::uint8_t* __restrict__ dst, std::int64_t ldd,
                                 const std::uint8_t* __restrict__ src, std::int64_t lds,
                                 std::int64_t rows, int wd, int width) {
  pdl_wait_and_release();
  const int nv = width / 16;
  for (std::int64_t e = std::int64_t(blockIdx.x) * blockDim.x + threadIdx.x; e < rows * nv;
       e += std::int64_t(gridDim.x) * blockDim.x) {
    const std::int64_t i = e / nv;
    const int c = int(e % nv) * 16;
    uint4 v = make_uint4(0, 0, 0, 0);
    if (c + 16 <= wd) {
      v = *reinterpret_cast<const uint4*>(src + i * lds + c);
    } else if (c < wd) {
      std::uint8_t b[16] = {};
      for (int t = 0; c + t < wd; ++t) b[t] = src[i * lds + c + t];
      std::memcpy(&v, b, 16);
    }
    *reinterpret_cast<uint4*>(dst + i * ldd + c) = v;
  }
}

void copy_cols(std::uint8_t* dst, std::int64_t ldd, const std::uint8_t* src, std::int64_t lds,
               std::int64_t rows, std::int64_t wd, std::int64_t width, cudaStream_t s) {
  if (rows == 0 || width == 0) return;
  if (width % 16 || (ldd & 15) || (reinterpret_cast<std::uintptr_t>(dst) & 15) ||
      (wd >= 16 && ((lds & 15) || (reinterpret_cast<std::uintptr_t>(src) & 15))))
    throw std::invalid_argument("copy_cols: unaligned");
  const std::int64_t work = rows * (width / 16);
  const unsigned grid = unsigned(std::min<std::int64_t>((work + 255) / 256, 8 * sm_count()));
  GFQ_CUDA(launch_pdl(copy_cols_kernel, dim3(grid), dim3(256), 0, s, dst, ldd, src, lds, rows, int(wd),
                      int(width)));
  count_launch();
}

void scatter_rows(std::uint8_t* dst, std::int64_t ldd, std::int64_t rows, std::int64_t cols,
                  const std::uint8_t* src, std::int64_t lds, const std::int32_t* rmap,
                  cudaStream_t s) {
  if (rows == 0 || cols == 0) return;
  const unsigned gx = unsigned((cols + 255) / 256), gy = unsigned(rows < 65535 ? rows : 65535);
  scatter_rows_kernel<<<dim3(gx, gy), 256, 0, s>>>(dst, ldd, rows, cols, src, lds, rmap);
  GFQ_CUDA(cudaGetLastError());
  count_launch();
}

}  // namespace gfq::dev
