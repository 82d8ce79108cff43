// ech_gf2.cu -- K2 for GF(2): a whole block ECH in ONE cooperative launch.
//
// GF(2) is the field of configs[1] and configs[4].  The augmented block
// Aug = [H | I] (rows <= 1024, cols + rows <= 8192) is bit-packed (32
// columns per word; 256 KB for 1024 x 2048, L2-resident) and eliminated by
// right-looking Gauss-Jordan over 32-column panels.  Per panel:
//   * CTA 0, warp 0 runs the pivot chain with the reference's column-wise
//     rule (first non-pivotal row with a set bit; reference
//     src/chief.cpp:436-460): lane l owns rows 32r + l transposed into 32
//     column masks, so a column step is a mask AND, a warp min-reduction, a
//     shuffle of the pivot row and 32 masked XORs -- no block barriers; it
//     inverts the 32 x 32 pivot block in registers and CTA 0 publishes every
//     row's multiplier word G[i] = Ap[i].N2 and a snapshot of the pivot rows;
//   * grid barrier; every CTA applies Aug[i] ^= XOR_{q in G[i]} pivot_q to
//     its rows (warp per row, lanes over words, coalesced); grid barrier.
// The blocks of this cooperative launch wait on one another only through the
// grid barrier, and cudaLaunchCooperativeKernel guarantees they are
// co-resident.  The reduced block is unpacked to u8 at the end; pivots go
// to info = [rank, cols[cap], rows[cap]] like the multi-launch path.
#include <algorithm>
#include <cstdio>
#include <cstdlib>

#include "../common.hpp"
#include "kernels.hpp"

namespace gfq::dev {
namespace {

constexpr int kMaxWords = 256;  // cols + rows <= 8192
constexpr int kCoopBlocks = 64;

__device__ __forceinline__ void transpose32(std::uint32_t (&a)[32]) {
  // a[r] bit c  ->  a[c] bit r   (LSB-first block swaps)
#pragma unroll
  for (int j = 16; j >= 1; j >>= 1) {
    const std::uint32_t m = j == 16 ? 0x0000FFFFu : j == 8 ? 0x00FF00FFu : j == 4 ? 0x0F0F0F0Fu
                          : j == 2  ? 0x33333333u : 0x55555555u;
#pragma unroll
    for (int k = 0; k < 32; ++k) {
      if (k & j) continue;
      const std::uint32_t t = ((a[k] >> j) ^ a[k + j]) & m;
      a[k] ^= t << j;
      a[k + j] ^= t;
    }
  }
}

// Sense-counting grid barrier for a cooperative launch (bar[0] = arrivals,
// bar[1] = generation; zeroed before the launch).
__device__ __forceinline__ void grid_barrier(unsigned* bar) {
  __syncthreads();
  if (threadIdx.x == 0) {
    volatile unsigned* vb = bar;
    const unsigned gen = vb[1];
    __threadfence();
    if (atomicAdd(&bar[0], 1u) == gridDim.x - 1) {
      bar[0] = 0;
      __threadfence();
      atomicAdd(&bar[1], 1u);
    } else {
      while (vb[1] == gen) __nanosleep(64);
    }
    __threadfence();
  }
  __syncthreads();
}

struct Gf2Args {
  int rows, cols, Wd, cap;
  const std::uint8_t* H;
  std::int64_t ldh;
  std::uint32_t* A;    // rows x Wd packed [W | T]
  std::uint32_t* gw;   // rows multiplier words
  std::uint32_t* bpg;  // 32 x Wd pivot-row snapshot
  std::uint8_t* Out;
  std::int64_t ldo;
  std::int32_t* info;
  unsigned* bar;       // [arrivals, generation, r2 of the current panel]
  unsigned long long* dbg;  // optional phase timestamps (GFQ_GF2_DEBUG)
};

__device__ __forceinline__ unsigned long long gtime() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
  return t;
}
#define GF2_STAMP(k)                                                              \
  do {                                                                            \
    if (g.dbg && blockIdx.x == 0 && threadIdx.x == 0 && (c0 >> 5) < 8)           \
      g.dbg[(c0 >> 5) * 8 + (k)] = gtime();                                       \
  } while (0)

__global__ void __launch_bounds__(1024, 1) ech_gf2_coop_kernel(Gf2Args g) {
  __shared__ std::uint32_t orig[1024];
  __shared__ std::uint32_t bp[32 * kMaxWords];
  __shared__ std::uint8_t fl[1024];
  __shared__ int pc[32], pr[32];
  __shared__ std::uint32_t n2[32];
  __shared__ int r2_sh;
  const int tid = threadIdx.x, nt = blockDim.x, lane = tid & 31, warp = tid >> 5;
  const int nwarps = nt >> 5;
  const int gwarp = blockIdx.x * nwarps + warp, gnwarps = gridDim.x * nwarps;
  const int rows = g.rows, cols = g.cols, Wd = g.Wd;

  if (g.dbg && blockIdx.x == 0 && tid == 0) g.dbg[63] = gtime();
  // ---- pack [H | I] (warp per row, lane per word)
  for (int i = gwarp; i < rows; i += gnwarps) {
    const std::uint8_t* h = g.H + std::int64_t(i) * g.ldh;
    for (int w = lane; w < Wd; w += 32) {
      std::uint32_t word = 0;
      const int j0 = 32 * w;
      if (j0 + 32 <= cols && (reinterpret_cast<std::uintptr_t>(h + j0) & 15) == 0) {
        const uint4 a = reinterpret_cast<const uint4*>(h + j0)[0];
        const uint4 b = reinterpret_cast<const uint4*>(h + j0)[1];
        const std::uint32_t wds[8] = {a.x, a.y, a.z, a.w, b.x, b.y, b.z, b.w};
#pragma unroll
        for (int q = 0; q < 8; ++q) {
          const std::uint32_t v = wds[q] & 0x01010101u;
          word |= ((v & 1u) | ((v >> 7) & 2u) | ((v >> 14) & 4u) | ((v >> 21) & 8u)) << (4 * q);
        }
      } else {
        for (int b = 0; b < 32; ++b) {
          const int j = j0 + b;
          if (j < cols) word |= std::uint32_t(h[j] & 1u) << b;
        }
        if (j0 <= cols + i && cols + i < j0 + 32) word |= 1u << (cols + i - j0);
      }
      g.A[std::int64_t(i) * Wd + w] = word;
    }
  }
  if (blockIdx.x == 0)
    for (int i = tid; i < 1024; i += nt) fl[i] = i < rows ? 0 : 1;
  grid_barrier(g.bar);

  // CTA 0: load panel word `wi` of every row, run the pivot chain in warp 0
  // and invert the pivot block; results in shared memory (pc, pr, n2, r2_sh).
  // `orig` must already hold the panel words (masked to the panel width).
  auto pmask_of = [&](int wi) {
    const int wc = cols - 32 * wi < 32 ? cols - 32 * wi : 32;
    return wc == 32 ? 0xFFFFFFFFu : ((1u << wc) - 1u);
  };
  auto factorize = [&](int wi, int info_off) {
    const int c0 = 32 * wi;
    {
      const int wc = cols - c0 < 32 ? cols - c0 : 32;
      if (warp == 0) {
        std::uint32_t col[32];
        std::uint32_t fm = 0;
#pragma unroll
        for (int r = 0; r < 32; ++r) {
          col[r] = orig[32 * r + lane];
          fm |= std::uint32_t(fl[32 * r + lane]) << r;
        }
        transpose32(col);  // col[c] bit r: row 32r + lane has bit c
        int r2 = 0;
        // Fully unrolled: col[c] and col[q > c] are static registers; columns
        // <= c are finished and skipped at compile time.
#pragma unroll
        for (int c = 0; c < 32; ++c) {
          if (c < wc) {
            std::uint32_t cm = col[c] & ~fm;
            unsigned cand = cm ? unsigned(32 * (__ffs(cm) - 1) + lane) : 0xFFFFFFFFu;
            cand = __reduce_min_sync(0xffffffffu, cand);
            if (cand != 0xFFFFFFFFu) {
              const int sl = int(cand & 31), sr = int(cand >> 5);
              // pivot row bits of the remaining columns, OR-reduced as a tree
              std::uint32_t part[4] = {0, 0, 0, 0};
#pragma unroll
              for (int q = c + 1; q < 32; ++q) part[q & 3] |= ((col[q] >> sr) & 1u) << q;
              const std::uint32_t mine = (part[0] | part[1]) | (part[2] | part[3]);
              const std::uint32_t ps = __shfl_sync(0xffffffffu, mine, sl);
              if (lane == sl) {
                cm &= ~(1u << sr);
                fm |= 1u << sr;
              }
#pragma unroll
              for (int q = c + 1; q < 32; ++q) col[q] ^= cm & (0u - ((ps >> q) & 1u));
              if (lane == 0) {
                pc[r2] = c;
                pr[r2] = int(cand);
              }
              ++r2;
            }
          }
        }
        __syncwarp();
        // N2 = inv(X), X[q][t] = bit pc[t] of the original word of row pr[q]:
        // swap-free Gauss-Jordan, lane = row of [X | I]; the pivot of column
        // q is the first unused lane with bit q, and N2 row q is the inverse
        // row of that lane.
        std::uint32_t x = 0, inv = 0, used = 0;
        if (lane < r2) {
          const std::uint32_t ow = orig[pr[lane]];
          for (int t = 0; t < r2; ++t) x |= ((ow >> pc[t]) & 1u) << t;
          inv = 1u << lane;
        }
        int myq = 0;
        for (int q = 0; q < r2; ++q) {
          const unsigned bal =
              __ballot_sync(0xffffffffu, lane < r2 && !((used >> lane) & 1u) && ((x >> q) & 1u));
          const int pv = __ffs(bal) - 1;
          used |= 1u << pv;
          const std::uint32_t px = __shfl_sync(0xffffffffu, x, pv), pi = __shfl_sync(0xffffffffu, inv, pv);
          if (lane != pv && ((x >> q) & 1u)) {
            x ^= px;
            inv ^= pi;
          }
          if (lane == pv) myq = q;
        }
        n2[lane] = 0u;
        __syncwarp();
        if (lane < r2) n2[myq] = inv;
        if (lane < r2) {
          g.info[1 + info_off + lane] = c0 + pc[lane];
          g.info[1 + g.cap + info_off + lane] = pr[lane];
          fl[pr[lane]] = 1;
        }
        if (lane == 0) r2_sh = r2;
      }
      __syncthreads();
    }
  };

  // Look-ahead schedule: CTA 0 publishes panel k's multipliers and updates
  // the words of panels k and k+1 itself, so after the first barrier it can
  // factorize panel k+1 while the other CTAs update the remaining words.
  const int npan = (cols + 31) / 32;
  const int upd_first = gridDim.x > 1 ? 1 : 0;  // CTAs that run the wide update
  const int uwarp = (int(blockIdx.x) - upd_first) * nwarps + warp;
  const int unwarps = (int(gridDim.x) - upd_first) * nwarps;
  int rtot = 0;
  if (blockIdx.x == 0) {
    const std::uint32_t pm = pmask_of(0);
    for (int i = tid; i < 1024; i += nt) orig[i] = i < rows ? (g.A[std::int64_t(i) * Wd] & pm) : 0u;
    __syncthreads();
    factorize(0, 0);
  }
  for (int k = 0; k < npan; ++k) {
    const int wi = k, c0 = 32 * k;
    GF2_STAMP(0);
    if (blockIdx.x == 0) {
      const int r2 = r2_sh;
      const bool has_next = k + 1 < npan;
      const std::uint32_t pm_next = has_next ? pmask_of(k + 1) : 0u;
      if (r2 > 0) {
        // pivot-row snapshot (global, words >= wi) and words wi, wi+1 in smem
        const int nw = Wd - wi;
        for (int e = tid; e < r2 * nw; e += nt) {
          const int q = e / nw, w = wi + e % nw;
          const std::uint32_t v = g.A[std::int64_t(pr[q]) * Wd + w];
          g.bpg[q * Wd + w] = v;
          if (w < wi + 2) bp[q * 2 + (w - wi)] = v;
        }
        __syncthreads();
        // G words, and words wi, wi+1 of every row (the next panel becomes
        // final here and is left in `orig` for the look-ahead factorization)
        for (int i = tid; i < rows; i += nt) {
          const std::uint32_t ow = orig[i];
          std::uint32_t gv = 0;
          for (int q = 0; q < r2; ++q)
            if (((ow >> pc[q]) & 1u) ^ (pr[q] == i ? 1u : 0u)) gv ^= n2[q];
          g.gw[i] = gv;
          // word wi+1 exists whenever [W | T] is wider than this panel, even
          // on the last panel (it then holds T columns)
          const bool has_w1 = wi + 1 < Wd;
          std::uint32_t x0 = g.A[std::int64_t(i) * Wd + wi];
          std::uint32_t x1 = has_w1 ? g.A[std::int64_t(i) * Wd + wi + 1] : 0u;
          std::uint32_t gg = gv;
          while (gg) {
            const int q = __ffs(gg) - 1;
            gg &= gg - 1;
            x0 ^= bp[2 * q];
            x1 ^= bp[2 * q + 1];
          }
          if (gv) {
            g.A[std::int64_t(i) * Wd + wi] = x0;
            if (has_w1) g.A[std::int64_t(i) * Wd + wi + 1] = x1;
          }
          if (has_next) orig[i] = x1 & pm_next;
        }
      } else if (has_next) {
        for (int i = tid; i < rows; i += nt) orig[i] = g.A[std::int64_t(i) * Wd + wi + 1] & pm_next;
      }
      if (has_next)
        for (int i = rows + tid; i < 1024; i += nt) orig[i] = 0u;
      if (tid == 0) g.bar[2] = unsigned(r2);
    }
    GF2_STAMP(1);
    grid_barrier(g.bar);
    GF2_STAMP(2);
    const int r2 = int(*reinterpret_cast<volatile unsigned*>(&g.bar[2]));
    if (r2 > 0 && int(blockIdx.x) >= upd_first && wi + 2 < Wd) {
      const int nw = Wd - (wi + 2);
      for (int e = tid; e < r2 * nw; e += nt) {
        const int q = e / nw, w = wi + 2 + e % nw;
        bp[q * kMaxWords + w] = g.bpg[q * Wd + w];
      }
      __syncthreads();
      for (int i = uwarp; i < rows; i += unwarps) {
        const std::uint32_t gv = g.gw[i];
        if (!gv) continue;
        std::uint32_t* arow = g.A + std::int64_t(i) * Wd;
        for (int w = wi + 2 + lane; w < Wd; w += 32) {
          std::uint32_t x = arow[w];
          std::uint32_t gg = gv;
          while (gg) {
            const int q = __ffs(gg) - 1;
            gg &= gg - 1;
            x ^= bp[q * kMaxWords + w];
          }
          arow[w] = x;
        }
      }
    }
    if (blockIdx.x == 0 && k + 1 < npan) factorize(k + 1, rtot + r2);  // overlaps the update
    rtot += r2;
    GF2_STAMP(3);
    grid_barrier(g.bar);
    GF2_STAMP(4);
  }

  // ---- unpack the reduced [W | T] to u8 (warp per row)
  const int tot = cols + rows;
  for (int i = gwarp; i < rows; i += gnwarps) {
    const std::uint32_t* arow = g.A + std::int64_t(i) * Wd;
    std::uint8_t* orow = g.Out + std::int64_t(i) * g.ldo;
    for (int w = lane; w < Wd; w += 32) {
      const std::uint32_t word = arow[w];
      const int j0 = 32 * w;
      if (j0 + 32 <= tot && (reinterpret_cast<std::uintptr_t>(orow + j0) & 15) == 0) {
        std::uint32_t outw[8];
#pragma unroll
        for (int q = 0; q < 8; ++q) {
          const std::uint32_t nib = (word >> (4 * q)) & 0xFu;
          outw[q] = (nib & 1u) | ((nib & 2u) << 7) | ((nib & 4u) << 14) | ((nib & 8u) << 21);
        }
        reinterpret_cast<uint4*>(orow + j0)[0] = make_uint4(outw[0], outw[1], outw[2], outw[3]);
        reinterpret_cast<uint4*>(orow + j0)[1] = make_uint4(outw[4], outw[5], outw[6], outw[7]);
      } else {
        for (int b = 0; b < 32 && j0 + b < tot; ++b) orow[j0 + b] = (word >> b) & 1u;
      }
    }
  }
  if (blockIdx.x == 0 && tid == 0) g.info[0] = rtot;
}

}  // namespace

std::int64_t ech_gf2_scratch_words(std::int64_t rows, std::int64_t cols) {
  const std::int64_t Wd = (cols + rows + 31) / 32;
  return rows * Wd + rows + 32 * Wd + 4;
}

bool ech_gf2_block(std::int64_t rows, std::int64_t cols, const std::uint8_t* H, std::int64_t ldh,
                   std::uint32_t* scratch, std::uint8_t* Out, std::int64_t ldo, std::int32_t* info,
                   std::int64_t cap, cudaStream_t s) {
  const std::int64_t Wd = (cols + rows + 31) / 32;
  if (rows > 1024 || Wd > kMaxWords) return false;
  static int blocks = 0;
  if (blocks == 0) {
    int per_sm = 0;
    GFQ_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, ech_gf2_coop_kernel, 1024, 0));
    const char* e = std::getenv("GFQ_GF2_BLOCKS");
    const int want = e ? std::atoi(e) : kCoopBlocks;
    blocks = std::max(1, std::min(want > 0 ? want : kCoopBlocks, per_sm * sm_count()));
  }
  Gf2Args g;
  g.rows = int(rows);
  g.cols = int(cols);
  g.Wd = int(Wd);
  g.cap = int(cap);
  g.H = H;
  g.ldh = ldh;
  g.A = scratch;
  g.gw = scratch + rows * Wd;
  g.bpg = g.gw + rows;
  g.bar = reinterpret_cast<unsigned*>(g.bpg + 32 * Wd);
  g.Out = Out;
  g.ldo = ldo;
  g.info = info;
  static const bool debug = std::getenv("GFQ_GF2_DEBUG") != nullptr;
  static unsigned long long* dbg = nullptr;
  if (debug && !dbg) GFQ_CUDA(cudaMallocManaged(&dbg, 64 * sizeof(unsigned long long)));
  g.dbg = debug ? dbg : nullptr;
  fill2d(reinterpret_cast<std::uint8_t*>(g.bar), 16, 1, 4 * sizeof(unsigned), 0, s);
  void* args[] = {&g};
  GFQ_CUDA(cudaLaunchCooperativeKernel(reinterpret_cast<const void*>(ech_gf2_coop_kernel),
                                       dim3(unsigned(blocks)), dim3(1024), args, 0, s));
  count_launch();
  if (debug) {
    GFQ_CUDA(cudaStreamSynchronize(s));
    std::fprintf(stderr, "gf2 prologue %lld ns\n", static_cast<long long>(dbg[0] - dbg[63]));
    for (int pnl = 0; pnl < 4; ++pnl) {
      std::fprintf(stderr, "gf2 panel %d:", pnl);
      for (int k = 1; k < 5; ++k)
        std::fprintf(stderr, " %lld", static_cast<long long>(dbg[pnl * 8 + k] - dbg[pnl * 8 + k - 1]));
      std::fprintf(stderr, " ns\n");
    }
  }
  return true;
}

}  // namespace gfq::dev
