// ech_gf2_cluster.cu -- K2 for GF(2), cluster-resident: the whole
// bit-packed block [H | I] (rows <= 1024, cols + rows <= 8192) lives in the
// shared memory of ONE 8-CTA thread-block cluster (each CTA holds a stripe of
// <= 128 rows), and every exchange between CTAs goes through distributed
// shared memory with cluster barriers instead of global memory and grid
// barriers.  Per 32-column panel (right-looking Gauss-Jordan with the
// reference's column-wise pivot rule, src/chief.cpp:436-460):
//   a. every CTA pushes word `wi` of its rows into the leader's `orig`;
//   b. the leader finds the panel's pivots and each row's multiplier word
//      G[i] (which pivot rows' ORIGINAL values to add): warp 0 runs the chain
//      on a 64-row window starting at the first non-pivotal row, tracking per
//      row the set of pivots added (Gauss-Jordan, so pivot rows are reduced
//      too); rows outside the window get G from nibble tables of the pivots'
//      coefficient sets.  A column without a window candidate sends the panel
//      to a CTA-wide chain over all rows.  G and the pivot list are pushed to
//      the owning CTAs;
//   c. every CTA pulls the panel's pivot rows from their owners (DSMEM loads);
//   d. every CTA updates its stripe: row ^= XOR_{q in G} pivot_q, through
//      per-panel nibble tables of pivot-row combinations (8 lookups a word).
// The reduced block is unpacked to u8 at the end; pivots go to
// info = [rank, cols[cap], rows[cap]] like the other ECH paths.
#include <cooperative_groups.h>

#include <algorithm>

#include <cstdio>
#include <cstdlib>

#include "../common.hpp"
#include "kernels.hpp"

namespace gfq::dev {
namespace {

namespace cg = cooperative_groups;

constexpr int kCl = 8;          // CTAs per cluster (portable maximum)
constexpr int kThreads = 1024;  // 32 warps per CTA
constexpr int kStripe = 128;    // rows per CTA (1024 / kCl)
constexpr int kMaxWd = 256;     // cols + rows <= 8192
constexpr int kTabWd = 96;      // nibble tables (128 x Wd words) up to here

struct ClArgs {
  int rows, cols, Wd, cap;
  const std::uint8_t* H;
  std::int64_t ldh;
  std::uint8_t* Out;
  std::int64_t ldo;
  std::int32_t* info;
  unsigned long long* dbg;  // developer phase stamps (GFQ_GF2_DEBUG)
};

__device__ __forceinline__ unsigned long long gtime() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}

__global__ void __launch_bounds__(kThreads, 1) ech_gf2_cluster_kernel(ClArgs g) {
  extern __shared__ __align__(16) std::uint32_t sm[];
  const int Wd = g.Wd, rows = g.rows, cols = g.cols;
  std::uint32_t* A = sm;                       // kStripe x Wd   (my rows)
  std::uint32_t* bp = A + kStripe * Wd;        // 32 x Wd        (pivot rows of the panel)
  std::uint32_t* orig = bp + 32 * Wd;          // 1024           (leader: panel word per row)
  std::uint32_t* gl = orig + 1024;             // kStripe        (multiplier word per my row)
  std::uint8_t* fl = reinterpret_cast<std::uint8_t*>(gl + kStripe);  // 1024 (leader)
  std::uint32_t* gall = reinterpret_cast<std::uint32_t*>(fl + 1024);  // 1024 (leader: G per row)
  std::uint32_t* tab = gall + 1024;  // 128 x Wd nibble tables (when Wd <= kTabWd)
  const bool use_tab = Wd <= kTabWd;
  __shared__ int pc[32], pr[32];
  __shared__ int r2_sh;
  __shared__ std::uint32_t nomw[2][32], nomc[2][32];
  __shared__ unsigned best[3];
  __shared__ int lo_sh, win_ok;
  __shared__ std::uint32_t pcoef[32], ntab[128];
  __shared__ std::uint8_t thisp[1024];

  cg::cluster_group cluster = cg::this_cluster();
  const int cr = int(cluster.block_rank());
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int row0 = cr * kStripe;
  const int nloc = rows - row0 < 0 ? 0 : (rows - row0 < kStripe ? rows - row0 : kStripe);
  std::uint32_t* lead_orig = cluster.map_shared_rank(orig, 0);

  // ---- pack my stripe of [H | I] (warp per row, lane per word)
  for (int li = warp; li < nloc; li += kThreads / 32) {
    const int i = row0 + li;
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
      A[li * Wd + w] = word;
    }
  }
  if (cr == 0) {
    for (int i = tid; i < 1024; i += kThreads) {
      fl[i] = i < rows ? 0 : 1;
      orig[i] = 0u;
    }
    if (tid == 0) lo_sh = 0;
    for (int i = tid; i < 1024; i += kThreads) thisp[i] = 0;
  }
  cluster.sync();

  const int npan = (cols + 31) / 32;
  int rtot = 0;
  for (int k = 0; k < npan; ++k) {
    const int wi = k, c0 = 32 * k;
    const int wc = cols - c0 < 32 ? cols - c0 : 32;
    const std::uint32_t pm = wc == 32 ? 0xFFFFFFFFu : ((1u << wc) - 1u);
    auto stamp = [&](int ph) {
      if (g.dbg && cr == 0 && tid == 0 && k < 8) {
        g.dbg[k * 16 + ph] = gtime();
        if (ph == 0) g.dbg[k * 16 + 15] = clock64();
        if (ph == 7) g.dbg[k * 16 + 14] = clock64();
      }
    };
    stamp(0);
    // a. panel word of my rows -> leader
    for (int li = tid; li < nloc; li += kThreads) lead_orig[row0 + li] = A[li * Wd + wi] & pm;
    cluster.sync();
    stamp(1);

    // b. leader: the pivot chain, CTA-wide.  Thread t owns row t: its
    // current panel word and `coef`, the set of this panel's pivot rows (by
    // pivot index) whose ORIGINAL rows have been added to it.  Per column,
    // every warp nominates its first non-pivotal row with the bit set (word
    // and coef), one barrier, every warp min-reduces the nominations, and
    // EVERY other row with the bit set (pivotal ones too: Gauss-Jordan) adds
    // the pivot row.  Selection only looks at non-pivotal rows, so the pivots
    // are the reference's; at the end row t = orig_t + sum_{q in coef_t}
    // orig(pivot q) is reduced on all pivot columns, i.e. coef_t is its
    // multiplier word G[t].
    if (cr == 0) {
      // Fast path: the first 64 rows from the first non-pivotal one hold
      // every pivot of a full-rank panel (the chosen row is the FIRST
      // non-pivotal one with the bit), so warp 0 runs the chain on that
      // window alone (2 rows per lane, no barriers).  If some column has no
      // candidate inside the window the whole panel goes to the CTA-wide
      // chain instead (free columns, rank-deficient blocks).
      if (warp == 0) {
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
        std::uint32_t w0 = i0 < 1024 ? orig[i0] : 0u, w1 = i1 < 1024 ? orig[i1] : 0u;
        bool p0 = i0 >= rows || fl[i0] != 0, p1 = i1 >= rows || fl[i1] != 0;
        std::uint32_t cf0 = 0, cf1 = 0;
        int r2 = 0, ok = 1;
        for (int c = 0; c < wc; ++c) {
          const unsigned b0 = __ballot_sync(0xffffffffu, ((w0 >> c) & 1u) && !p0);
          const unsigned b1 = __ballot_sync(0xffffffffu, ((w1 >> c) & 1u) && !p1);
          if (!(b0 | b1)) {
            ok = 0;
            break;
          }
          const int hi = b0 ? 0 : 1;
          const int sl = __ffs(hi ? b1 : b0) - 1;
          const std::uint32_t pw = __shfl_sync(0xffffffffu, hi ? w1 : w0, sl);
          const std::uint32_t pcf = __shfl_sync(0xffffffffu, hi ? cf1 : cf0, sl) ^ (1u << r2);
          const bool me0 = !hi && lane == sl, me1 = hi && lane == sl;
          if (me0) p0 = true;
          else if ((w0 >> c) & 1u) {
            w0 ^= pw;
            cf0 ^= pcf;
          }
          if (me1) p1 = true;
          else if ((w1 >> c) & 1u) {
            w1 ^= pw;
            cf1 ^= pcf;
          }
          if (lane == 0) {
            pc[r2] = c;
            pr[r2] = lo + 32 * hi + sl;
          }
          ++r2;
        }
        if (lane == 0) {
          win_ok = ok;
          r2_sh = r2;
          lo_sh = lo;
        }
        if (ok) {
          // the pivots' own multipliers (others are recomputed below)
          if (i0 < rows) gall[i0] = cf0;
          if (i1 < rows) gall[i1] = cf1;
          __syncwarp();
          if (lane < r2) pcoef[lane] = gall[pr[lane]] ^ (1u << lane);
        }
      }
      __syncthreads();
      if (win_ok) {
        // G[i] = XOR over the pivot columns set in orig_i of (own original +
        // coef) of that column's pivot, via 8 nibble tables
        // ntab[k][m] = XOR_{b in m} pcoef(pivot of column 4k+b).  This
        // panel's pivot rows keep their chain coef.
        const int r2 = r2_sh;
        if (tid < 128) {
          const int kq = tid >> 4, m = tid & 15;
          std::uint32_t v = 0;
          for (int q = 0; q < r2; ++q) {
            const int cq = pc[q];
            if ((cq >> 2) == kq && ((m >> (cq & 3)) & 1)) v ^= pcoef[q];
          }
          ntab[tid] = v;
        }
        if (tid < r2) thisp[pr[tid]] = 1;
        __syncthreads();
        for (int i = tid; i < rows; i += kThreads) {
          if (thisp[i]) continue;
          const std::uint32_t ow = orig[i];
          std::uint32_t gv = 0;
#pragma unroll
          for (int kq = 0; kq < 8; ++kq) gv ^= ntab[16 * kq + ((ow >> (4 * kq)) & 15u)];
          gall[i] = gv;
        }
        __syncthreads();
        if (tid < r2) {
          fl[pr[tid]] = 1;
          thisp[pr[tid]] = 0;
        }
      } else {
      constexpr int kChainWarps = 8, kRowsPerLane = 1024 / (32 * kChainWarps);
        if (warp < kChainWarps) {
          std::uint32_t word[kRowsPerLane], coef[kRowsPerLane];
          std::uint32_t pivm = 0;  // bit s: row 256*s + tid is pivotal
#pragma unroll
          for (int s2 = 0; s2 < kRowsPerLane; ++s2) {
            word[s2] = orig[256 * s2 + tid];
            coef[s2] = 0u;
            pivm |= std::uint32_t(fl[256 * s2 + tid] != 0) << s2;
          }
          int r2 = 0;
          if (tid < 3) best[tid] = 0xFFFFFFFFu;
          asm volatile("bar.sync 1, 256;" ::: "memory");
#pragma unroll 1
          for (int c = 0; c < wc; ++c) {
            const int par = c & 1, b3 = c % 3;
            // this warp's first non-pivotal row with bit c: rows 256*s + tid,
            // so the smallest s with any candidate lane, then the lowest lane
            int ws = -1, wl = 0;
#pragma unroll
            for (int s2 = 0; s2 < kRowsPerLane; ++s2) {
              const unsigned b =
                  __ballot_sync(0xffffffffu, ((word[s2] >> c) & 1u) && !((pivm >> s2) & 1u));
              if (ws < 0 && b) {
                ws = s2;
                wl = __ffs(b) - 1;
              }
            }
            if (ws >= 0 && lane == wl) {
              std::uint32_t wv = 0, cv = 0;
#pragma unroll
              for (int t = 0; t < kRowsPerLane; ++t)
                if (t == ws) {
                  wv = word[t];
                  cv = coef[t];
                }
              nomw[par][warp] = wv;
              nomc[par][warp] = cv;
              atomicMin(&best[b3], unsigned(256 * ws + 32 * warp + wl));
            }
            asm volatile("bar.sync 1, 256;" ::: "memory");
            const unsigned m = best[b3];
            // column c-1's buffer: its readers all passed this barrier, and
            // column c+2's nominations come after the next one
            if (tid == 0) best[(c + 2) % 3] = 0xFFFFFFFFu;
            if (m == 0xFFFFFFFFu) continue;  // uniform: no pivot in column c
            const unsigned owner = (m & 255u) >> 5;
            const std::uint32_t pw = nomw[par][owner], pcf = nomc[par][owner] ^ (1u << r2);
#pragma unroll
            for (int s2 = 0; s2 < kRowsPerLane; ++s2) {
              const unsigned row = unsigned(256 * s2 + tid);
              if (row == m) {
                pivm |= 1u << s2;
              } else if ((word[s2] >> c) & 1u) {
                word[s2] ^= pw;
                coef[s2] ^= pcf;
              }
            }
            if (tid == 0) {
              pc[r2] = c;
              pr[r2] = int(m);
            }
            ++r2;
            }
  #pragma unroll
          for (int s2 = 0; s2 < kRowsPerLane; ++s2) {
            const int i = 256 * s2 + tid;
            gall[i] = coef[s2];
            if ((pivm >> s2) & 1u) fl[i] = 1;
          }
          if (tid == 0) r2_sh = r2;
        }
      }
      __syncthreads();  // gall, pc / pr / r2 complete
      const int r2 = r2_sh;
      for (int i = tid; i < rows; i += kThreads)
        *cluster.map_shared_rank(&gl[i % kStripe], unsigned(i / kStripe)) = gall[i];
      if (tid < r2) {
        g.info[1 + rtot + tid] = c0 + pc[tid];
        g.info[1 + g.cap + rtot + tid] = pr[tid];
      }
      // pivot list -> every CTA
      if (tid < kCl * 32) {
        const unsigned dst = unsigned(tid >> 5);
        const int q = tid & 31;
        if (q < r2) *cluster.map_shared_rank(&pr[q], dst) = pr[q];
        if (q == 0) *cluster.map_shared_rank(&r2_sh, dst) = r2;
      }
      stamp(2);
    }
    stamp(3);
    cluster.sync();
    stamp(4);

    const int r2 = r2_sh;
    if (r2 > 0) {
      // c. pull the pivot rows (words >= wi) from their owners' stripes
      const int nw = Wd - wi;
      for (int e = tid; e < r2 * nw; e += kThreads) {
        const int q = e / nw, w = wi + e % nw;
        const int row = pr[q];
        const std::uint32_t* src =
            cluster.map_shared_rank(&A[(row % kStripe) * Wd + w], unsigned(row / kStripe));
        bp[q * Wd + w] = *src;
      }
      stamp(5);
      cluster.sync();  // every pull done before any owner rewrites a pivot row
      stamp(6);
      // d. update my stripe.  With the nibble tables (Wd <= kTabWd):
      // tab[k][m][w] = XOR_{b in m} pivot_{4k+b}[w], so a row's update is 8
      // lookups per word instead of one XOR per set multiplier bit.
      if (use_tab) {
        for (int e = tid; e < 128 * nw; e += kThreads) {
          const int km = e / nw, w = wi + e % nw;
          const int kq = km >> 4, m = km & 15;
          std::uint32_t v = 0;
#pragma unroll
          for (int b2 = 0; b2 < 4; ++b2)
            if (((m >> b2) & 1) && 4 * kq + b2 < r2) v ^= bp[(4 * kq + b2) * Wd + w];
          tab[km * Wd + w] = v;
        }
        __syncthreads();
        for (int li = warp; li < nloc; li += kThreads / 32) {
          const std::uint32_t gv = gl[li];
          if (!gv) continue;
          std::uint32_t* arow = A + li * Wd;
          for (int w = wi + lane; w < Wd; w += 32) {
            std::uint32_t x = arow[w];
#pragma unroll
            for (int kq = 0; kq < 8; ++kq) x ^= tab[(16 * kq + ((gv >> (4 * kq)) & 15u)) * Wd + w];
            arow[w] = x;
          }
        }
      } else {
        for (int li = warp; li < nloc; li += kThreads / 32) {
          const std::uint32_t gv = gl[li];
          if (!gv) continue;
          std::uint32_t* arow = A + li * Wd;
          for (int w = wi + lane; w < Wd; w += 32) {
            std::uint32_t x = arow[w];
            std::uint32_t gg = gv;
            while (gg) {
              const int q = __ffs(gg) - 1;
              gg &= gg - 1;
              x ^= bp[q * Wd + w];
            }
            arow[w] = x;
          }
        }
      }
      __syncthreads();
      stamp(7);
    }
    rtot += r2;
  }

  // ---- unpack my stripe of the reduced [W | T] to u8 (warp per row)
  const int tot = cols + rows;
  for (int li = warp; li < nloc; li += kThreads / 32) {
    const std::uint32_t* arow = A + li * Wd;
    std::uint8_t* orow = g.Out + std::int64_t(row0 + li) * g.ldo;
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
  if (cr == 0 && tid == 0) g.info[0] = rtot;
  cluster.sync();  // no CTA may exit while others still address its shared memory
}

}  // namespace

bool ech_gf2_cluster(std::int64_t rows, std::int64_t cols, const std::uint8_t* H, std::int64_t ldh,
                     std::uint8_t* Out, std::int64_t ldo, std::int32_t* info, std::int64_t cap,
                     cudaStream_t s) {
  static const bool off = std::getenv("GFQ_NO_GF2_CLUSTER") != nullptr;
  const std::int64_t Wd = (cols + rows + 31) / 32;
  if (off || rows > kCl * kStripe || Wd > kMaxWd || rows <= 0 || cols <= 0) return false;
  const std::size_t smem =
      std::size_t(kStripe * Wd + 32 * Wd + 1024 + kStripe) * 4 + 1024 + 4096 +
      (Wd <= kTabWd ? std::size_t(128 * Wd) * 4 : 0);
  static bool attr = false;
  if (!attr) {
    GFQ_CUDA(cudaFuncSetAttribute(ech_gf2_cluster_kernel,
                                  cudaFuncAttributeMaxDynamicSharedMemorySize,
                                  int(std::max(std::size_t(kStripe * kMaxWd + 32 * kMaxWd + 1024 + kStripe) * 4 + 1024 + 4096,
                                               std::size_t(kStripe * kTabWd + 32 * kTabWd + 1024 + kStripe) * 4 +
                                                   1024 + 4096 + std::size_t(128 * kTabWd) * 4))));
    attr = true;
  }
  static const bool debug = std::getenv("GFQ_GF2_DEBUG") != nullptr;
  static unsigned long long* dbg = nullptr;
  if (debug && !dbg) GFQ_CUDA(cudaMalloc(&dbg, 8 * 16 * sizeof(unsigned long long)));
  ClArgs g{int(rows), int(cols), int(Wd), int(cap), H, ldh, Out, ldo, info, debug ? dbg : nullptr};
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(kCl);
  cfg.blockDim = dim3(kThreads);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = s;
  cudaLaunchAttribute attrs[1];
  attrs[0].id = cudaLaunchAttributeClusterDimension;
  attrs[0].val.clusterDim.x = kCl;
  attrs[0].val.clusterDim.y = 1;
  attrs[0].val.clusterDim.z = 1;
  cfg.attrs = attrs;
  cfg.numAttrs = 1;
  GFQ_CUDA(cudaLaunchKernelEx(&cfg, ech_gf2_cluster_kernel, g));
  count_launch();
  if (debug) {
    GFQ_CUDA(cudaStreamSynchronize(s));
    unsigned long long hd[8 * 16];
    GFQ_CUDA(cudaMemcpy(hd, dbg, sizeof hd, cudaMemcpyDeviceToHost));
    const unsigned long long* dbg = hd;
    for (int k = 0; k < 4; ++k) {
      std::fprintf(stderr, "gf2cl panel %d:", k);
      for (int ph = 1; ph < 8; ++ph)
        std::fprintf(stderr, " %lld", static_cast<long long>(dbg[k * 16 + ph] - dbg[k * 16 + ph - 1]));
      std::fprintf(stderr, " | clk %.0f MHz", double(dbg[k * 16 + 14] - dbg[k * 16 + 15]) * 1e3 /
                                              double(dbg[k * 16 + 7] - dbg[k * 16]));
      std::fprintf(stderr, " | total %lld ns\n",
                   static_cast<long long>(dbg[(k + 1) * 16] - dbg[k * 16]));
    }
  }
  return true;
}

}  // namespace gfq::dev
