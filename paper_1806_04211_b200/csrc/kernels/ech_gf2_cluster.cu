// ech_gf2_cluster.cu -- K2 for GF(2), cluster-resident: the whole
// bit-packed block [H | I] (rows <= 1024, cols + rows <= 8192) lives in the
// shared memory of ONE 8-CTA thread-block cluster (each CTA holds a stripe of
// <= 128 rows), and every exchange between CTAs goes through distributed
// shared memory with cluster barriers instead of global memory and grid
// barriers.  Right-looking Gauss-Jordan over 32-column panels with the
// reference's column-wise pivot rule (src/chief.cpp:436-460).
//
// The leader (CTA 0) finds a panel's pivots from the rows' panel words: warp
// 0 runs the chain on a 64-row window from the first non-pivotal row (the
// chosen row is the FIRST non-pivotal one with the bit, so a full-rank
// panel's pivots are all there), in column layout (lane q holds column q as
// a 64-bit row mask: a pivot step is one broadcast and one masked XOR per
// lane), tracking for every window row the set of pivots added to it.
// Gauss-Jordan, so a pivot row's set is its multiplier word G; any other
// row's G is the XOR, over the pivot columns set in its panel word, of that
// pivot's (own + set) -- evaluated by every CTA for its own rows from nibble
// tables.  A column without a window candidate sends the panel to a
// CTA-wide chain over all rows.
//
// Per panel k (one-panel look-ahead):
//   1. every CTA: G for its rows; pull the panel's pivot rows (DSMEM loads)
//      and build nibble tables of pivot-row combinations;  -- barrier Y
//   2. every CTA updates word k+1 of its rows and pushes it to the leader;
//      arrive Z; the leader's warp 0 waits on Z and factorizes panel k+1
//      while all other warps update the rest of their stripes (8 table
//      lookups a word); wait Z;
//   3. the leader publishes panel k+1's pivots to every CTA;  -- barrier X.
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
  // extraction mode (Out == nullptr): the reduced rows stay bit-packed
  // (P, Wd words a row) and the leader writes the index maps the extraction
  // kernel needs: sorted pivot rows (RS), row -> pivot index q or -(u+1)
  // for the u-th non-pivot row (QK), non-pivot columns (GC)
  std::uint32_t* P;
  std::int16_t *RS, *QK, *GC;
  int serial;  // developer experiment (GFQ_GF2_SERIAL): leader updates after its chain
};

// leader scratch of the extraction epilogue (pivot-column flags, bytes)
constexpr int kExBytes = 8192;

__device__ __forceinline__ unsigned long long gtime() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}

__device__ __forceinline__ void cl_arrive() {
  asm volatile("barrier.cluster.arrive.release.aligned;" ::: "memory");
}
__device__ __forceinline__ void cl_wait() {
  asm volatile("barrier.cluster.wait.acquire.aligned;" ::: "memory");
}

__global__ void __launch_bounds__(kThreads, 1) ech_gf2_cluster_kernel(ClArgs g) {
  extern __shared__ __align__(16) std::uint32_t sm[];
  const int Wd = g.Wd, rows = g.rows, cols = g.cols;
  std::uint32_t* A = sm;                        // kStripe x Wd   (my rows)
  std::uint32_t* bp = A + kStripe * Wd;         // 32 x Wd        (pivot rows of the panel)
  std::uint32_t* orig = bp + 32 * Wd;           // 1024           (leader: panel word per row)
  std::uint32_t* gl = orig + 1024;              // kStripe        (multiplier word per my row)
  std::uint8_t* fl = reinterpret_cast<std::uint8_t*>(gl + kStripe);   // 1024 (leader: pivotal)
  std::uint32_t* gall = reinterpret_cast<std::uint32_t*>(fl + 1024);  // 1024 (leader fallback)
  // 128 x Wd nibble tables (when Wd <= kTabWd), rows at an odd stride so the
  // look-ahead word's lookups (every thread the same word) spread over banks
  const int Ts = Wd + 1;
  std::uint32_t* tab = gall + 1024;
  const bool use_tab = Wd <= kTabWd;
  std::uint8_t* ex = reinterpret_cast<std::uint8_t*>(tab + (use_tab ? 128 * Ts : 0));
  std::uint8_t* ex_cf = ex;  // pivot-column flags (leader, extraction mode)
  // the current panel's pivots (the leader's copy is authoritative)
  __shared__ int pc[32], pr[32], r2_sh, ok_sh, lo_sh, npiv_sh;
  __shared__ std::uint32_t pcoef[32], ntab[128];
  __shared__ int colq[32], qof[kStripe];
  __shared__ std::uint32_t nomw[2][32], nomc[2][32];
  __shared__ unsigned best[3];

  cg::cluster_group cluster = cg::this_cluster();
  const int cr = int(cluster.block_rank());
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int row0 = cr * kStripe;
  const int nloc = rows - row0 < 0 ? 0 : (rows - row0 < kStripe ? rows - row0 : kStripe);
  std::uint32_t* lead_orig = cluster.map_shared_rank(orig, 0);
  const int npan = (cols + 31) / 32;
  auto pmask = [&](int k) {
    const int wc = cols - 32 * k < 32 ? cols - 32 * k : 32;
    return wc == 32 ? 0xFFFFFFFFu : ((1u << wc) - 1u);
  };
  auto stamp = [&](int k, int ph) {
    if (g.dbg && cr == 0 && tid == 0 && k >= 0 && k < 8) g.dbg[k * 16 + ph] = gtime();
  };

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
    if (tid == 0) {
      lo_sh = 0;
      npiv_sh = 0;
    }
  }
  cluster.sync();

  // ---- leader: pivots of panel k from `orig` (window chain in warp 0; the
  // caller falls back to full_chain when ok_sh == 0)
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
    stamp(k - 1, 9);
    // row layout: lane l holds window rows lo + l and lo + 32 + l as their
    // panel word w and coefficient word kk (bit q: pivot q's ORIGINAL row
    // has been added).  Per column: two ballots pick the first open row
    // with the bit, one shuffle pair broadcasts its (w, kk), and every other
    // window row with the bit adds it (kk ^= kk_s ^ e_q) -- no barriers, no
    // shared memory on the chain.
    const int i0 = lo + lane, i1 = lo + 32 + lane;
    std::uint32_t w0 = i0 < rows ? orig[i0] : 0u, w1 = i1 < rows ? orig[i1] : 0u;
    bool p0 = i0 >= rows || fl[i0] != 0, p1 = i1 >= rows || fl[i1] != 0;
    std::uint32_t k0 = 0, k1 = 0;
    const int open_in = __popc(__ballot_sync(0xffffffffu, !p0)) + __popc(__ballot_sync(0xffffffffu, !p1));
    // the window holds every non-pivotal row: a column without a candidate
    // is then a free column, not a reason to fall back
    const bool covers_all = open_in == rows - npiv_sh;
    stamp(k - 1, 10);
    const long long ck0 = clock64();
    int r2 = 0, ok = 1, q0 = -1, q1 = -1, mpc = 0, mpr = 0;
    const unsigned lanebit = 1u << lane;
#pragma unroll 1
    for (int c = 0; c < wc; ++c) {
      const unsigned b0 = __ballot_sync(0xffffffffu, !p0 && ((w0 >> c) & 1u));
      const unsigned b1 = __ballot_sync(0xffffffffu, !p1 && ((w1 >> c) & 1u));
      if (!(b0 | b1)) {
        if (covers_all) continue;
        ok = 0;
        break;
      }
      const bool hi = b0 == 0;
      const unsigned bb = hi ? b1 : b0;
      const int sl = __ffs(bb) - 1;
      const std::uint32_t pw = __shfl_sync(0xffffffffu, hi ? w1 : w0, sl);
      const std::uint32_t pk = __shfl_sync(0xffffffffu, hi ? k1 : k0, sl) ^ (1u << r2);
      // "am I the pivot lane" from the ballot's lowest bit (no lane id in the loop)
      const bool mine = (bb & (0u - bb) & lanebit) != 0;
      const bool me0 = !hi && mine, me1 = hi && mine;
      if (!me0 && ((w0 >> c) & 1u)) {
        w0 ^= pw;
        k0 ^= pk;
      }
      if (!me1 && ((w1 >> c) & 1u)) {
        w1 ^= pw;
        k1 ^= pk;
      }
      if (me0) {
        p0 = true;
        q0 = r2;
      }
      if (me1) {
        p1 = true;
        q1 = r2;
      }
      if ((lanebit >> r2) & 1u) {  // kept in registers: no shared stores on the chain
        mpc = c;
        mpr = lo + (hi ? 32 : 0) + sl;
      }
      ++r2;
    }
    if (lane < r2) {
      pc[lane] = mpc;
      pr[lane] = mpr;
    }
    __syncwarp();
    stamp(k - 1, 11);
    if (g.dbg && cr == 0 && tid == 0 && k >= 1 && k < 9) g.dbg[(k - 1) * 16 + 13] = clock64() - ck0;
    // a pivot row's multiplier word: its own bit plus the pivots added to it
    if (ok) {
      if (q0 >= 0) pcoef[q0] = k0 ^ (1u << q0);
      if (q1 >= 0) pcoef[q1] = k1 ^ (1u << q1);
    }
    __syncwarp();
    if (lane == 0) {
      ok_sh = ok;
      r2_sh = r2;
      lo_sh = lo;
    }
    stamp(k - 1, 12);
  };
  // CTA-wide chain over all rows (warps 0..7, 4 rows per lane); leader CTA,
  // every thread calls it
  auto full_chain = [&](int k) {
    const int wc = cols - 32 * k < 32 ? cols - 32 * k : 32;
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
      for (int s2 = 0; s2 < kRowsPerLane; ++s2) gall[256 * s2 + tid] = coef[s2];
      if (tid == 0) r2_sh = r2;
    }
    __syncthreads();
    if (tid < r2_sh) pcoef[tid] = gall[pr[tid]] ^ (1u << tid);
    __syncthreads();
  };
  // leader, every thread: record panel k's pivots and send them to CTAs 1..7
  auto publish = [&](int k, int rtot) {
    const int r2 = r2_sh;
    __syncthreads();
    if (tid == 0) npiv_sh = rtot + r2;
    if (tid < r2) {
      g.info[1 + rtot + tid] = 32 * k + pc[tid];
      g.info[1 + g.cap + rtot + tid] = pr[tid];
      fl[pr[tid]] = 1;
    }
    if (tid >= 32 && tid < kCl * 32) {
      const unsigned dst = unsigned(tid >> 5);
      const int q = tid & 31;
      if (q < r2) {
        *cluster.map_shared_rank(&pr[q], dst) = pr[q];
        *cluster.map_shared_rank(&pc[q], dst) = pc[q];
        *cluster.map_shared_rank(&pcoef[q], dst) = pcoef[q];
      }
      if (q == 0) *cluster.map_shared_rank(&r2_sh, dst) = r2;
    }
  };

  // ---- panel 0 pivots (no look-ahead yet)
  {
    const std::uint32_t pm = pmask(0);
    for (int li = tid; li < nloc; li += kThreads) lead_orig[row0 + li] = A[li * Wd] & pm;
  }
  cluster.sync();
  if (cr == 0) {
    if (warp == 0) window_chain(0);
    __syncthreads();
    if (!ok_sh) full_chain(0);
    __syncthreads();
    publish(0, 0);
  }
  cluster.sync();

  int rtot = 0;
  for (int k = 0; k < npan; ++k) {
    const int wi = k;
    const int r2 = r2_sh;
    const std::uint32_t pm = pmask(k);
    const bool has_next = k + 1 < npan;
    const int nw = Wd - wi;
    stamp(k, 0);
    // 1. G for my rows, pivot rows, tables
    if (r2 > 0) {
      // column -> pivot index of the panel, my row -> pivot index (O(1)
      // lookups below instead of loops over the r2 pivots)
      if (tid < 32) colq[tid] = -1;
      if (tid < kStripe) qof[tid] = -1;
      __syncthreads();
      if (tid < r2) {
        colq[pc[tid]] = tid;
        const int li = pr[tid] - row0;
        if (li >= 0 && li < kStripe) qof[li] = tid;
      }
      __syncthreads();
      if (tid < 128) {
        const int kq = tid >> 4, m = tid & 15;
        std::uint32_t v = 0;
#pragma unroll
        for (int b2 = 0; b2 < 4; ++b2) {
          const int q = colq[4 * kq + b2];
          if (((m >> b2) & 1) && q >= 0) v ^= pcoef[q];
        }
        ntab[tid] = v;
      }
      for (int e = tid; e < r2 * nw; e += kThreads) {
        const int q = e / nw, w = wi + e % nw;
        const int row = pr[q];
        bp[q * Wd + w] =
            *cluster.map_shared_rank(&A[(row % kStripe) * Wd + w], unsigned(row / kStripe));
      }
      __syncthreads();
      for (int li = tid; li < nloc; li += kThreads) {
        const std::uint32_t ow = A[li * Wd + wi] & pm;
        std::uint32_t gv = 0;
#pragma unroll
        for (int kq = 0; kq < 8; ++kq) gv ^= ntab[16 * kq + ((ow >> (4 * kq)) & 15u)];
        const int q = qof[li];
        if (q >= 0) gv = pcoef[q] ^ (1u << q);
        gl[li] = gv;
      }
      if (use_tab)
        for (int e = tid; e < 128 * nw; e += kThreads) {
          const int km = e / nw, w = wi + e % nw;
          const int kq = km >> 4, m = km & 15;
          std::uint32_t v = 0;
#pragma unroll
          for (int b2 = 0; b2 < 4; ++b2)
            if (((m >> b2) & 1) && 4 * kq + b2 < r2) v ^= bp[(4 * kq + b2) * Wd + w];
          tab[km * Ts + w] = v;
        }
      __syncthreads();
    }
    stamp(k, 1);
    cluster.sync();  // Y: every pull done before any stripe changes
    stamp(k, 2);

    // word w of my row li after this panel
    auto upd = [&](int li, int w) {
      const std::uint32_t gv = gl[li];
      std::uint32_t x = A[li * Wd + w];
      if (use_tab) {
#pragma unroll
        for (int kq = 0; kq < 8; ++kq) x ^= tab[(16 * kq + ((gv >> (4 * kq)) & 15u)) * Ts + w];
      } else {
        std::uint32_t gg = gv;
        while (gg) {
          const int q = __ffs(gg) - 1;
          gg &= gg - 1;
          x ^= bp[q * Wd + w];
        }
      }
      return x;
    };
    // 2. word k+1 first (the next panel's chain input), pushed to the leader
    if (has_next) {
      const std::uint32_t pmn = pmask(k + 1);
      for (int li = tid; li < nloc; li += kThreads) {
        const std::uint32_t x = r2 > 0 ? upd(li, wi + 1) : A[li * Wd + wi + 1];
        A[li * Wd + wi + 1] = x;
        lead_orig[row0 + li] = x & pmn;
      }
    }
    __syncthreads();
    cl_arrive();  // Z: my panel-(k+1) words are with the leader
    stamp(k, 3);
    const bool chain_warp = has_next && cr == 0 && warp == 0;
    if (chain_warp) {
      cl_wait();
      stamp(k, 8);
      window_chain(k + 1);
      stamp(k, 4);
    }
    if (g.serial && cr == 0 && has_next) __syncthreads();
    // the rest of panel k's update: word wi and words wi+2.. (the leader's
    // warp 0 is busy with the chain, so its rows go to warps 1..31)
    if (r2 > 0) {
      // in the leader the chain warp (warp 0, SMSP 0) would get one issue
      // slot in eight next to the other SMSP-0 warps, so SMSP 0's other
      // warps sit this phase out and warps on SMSPs 1-3 share the rows
      const bool lead = cr == 0 && has_next;
      const int nwarps = lead ? 24 : 32;
      const int widx = lead ? warp - (warp >> 2) - 1 : warp;
      if (!lead || (warp & 3) != 0)
        for (int li = widx; li < nloc; li += nwarps)
          for (int t = lane; t < nw; t += 32) {
            const int w = wi + t;
            if (has_next && w == wi + 1) continue;
            A[li * Wd + w] = upd(li, w);
          }
    }
    if (!chain_warp) cl_wait();
    stamp(k, 5);
    if (cr == 0 && has_next) {
      __syncthreads();
      if (!ok_sh) full_chain(k + 1);
      publish(k + 1, rtot + r2);
    }
    cluster.sync();  // X: panel k done everywhere, panel k+1's pivots published
    stamp(k, 6);
    rtot += r2;
    // every row pivotal: the remaining panels can hold no pivot and their
    // updates are empty (rtot is the same in every CTA)
    if (rtot >= rows) break;
  }

  if (g.dbg && cr == 0 && tid == 0) g.dbg[8 * 16 + 0] = gtime();
  if (g.Out) {
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
  } else {
    // ---- extraction, part 1 (reference src/jobs.cpp:104-121 conventions):
    // packed rows to global, and the leader's index maps
    for (int e = tid; e < nloc * Wd; e += kThreads)
      g.P[std::int64_t(row0 + e / Wd) * Wd + e % Wd] = A[e];
    const int r = rtot;
    if (cr == 0) {
      for (int c = tid; c < cols; c += kThreads) ex_cf[c] = 0;
      __syncthreads();
      for (int q = tid; q < r; q += kThreads) {
        ex_cf[g.info[1 + q]] = 1;
        g.QK[g.info[1 + g.cap + q]] = std::int16_t(q);
      }
      // rows: one per thread, block prefix of the pivot flags
      const int i = tid;
      const bool pv = i < rows && fl[i] != 0;
      const unsigned bal = __ballot_sync(0xffffffffu, pv);
      if (lane == 0) nomw[0][warp] = __popc(bal);
      __syncthreads();
      if (warp == 0) {
        std::uint32_t v = nomw[0][lane], x = v;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
          const std::uint32_t y = __shfl_up_sync(0xffffffffu, x, o);
          if (lane >= o) x += y;
        }
        nomc[0][lane] = x - v;  // exclusive prefix per warp
      }
      __syncthreads();
      const int before = int(nomc[0][warp]) + __popc(bal & ((1u << lane) - 1u));
      if (i < rows) {
        if (pv) g.RS[before] = std::int16_t(i);
        else g.QK[i] = std::int16_t(-(i - before) - 1);
      }
      // non-pivot columns: 8 per thread, block prefix of the counts
      int cnt = 0;
      for (int t = 0; t < 8; ++t) {
        const int c = 8 * tid + t;
        cnt += (c < cols && !ex_cf[c]) ? 1 : 0;
      }
      std::uint32_t x = std::uint32_t(cnt);
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const std::uint32_t y = __shfl_up_sync(0xffffffffu, x, o);
        if (lane >= o) x += y;
      }
      if (lane == 31) nomw[1][warp] = x;
      __syncthreads();
      if (warp == 0) {
        std::uint32_t v = nomw[1][lane], y2 = v;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
          const std::uint32_t z = __shfl_up_sync(0xffffffffu, y2, o);
          if (lane >= o) y2 += z;
        }
        nomc[1][lane] = y2 - v;
      }
      __syncthreads();
      int pos = int(nomc[1][warp] + x) - cnt;
      for (int t = 0; t < 8; ++t) {
        const int c = 8 * tid + t;
        if (c < cols && !ex_cf[c]) g.GC[pos++] = std::int16_t(c);
      }
    }
  }
  if (g.dbg && cr == 0 && tid == 0) g.dbg[8 * 16 + 1] = gtime();
  if (cr == 0 && tid == 0) g.info[0] = rtot;
  cluster.sync();  // no CTA may exit while others still address its shared memory
}

// Extraction, part 2: one block per row of the reduced packed [W | T].
// Row i with pivot index q writes M row q (T bits at the sorted pivot rows)
// and R row q (W bits at the non-pivot columns); the u-th non-pivot row
// writes K row u.
__global__ void __launch_bounds__(128) gf2_extract_kernel(int rows, int cols, int Wd,
                                                          const std::uint32_t* P,
                                                          const std::int32_t* info, int cap,
                                                          const std::int16_t* RS,
                                                          const std::int16_t* QK,
                                                          const std::int16_t* GC, EchExtract ex) {
  (void)cap;
  const int i = blockIdx.x;
  const int r = info[0];
  const std::uint32_t* prow = P + std::int64_t(i) * Wd;
  auto bit = [&](int pos) { return std::uint8_t((prow[pos >> 5] >> (pos & 31)) & 1u); };
  const int qk = QK[i];
  if (qk >= 0) {
    std::uint8_t* m = ex.M + std::int64_t(qk) * ex.ldm;
    for (int t = threadIdx.x; t < r; t += blockDim.x) m[t] = bit(cols + RS[t]);
    std::uint8_t* rr = ex.R + std::int64_t(qk) * ex.ldr;
    for (int t = threadIdx.x; t < cols - r; t += blockDim.x) rr[t] = bit(GC[t]);
  } else {
    std::uint8_t* k = ex.K + std::int64_t(-qk - 1) * ex.ldk;
    for (int t = threadIdx.x; t < r; t += blockDim.x) k[t] = bit(cols + RS[t]);
  }
}

}  // namespace

bool ech_gf2_cluster(std::int64_t rows, std::int64_t cols, const std::uint8_t* H, std::int64_t ldh,
                     std::uint8_t* Out, std::int64_t ldo, std::int32_t* info, std::int64_t cap,
                     cudaStream_t s, const EchExtract* ex) {
  static const bool off = std::getenv("GFQ_NO_GF2_CLUSTER") != nullptr;
  const std::int64_t Wd = (cols + rows + 31) / 32;
  if (off || rows > kCl * kStripe || Wd > kMaxWd || rows <= 0 || cols <= 0) return false;
  const std::size_t smem =
      std::size_t(kStripe * Wd + 32 * Wd + 1024 + kStripe) * 4 + 1024 + 4096 +
      (Wd <= kTabWd ? std::size_t(128 * (Wd + 1)) * 4 : 0) + kExBytes;
  static bool attr = false;
  if (!attr) {
    GFQ_CUDA(cudaFuncSetAttribute(ech_gf2_cluster_kernel,
                                  cudaFuncAttributeMaxDynamicSharedMemorySize,
                                  int(std::max(std::size_t(kStripe * kMaxWd + 32 * kMaxWd + 1024 + kStripe) * 4 + 1024 + 4096,
                                               std::size_t(kStripe * kTabWd + 32 * kTabWd + 1024 + kStripe) * 4 +
                                                   1024 + 4096 + std::size_t(128 * (kTabWd + 1)) * 4) +
                                      kExBytes)));
    attr = true;
  }
  // algorithmic bytes: H read, M / K / R written (rank taken as min(rows, cols))
  const double rk = double(std::min(rows, cols));
  ProfScope ps(kProfEchGf2, double(rows) * double(cols) + rk * (double(rows) + double(cols) - rk), s);
  static const bool debug = std::getenv("GFQ_GF2_DEBUG") != nullptr;
  static unsigned long long* dbg = nullptr;
  if (debug && !dbg) GFQ_CUDA(cudaMalloc(&dbg, 9 * 16 * sizeof(unsigned long long)));
  ClArgs g{int(rows), int(cols), int(Wd), int(cap), H, ldh, Out, ldo, info, debug ? dbg : nullptr,
            ex ? ex->P : nullptr, ex ? ex->RS : nullptr, ex ? ex->QK : nullptr,
            ex ? ex->GC : nullptr, std::getenv("GFQ_GF2_SERIAL") ? 1 : 0};
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
  if (ex) {
    gf2_extract_kernel<<<unsigned(rows), 128, 0, s>>>(int(rows), int(cols), int(Wd), ex->P, info,
                                                       int(cap), ex->RS, ex->QK, ex->GC, *ex);
    GFQ_CUDA(cudaGetLastError());
    count_launch();
  }
  if (debug) {
    GFQ_CUDA(cudaStreamSynchronize(s));
    unsigned long long hd[9 * 16];
    GFQ_CUDA(cudaMemcpy(hd, dbg, sizeof hd, cudaMemcpyDeviceToHost));
    const unsigned long long* dbg = hd;
    std::fprintf(stderr, "gf2cl rows %lld cols %lld Wd %lld epilogue %lld ns\n", static_cast<long long>(rows),
                 static_cast<long long>(cols), static_cast<long long>(Wd),
                 static_cast<long long>(hd[8 * 16 + 1] - hd[8 * 16]));
    for (int k = 0; k < 4 && k < (cols + 31) / 32; ++k) {
      std::fprintf(stderr, "gf2cl panel %d:", k);
      for (int ph = 1; ph < 7; ++ph)
        std::fprintf(stderr, " %lld", static_cast<long long>(dbg[k * 16 + ph] - dbg[k * 16 + ph - 1]));

      std::fprintf(stderr, " | zwait %lld chain %lld", static_cast<long long>(dbg[k * 16 + 8] - dbg[k * 16 + 3]),
                   static_cast<long long>(dbg[k * 16 + 4] - dbg[k * 16 + 8]));
      std::fprintf(stderr, " | rounds %lld cyc", static_cast<long long>(dbg[k * 16 + 13]));
      std::fprintf(stderr, " | scan %lld masks %lld rounds %lld coef %lld",
                   static_cast<long long>(dbg[k * 16 + 9] - dbg[k * 16 + 8]),
                   static_cast<long long>(dbg[k * 16 + 10] - dbg[k * 16 + 9]),
                   static_cast<long long>(dbg[k * 16 + 11] - dbg[k * 16 + 10]),
                   static_cast<long long>(dbg[k * 16 + 12] - dbg[k * 16 + 11]));
      std::fprintf(stderr, " | total %lld ns\n",
                   static_cast<long long>(dbg[(k + 1) * 16] - dbg[k * 16]));
    }
  }
  return true;
}

}  // namespace gfq::dev

// ---------------------------------------------------------------- few rows
// GF(2) ECH of a block with at most 32 rows (the ClearDowns of a block row
// that has all but a few of its pivots already): one warp, one row per lane,
// the bit-packed [W | T] rows in shared memory; column by column, the first
// non-pivotal row with the bit is the pivot and every other row with the bit
// adds it (Gauss-Jordan); the loop stops once every row is pivotal.  Writes
// info and the EchResult blocks like the extraction mode above.
namespace gfq::dev {
namespace {

__global__ void __launch_bounds__(32) ech_gf2_small_kernel(int rows, int cols, const std::uint8_t* H,
                                                           std::int64_t ldh, std::int32_t* info,
                                                           int cap, EchExtract ex) {
  extern __shared__ std::uint32_t sw[];
  const int lane = threadIdx.x;
  const int Wd = (cols + rows + 31) / 32, st = Wd + 1;  // padded row stride: no bank conflicts
  std::uint32_t* row = sw + lane * st;
  std::uint8_t* colpiv = reinterpret_cast<std::uint8_t*>(sw + 32 * st);  // cols bytes
  __shared__ int pc[32], pr[32];
  // pack [H | I] warp-cooperatively: lane w builds word w of each row from
  // 32 consecutive bytes (coalesced 16-byte loads when aligned)
  const bool vec = (reinterpret_cast<std::uintptr_t>(H) & 15) == 0 && (ldh & 15) == 0;
  for (int i = 0; i < rows; ++i) {
    const std::uint8_t* h = H + std::int64_t(i) * ldh;
    for (int w = lane; w < Wd; w += 32) {
      std::uint32_t word = 0;
      const int j0 = 32 * w;
      if (vec && j0 + 32 <= cols) {
        const uint4 a = reinterpret_cast<const uint4*>(h + j0)[0], b = reinterpret_cast<const uint4*>(h + j0)[1];
        const std::uint32_t v[8] = {a.x, a.y, a.z, a.w, b.x, b.y, b.z, b.w};
#pragma unroll
        for (int q = 0; q < 8; ++q) {
          const std::uint32_t x = v[q] & 0x01010101u;  // one bit per byte
          word |= ((x & 1u) | ((x >> 7) & 2u) | ((x >> 14) & 4u) | ((x >> 21) & 8u)) << (4 * q);
        }
      } else {
        for (int b = 0; b < 32; ++b) {
          const int j = j0 + b;
          if (j < cols) word |= std::uint32_t(h[j] & 1u) << b;
        }
      }
      if (j0 <= cols + i && cols + i < j0 + 32) word |= 1u << (cols + i - j0);
      sw[i * st + w] = word;
    }
  }
  for (int c = lane; c < cols; c += 32) colpiv[c] = 0;
  __syncwarp();
  bool piv = lane >= rows;
  int r = 0;
  for (int c = 0; c < cols; ++c) {
    const unsigned open = __ballot_sync(0xffffffffu, !piv);
    if (!open) break;
    const bool has = lane < rows && ((row[c >> 5] >> (c & 31)) & 1u);
    const unsigned cand = __ballot_sync(0xffffffffu, has && !piv);
    if (!cand) continue;
    const int p = __ffs(cand) - 1;
    const std::uint32_t* prow = sw + p * st;
    if (has && lane != p)
      for (int w = c >> 5; w < Wd; ++w) row[w] ^= prow[w];
    __syncwarp();
    if (lane == p) piv = true;
    if (lane == 0) {
      pc[r] = c;
      pr[r] = p;
      colpiv[c] = 1;
    }
    ++r;
  }
  __syncwarp();
  if (lane < r) {
    info[1 + lane] = pc[lane];
    info[1 + cap + lane] = pr[lane];
  }
  if (lane == 0) info[0] = r;
  // sorted pivot rows (= pivotal lanes in order) and each row's output index
  const unsigned pivmask = __ballot_sync(0xffffffffu, lane < rows && piv);
  int q = -1;
  for (int t = 0; t < r; ++t)
    if (pr[t] == lane) q = t;
  const int below = __popc(pivmask & ((1u << lane) - 1u));  // pivot rows before me
  // M / K rows: the T columns at the sorted pivot rows
  if (lane < rows) {
    std::uint8_t* out = q >= 0 ? ex.M + std::int64_t(q) * ex.ldm : ex.K + std::int64_t(lane - below) * ex.ldk;
    unsigned m = pivmask;
    for (int s = 0; s < r; ++s) {
      const int pos = cols + (__ffs(m) - 1);
      m &= m - 1;
      out[s] = std::uint8_t((row[pos >> 5] >> (pos & 31)) & 1u);
    }
  }
  // R rows (the non-pivot columns of the pivot rows), warp-cooperatively:
  // column c goes to position c - #(pivot columns < c); pc is increasing
  __syncwarp();
  for (int t2 = 0; t2 < r; ++t2) {
    const int prw = pr[t2];
    const std::uint32_t* src = sw + prw * st;
    std::uint8_t* rr = ex.R + std::int64_t(t2) * ex.ldr;
    int below_c = 0;  // pivot columns < c (c increases, so it only advances)
    for (int c = lane; c < cols; c += 32) {
      while (below_c < r && pc[below_c] < c) ++below_c;
      if (colpiv[c]) continue;
      rr[c - below_c] = std::uint8_t((src[c >> 5] >> (c & 31)) & 1u);
    }
  }
}

}  // namespace

bool ech_gf2_small(std::int64_t rows, std::int64_t cols, const std::uint8_t* H, std::int64_t ldh,
                   std::int32_t* info, std::int64_t cap, cudaStream_t s, const EchExtract& ex) {
  if (rows < 1 || rows > 32 || cols < 1) return false;
  const std::int64_t Wd = (cols + rows + 31) / 32;
  const std::size_t smem = std::size_t(32 * (Wd + 1)) * 4 + std::size_t(cols) + 16;
  if (smem > 200 * 1024) return false;
  static bool attr = false;
  if (!attr) {
    GFQ_CUDA(cudaFuncSetAttribute(ech_gf2_small_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                  200 * 1024));
    attr = true;
  }
  const double rk = double(std::min(rows, cols));
  ProfScope ps(kProfEchGf2, double(rows) * double(cols) + rk * (double(rows) + double(cols) - rk), s);
  ech_gf2_small_kernel<<<1, 32, smem, s>>>(int(rows), int(cols), H, ldh, info, int(cap), ex);
  GFQ_CUDA(cudaGetLastError());
  count_launch();
  return true;
}

}  // namespace gfq::dev
