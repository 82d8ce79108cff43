// ech_gf2_outer.cu -- K2 for tall GF(2) blocks: one outer panel of the
// two-level device ECH (jobs.cpp panel_ech) in ONE cluster launch.
//
// The two-level ECH keeps Aug = [W | T] in HBM and eliminates it in outer
// panels of `ow` columns: the panel is copied into the scratch Z = [X | Y]
// (Y zero), eliminated there, and the rest of Aug then gets one deep-K
// contraction on the tensor cores.  For GF(2) the elimination of the panel
// (the column-wise pivot rule of src/chief.cpp:436-460 over up to 8192 rows,
// Gauss-Jordan, the outer row operator tracked in Y) runs here with the whole
// bit-packed [X | Y] (rows x 2 ow bits: 75 KB per CTA at 8192 rows and
// ow = 256) resident in the distributed shared memory of one 8-CTA cluster,
// CTA c >= 1 holding rows [(c-1) S, c S), S = ceil(rows / 7); the leader
// CTA 0 holds the pivot search state.  Per 32-column
// sub-panel k (one-panel look-ahead, as in ech_gf2_cluster.cu):
//   1. every CTA pulls the sub-panel's pivot rows from their owners over
//      DSMEM, plants each pivot's tracking unit Y[p, slot] in its copies,
//      computes every own row's multiplier word G from nibble tables of the
//      pivots' coefficient words, and builds nibble tables of pivot-row
//      combinations;                                         -- barrier
//   2. word k+1 of every row is updated first and pushed to the leader,
//      whose warp 0 runs the pivot chain of sub-panel k+1 while every other
//      warp finishes sub-panel k's update (8 table lookups a word); the
//      leader then publishes the pivots.                     -- barrier
// The chain runs on a 64-row window from the first non-pivotal row; a
// column with no window candidate scans the rows below the window (each
// row's word brought up to date by replaying the sub-panel's pivots so far)
// for the first one with the bit -- a "far" pivot, tracked in the lane of its
// pivot number for the rest of the chain -- so no column ever needs a
// CTA-wide chain over all rows.
//
// Contract (the same state the 32-wide ech_step launches leave):
// Z[:, 0:wd] = X, Z[:, ow:2 ow] = Y (zero on entry; Y[p, g - base] = 1 for
// the g-th pivot, then carried by the row operations); flags[i] = 1 for
// pivotal rows; info = [rank, cols[cap], rows[cap]] with the new pivots
// appended (columns panel-local, ech_outer_finish shifts them by the panel's
// first column) and info[0] advanced; *base = rank at the outer panel's start.
#include <cooperative_groups.h>

#include <algorithm>
#include <cstdio>
#include <cstdlib>

#include "../common.hpp"
#include "kernels.hpp"

namespace gfq::dev {
namespace {

namespace cg = cooperative_groups;

constexpr int kOCl = 8;          // CTAs per cluster
constexpr int kOThreads = 1024;  // 32 warps per CTA
constexpr int kORowsMax = 8192;  // rows <= 8 x 1024

struct OuterArgs {
  int rows, wd, ow;  // rows, panel columns (<= ow), outer width (256 or 512)
  std::uint8_t* Z;
  std::int64_t ldz;
  std::uint8_t* flags;
  std::int32_t* info;
  int cap;
  unsigned long long* dbg;  // developer phase stamps (GFQ_GF2_DEBUG): leader, per sub-panel
};
__device__ __forceinline__ unsigned long long gtime_o() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}

__device__ __forceinline__ void cl_arrive_o() {
  asm volatile("barrier.cluster.arrive.release.aligned;" ::: "memory");
}
__device__ __forceinline__ void cl_wait_o() {
  asm volatile("barrier.cluster.wait.acquire.aligned;" ::: "memory");
}

__global__ void __launch_bounds__(kOThreads, 1) ech_gf2_outer_kernel(OuterArgs g) {
  extern __shared__ __align__(16) std::uint32_t sm[];
  const int rows = g.rows, Xw = g.ow / 32, Wd = 2 * Xw;
  // the leader (CTA 0) holds no rows: its warp 0 runs the pivot chain while
  // the other CTAs update, and shuffles share the shared-memory pipe with
  // table lookups -- a leader updating rows of its own doubles the chain
  const int S = (rows + kOCl - 2) / (kOCl - 1);
  // table rows padded to an odd stride: the 16 entries of a nibble group hit
  // 16 different banks when every thread looks up the same word (stride Wd,
  // a multiple of 16, put them on two banks)
  const int Ts = Wd + 1;
  std::uint32_t* A = sm;                     // S x Wd       (my rows)
  std::uint32_t* bp = A + S * Wd;            // 32 x Wd      (the sub-panel's pivot rows)
  std::uint32_t* tab = bp + 32 * Wd;         // 128 x Wd     (nibble tables)
  std::uint32_t* gl = tab + 128 * Ts;        // S            (multiplier word of my rows)
  int* qof = reinterpret_cast<int*>(gl + S); // S            (my row -> pivot index, -1)
  std::uint32_t* orig = reinterpret_cast<std::uint32_t*>(qof + S);  // rows (leader: sub-panel words)
  std::uint8_t* fl = reinterpret_cast<std::uint8_t*>(orig + rows);   // rows (leader: pivotal)
  __shared__ int pc[32], pr[32], colq[32];
  __shared__ std::uint32_t pcoef[32], ntab[128];
  __shared__ int spc[32];
  __shared__ std::uint32_t spw[32], spk[32];
  __shared__ int r2_sh, lo_sh, npiv_sh, rbase_sh;

  cg::cluster_group cluster = cg::this_cluster();
  const int cr = int(cluster.block_rank());
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int row0 = cr == 0 ? 0 : (cr - 1) * S;
  const int nloc = cr == 0 ? 0 : (rows - row0 < 0 ? 0 : (rows - row0 < S ? rows - row0 : S));
  std::uint32_t* lead_orig = cluster.map_shared_rank(orig, 0);
  const int npan = (g.wd + 31) / 32;
  auto pmask = [&](int k) {
    const int wc = g.wd - 32 * k < 32 ? g.wd - 32 * k : 32;
    return wc == 32 ? 0xFFFFFFFFu : ((1u << wc) - 1u);
  };
  auto stamp = [&](int slot) {
    if (g.dbg && cr == 0 && tid == 0 && slot < 256) g.dbg[slot] = gtime_o();
  };
  auto cstamp = [&](int slot) {  // chain warp
    if (g.dbg && cr == 0 && lane == 0 && slot < 256) g.dbg[slot] = gtime_o();
  };
  stamp(0);

  // ---- pack my rows: X words from Z, Y words zero
  for (int e = tid; e < nloc * Wd; e += kOThreads) {
    const int li = e / Wd, w = e - li * Wd;
    std::uint32_t word = 0;
    if (w < Xw) {
      const std::uint8_t* z = g.Z + std::int64_t(row0 + li) * g.ldz + 32 * w;
      const int j0 = 32 * w;
      if (j0 + 32 <= g.wd && (reinterpret_cast<std::uintptr_t>(z) & 15) == 0) {
        const uint4 a = reinterpret_cast<const uint4*>(z)[0];
        const uint4 b = reinterpret_cast<const uint4*>(z)[1];
        const std::uint32_t wds[8] = {a.x, a.y, a.z, a.w, b.x, b.y, b.z, b.w};
#pragma unroll
        for (int q = 0; q < 8; ++q) {
          const std::uint32_t v = wds[q] & 0x01010101u;
          word |= ((v & 1u) | ((v >> 7) & 2u) | ((v >> 14) & 4u) | ((v >> 21) & 8u)) << (4 * q);
        }
      } else {
        for (int b = 0; b < 32 && j0 + b < g.wd; ++b) word |= std::uint32_t(z[b] & 1u) << b;
      }
    }
    A[e] = word;
  }
  if (cr == 0) {
    for (int i = tid; i < rows; i += kOThreads) fl[i] = g.flags[i];
    if (tid == 0) {
      lo_sh = 0;
      npiv_sh = g.info[0];
      rbase_sh = g.info[0];
    }
  }
  cluster.sync();
  stamp(1);

  // ---- leader warp 0: pivots of sub-panel k from `orig`
  auto window_chain = [&](int k) {
    const int wc = g.wd - 32 * k < 32 ? g.wd - 32 * k : 32;
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
    std::uint32_t w0 = i0 < rows ? orig[i0] : 0u, w1 = i1 < rows ? orig[i1] : 0u;
    bool p0 = i0 >= rows || fl[i0] != 0, p1 = i1 >= rows || fl[i1] != 0;
    std::uint32_t k0 = 0, k1 = 0;
    const unsigned open0 = __ballot_sync(0xffffffffu, !p0), open1 = __ballot_sync(0xffffffffu, !p1);
    const bool covers_all = __popc(open0) + __popc(open1) == rows - npiv_sh;
    int r2 = 0, q0 = -1, q1 = -1, mpc = 0, mpr = 0;
    const unsigned lanebit = 1u << lane;
    const long long ck0 = clock64();
    int nfar = 0;
    // ---- fast path, column layout: lane c holds column c of the window as
    // a 64-bit row mask (cm) and lane q the rows whose coefficient word has
    // pivot q (km).  A pivot step: broadcast column c's mask, the first open
    // row is the pivot p, every row of the mask but p adds row p (a lane
    // flips its mask by them iff row p has its bit) -- one 64-bit shuffle
    // and a few ALU operations a column.
    std::uint64_t cm = 0, km = 0;
    for (int i = 0; i < 32; ++i) {
      const unsigned blo = __ballot_sync(0xffffffffu, (w0 >> i) & 1u);
      const unsigned bhi = __ballot_sync(0xffffffffu, (w1 >> i) & 1u);
      if (lane == i) cm = std::uint64_t(blo) | (std::uint64_t(bhi) << 32);
    }
    std::uint64_t openm = std::uint64_t(open0) | (std::uint64_t(open1) << 32);
    int myslot = -1;  // window slot of pivot number lane
    int c = 0;
#pragma unroll 1
    for (; c < wc; ++c) {
      const std::uint64_t M = __shfl_sync(0xffffffffu, cm, c);
      const std::uint64_t cand = M & openm;
      if (cand == 0) {
        if (covers_all) continue;
        break;  // no window candidate: the row-layout path below takes over
      }
      const int pidx = __ffsll(static_cast<long long>(cand)) - 1;
      const std::uint64_t pbit = std::uint64_t(1) << pidx;
      const std::uint64_t R = M & ~pbit;
      if (cm & pbit) cm ^= R;
      if (km & pbit) km ^= R;
      if (lane == r2) {
        km ^= R;
        myslot = pidx;
        mpc = c;
        mpr = lo + pidx;
      }
      openm &= ~pbit;
      ++r2;
    }
    if (c < wc) {
      // ---- slow path (a column without a window candidate): back to row
      // layout -- row i's word is bit i of every lane's column mask, its
      // coefficient bit i of every lane's km -- and continue with far pivots
      for (int i = 0; i < 64; ++i) {
        const unsigned bw = __ballot_sync(0xffffffffu, (cm >> i) & 1u);
        const unsigned bk = __ballot_sync(0xffffffffu, (km >> i) & 1u);
        if (i == lane) {
          w0 = bw;
          k0 = bk;
        }
        if (i == lane + 32) {
          w1 = bw;
          k1 = bk;
        }
      }
      // pivot numbers of the window rows chosen so far
      for (int q = 0; q < r2; ++q) {
        const int sl = __shfl_sync(0xffffffffu, myslot, q);
        if (sl == lane) {
          p0 = true;
          q0 = q;
        }
        if (sl == lane + 32) {
          p1 = true;
          q1 = q;
        }
      }
      bool fv = false;  // this lane's pivot (number == lane) is a far row
      std::uint32_t fw = 0, fk = 0;
#pragma unroll 1
      for (; c < wc; ++c) {
        const unsigned b0 = __ballot_sync(0xffffffffu, !p0 && ((w0 >> c) & 1u));
        const unsigned b1 = __ballot_sync(0xffffffffu, !p1 && ((w1 >> c) & 1u));
        std::uint32_t pw, pk;
        bool me0 = false, me1 = false;
        if (b0 | b1) {
          const bool hi = b0 == 0;
          const unsigned bb = hi ? b1 : b0;
          const int sl = __ffs(bb) - 1;
          pw = __shfl_sync(0xffffffffu, hi ? w1 : w0, sl);
          pk = __shfl_sync(0xffffffffu, hi ? k1 : k0, sl) ^ (1u << r2);
          const bool mine = (bb & (0u - bb) & lanebit) != 0;
          me0 = !hi && mine;
          me1 = hi && mine;
          if ((lanebit >> r2) & 1u) {
            mpc = c;
            mpr = lo + (hi ? 32 : 0) + sl;
          }
        } else {
          if (covers_all) continue;
          // far scan: the pivot rows' CURRENT words and coefficients (they
          // are reduced among themselves, so a row's word is its original
          // word plus the current pivot rows of the pivot columns it has)
          ++nfar;
          if (q0 >= 0) {
            spc[q0] = 0;
            spw[q0] = w0;
            spk[q0] = k0 ^ (1u << q0);
          }
          if (q1 >= 0) {
            spw[q1] = w1;
            spk[q1] = k1 ^ (1u << q1);
          }
          if (fv) {
            spw[lane] = fw;
            spk[lane] = fk ^ lanebit;
          }
          if (lane < r2) spc[lane] = mpc;
          __syncwarp();
          int found = -1;
          std::uint32_t fwv = 0, fkv = 0;
          for (int jb = lo + 64; jb < rows && found < 0; jb += 32) {
            const int j = jb + lane;
            std::uint32_t w = 0, kk = 0;
            bool hit = false;
            if (j < rows && fl[j] == 0) {
              const std::uint32_t o = orig[j];
              w = o;
              for (int q = 0; q < r2; ++q)
                if ((o >> spc[q]) & 1u) {
                  w ^= spw[q];
                  kk ^= spk[q];
                }
              hit = (w >> c) & 1u;
            }
            const unsigned hb = __ballot_sync(0xffffffffu, hit);
            if (hb) {
              const int sl = __ffs(hb) - 1;
              found = jb + sl;
              fwv = __shfl_sync(0xffffffffu, w, sl);
              fkv = __shfl_sync(0xffffffffu, kk, sl);
            }
          }
          __syncwarp();
          if (found < 0) continue;  // no pivot in column c
          pw = fwv;
          pk = fkv ^ (1u << r2);
          if (lane == r2) {
            fv = true;
            fw = fwv;
            fk = fkv;
            mpc = c;
            mpr = found;
            fl[found] = 1;  // below the window: no window flag depends on it
          }
        }
        // every other row with the bit adds the pivot (window rows, earlier
        // far pivots; the far pivot itself just became lane r2's)
        if (!me0 && ((w0 >> c) & 1u)) {
          w0 ^= pw;
          k0 ^= pk;
        }
        if (!me1 && ((w1 >> c) & 1u)) {
          w1 ^= pw;
          k1 ^= pk;
        }
        if (fv && lane != r2 && ((fw >> c) & 1u)) {
          fw ^= pw;
          fk ^= pk;
        }
        if (me0) {
          p0 = true;
          q0 = r2;
        }
        if (me1) {
          p1 = true;
          q1 = r2;
        }
        ++r2;
      }
      if (q0 >= 0) pcoef[q0] = k0 ^ (1u << q0);
      if (q1 >= 0) pcoef[q1] = k1 ^ (1u << q1);
      if (fv) pcoef[lane] = fk ^ lanebit;
    } else {
      // a pivot row's multiplier word: its own bit plus the pivots added to
      // it -- bit q' of row p's coefficient is bit p of lane q''s km
      for (int q = 0; q < r2; ++q) {
        const int sl = __shfl_sync(0xffffffffu, myslot, q);
        const unsigned b = __ballot_sync(0xffffffffu, (km >> sl) & 1u);
        if (lane == 0) pcoef[q] = b ^ (1u << q);
      }
    }
    if (g.dbg && lane == 0 && k < 8) {
      g.dbg[200 + k] = clock64() - ck0;
      g.dbg[220 + k] = nfar;
    }
    if (lane < r2) {
      pc[lane] = mpc;
      pr[lane] = mpr;
    }
    __syncwarp();
    if (lane == 0) {
      r2_sh = r2;
      lo_sh = lo;
    }
  };
  // leader, every thread: record sub-panel k's pivots and send them to CTAs 1..7
  auto publish = [&](int k, int rtot) {
    const int r2 = r2_sh;
    __syncthreads();
    const int rb = rbase_sh;
    if (tid == 0) npiv_sh = rb + rtot + r2;
    if (tid < r2) {
      g.info[1 + rb + rtot + tid] = 32 * k + pc[tid];
      g.info[1 + g.cap + rb + rtot + tid] = pr[tid];
      g.flags[pr[tid]] = 1;
      fl[pr[tid]] = 1;
    }
    if (tid >= 32 && tid < kOCl * 32) {
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

  // ---- sub-panel 0's pivots (no look-ahead yet)
  {
    const std::uint32_t pm = pmask(0);
    for (int li = tid; li < nloc; li += kOThreads) lead_orig[row0 + li] = A[li * Wd] & pm;
  }
  cluster.sync();
  if (cr == 0) {
    if (warp == 0) window_chain(0);
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
    stamp(8 + 8 * k);
    // 1. G for my rows, the pivot rows (with their planted units), tables
    if (r2 > 0) {
      if (tid < 32) colq[tid] = -1;
      for (int li = tid; li < S; li += kOThreads) qof[li] = -1;
      __syncthreads();
      if (tid < r2) {
        colq[pc[tid]] = tid;
        const int li = pr[tid] - row0;
        if (li >= 0 && li < S) qof[li] = tid;
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
      for (int e = tid; e < r2 * nw; e += kOThreads) {
        const int q = e / nw, w = wi + e % nw;
        const int row = pr[q];
        std::uint32_t x = *cluster.map_shared_rank(&A[(row % S) * Wd + w], unsigned(row / S + 1));
        const int slot = rtot + q;  // the pivot's tracking unit Y[row, slot]
        if (w == Xw + (slot >> 5)) x |= 1u << (slot & 31);
        bp[q * Wd + w] = x;
      }
      __syncthreads();
      for (int li = tid; li < nloc; li += kOThreads) {
        const std::uint32_t ow = A[li * Wd + wi] & pm;
        std::uint32_t gv = 0;
#pragma unroll
        for (int kq = 0; kq < 8; ++kq) gv ^= ntab[16 * kq + ((ow >> (4 * kq)) & 15u)];
        const int q = qof[li];
        if (q >= 0) gv = pcoef[q] ^ (1u << q);
        gl[li] = gv;
      }
      for (int e = tid; e < 128 * nw; e += kOThreads) {
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
    stamp(9 + 8 * k);
    cluster.sync();  // every pull done before any stripe changes
    stamp(10 + 8 * k);

    // word w of my row li after this sub-panel
    auto upd = [&](int li, int w) {
      const std::uint32_t gv = gl[li];
      std::uint32_t x = A[li * Wd + w];
#pragma unroll
      for (int kq = 0; kq < 8; ++kq) x ^= tab[(16 * kq + ((gv >> (4 * kq)) & 15u)) * Ts + w];
      const int q = qof[li];
      if (q >= 0 && w == Xw + ((rtot + q) >> 5)) x ^= 1u << ((rtot + q) & 31);  // own unit
      return x;
    };
    // 2. word k+1 first (the next sub-panel's chain input), pushed to the leader
    if (has_next) {
      const std::uint32_t pmn = pmask(k + 1);
      for (int li = tid; li < nloc; li += kOThreads) {
        const std::uint32_t x = r2 > 0 ? upd(li, wi + 1) : A[li * Wd + wi + 1];
        A[li * Wd + wi + 1] = x;
        lead_orig[row0 + li] = x & pmn;
      }
    }
    __syncthreads();
    cl_arrive_o();
    const bool chain_warp = has_next && cr == 0 && warp == 0;
    stamp(11 + 8 * k);
    if (chain_warp) {
      cl_wait_o();
      cstamp(12 + 8 * k);
      window_chain(k + 1);
      cstamp(13 + 8 * k);
    }
    if (r2 > 0) {
      // the leader's SMSP-0 warps sit out while warp 0 runs the chain
      const bool lead = cr == 0 && has_next;
      const int nthr = lead ? 768 : kOThreads;
      const int t0 = lead ? (warp - (warp >> 2) - 1) * 32 + lane : tid;
      if (!lead || (warp & 3) != 0)
        for (int e = t0; e < nloc * nw; e += nthr) {
          const int li = e / nw, w = wi + e % nw;
          if (has_next && w == wi + 1) continue;
          A[li * Wd + w] = upd(li, w);
        }
    }
    stamp(14 + 8 * k);
    if (!chain_warp) cl_wait_o();
    if (cr == 0 && has_next) {
      __syncthreads();
      publish(k + 1, rtot + r2);
    }
    cluster.sync();  // sub-panel k done everywhere, k+1's pivots published
    rtot += r2;
  }

  stamp(2);
  // ---- unpack my rows: X to Z[:, 0:ow], Y to Z[:, ow:2 ow]
  for (int e = tid; e < nloc * Wd; e += kOThreads) {
    const int li = e / Wd, w = e - li * Wd;
    const std::uint32_t word = A[e];
    std::uint8_t* orow = g.Z + std::int64_t(row0 + li) * g.ldz + 32 * w;
    if ((reinterpret_cast<std::uintptr_t>(orow) & 15) == 0) {
      std::uint32_t outw[8];
#pragma unroll
      for (int q = 0; q < 8; ++q) {
        const std::uint32_t nib = (word >> (4 * q)) & 0xFu;
        outw[q] = (nib & 1u) | ((nib & 2u) << 7) | ((nib & 4u) << 14) | ((nib & 8u) << 21);
      }
      reinterpret_cast<uint4*>(orow)[0] = make_uint4(outw[0], outw[1], outw[2], outw[3]);
      reinterpret_cast<uint4*>(orow)[1] = make_uint4(outw[4], outw[5], outw[6], outw[7]);
    } else {
      for (int b = 0; b < 32; ++b) orow[b] = (word >> b) & 1u;
    }
  }
  if (cr == 0 && tid == 0) g.info[0] = rbase_sh + rtot;
  stamp(3);
  cluster.sync();  // no CTA may exit while others still address its shared memory
}

std::size_t outer_smem(int rows, int ow) {
  const int Wd = 2 * (ow / 32), S = (rows + kOCl - 2) / (kOCl - 1);
  return std::size_t(S * Wd + 32 * Wd + 128 * (Wd + 1) + 2 * S + rows) * 4 + std::size_t(rows) + 16;
}

}  // namespace

bool ech_gf2_outer(std::int64_t rows, std::int64_t wd, std::int64_t ow, std::uint8_t* Z, std::int64_t ldz,
                   std::uint8_t* flags, std::int32_t* info, std::int64_t cap, cudaStream_t s) {
  static const bool off = std::getenv("GFQ_NO_GF2_OUTER") != nullptr;
  if (off || rows <= 0 || rows > kORowsMax || wd <= 0 || wd > ow || (ow != 256 && ow != 512)) return false;
  if ((ldz & 15) || (reinterpret_cast<std::uintptr_t>(Z) & 15)) return false;
  const std::size_t smem = outer_smem(int(rows), int(ow));
  if (smem > 212 * 1024) return false;
  static bool attr = false;
  if (!attr) {
    GFQ_CUDA(cudaFuncSetAttribute(ech_gf2_outer_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                  212 * 1024));
    attr = true;
  }
  // algorithmic bytes: the panel read and [X | Y] written back
  ProfScope ps(kProfEchGf2, double(rows) * double(wd + 2 * ow), s);
  static const bool debug = std::getenv("GFQ_GF2_DEBUG") != nullptr;
  static unsigned long long* dbg = nullptr;
  if (debug && !dbg) GFQ_CUDA(cudaMalloc(&dbg, 256 * sizeof(unsigned long long)));
  OuterArgs g{int(rows), int(wd), int(ow), Z, ldz, flags, info, int(cap), debug ? dbg : nullptr};
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(kOCl);
  cfg.blockDim = dim3(kOThreads);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = s;
  cudaLaunchAttribute attrs[1];
  attrs[0].id = cudaLaunchAttributeClusterDimension;
  attrs[0].val.clusterDim.x = kOCl;
  attrs[0].val.clusterDim.y = 1;
  attrs[0].val.clusterDim.z = 1;
  cfg.attrs = attrs;
  cfg.numAttrs = 1;
  GFQ_CUDA(cudaLaunchKernelEx(&cfg, ech_gf2_outer_kernel, g));
  count_launch();
  if (debug) {
    GFQ_CUDA(cudaStreamSynchronize(s));
    unsigned long long h[256];
    GFQ_CUDA(cudaMemcpy(h, dbg, sizeof h, cudaMemcpyDeviceToHost));
    const auto d = [&](int a, int b) { return static_cast<long long>(h[b] - h[a]); };
    std::fprintf(stderr, "gf2outer rows %lld wd %lld: pack %lld, panels %lld, unpack %lld ns\n",
                 static_cast<long long>(rows), static_cast<long long>(wd), d(0, 1), d(1, 2), d(2, 3));
    for (int k = 0; k + 1 < (wd + 31) / 32 && k < 4; ++k)
      std::fprintf(stderr, "  sub %d: tables %lld sync %lld word+1 %lld | chainwait %lld chain %lld | rest %lld next %lld\n", k,
                   d(8 + 8 * k, 9 + 8 * k), d(9 + 8 * k, 10 + 8 * k), d(10 + 8 * k, 11 + 8 * k),
                   d(11 + 8 * k, 12 + 8 * k), d(12 + 8 * k, 13 + 8 * k), d(11 + 8 * k, 14 + 8 * k),
                   d(8 + 8 * k, 16 + 8 * k));
    std::fprintf(stderr, "  chain loop cycles:");
    for (int k = 0; k < 8; ++k) std::fprintf(stderr, " %llu(far %llu)", h[200 + k], h[220 + k]);
    std::fprintf(stderr, "\n");
  }
  return true;
}

}  // namespace gfq::dev
