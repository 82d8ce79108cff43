// gf_mad_f4.cu -- K1f: the block multiply-accumulate D = Cin + A.B mod p for
// the small primes p in {2, 3, 5, 7} on the FP4 tensor-core path
// (tcgen05.mma kind::mxf4, block-scaled E2M1 operands, fp32 accumulators in
// TMEM), which issues twice the multiply-adds per instruction of kind::i8
// for the same 32 operand bytes.  Same contract as K1 (gf_mad_tc.cu), which
// replaces the reference's scalar mul_add_kernel (src/matrix.cpp:81-133).
//
// Exactness.  Every residue is encoded as the E2M1 value of its symmetric
// representative s in [-(p-1)/2, (p-1)/2] (p = 2: 0 / 1), which is exact for
// |s| <= 3 (E2M1 holds 0, 0.5, 1, 1.5, 2, 3, 4, 6).  The block scales are all
// 2^0 (UE8M0 127), so each product s_a.s_b is an integer with |.| <= 9 and the
// fp32 accumulator holds the exact integer sum while |sum| <= 9.k < 2^24; the
// host keeps k below that per launch (k <= 1.8M, never reached by the
// Chief).  The epilogue rounds the accumulator to an int32 (exact), adds a
// multiple of p that makes it non-negative, the addend, and reduces mod p.
//
// Operand layout.  kind::mxf4 reads both operands K-major with two E2M1
// values per byte, so each contraction first packs A (m x k -> m x kp/2
// bytes) and transposes + packs B (k x n -> n x kp/2 bytes), kp = k rounded
// up to 64, zero padded; pack kernels below (HBM-bound, 1.5 B moved per
// element).  The MMA kernel then mirrors K1: 128 x 224 tiles, K-block 128
// bytes (256 elements) per stage, 5-stage TMA ring (SWIZZLE_128B, both
// operands K-major), one MMA-issuing thread, fp32 accumulators
// double-buffered in TMEM (2 x 224 columns) and released once in registers,
// the scale factors (all 0x7F) planted once per CTA in 32 further TMEM
// columns, 8 epilogue warps.  224 rather than 256 columns because 2 x 256
// accumulator columns would leave no TMEM for the scale factors.
#include <cuda.h>

#include <algorithm>
#include <atomic>
#include <cstdlib>
#include <mutex>
#include <stdexcept>
#include <type_traits>
#include <vector>

#include "../common.hpp"
#include "kernels.hpp"
#include "tc_ptx.cuh"

namespace gfq::dev {
namespace f4 {
using namespace tc;

constexpr int BM = 128, BKB = 128;  // BKB: packed bytes of K per stage (256 elements)
constexpr int A_STAGE = BM * BKB;   // 16 KB
constexpr int EPI_WARPS = 8;
constexpr int NUM_THREADS = 64 + 32 * EPI_WARPS;
constexpr int TMEM_COLS = 512;
// Tile variants: BN output columns, STAGES ring depth, ACCS accumulators in
// TMEM (2 = the epilogue of tile i overlaps the MMAs of tile i+1); the
// scale factors take 32 TMEM columns after the accumulators.
template <int BN_, int STAGES_, int ACCS_>
struct Cfg {
  static constexpr int BN = BN_, STAGES = STAGES_, ACCS = ACCS_;
  static constexpr int B_STAGE = BN * BKB;
  static constexpr int STAGE_BYTES = A_STAGE + B_STAGE;
  static constexpr int SMEM_BYTES = STAGES * STAGE_BYTES + 1024 + 256;
  static constexpr int SF_COL = ACCS * BN;  // scale factors of A (16 columns), then of B (16)
  static_assert(SF_COL + 32 <= TMEM_COLS, "TMEM: accumulators + scale factors");
  static_assert(SMEM_BYTES <= 227 * 1024, "shared memory");
  // kind::mxf4 instruction descriptor: A = B = E2M1 (MXF4 format 1, bits 7-9
  // and 10-12), both K-major, N >> 3 at bit 17, scale format UE8M0 (bit 23),
  // M >> 4 at bit 24, scale-factor ids 0, dense K = 64.
  static constexpr std::uint32_t IDESC = (1u << 7) | (1u << 10) | ((std::uint32_t(BN) >> 3) << 17) |
                                         (1u << 23) | ((std::uint32_t(BM) >> 4) << 24);
};
// measured on 8192 x 8192 x 65536 GF(2) (tools/f4_bench.py, kernel only):
// 192 x 2: 6.33 POPS, 224 x 2: 6.64, 256 x 1: 6.59
using CfgA = Cfg<224, 5, 2>;  // default
using CfgB = Cfg<192, 5, 2>;
using CfgC = Cfg<256, 4, 1>;

__device__ __forceinline__ void mma_f4(std::uint32_t d_tmem, std::uint64_t adesc, std::uint64_t bdesc,
                                       std::uint32_t idesc, std::uint32_t accumulate, std::uint32_t sfa,
                                       std::uint32_t sfb) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::mxf4.block_scale.block32 [%0], %1, %2, %3, [%5], [%6], p;\n\t}" ::"r"(
          d_tmem),
      "l"(adesc), "l"(bdesc), "r"(idesc), "r"(accumulate), "r"(sfa), "r"(sfb));
}

__device__ __forceinline__ void tmem_ld16(std::uint32_t taddr, std::uint32_t (&v)[16]) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x16.b32 "
      "{%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
      : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7]),
        "=r"(v[8]), "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]), "=r"(v[14]), "=r"(v[15])
      : "r"(taddr));
  asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
}

__device__ __forceinline__ void tmem_st32_const(std::uint32_t taddr, std::uint32_t x) {
  asm volatile(
      "tcgen05.st.sync.aligned.32x32b.x32.b32 [%0], "
      "{%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,"
      "%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,%1};" ::"r"(taddr),
      "r"(x));
  asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
}

// Clusters of CM x CN CTAs on a CM x CN block of tiles: the CM CTAs of one
// N-tile share its B tile and the CN CTAs of one M-tile share its A tile, so
// each CTA loads 1/CM of the B tile and 1/CN of the A tile and multicasts
// each part into the rings of the CTAs sharing it -- L2 -> SM operand traffic
// per tile drops from A + B to A/CN + B/CM.  A stage may be refilled only
// once every CTA of the cluster has drained it, so each CTA's MMA commit
// arrives on the `empty` barrier of all of them (count CM.CN).
template <class C, int CM, int CN>
__global__ void __launch_bounds__(NUM_THREADS, 1)
gf_mad_f4_kernel(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB, int m,
                 int n, int kpb, std::uint32_t p, std::uint32_t magic, std::uint32_t bias,
                 const std::uint8_t* Cin, std::int64_t ldc, std::uint8_t* D, std::int64_t ldd, int gm) {
  pdl_wait();
  constexpr int BN = C::BN, STAGES = C::STAGES, ACCS = C::ACCS, B_STAGE = C::B_STAGE,
                STAGE_BYTES = C::STAGE_BYTES, SF_COL = C::SF_COL;
  extern __shared__ __align__(1024) std::uint8_t smem_raw[];
  std::uint8_t* smem = reinterpret_cast<std::uint8_t*>(
      (reinterpret_cast<std::uintptr_t>(smem_raw) + 1023) & ~std::uintptr_t(1023));
  std::uint8_t* sA = smem;
  std::uint8_t* sB = smem + STAGES * A_STAGE;
  std::uint64_t* bars = reinterpret_cast<std::uint64_t*>(smem + STAGES * STAGE_BYTES);
  std::uint64_t* full = bars;
  std::uint64_t* empty = bars + STAGES;
  std::uint64_t* tfull = bars + 2 * STAGES;
  std::uint64_t* tempty = bars + 2 * STAGES + 2;
  std::uint32_t* tmem_slot = reinterpret_cast<std::uint32_t*>(bars + 2 * STAGES + 4);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int num_m = (m + BM - 1) / BM, num_n = (n + BN - 1) / BN;
  // work units: CM x CN blocks of tiles; this CTA takes tile
  // (CM.um + rm, CN.un + rn) of unit (um, un) -- a phantom past num_m or
  // num_n at a ragged edge (its loads fill zeros, its outputs are all out of
  // range)
  constexpr int CL = CM * CN;
  const int num_um = (num_m + CM - 1) / CM, num_un = (num_n + CN - 1) / CN;
  const int num_tiles = num_um * num_un;
  const int num_kb = (kpb + BKB - 1) / BKB;
  const int rank = CL > 1 ? int(cluster_ctarank()) : 0;
  const int rm = rank % CM, rn = rank / CM;
  std::uint16_t a_mask = 0, b_mask = 0;  // the CTAs sharing this CTA's A / B tile
  for (int j = 0; j < CN; ++j) a_mask |= std::uint16_t(1u << (rm + CM * j));
  for (int j = 0; j < CM; ++j) b_mask |= std::uint16_t(1u << (j + CM * rn));
  const int first = int(blockIdx.x) / CL, stride = int(gridDim.x) / CL;
  const int gu = gm / CM > 0 ? gm / CM : 1;

  if (warp == 0 && lane == 0) {
    prefetch_tmap(&tmA);
    prefetch_tmap(&tmB);
    for (int s = 0; s < STAGES; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], CL);
    }
    for (int a = 0; a < 2; ++a) {
      mbar_init(&tfull[a], 1);
      mbar_init(&tempty[a], EPI_WARPS);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  }
  if (warp == 1) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(tmem_slot)),
                 "r"(TMEM_COLS));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  fence_before();
  __syncthreads();
  fence_after();
  const std::uint32_t tmem_base = *tmem_slot;
  // plant the scale factors: every byte of TMEM columns [SF_COL, SF_COL+32)
  // = UE8M0 127 (2^0), whatever lanes / bytes the MMA reads them from
  if (warp >= 2 && warp < 6) {
    const int quarter = warp & 3;
    tmem_st32_const(tmem_base + (std::uint32_t(quarter * 32) << 16) + std::uint32_t(SF_COL), 0x7F7F7F7Fu);
  }
  fence_before();
  __syncthreads();
  // the peer's barriers must be initialised before its first multicast
  if constexpr (CL > 1) cluster_sync_all();
  fence_after();
  const std::uint32_t sfa = tmem_base + std::uint32_t(SF_COL);
  const std::uint32_t sfb = tmem_base + std::uint32_t(SF_COL + 16);

  if (warp == 0) {
    if (lane == 0) {
      int stage = 0;
      std::uint32_t phase = 0;
      for (int tile = first; tile < num_tiles; tile += stride) {
        int um, un;
        tile_coords(tile, num_um, num_un, gu, um, un);
        const int mb = um * CM + rm, nb = un * CN + rn;
        for (int kb = 0; kb < num_kb; ++kb) {
          mbar_wait(&empty[stage], phase ^ 1);
          mbar_arrive_expect_tx(&full[stage], STAGE_BYTES);
          if constexpr (CN > 1)
            tma_load_2d_mc(&tmA, &full[stage], sA + stage * A_STAGE + rn * (A_STAGE / CN), kb * BKB,
                           mb * BM + rn * (BM / CN), a_mask);
          else
            tma_load_2d(&tmA, &full[stage], sA + stage * A_STAGE, kb * BKB, mb * BM);
          if constexpr (CM > 1)
            tma_load_2d_mc(&tmB, &full[stage], sB + stage * B_STAGE + rm * (B_STAGE / CM), kb * BKB,
                           nb * BN + rm * (BN / CM), b_mask);
          else
            tma_load_2d(&tmB, &full[stage], sB + stage * B_STAGE, kb * BKB, nb * BN);
          if (++stage == STAGES) {
            stage = 0;
            phase ^= 1;
          }
        }
      }
    }
  } else if (warp == 1) {
    if (lane == 0) {
      int stage = 0;
      std::uint32_t phase = 0;
      int it = 0;
      for (int tile = first; tile < num_tiles; tile += stride, ++it) {
        const int acc = ACCS == 2 ? (it & 1) : 0;
        const std::uint32_t acc_phase = ACCS == 2 ? ((it >> 1) & 1) : (it & 1);
        mbar_wait(&tempty[acc], acc_phase ^ 1);
        fence_after();
        const std::uint32_t d_tmem = tmem_base + std::uint32_t(acc * BN);
        for (int kb = 0; kb < num_kb; ++kb) {
          mbar_wait(&full[stage], phase);
          fence_after();
          const std::uint32_t a0 = smem_u32(sA + stage * A_STAGE);
          const std::uint32_t b0 = smem_u32(sB + stage * B_STAGE);
#pragma unroll
          for (int kk = 0; kk < BKB / 32; ++kk) {
            // both operands K-major SW128: 32 bytes (64 E2M1 values) per MMA
            const std::uint64_t ad = umma_desc(a0 + kk * 32, 16, 1024);
            const std::uint64_t bd = umma_desc(b0 + kk * 32, 16, 1024);
            mma_f4(d_tmem, ad, bd, C::IDESC, (kb | kk) != 0, sfa, sfb);
          }
          if constexpr (CL > 1)
            mma_commit_mc(&empty[stage], std::uint16_t((1u << CL) - 1));
          else
            mma_commit(&empty[stage]);
          if (++stage == STAGES) {
            stage = 0;
            phase ^= 1;
          }
        }
        mma_commit(&tfull[acc]);
      }
    }
  } else {
    // epilogue: warp w reads TMEM lane quarter w % 4 and one half of the
    // tile's columns, in chunks of 32 columns (+ one of 16)
    constexpr int HALF = BN / 2, C32 = HALF / 32, TAIL = HALF % 32;
    static_assert(TAIL == 0 || TAIL == 16, "epilogue chunks");
    constexpr int NCH = C32 + (TAIL ? 1 : 0);
    const int quarter = warp & 3;
    const int half = (warp - 2) >> 2;
    const int row_in_tile = quarter * 32 + lane;
    const bool p2 = p == 2;
    int it = 0;
    for (int tile = first; tile < num_tiles; tile += stride, ++it) {
      int um, un;
      tile_coords(tile, num_um, num_un, gu, um, un);
      const int mb = um * CM + rm, nb = un * CN + rn;
      const int acc = ACCS == 2 ? (it & 1) : 0;
      const std::uint32_t acc_phase = ACCS == 2 ? ((it >> 1) & 1) : (it & 1);
      const int row = mb * BM + row_in_tile;
      const bool row_ok = row < m;
      const int cbase = nb * BN + half * HALF;
      const std::uint8_t* crow = (Cin && row_ok) ? Cin + std::int64_t(row) * ldc : nullptr;
      std::uint8_t* drow = row_ok ? D + std::int64_t(row) * ldd : nullptr;
      const bool vec = row_ok && cbase + HALF <= n &&
                       (reinterpret_cast<std::uintptr_t>(drow + cbase) & 15) == 0 &&
                       (!crow || (reinterpret_cast<std::uintptr_t>(crow + cbase) & 15) == 0);
      uint4 cpre[HALF / 16];
#pragma unroll
      for (int q = 0; q < HALF / 16; ++q) cpre[q] = make_uint4(0, 0, 0, 0);
      if (vec && crow) {
#pragma unroll
        for (int q = 0; q < HALF / 16; ++q) cpre[q] = reinterpret_cast<const uint4*>(crow + cbase)[q];
      }
      mbar_wait(&tfull[acc], acc_phase);
      fence_after();
      // W columns (16 or 32) of accumulators at column offset c0 of the half
      auto process = [&](std::uint32_t* v, auto wtag, int c0, bool last) {
        constexpr int W = decltype(wtag)::value;
        if (last) {
          fence_before();
          __syncwarp();
          if (lane == 0) mbar_arrive(&tempty[acc]);
        }
        // the exact integer sums (fp32 -> int32 is exact below 2^24), made
        // non-negative by `bias` (a multiple of p; 0 for p = 2)
#pragma unroll
        for (int c = 0; c < W; ++c) v[c] = std::uint32_t(__float2int_rn(__uint_as_float(v[c]))) + bias;
        const int col0 = cbase + c0;
        if (vec) {
#pragma unroll
          for (int h = 0; h < W / 16; ++h) {
            const uint4 cq = cpre[c0 / 16 + h];
            const std::uint32_t cw[4] = {cq.x, cq.y, cq.z, cq.w};
            std::uint32_t ow[4];
            if (p2) {
#pragma unroll
              for (int w = 0; w < 4; ++w)
                ow[w] = (pack_low_bytes(v[16 * h + 4 * w], v[16 * h + 4 * w + 1], v[16 * h + 4 * w + 2],
                                        v[16 * h + 4 * w + 3]) ^ cw[w]) & 0x01010101u;
            } else {
#pragma unroll
              for (int w = 0; w < 4; ++w) {
                std::uint32_t r[4];
#pragma unroll
                for (int b = 0; b < 4; ++b)
                  r[b] = modp(v[16 * h + 4 * w + b] + __byte_perm(cw[w], 0, 0x4440 + b), p, magic);
                ow[w] = pack_low_bytes(r[0], r[1], r[2], r[3]);
              }
            }
            reinterpret_cast<uint4*>(drow + col0)[h] = make_uint4(ow[0], ow[1], ow[2], ow[3]);
          }
        } else if (row_ok) {
#pragma unroll
          for (int c = 0; c < W; ++c) {
            if (col0 + c < n) {
              std::uint32_t x = v[c];
              if (crow) x += crow[col0 + c];
              drow[col0 + c] = static_cast<std::uint8_t>(modp(x, p, magic));
            }
          }
        }
      };
      const std::uint32_t tbase =
          tmem_base + (std::uint32_t(quarter * 32) << 16) + std::uint32_t(acc * BN + half * HALF);
#pragma unroll
      for (int ch = 0; ch < C32; ++ch) {
        std::uint32_t v[32];
        tmem_ld32(tbase + std::uint32_t(ch * 32), v);
        process(v, std::integral_constant<int, 32>{}, ch * 32, ch == NCH - 1);
      }
      if constexpr (TAIL != 0) {
        std::uint32_t v[16];
        tmem_ld16(tbase + std::uint32_t(C32 * 32), v);
        process(v, std::integral_constant<int, 16>{}, C32 * 32, true);
      }
    }
  }

  fence_before();
  __syncthreads();
  // the peer's last commits arrive on this CTA's barriers
  if constexpr (CL > 1) cluster_sync_all();
  if (warp == 1) {
    fence_after();
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem_base), "r"(TMEM_COLS));
  }
}

// E2M1 codes of the residues 0..7 as nibbles of one word: residue v maps to
// its symmetric representative s (v <= (p-1)/2 ? v : v - p), encoded as
// sign bit 3 | magnitude code (0 -> 0, 1 -> 2, 2 -> 4, 3 -> 5).
__host__ __device__ constexpr std::uint32_t e2m1_of_mag(std::uint32_t a) {
  return a == 0 ? 0u : a == 1 ? 2u : a == 2 ? 4u : 5u;
}
std::uint32_t code_word(std::uint32_t p) {
  std::uint32_t w = 0;
  for (std::uint32_t v = 0; v < p && v < 8; ++v) {
    const bool neg = p > 2 && v > (p - 1) / 2;
    const std::uint32_t mag = neg ? p - v : v;
    w |= ((neg ? 8u : 0u) | e2m1_of_mag(mag)) << (4 * v);
  }
  return w;
}

// two residue bytes -> one byte of two E2M1 codes (element 2j low nibble)
__device__ __forceinline__ std::uint32_t pack4(std::uint32_t x, std::uint32_t codes) {
  // x holds 4 residues (bytes); returns 2 packed bytes in the low 16 bits
  const std::uint32_t c0 = (codes >> (4 * (x & 0xFF))) & 0xF;
  const std::uint32_t c1 = (codes >> (4 * ((x >> 8) & 0xFF))) & 0xF;
  const std::uint32_t c2 = (codes >> (4 * ((x >> 16) & 0xFF))) & 0xF;
  const std::uint32_t c3 = (codes >> (4 * (x >> 24))) & 0xF;
  return c0 | (c1 << 4) | (c2 << 8) | (c3 << 12);
}

// A (m x k residues, row-major) -> Ap (m x kpb bytes): one thread per 32
// elements (16 output bytes), columns >= k zero.
__global__ void __launch_bounds__(256) pack_rows_f4_kernel(const std::uint8_t* A, std::int64_t lda, int m, int k,
                                                           std::uint8_t* out, int kpb, std::uint32_t codes) {
  pdl_wait_and_release();
  const int per_row = kpb / 16;
  const std::int64_t total = std::int64_t(m) * per_row;
  const bool al = ((reinterpret_cast<std::uintptr_t>(A) | std::uintptr_t(lda)) & 15) == 0;
  for (std::int64_t t = std::int64_t(blockIdx.x) * blockDim.x + threadIdx.x; t < total;
       t += std::int64_t(gridDim.x) * blockDim.x) {
    const int r = int(t / per_row), q = int(t - std::int64_t(r) * per_row);
    const int c0 = q * 32;
    const std::uint8_t* src = A + std::int64_t(r) * lda;
    std::uint32_t w[8];
    if (al && c0 + 32 <= k) {
      const uint4 lo = reinterpret_cast<const uint4*>(src + c0)[0];
      const uint4 hi = reinterpret_cast<const uint4*>(src + c0)[1];
      w[0] = lo.x; w[1] = lo.y; w[2] = lo.z; w[3] = lo.w;
      w[4] = hi.x; w[5] = hi.y; w[6] = hi.z; w[7] = hi.w;
    } else {
#pragma unroll
      for (int u = 0; u < 8; ++u) {
        std::uint32_t x = 0;
#pragma unroll
        for (int b = 0; b < 4; ++b) {
          const int c = c0 + 4 * u + b;
          if (c < k) x |= std::uint32_t(src[c]) << (8 * b);
        }
        w[u] = x;
      }
    }
    // residue 0 codes to 0, so the zero padding packs to zero bytes
    uint4 o;
    o.x = pack4(w[0], codes) | (pack4(w[1], codes) << 16);
    o.y = pack4(w[2], codes) | (pack4(w[3], codes) << 16);
    o.z = pack4(w[4], codes) | (pack4(w[5], codes) << 16);
    o.w = pack4(w[6], codes) | (pack4(w[7], codes) << 16);
    reinterpret_cast<uint4*>(out + std::int64_t(r) * kpb)[q] = o;
  }
}

// B (k x n residues, row-major) -> Bt (n x kpb bytes, K-major): a CTA packs
// a 128 (k) x 512 (n) tile staged in shared memory (16 coalesced 16-byte
// loads a thread, all in flight together); thread t then reads 4 adjacent
// columns (one 32-bit word a row: a warp covers 128 consecutive bytes, no
// bank conflicts) over 64 rows and writes each column's 64 codes as one
// 32-byte sector.
constexpr int PC_K = 128, PC_N = 512, PC_LD = PC_N + 16;
constexpr int PC_SMEM = PC_K * PC_LD;
__global__ void __launch_bounds__(256) pack_cols_f4_kernel(const std::uint8_t* B, std::int64_t ldb, int k, int n,
                                                           std::uint8_t* out, int kpb, std::uint32_t codes) {
  pdl_wait_and_release();
  extern __shared__ __align__(16) std::uint8_t tile[];
  const int n0 = blockIdx.x * PC_N, k0 = blockIdx.y * PC_K;
  const bool al = ((reinterpret_cast<std::uintptr_t>(B) | std::uintptr_t(ldb)) & 15) == 0;
  uint4 x[16];
#pragma unroll
  for (int q = 0; q < 16; ++q) {
    const int v = threadIdx.x + 256 * q;  // 128 rows x 32 vectors
    const int r = v >> 5, c = (v & 31) * 16;
    const int kr = k0 + r, nc = n0 + c;
    x[q] = make_uint4(0, 0, 0, 0);
    if (kr < k) {
      const std::uint8_t* src = B + std::int64_t(kr) * ldb + nc;
      if (al && nc + 16 <= n) {
        x[q] = *reinterpret_cast<const uint4*>(src);
      } else {
        std::uint32_t w[4] = {0, 0, 0, 0};
        for (int b = 0; b < 16; ++b)
          if (nc + b < n) w[b >> 2] |= std::uint32_t(src[b]) << (8 * (b & 3));
        x[q] = make_uint4(w[0], w[1], w[2], w[3]);
      }
    }
  }
#pragma unroll
  for (int q = 0; q < 16; ++q) {
    const int v = threadIdx.x + 256 * q;
    *reinterpret_cast<uint4*>(tile + (v >> 5) * PC_LD + (v & 31) * 16) = x[q];
  }
  __syncthreads();
  const int cg = threadIdx.x & 127, rh = threadIdx.x >> 7;  // 4 columns, 64 rows
  const int j0 = n0 + 4 * cg;
  if (j0 >= n) return;
  std::uint32_t o[4][8];
#pragma unroll
  for (int u = 0; u < 8; ++u) {
    std::uint32_t a0 = 0, a1 = 0, a2 = 0, a3 = 0;
#pragma unroll
    for (int b = 0; b < 8; ++b) {
      const std::uint32_t w = *reinterpret_cast<const std::uint32_t*>(tile + (64 * rh + 8 * u + b) * PC_LD + 4 * cg);
      a0 |= ((codes >> (4 * (w & 0xFF))) & 0xF) << (4 * b);
      a1 |= ((codes >> (4 * ((w >> 8) & 0xFF))) & 0xF) << (4 * b);
      a2 |= ((codes >> (4 * ((w >> 16) & 0xFF))) & 0xF) << (4 * b);
      a3 |= ((codes >> (4 * (w >> 24))) & 0xF) << (4 * b);
    }
    o[0][u] = a0;
    o[1][u] = a1;
    o[2][u] = a2;
    o[3][u] = a3;
  }
  const int kb = (k0 + 64 * rh) / 2;  // byte offset of these 64 codes
  if (kb >= kpb) return;
#pragma unroll
  for (int c = 0; c < 4; ++c) {
    if (j0 + c >= n) break;
    uint4* dst = reinterpret_cast<uint4*>(out + std::int64_t(j0 + c) * kpb + kb);
    dst[0] = make_uint4(o[c][0], o[c][1], o[c][2], o[c][3]);
    dst[1] = make_uint4(o[c][4], o[c][5], o[c][6], o[c][7]);
  }
}

}  // namespace f4

bool f4_field(std::uint32_t p) { return p == 2 || p == 3 || p == 5 || p == 7; }

std::int64_t mad_f4_scratch_bytes(std::int64_t m, std::int64_t n, std::int64_t k) {
  const std::int64_t kpb = (k + 63) / 64 * 32;
  return (m + n) * kpb + 256;
}

std::int64_t mad_f4_bt_bytes(std::int64_t n, std::int64_t k) {
  const std::int64_t kpb = (k + 63) / 64 * 32;
  return n * kpb + 256;
}

void pack_b_f4(std::uint32_t p, std::int64_t n, std::int64_t k, const std::uint8_t* B, std::int64_t ldb,
               std::uint8_t* bt, cudaStream_t s) {
  using namespace f4;
  static const bool once = [] {
    GFQ_CUDA(cudaFuncSetAttribute(pack_cols_f4_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, PC_SMEM));
    return true;
  }();
  (void)once;
  const std::int64_t kpb = (k + 63) / 64 * 32;
  ProfScope ps(kProfSelect, double(n) * double(k) * 1.5, s);
  GFQ_CUDA(launch_pdl(pack_cols_f4_kernel, dim3(unsigned((n + PC_N - 1) / PC_N), unsigned((kpb + 63) / 64)),
                      dim3(256), std::size_t(PC_SMEM), s, B, ldb, int(k), int(n), bt, int(kpb), code_word(p)));
  count_launch();
}

bool mad_f4(std::uint32_t p, std::int64_t m, std::int64_t n, std::int64_t k, const std::uint8_t* A,
            std::int64_t lda, const std::uint8_t* B, std::int64_t ldb, const std::uint8_t* Cin, std::int64_t ldc,
            std::uint8_t* D, std::int64_t ldd, std::uint8_t* scratch, cudaStream_t s,
            const std::uint8_t* bt_packed) {
  using namespace f4;
  if (!f4_field(p) || m <= 0 || n <= 0 || k <= 0) return false;
  if ((reinterpret_cast<std::uintptr_t>(bt_packed) & 15) != 0) return false;
  // |sum| <= h^2 k must stay below 2^24 (h = (p-1)/2, 1 for p = 2)
  const std::int64_t h = p == 2 ? 1 : (p - 1) / 2;
  if (h * h * k >= (std::int64_t(1) << 24) || m >= (1LL << 31) || n >= (1LL << 31)) return false;
  if ((reinterpret_cast<std::uintptr_t>(scratch) & 15) != 0) return false;
  static const int variant = [] {
    const char* e = std::getenv("GFQ_F4_VARIANT");
    return e ? std::atoi(e) : 0;
  }();
  // operand-sharing clusters (see the kernel): GFQ_F4_CLUSTER = 1 (none),
  // 2 (CTA pairs sharing B), 4 (2 x 2), 12 (pairs sharing A); tile 224 only
  static const int clv = [] {
    const char* e = std::getenv("GFQ_F4_CLUSTER");
    const int v = e ? std::atoi(e) : 2;
    return v == 1 || v == 4 || v == 12 ? v : 2;
  }();
  const int cm = variant != 0 ? 1 : clv == 2 || clv == 4 ? 2 : 1;
  const int cn = variant != 0 ? 1 : clv == 4 || clv == 12 ? 2 : 1;
  using KernT = void (*)(CUtensorMap, CUtensorMap, int, int, int, std::uint32_t, std::uint32_t, std::uint32_t,
                         const std::uint8_t*, std::int64_t, std::uint8_t*, std::int64_t, int);
  KernT kern = variant == 1   ? gf_mad_f4_kernel<CfgB, 1, 1>
               : variant == 2 ? gf_mad_f4_kernel<CfgC, 1, 1>
               : cm == 2 && cn == 2 ? gf_mad_f4_kernel<CfgA, 2, 2>
               : cm == 2            ? gf_mad_f4_kernel<CfgA, 2, 1>
               : cn == 2            ? gf_mad_f4_kernel<CfgA, 1, 2>
                                    : gf_mad_f4_kernel<CfgA, 1, 1>;
  const int smem = variant == 1 ? CfgB::SMEM_BYTES : variant == 2 ? CfgC::SMEM_BYTES : CfgA::SMEM_BYTES;
  const int cl = cm * cn;
  const int BN = variant == 1 ? CfgB::BN : variant == 2 ? CfgC::BN : CfgA::BN;
  // co-resident clusters of this shape (a persistent grid must not exceed it)
  static const int max_clusters = [&] {
    auto big = [](auto k, int bytes) {
      GFQ_CUDA(cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes));
    };
    big(gf_mad_f4_kernel<CfgA, 1, 1>, CfgA::SMEM_BYTES);
    big(gf_mad_f4_kernel<CfgB, 1, 1>, CfgB::SMEM_BYTES);
    big(gf_mad_f4_kernel<CfgC, 1, 1>, CfgC::SMEM_BYTES);
    big(gf_mad_f4_kernel<CfgA, 2, 1>, CfgA::SMEM_BYTES);
    big(gf_mad_f4_kernel<CfgA, 1, 2>, CfgA::SMEM_BYTES);
    big(gf_mad_f4_kernel<CfgA, 2, 2>, CfgA::SMEM_BYTES);
    big(pack_cols_f4_kernel, PC_SMEM);
    if (cl == 1) return 1 << 30;
    cudaLaunchAttribute at;
    at.id = cudaLaunchAttributeClusterDimension;
    at.val.clusterDim.x = unsigned(cl);
    at.val.clusterDim.y = 1;
    at.val.clusterDim.z = 1;
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(unsigned(cl * 256));
    cfg.blockDim = dim3(NUM_THREADS);
    cfg.dynamicSmemBytes = std::size_t(smem);
    cfg.attrs = &at;
    cfg.numAttrs = 1;
    int n = 0;
    GFQ_CUDA(cudaOccupancyMaxActiveClusters(&n, kern, &cfg));
    return n > 0 ? n : 1;
  }();
  const std::int64_t kpb = (k + 63) / 64 * 32;
  std::uint8_t* Ap = scratch;
  // B already packed (pack_b_f4 into a mad_f4_bt_bytes block, ordered before
  // this call on s): the scratch then only holds A
  const std::uint8_t* Bt = bt_packed ? bt_packed : scratch + (m * kpb + 127) / 128 * 128;
  CUtensorMap mA, mB;
  if (!make_map_box(&mA, Ap, kpb, m, kpb, BKB, std::uint32_t(BM / cn))) return false;
  if (!make_map_box(&mB, Bt, kpb, n, kpb, BKB, std::uint32_t(BN / cm))) return false;
  const std::uint32_t codes = code_word(p);
  {
    ProfScope ps(kProfSelect, double(m) * double(k) * 1.5, s);
    const std::int64_t total = m * (kpb / 16);
    const std::int64_t cap = std::int64_t(sm_count()) * 8;
    const unsigned grid = unsigned(std::min<std::int64_t>((total + 255) / 256, cap));
    GFQ_CUDA(launch_pdl(pack_rows_f4_kernel, dim3(grid), dim3(256), 0, s, A, lda, int(m), int(k), Ap, int(kpb),
                        codes));
    count_launch();
  }
  if (!bt_packed) pack_b_f4(p, n, k, B, ldb, scratch + (m * kpb + 127) / 128 * 128, s);
  const std::int64_t sms = k1_sms(s);
  const std::int64_t tiles_per_rowtile = (n + BN - 1) / BN;
  // row pieces of <= GFQ_K1_MAX_WAVES tile waves each (see mad_tc)
  static const std::int64_t max_waves = [] {
    const char* e = std::getenv("GFQ_K1_MAX_WAVES");
    return e ? std::int64_t(std::atoll(e)) : std::int64_t(0);
  }();
  std::int64_t mp = m;
  if (max_waves > 0 && (m + BM - 1) / BM * tiles_per_rowtile > max_waves * sms)
    mp = std::max<std::int64_t>(1, (max_waves * sms) / tiles_per_rowtile) * BM;
  const std::uint32_t magic = static_cast<std::uint32_t>((0x100000000ULL / p) + 1);
  const std::uint32_t bias = p == 2 ? 0u : std::uint32_t((h * h * k + p - 1) / p * p);
  ProfScope ps(kProfF4, 2.0 * double(m) * double(n) * double(k), s);
  K1Lane lane(s);
  for (std::int64_t m0 = 0; m0 < m; m0 += mp) {
    const std::int64_t mm = std::min(mp, m - m0);
    CUtensorMap mA;
    if (!make_map_box(&mA, Ap + m0 * kpb, kpb, mm, kpb, BKB, std::uint32_t(BM / cn))) throw std::runtime_error("mad_f4: tensor map");
    const std::int64_t num_m = (mm + BM - 1) / BM;
    const std::int64_t units_all = (num_m + cm - 1) / cm * ((tiles_per_rowtile + cn - 1) / cn);
    const std::int64_t cap = std::min<std::int64_t>(sms / cl, max_clusters);
    const int units = int(units_all < cap ? units_all : cap);
    // raster group: the A slice of gm M-tiles within ~32 MB
    const std::int64_t gm = std::max<std::int64_t>(
        1, std::min<std::int64_t>(num_m, (std::int64_t(32) << 20) / (std::int64_t(BM) * kpb)));
    const std::uint8_t* cin = Cin ? Cin + m0 * ldc : nullptr;
    std::uint8_t* d = D + m0 * ldd;
    cudaLaunchAttribute at[2];
    at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    at[0].val.programmaticStreamSerializationAllowed = 1;
    at[1].id = cudaLaunchAttributeClusterDimension;
    at[1].val.clusterDim.x = unsigned(cl);
    at[1].val.clusterDim.y = 1;
    at[1].val.clusterDim.z = 1;
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(unsigned(units * cl));
    cfg.blockDim = dim3(NUM_THREADS);
    cfg.stream = s;
    cfg.attrs = pdl_enabled() ? at : at + 1;
    cfg.numAttrs = pdl_enabled() ? 2 : 1;
    cfg.dynamicSmemBytes = std::size_t(smem);
    GFQ_CUDA(cudaLaunchKernelEx(&cfg, kern, mA, mB, int(mm), int(n), int(kpb), p, magic, bias, cin, ldc, d, ldd,
                                int(gm)));
    GFQ_CUDA(cudaGetLastError());
    count_launch();
  }
  return true;
}

}  // namespace gfq::dev
