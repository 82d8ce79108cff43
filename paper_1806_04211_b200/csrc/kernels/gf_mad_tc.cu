// gf_mad_tc.cu -- K1: the block multiply-accumulate D = Cin + A.B mod p on
// the 5th-generation tensor cores (tcgen05.mma kind::i8, u8 x u8 -> s32 in
// TMEM), fed by TMA, with the mod-p reduction and the addend fused into the
// epilogue.  Replaces the reference's scalar mul_add_kernel
// (src/matrix.cpp:81-133) on the UpdateRow / UpdateRowTrafo / ClearUp path.
//
// Layout: A (m x k, row-major = K-major), B (k x n, row-major = MN-major,
// legal for INT8 UMMA), residues 0..p-1 as u8.  Tile 128 x 256 (or 128 x 128
// when that fills more SMs), K-block 128 bytes, 4- (6-) stage smem ring,
// persistent CTAs (one per SM), TMEM double-buffered (2 x BN columns) so the
// epilogue of tile i overlaps the MMAs of tile i+1, and released as soon as
// the accumulator is in registers.  Warp roles: 0 = TMA producer, 1 = MMA
// issuer + TMEM owner, 2..9 = epilogue (two warps per TMEM lane quarter,
// each a half row of the tile; p = 2 packs with byte permutes, other p
// use a Barrett reduction).
//
// Exactness: (p-1)^2 * k + (p-1) < 2^31 is required per launch; the host
// splits K into chunks and chains them through the addend (mod p between).
#include <vector>
#include <cuda.h>
#include <cudaTypedefs.h>

#include <atomic>
#include <cstdlib>
#include <cstring>
#include <mutex>

#include "../common.hpp"
#include "kernels.hpp"
#include "tc_ptx.cuh"

namespace gfq::dev {
namespace tc {

constexpr int BM = 128, BK = 128;
constexpr int A_STAGE = BM * BK;           // 16 KB
constexpr int B_HALF = BK * 128;           // 16 KB (128 k-rows x 128 n-bytes, one TMA box)
constexpr int EPI_WARPS = 8;               // two per TMEM lane quarter
constexpr int NUM_THREADS = 64 + 32 * EPI_WARPS;

// Per N-tile geometry: BN = 256 (4 stages of 48 KB) for large problems,
// BN = 128 (6 stages of 32 KB) when the 256-wide tiling leaves SMs idle.
template <int BN>
struct Geo {
  static constexpr int B_STAGE = BK * BN;
  static constexpr int STAGE_BYTES = A_STAGE + B_STAGE;
  static constexpr int STAGES = BN == 256 ? 4 : 6;
  static constexpr int SMEM_BYTES = STAGES * STAGE_BYTES + 1024 /*align*/ + 256 /*barriers*/;
  static constexpr int TMEM_COLS = 2 * BN;  // double-buffered accumulator
  // kind::i8 instruction descriptor: D=S32 (bits 4-5 = 2), A=B=UINT8,
  // A K-major, B MN-major (bit 16), N>>3 at bit 17, M>>4 at bit 24.
  static constexpr std::uint32_t IDESC = (2u << 4) | (1u << 16) |
                                         ((std::uint32_t(BN) >> 3) << 17) |
                                         ((std::uint32_t(BM) >> 4) << 24);
};

template <int BN>
__global__ void __launch_bounds__(NUM_THREADS, 1)
gf_mad_tc_kernel(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB,
                 int m, int n, int k, std::uint32_t p, std::uint32_t magic,
                 const std::uint8_t* Cin, std::int64_t ldc, std::uint8_t* D, std::int64_t ldd,
                 int gm, unsigned long long* dbg) {
  // PDL: wait for the predecessor grid before any global access; dependents
  // are released only at exit (a waiting 200 KB-smem K1 CTA would hold an SM
  // other streams could use)
  pdl_wait();
  using G = Geo<BN>;
  constexpr int STAGES = G::STAGES;
  // dbg (developer timing, GFQ_TC_DEBUG): per CTA 8 globaltimer stamps.
  auto stamp = [&](int slot) {
    if (dbg && threadIdx.x % 32 == 0) {
      unsigned long long t;
      asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
      dbg[blockIdx.x * 8 + slot] = t;
    }
  };
  if (threadIdx.x == 0) stamp(0);
  extern __shared__ __align__(1024) std::uint8_t smem_raw[];
  std::uint8_t* smem = reinterpret_cast<std::uint8_t*>(
      (reinterpret_cast<std::uintptr_t>(smem_raw) + 1023) & ~std::uintptr_t(1023));
  std::uint8_t* sA = smem;                            // STAGES x 16 KB
  std::uint8_t* sB = smem + STAGES * A_STAGE;         // STAGES x BN * 128 B
  std::uint64_t* bars = reinterpret_cast<std::uint64_t*>(smem + STAGES * G::STAGE_BYTES);
  std::uint64_t* full = bars;                         // [STAGES]
  std::uint64_t* empty = bars + STAGES;               // [STAGES]
  std::uint64_t* tfull = bars + 2 * STAGES;           // [2]
  std::uint64_t* tempty = bars + 2 * STAGES + 2;      // [2]
  std::uint32_t* tmem_slot = reinterpret_cast<std::uint32_t*>(bars + 2 * STAGES + 4);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int num_m = (m + BM - 1) / BM, num_n = (n + BN - 1) / BN;
  const int num_tiles = num_m * num_n;
  const int num_kb = (k + BK - 1) / BK;

  if (warp == 0 && lane == 0) {
    prefetch_tmap(&tmA);
    prefetch_tmap(&tmB);
    for (int s = 0; s < STAGES; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);
    }
    for (int a = 0; a < 2; ++a) {
      mbar_init(&tfull[a], 1);
      mbar_init(&tempty[a], EPI_WARPS);  // one arrive per epilogue warp
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  }
  if (warp == 1) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                     smem_u32(tmem_slot)),
                 "r"(G::TMEM_COLS));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  fence_before();
  __syncthreads();
  fence_after();
  const std::uint32_t tmem_base = *tmem_slot;
  if (threadIdx.x == 0) stamp(1);

  if (warp == 0) {
    // ---------------- TMA producer
    if (lane == 0) {
      int stage = 0;
      std::uint32_t phase = 0;
      for (int tile = blockIdx.x; tile < num_tiles; tile += gridDim.x) {
        int mb, nb;
        tile_coords(tile, num_m, num_n, gm, mb, nb);
        for (int kb = 0; kb < num_kb; ++kb) {
          mbar_wait(&empty[stage], phase ^ 1);
          mbar_arrive_expect_tx(&full[stage], G::STAGE_BYTES);
          tma_load_2d(&tmA, &full[stage], sA + stage * A_STAGE, kb * BK, mb * BM);
#pragma unroll
          for (int h = 0; h < BN / 128; ++h)
            tma_load_2d(&tmB, &full[stage], sB + stage * G::B_STAGE + h * B_HALF, nb * BN + h * 128,
                        kb * BK);
          if (++stage == STAGES) {
            stage = 0;
            phase ^= 1;
          }
        }
      }
    }
  } else if (warp == 1) {
    // ---------------- MMA issuer (single thread)
    if (lane == 0) {
      int stage = 0;
      std::uint32_t phase = 0;
      int it = 0;
      for (int tile = blockIdx.x; tile < num_tiles; tile += gridDim.x, ++it) {
        const int acc = it & 1;
        const std::uint32_t acc_phase = (it >> 1) & 1;
        mbar_wait(&tempty[acc], acc_phase ^ 1);
        fence_after();
        const std::uint32_t d_tmem = tmem_base + std::uint32_t(acc * BN);
        for (int kb = 0; kb < num_kb; ++kb) {
          mbar_wait(&full[stage], phase);
          fence_after();
          if (kb == 0 && it == 0) stamp(2);
          const std::uint32_t a0 = smem_u32(sA + stage * A_STAGE);
          const std::uint32_t b0 = smem_u32(sB + stage * G::B_STAGE);
#pragma unroll
          for (int kk = 0; kk < BK / 32; ++kk) {
            // A: K-major SW128, 32 bytes of K per MMA -> advance start by 32 B.
            const std::uint64_t ad = umma_desc(a0 + kk * 32, 16, 1024);
            // B: MN-major SW128, 32 K-rows per MMA -> advance by 32 x 128 B;
            // the 128-column halves are B_HALF apart (LBO).
            const std::uint64_t bd = umma_desc(b0 + kk * 32 * 128, B_HALF, 1024);
            mma_i8(d_tmem, ad, bd, G::IDESC, (kb | kk) != 0);
          }
          mma_commit(&empty[stage]);
          if (++stage == STAGES) {
            stage = 0;
            phase ^= 1;
          }
        }
        mma_commit(&tfull[acc]);
      }
      stamp(3);
    }
  } else {
    // ---------------- epilogue: 8 warps; warp w reads TMEM lane quarter
    // w % 4 (the tcgen05.ld rule) and one half of the tile's columns.
    constexpr int HALF = BN / 2, CHUNKS = HALF / 32;
    const int quarter = warp & 3;
    const int half = (warp - 2) >> 2;
    const int row_in_tile = quarter * 32 + lane;
    const bool p2 = p == 2;
    int it = 0;
    for (int tile = blockIdx.x; tile < num_tiles; tile += gridDim.x, ++it) {
      int mb, nb;
        tile_coords(tile, num_m, num_n, gm, mb, nb);
      const int acc = it & 1;
      const std::uint32_t acc_phase = (it >> 1) & 1;
      const int row = mb * BM + row_in_tile;
      const bool row_ok = row < m;
      const int cbase = nb * BN + half * HALF;
      const std::uint8_t* crow = (Cin && row_ok) ? Cin + std::int64_t(row) * ldc : nullptr;
      std::uint8_t* drow = row_ok ? D + std::int64_t(row) * ldd : nullptr;
      // The whole half-row is in range and 16 B aligned (the common case):
      // prefetch its addend before waiting on the MMAs.
      const bool vec = row_ok && cbase + HALF <= n &&
                       (reinterpret_cast<std::uintptr_t>(drow + cbase) & 15) == 0 &&
                       (!crow || (reinterpret_cast<std::uintptr_t>(crow + cbase) & 15) == 0);
      uint4 cpre[HALF / 16];
#pragma unroll
      for (int q = 0; q < HALF / 16; ++q) cpre[q] = make_uint4(0, 0, 0, 0);
      if (vec && crow) {
#pragma unroll
        for (int q = 0; q < HALF / 16; ++q)
          cpre[q] = reinterpret_cast<const uint4*>(crow + cbase)[q];
      }
      mbar_wait(&tfull[acc], acc_phase);
      fence_after();
      if (warp == 2 && it == 0) stamp(4);
#pragma unroll
      for (int ch = 0; ch < CHUNKS; ++ch) {
        std::uint32_t v[32];
        const std::uint32_t taddr = tmem_base + (std::uint32_t(quarter * 32) << 16) +
                                    std::uint32_t(acc * BN + half * HALF + ch * 32);
        tmem_ld32(taddr, v);
        if (ch == CHUNKS - 1) {
          // accumulator fully in registers: hand it back to the MMA warp
          fence_before();
          __syncwarp();
          if (lane == 0) mbar_arrive(&tempty[acc]);
        }
        const int col0 = cbase + ch * 32;
        if (vec) {
          const std::uint32_t cw[8] = {cpre[2 * ch].x,     cpre[2 * ch].y,     cpre[2 * ch].z,
                                       cpre[2 * ch].w,     cpre[2 * ch + 1].x, cpre[2 * ch + 1].y,
                                       cpre[2 * ch + 1].z, cpre[2 * ch + 1].w};
          std::uint32_t ow[8];
          if (p2) {
#pragma unroll
            for (int w = 0; w < 8; ++w)
              ow[w] = (pack_low_bytes(v[4 * w], v[4 * w + 1], v[4 * w + 2], v[4 * w + 3]) ^ cw[w]) &
                      0x01010101u;
          } else {
#pragma unroll
            for (int w = 0; w < 8; ++w) {
              std::uint32_t r[4];
#pragma unroll
              for (int b = 0; b < 4; ++b)
                r[b] = modp(v[4 * w + b] + __byte_perm(cw[w], 0, 0x4440 + b), p, magic);
              ow[w] = pack_low_bytes(r[0], r[1], r[2], r[3]);
            }
          }
          reinterpret_cast<uint4*>(drow + col0)[0] = make_uint4(ow[0], ow[1], ow[2], ow[3]);
          reinterpret_cast<uint4*>(drow + col0)[1] = make_uint4(ow[4], ow[5], ow[6], ow[7]);
        } else if (row_ok) {
#pragma unroll
          for (int c = 0; c < 32; ++c) {
            if (col0 + c < n) {
              std::uint32_t x = v[c];
              if (crow) x += crow[col0 + c];
              drow[col0 + c] = static_cast<std::uint8_t>(modp(x, p, magic));
            }
          }
        }
      }
    }
    if (warp == 2) stamp(5);
  }

  fence_before();
  __syncthreads();
  if (warp == 1) {
    fence_after();
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem_base),
                 "r"(G::TMEM_COLS));
    stamp(6);
  }
}

// ------------------------------------------------------------------ host side
PFN_cuTensorMapEncodeTiled_v12000 encode_fn() {
  static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
  static std::once_flag once;
  std::call_once(once, [] {
    void* ptr = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &ptr, cudaEnableDefault, &q) ==
            cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(ptr);
  });
  return fn;
}

bool encode_map(CUtensorMap* map, const std::uint8_t* base, std::int64_t inner,
                std::int64_t outer, std::int64_t ld, std::uint32_t box_inner, std::uint32_t box_outer) {
  auto fn = encode_fn();
  if (!fn) return false;
  cuuint64_t dims[2] = {cuuint64_t(inner), cuuint64_t(outer)};
  cuuint64_t strides[1] = {cuuint64_t(ld)};
  cuuint32_t box[2] = {box_inner, box_outer};
  cuuint32_t estr[2] = {1, 1};
  CUresult r = fn(map, CU_TENSOR_MAP_DATA_TYPE_UINT8, 2, const_cast<std::uint8_t*>(base), dims,
                  strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                  CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  return r == CUDA_SUCCESS;
}

// Encoded maps are a pure function of (base, inner, outer, ld, box): a small
// per-thread direct-mapped cache skips re-encoding for recycled buffers.
bool make_map_box(CUtensorMap* map, const std::uint8_t* base, std::int64_t inner, std::int64_t outer,
                  std::int64_t ld, std::uint32_t box_inner, std::uint32_t box_outer) {
  struct Entry {
    const std::uint8_t* base = nullptr;
    std::int64_t inner = 0, outer = 0, ld = 0;
    std::uint32_t box = 0;
    CUtensorMap map;
  };
  constexpr int kEntries = 256;
  thread_local Entry cache[kEntries];
  static const bool off = std::getenv("GFQ_NO_TMAP_CACHE") != nullptr;
  if (off) return encode_map(map, base, inner, outer, ld, box_inner, box_outer);
  const std::uint32_t box = box_inner << 16 | box_outer;
  const std::uint64_t h = (reinterpret_cast<std::uintptr_t>(base) >> 4) * 0x9E3779B97F4A7C15ull ^
                          std::uint64_t(inner) * 0xC2B2AE3D27D4EB4Full ^ std::uint64_t(outer) * 31 ^
                          std::uint64_t(ld) ^ std::uint64_t(box) * 0x165667B19E3779F9ull;
  Entry& e = cache[(h >> 32) % kEntries];
  if (e.base == base && e.inner == inner && e.outer == outer && e.ld == ld && e.box == box) {
    *map = e.map;
    return true;
  }
  if (!encode_map(map, base, inner, outer, ld, box_inner, box_outer)) return false;
  e.base = base;
  e.inner = inner;
  e.outer = outer;
  e.ld = ld;
  e.box = box;
  e.map = *map;
  return true;
}
bool make_map(CUtensorMap* map, const std::uint8_t* base, std::int64_t inner,
              std::int64_t outer, std::int64_t ld) {
  return make_map_box(map, base, inner, outer, ld, 128, 128);
}

// Developer timing: with GFQ_TC_DEBUG set, every launch stamps into one
// device buffer of 148 x 8 u64 (read back by gfq_tc_debug_take).
unsigned long long* g_dbg = nullptr;
unsigned long long* tc_debug_buf() {
  static std::once_flag once;
  std::call_once(once, [] {
    if (std::getenv("GFQ_TC_DEBUG")) {
      GFQ_CUDA(cudaMalloc(&g_dbg, 148 * 8 * sizeof(unsigned long long)));
      GFQ_CUDA(cudaMemset(g_dbg, 0, 148 * 8 * sizeof(unsigned long long)));
    }
  });
  return g_dbg;
}

}  // namespace tc

void tc_debug_take(unsigned long long* host) {
  if (!tc::g_dbg) return;
  GFQ_CUDA(cudaMemcpy(host, tc::g_dbg, 148 * 8 * sizeof(unsigned long long), cudaMemcpyDeviceToHost));
}

bool mad_tc(std::uint32_t p, std::int64_t m, std::int64_t n, std::int64_t k,
            const std::uint8_t* A, std::int64_t lda, const std::uint8_t* B,
            std::int64_t ldb, const std::uint8_t* Cin, std::int64_t ldc,
            std::uint8_t* D, std::int64_t ldd, cudaStream_t s) {
  using namespace tc;
  if (m <= 0 || n <= 0 || k <= 0) return false;
  const auto al16 = [](const void* q) { return (reinterpret_cast<std::uintptr_t>(q) & 15) == 0; };
  if (!al16(A) || !al16(B) || (lda & 15) || (ldb & 15)) return false;
  if (m >= (1LL << 31) || n >= (1LL << 31) || k >= (1LL << 31)) return false;
  static std::once_flag attr_once;
  std::call_once(attr_once, [] {
    GFQ_CUDA(cudaFuncSetAttribute(gf_mad_tc_kernel<256>,
                                  cudaFuncAttributeMaxDynamicSharedMemorySize, Geo<256>::SMEM_BYTES));
    GFQ_CUDA(cudaFuncSetAttribute(gf_mad_tc_kernel<128>,
                                  cudaFuncAttributeMaxDynamicSharedMemorySize, Geo<128>::SMEM_BYTES));
  });
  // K chunk: (p-1)^2 * kc + (p-1) < 2^31, multiple of BK.
  const std::uint64_t sq = std::uint64_t(p - 1) * (p - 1);
  std::int64_t kc = sq ? std::int64_t((0x7FFFFFFFULL - p) / sq) : (1LL << 40);
  kc = kc / BK * BK;
  if (kc <= 0) return false;
  const std::uint32_t magic = static_cast<std::uint32_t>((0x100000000ULL / p) + 1);
  // N tile: 128 wide when that cuts the tile-waves enough (a 128-wide tile
  // costs ~0.55 of a 256-wide one: A is re-read and the MMA is narrower).
  const std::int64_t sms = k1_sms(s);
  const std::int64_t mt = (m + BM - 1) / BM;
  const std::int64_t t256 = mt * ((n + 255) / 256), t128 = mt * ((n + 127) / 128);
  const bool narrow = 11 * ((t128 + sms - 1) / sms) < 18 * ((t256 + sms - 1) / sms);
  const std::int64_t tiles = narrow ? t128 : t256;
  const int grid = int(tiles < sms ? tiles : sms);
  // Every chunk's tensor maps are built (and validated) before the first
  // launch: returning false after a launch would let the caller's SIMT
  // fallback re-add A.B onto a D that already holds part of it (in-place
  // callers pass Cin == D).
  // Row pieces: a persistent launch holds every SM until its last tile, so
  // a long one starves the critical-path ECH on the high-priority stream;
  // GFQ_K1_MAX_WAVES = w cuts launches to <= w tile waves each (row pieces
  // of the output), letting the block scheduler interleave between them.
  static const std::int64_t max_waves = [] {
    const char* e = std::getenv("GFQ_K1_MAX_WAVES");
    return e ? std::int64_t(std::atoll(e)) : std::int64_t(0);
  }();
  const std::int64_t tiles_per_rowtile = narrow ? (n + 127) / 128 : (n + 255) / 256;
  std::int64_t mp = m;
  if (max_waves > 0 && tiles > max_waves * sms)
    mp = std::max<std::int64_t>(1, (max_waves * sms) / tiles_per_rowtile) * BM;
  struct Chunk {
    std::int64_t m0, mm, k0, kk;
    int grid;
    CUtensorMap mA, mB;
  };
  std::vector<Chunk> chunks;
  for (std::int64_t k0 = 0; k0 < k; k0 += kc) {
    for (std::int64_t m0 = 0; m0 < m; m0 += mp) {
      Chunk c;
      c.m0 = m0;
      c.mm = std::min(mp, m - m0);
      c.k0 = k0;
      c.kk = (k - k0) < kc ? (k - k0) : kc;
      const std::int64_t t = (c.mm + BM - 1) / BM * tiles_per_rowtile;
      c.grid = int(t < sms ? t : sms);
      // A sub-block starting at column k0 must stay 16B aligned.
      if ((k0 & 15) != 0) return false;
      if (!make_map(&c.mA, A + m0 * lda + k0, c.kk, c.mm, lda)) return false;
      if (!make_map(&c.mB, B + k0 * ldb, n, c.kk, ldb)) return false;
      chunks.push_back(c);
    }
  }
  (void)grid;
  static const std::int64_t group_mb = [] {
    const char* e = std::getenv("GFQ_K1_GROUP_MB");
    const std::int64_t v = e ? std::int64_t(std::atoll(e)) : 32;
    return v > 0 ? v : std::int64_t(1) << 20;  // <= 0: one group (plain M-fastest raster)
  }();
  K1Lane lane(s);
  for (const Chunk& c : chunks) {
    const std::int64_t k0 = c.k0, kk = c.kk, m0 = c.m0;
    const CUtensorMap& mA = c.mA;
    const CUtensorMap& mB = c.mB;
    const std::uint8_t* cin = k0 == 0 ? Cin : D;
    const std::int64_t ldcin = k0 == 0 ? ldc : ldd;
    if (cin) cin += m0 * ldcin;
    std::uint8_t* d = D + m0 * ldd;
    // raster group: the A slice of gm M-tiles within ~32 MB (GFQ_K1_GROUP_MB)
    const std::int64_t num_m = (c.mm + BM - 1) / BM;
    const std::int64_t gm = std::max<std::int64_t>(
        1, std::min<std::int64_t>(num_m, (group_mb << 20) / (std::int64_t(BM) * std::max<std::int64_t>(kk, 1))));
    if (narrow)
      GFQ_CUDA(launch_pdl(gf_mad_tc_kernel<128>, dim3(c.grid), dim3(NUM_THREADS), Geo<128>::SMEM_BYTES, s,
          mA, mB, int(c.mm), int(n), int(kk), p, magic, cin, ldcin, d, ldd, int(gm), tc_debug_buf()));
    else
      GFQ_CUDA(launch_pdl(gf_mad_tc_kernel<256>, dim3(c.grid), dim3(NUM_THREADS), Geo<256>::SMEM_BYTES, s,
          mA, mB, int(c.mm), int(n), int(kk), p, magic, cin, ldcin, d, ldd, int(gm), tc_debug_buf()));
    GFQ_CUDA(cudaGetLastError());
    count_launch();
  }
  return true;
}

}  // namespace gfq::dev
