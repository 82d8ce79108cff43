// tc_ptx.cuh -- inline-PTX helpers shared by the tcgen05 contraction kernels
// (K1 kind::i8 in gf_mad_tc.cu, K1 kind::mxf4 in gf_mad_f4.cu): mbarriers,
// TMA tile loads, UMMA shared-memory descriptors, MMA issue / commit,
// tcgen05 fences and TMEM loads, and the epilogue's byte packing / mod-p
// reduction.
#pragma once

#include <cuda.h>

#include <cstdint>

namespace gfq::dev::tc {

__device__ __forceinline__ std::uint32_t smem_u32(const void* p) {
  return static_cast<std::uint32_t>(__cvta_generic_to_shared(p));
}

__device__ __forceinline__ void mbar_init(std::uint64_t* bar, std::uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count));
}

__device__ __forceinline__ void mbar_wait(std::uint64_t* bar, std::uint32_t parity) {
  asm volatile(
      "{\n\t.reg .pred P1;\n"
      "WAIT_%=:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n\t"
      "@P1 bra DONE_%=;\n\t"
      "bra WAIT_%=;\n"
      "DONE_%=:\n\t}" ::"r"(smem_u32(bar)),
      "r"(parity));
}

__device__ __forceinline__ void mbar_arrive_expect_tx(std::uint64_t* bar, std::uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)),
               "r"(bytes));
}

__device__ __forceinline__ void mbar_arrive(std::uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)));
}

__device__ __forceinline__ void tma_load_2d(const CUtensorMap* map, std::uint64_t* bar,
                                            void* dst, int c0, int c1) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes"
      " [%0], [%1, {%3, %4}], [%2];" ::"r"(smem_u32(dst)),
      "l"(reinterpret_cast<std::uint64_t>(map)), "r"(smem_u32(bar)), "r"(c0), "r"(c1)
      : "memory");
}

// The same tile written at the same shared-memory offset of every CTA in
// `mask` (cluster ranks); each destination CTA's mbarrier at `bar`'s offset
// receives the bytes it got.
__device__ __forceinline__ void tma_load_2d_mc(const CUtensorMap* map, std::uint64_t* bar, void* dst, int c0,
                                               int c1, std::uint16_t mask) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes.multicast::cluster"
      " [%0], [%1, {%3, %4}], [%2], %5;" ::"r"(smem_u32(dst)),
      "l"(reinterpret_cast<std::uint64_t>(map)), "r"(smem_u32(bar)), "r"(c0), "r"(c1), "h"(mask)
      : "memory");
}

__device__ __forceinline__ std::uint32_t cluster_ctarank() {
  std::uint32_t r;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
  return r;
}

__device__ __forceinline__ void cluster_sync_all() {
  asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}

__device__ __forceinline__ void prefetch_tmap(const CUtensorMap* map) {
  asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<std::uint64_t>(map))
               : "memory");
}

// UMMA shared-memory descriptor: start | LBO | SBO | version=1 | SWIZZLE_128B.
__device__ __forceinline__ std::uint64_t umma_desc(std::uint32_t saddr, std::uint32_t lbo,
                                                   std::uint32_t sbo) {
  return (std::uint64_t((saddr >> 4) & 0x3FFF)) | (std::uint64_t((lbo >> 4) & 0x3FFF) << 16) |
         (std::uint64_t((sbo >> 4) & 0x3FFF) << 32) | (std::uint64_t(1) << 46) |
         (std::uint64_t(2) << 61);
}

__device__ __forceinline__ void mma_i8(std::uint32_t d_tmem, std::uint64_t adesc,
                                       std::uint64_t bdesc, std::uint32_t idesc,
                                       std::uint32_t accumulate) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %3, p;\n\t}" ::"r"(d_tmem),
      "l"(adesc), "l"(bdesc), "r"(idesc), "r"(accumulate));
}

__device__ __forceinline__ void mma_commit(std::uint64_t* bar) {
  asm volatile(
      "tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
          smem_u32(bar))
      : "memory");
}

// arrive on the mbarrier at `bar`'s offset in every CTA of `mask` once the
// MMAs issued so far have completed
__device__ __forceinline__ void mma_commit_mc(std::uint64_t* bar, std::uint16_t mask) {
  asm volatile(
      "tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;" ::"r"(
          smem_u32(bar)),
      "h"(mask)
      : "memory");
}

__device__ __forceinline__ void fence_after() {
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
}
__device__ __forceinline__ void fence_before() {
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
}

__device__ __forceinline__ void tmem_ld32(std::uint32_t taddr, std::uint32_t (&v)[32]) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x32.b32 "
      "{%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,"
      "%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
      : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]),
        "=r"(v[7]), "=r"(v[8]), "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]),
        "=r"(v[13]), "=r"(v[14]), "=r"(v[15]), "=r"(v[16]), "=r"(v[17]), "=r"(v[18]),
        "=r"(v[19]), "=r"(v[20]), "=r"(v[21]), "=r"(v[22]), "=r"(v[23]), "=r"(v[24]),
        "=r"(v[25]), "=r"(v[26]), "=r"(v[27]), "=r"(v[28]), "=r"(v[29]), "=r"(v[30]),
        "=r"(v[31])
      : "r"(taddr));
  asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
}

__device__ __forceinline__ std::uint32_t modp(std::uint32_t x, std::uint32_t p,
                                              std::uint32_t magic) {
  const std::uint32_t q = __umulhi(x, magic);
  const std::int32_t r = static_cast<std::int32_t>(x - q * p);
  return static_cast<std::uint32_t>(r < 0 ? r + static_cast<std::int32_t>(p) : r);
}

// 4 packed residues of a p = 2 tile chunk: bit 0 of v0..v3, xor the addend
// bits (c & 0x01010101 by construction).
__device__ __forceinline__ std::uint32_t pack_low_bytes(std::uint32_t v0, std::uint32_t v1,
                                                        std::uint32_t v2, std::uint32_t v3) {
  const std::uint32_t lo = __byte_perm(v0, v1, 0x0040);
  const std::uint32_t hi = __byte_perm(v2, v3, 0x0040);
  return __byte_perm(lo, hi, 0x5410);
}


// Tile raster: groups of `gm` M-tiles, M fastest inside a group, then N,
// then the next group.  The 148 tiles in flight span gm A row-panels and
// ~148/gm B column-panels, so the group's A slice (gm x 128 x K bytes, kept
// <= ~32 MB by the host) stays L2-resident while B streams through once per
// group; a plain M-fastest order over all M re-reads the whole of A every
// wave once A outgrows L2 (8192 x 65536 x 8192: 7.96 GB of DRAM reads for
// 1.14 GB of operands, profiles/r02_traffic.json).
__device__ __forceinline__ void tile_coords(int tile, int num_m, int num_n, int gm, int& mb, int& nb) {
  const int per_group = gm * num_n;
  const int g = tile / per_group;
  const int r = tile - g * per_group;
  const int m0 = g * gm;
  const int rows = num_m - m0 < gm ? num_m - m0 : gm;
  mb = m0 + r % rows;
  nb = r / rows;
}

// Host: encode a 2-D u8 tensor map (inner dim contiguous, row stride ld
// bytes) with a box of box_inner x box_outer and 128-byte swizzle
// (gf_mad_tc.cu; per-thread cached).
bool make_map_box(CUtensorMap* map, const std::uint8_t* base, std::int64_t inner, std::int64_t outer,
                  std::int64_t ld, std::uint32_t box_inner, std::uint32_t box_outer);

}  // namespace gfq::dev::tc
