// gf_mad_tc.cu -- K1: the block multiply-accumulate D = Cin + A.B mod p on
// the 5th-generation tensor cores (tcgen05.mma kind::i8, u8 x u8 -> s32 in
// TMEM), fed by TMA, with the mod-p reduction and the addend fused into the
// epilogue.  Replaces the reference's scalar mul_add_kernel
// (src/matrix.cpp:81-133) on the UpdateRow / UpdateRowTrafo / ClearUp path.
//
// Layout: A (m x k, row-major = K-major), B (k x n, row-major = MN-major,
// legal for INT8 UMMA), residues 0..p-1 as u8.  Tile 128 x 256, K-block 128
// bytes, 4-stage smem ring (48 KB/stage), persistent CTAs (one per SM), TMEM
// double-buffered (2 x 256 columns) so the epilogue of tile i overlaps the
// MMAs of tile i+1.  Warp roles: 0 = TMA producer, 1 = MMA issuer + TMEM
// owner, 2..5 = epilogue (one TMEM lane / output row per thread).
//
// Exactness: (p-1)^2 * k + (p-1) < 2^31 is required per launch; the host
// splits K into chunks and chains them through the addend (mod p between).
#include <cuda.h>
#include <cudaTypedefs.h>

#include <atomic>
#include <cstring>
#include <mutex>

#include "../common.hpp"
#include "kernels.hpp"

namespace gfq::dev {
namespace tc {

constexpr int BM = 128, BN = 256, BK = 128, STAGES = 4;
constexpr int A_STAGE = BM * BK;           // 16 KB
constexpr int B_HALF = BK * 128;           // 16 KB (128 k-rows x 128 n-bytes)
constexpr int B_STAGE = 2 * B_HALF;        // 32 KB
constexpr int STAGE_BYTES = A_STAGE + B_STAGE;
constexpr int SMEM_BYTES = STAGES * STAGE_BYTES + 1024 /*align*/ + 256 /*barriers*/;
constexpr int NUM_THREADS = 192;
constexpr int TMEM_COLS = 512;

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

// Instruction descriptor, kind::i8: D=S32, A=B=UINT8, A K-major, B MN-major,
// N=256 (bits 17..22 = N>>3), M=128 (bits 24..28 = M>>4).
constexpr std::uint32_t kIdesc = (2u << 4) | (0u << 7) | (0u << 10) | (0u << 15) | (1u << 16) |
                                 ((std::uint32_t(BN) >> 3) << 17) | ((std::uint32_t(BM) >> 4) << 24);

__global__ void __launch_bounds__(NUM_THREADS, 1)
gf_mad_tc_kernel(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB,
                 int m, int n, int k, std::uint32_t p, std::uint32_t magic,
                 const std::uint8_t* Cin, std::int64_t ldc, std::uint8_t* D, std::int64_t ldd) {
  extern __shared__ __align__(1024) std::uint8_t smem_raw[];
  std::uint8_t* smem = reinterpret_cast<std::uint8_t*>(
      (reinterpret_cast<std::uintptr_t>(smem_raw) + 1023) & ~std::uintptr_t(1023));
  std::uint8_t* sA = smem;                            // STAGES x 16 KB
  std::uint8_t* sB = smem + STAGES * A_STAGE;         // STAGES x 32 KB
  std::uint64_t* bars = reinterpret_cast<std::uint64_t*>(smem + STAGES * STAGE_BYTES);
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
      mbar_init(&tempty[a], 4);  // one arrive per epilogue warp
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  }
  if (warp == 1) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                     smem_u32(tmem_slot)),
                 "r"(TMEM_COLS));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  fence_before();
  __syncthreads();
  fence_after();
  const std::uint32_t tmem_base = *tmem_slot;

  if (warp == 0) {
    // ---------------- TMA producer
    if (lane == 0) {
      int stage = 0;
      std::uint32_t phase = 0;
      for (int tile = blockIdx.x; tile < num_tiles; tile += gridDim.x) {
        const int mb = tile % num_m, nb = tile / num_m;
        for (int kb = 0; kb < num_kb; ++kb) {
          mbar_wait(&empty[stage], phase ^ 1);
          mbar_arrive_expect_tx(&full[stage], STAGE_BYTES);
          tma_load_2d(&tmA, &full[stage], sA + stage * A_STAGE, kb * BK, mb * BM);
          tma_load_2d(&tmB, &full[stage], sB + stage * B_STAGE, nb * BN, kb * BK);
          tma_load_2d(&tmB, &full[stage], sB + stage * B_STAGE + B_HALF, nb * BN + 128, kb * BK);
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
          const std::uint32_t a0 = smem_u32(sA + stage * A_STAGE);
          const std::uint32_t b0 = smem_u32(sB + stage * B_STAGE);
#pragma unroll
          for (int kk = 0; kk < BK / 32; ++kk) {
            // A: K-major SW128, 32 bytes of K per MMA -> advance start by 32 B.
            const std::uint64_t ad = umma_desc(a0 + kk * 32, 16, 1024);
            // B: MN-major SW128, 32 K-rows per MMA -> advance by 32 x 128 B.
            const std::uint64_t bd = umma_desc(b0 + kk * 32 * 128, B_HALF, 1024);
            mma_i8(d_tmem, ad, bd, kIdesc, (kb | kk) != 0);
          }
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
    // ---------------- epilogue: warps 2..5, TMEM lane quarter = warp % 4
    const int quarter = warp & 3;
    const int row_in_tile = quarter * 32 + lane;
    int it = 0;
    for (int tile = blockIdx.x; tile < num_tiles; tile += gridDim.x, ++it) {
      const int mb = tile % num_m, nb = tile / num_m;
      const int acc = it & 1;
      const std::uint32_t acc_phase = (it >> 1) & 1;
      const int row = mb * BM + row_in_tile;
      const bool row_ok = row < m;
      const std::uint8_t* crow = (Cin && row_ok) ? Cin + std::int64_t(row) * ldc : nullptr;
      std::uint8_t* drow = row_ok ? D + std::int64_t(row) * ldd : nullptr;
      // Prefetch this row's addend segment before waiting on the MMAs, so
      // its HBM latency hides behind the mainloop.
      const bool pre = crow && nb * BN + BN <= n &&
                       (reinterpret_cast<std::uintptr_t>(crow + nb * BN) & 15) == 0;
      uint4 cpre[BN / 16];
      if (pre) {
#pragma unroll
        for (int q = 0; q < BN / 16; ++q)
          cpre[q] = reinterpret_cast<const uint4*>(crow + nb * BN)[q];
      }
      mbar_wait(&tfull[acc], acc_phase);
      fence_after();
#pragma unroll
      for (int ch = 0; ch < BN / 32; ++ch) {
        std::uint32_t v[32];
        const std::uint32_t taddr = tmem_base + (std::uint32_t(quarter * 32) << 16) +
                                    std::uint32_t(acc * BN + ch * 32);
        tmem_ld32(taddr, v);
        const int col0 = nb * BN + ch * 32;
        if (!row_ok || col0 >= n) continue;
        const int ncols = (n - col0) < 32 ? (n - col0) : 32;
        const bool vec = ncols == 32 &&
                         ((reinterpret_cast<std::uintptr_t>(drow + col0) & 15) == 0) &&
                         (!crow || (reinterpret_cast<std::uintptr_t>(crow + col0) & 15) == 0);
        if (vec) {
          uint4 cv[2] = {make_uint4(0, 0, 0, 0), make_uint4(0, 0, 0, 0)};
          if (pre) {
            cv[0] = cpre[2 * ch];
            cv[1] = cpre[2 * ch + 1];
          } else if (crow) {
            cv[0] = reinterpret_cast<const uint4*>(crow + col0)[0];
            cv[1] = reinterpret_cast<const uint4*>(crow + col0)[1];
          }
          const std::uint32_t* cw = reinterpret_cast<const std::uint32_t*>(cv);
          std::uint32_t ow[8];
#pragma unroll
          for (int w = 0; w < 8; ++w) {
            std::uint32_t word = 0;
#pragma unroll
            for (int b = 0; b < 4; ++b) {
              const std::uint32_t x = v[w * 4 + b] + ((cw[w] >> (8 * b)) & 0xFF);
              word |= modp(x, p, magic) << (8 * b);
            }
            ow[w] = word;
          }
          reinterpret_cast<uint4*>(drow + col0)[0] = make_uint4(ow[0], ow[1], ow[2], ow[3]);
          reinterpret_cast<uint4*>(drow + col0)[1] = make_uint4(ow[4], ow[5], ow[6], ow[7]);
        } else {
          for (int c = 0; c < ncols; ++c) {
            std::uint32_t x = v[c];
            if (crow) x += crow[col0 + c];
            drow[col0 + c] = static_cast<std::uint8_t>(modp(x, p, magic));
          }
        }
      }
      fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(&tempty[acc]);
    }
  }

  fence_before();
  __syncthreads();
  if (warp == 1) {
    fence_after();
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem_base),
                 "r"(TMEM_COLS));
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

bool make_map(CUtensorMap* map, const std::uint8_t* base, std::int64_t inner,
              std::int64_t outer, std::int64_t ld) {
  auto fn = encode_fn();
  if (!fn) return false;
  cuuint64_t dims[2] = {cuuint64_t(inner), cuuint64_t(outer)};
  cuuint64_t strides[1] = {cuuint64_t(ld)};
  cuuint32_t box[2] = {128, 128};
  cuuint32_t estr[2] = {1, 1};
  CUresult r = fn(map, CU_TENSOR_MAP_DATA_TYPE_UINT8, 2, const_cast<std::uint8_t*>(base), dims,
                  strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                  CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  return r == CUDA_SUCCESS;
}

}  // namespace tc

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
    GFQ_CUDA(cudaFuncSetAttribute(gf_mad_tc_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                  SMEM_BYTES));
  });
  // K chunk: (p-1)^2 * kc + (p-1) < 2^31, multiple of BK.
  const std::uint64_t sq = std::uint64_t(p - 1) * (p - 1);
  std::int64_t kc = sq ? std::int64_t((0x7FFFFFFFULL - p) / sq) : (1LL << 40);
  kc = kc / BK * BK;
  if (kc <= 0) return false;
  const std::uint32_t magic = static_cast<std::uint32_t>((0x100000000ULL / p) + 1);
  const int num_tiles = int(((m + BM - 1) / BM) * ((n + BN - 1) / BN));
  const int grid = num_tiles < sm_count() ? num_tiles : sm_count();
  for (std::int64_t k0 = 0; k0 < k; k0 += kc) {
    const std::int64_t kk = (k - k0) < kc ? (k - k0) : kc;
    CUtensorMap mA, mB;
    // A sub-block starting at column k0 must stay 16B aligned.
    if ((k0 & 15) != 0) return false;
    if (!make_map(&mA, A + k0, kk, m, lda)) return false;
    if (!make_map(&mB, B + k0 * ldb, n, kk, ldb)) return false;
    const std::uint8_t* cin = k0 == 0 ? Cin : D;
    const std::int64_t ldcin = k0 == 0 ? ldc : ldd;
    gf_mad_tc_kernel<<<grid, NUM_THREADS, SMEM_BYTES, s>>>(mA, mB, int(m), int(n), int(kk), p,
                                                           magic, cin, ldcin, D, ldd);
    GFQ_CUDA(cudaGetLastError());
    count_launch();
  }
  return true;
}

}  // namespace gfq::dev
