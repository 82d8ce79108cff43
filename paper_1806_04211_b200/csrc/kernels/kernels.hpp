// kernels.hpp -- launch wrappers for the sm_100a kernels of the GF(p) path.
//
// All matrices are u8 residues 0..p-1, row-major, with a row stride (ld) in
// bytes.  Every wrapper is stream-ordered and returns immediately.
#pragma once

#include <cuda_runtime.h>

#include <cstddef>
#include <cstdint>
#include <utility>

namespace gfq::dev {

// Programmatic dependent launch (PDL).  launch_pdl launches a kernel with
// programmatic stream serialization, so its CTAs may become resident while
// the previous kernel in the stream drains; every kernel launched this way
// calls pdl_wait() before its first global-memory access (it returns once
// the predecessor grid has completed and its writes are visible -- a no-op
// without a programmatic predecessor) and pdl_release() once its own
// dependents may be scheduled.  GFQ_NO_PDL=1 launches without the attribute.
#ifdef __CUDACC__
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
__device__ __forceinline__ void pdl_release() {
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
}
__device__ __forceinline__ void pdl_wait_and_release() {
  pdl_wait();
  pdl_release();
}
#endif
bool pdl_enabled();
template <typename... KArgs, typename... Args>
inline cudaError_t launch_pdl(void (*kernel)(KArgs...), dim3 grid, dim3 block, std::size_t smem,
                              cudaStream_t s, Args&&... args) {
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[0].val.programmaticStreamSerializationAllowed = 1;
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = s;
  cfg.attrs = at;
  cfg.numAttrs = pdl_enabled() ? 1 : 0;
  return cudaLaunchKernelEx(&cfg, kernel, std::forward<Args>(args)...);
}

// ---------------------------------------------------------------- K1
// D = (Cin ? Cin : 0) + A.B mod p   (A: m x k, B: k x n, Cin/D: m x n).
// Cin may alias D.  Dispatches to the tcgen05 kind::i8 kernel when the
// operands are TMA-legal and the contraction is large enough, else to the
// SIMT small-K kernel.  Exact for any k (K is split so the s32 accumulator
// cannot overflow: (p-1)^2 * k_chunk < 2^31).
void mad(std::uint32_t p, std::int64_t m, std::int64_t n, std::int64_t k,
         const std::uint8_t* A, std::int64_t lda, const std::uint8_t* B,
         std::int64_t ldb, const std::uint8_t* Cin, std::int64_t ldc,
         std::uint8_t* D, std::int64_t ldd, cudaStream_t s);

// The small-K contraction (k <= 32, 16-byte aligned B / Cin / D) with row
// maps, for the rank-r' updates fused with their gathers / riffles:
// D[drm[i]] = Cin[crm[i]] + sum_t A[i][t] * B[brm[t]] (each map may be
// null = identity; crm[i] = -1: no addend).  Maps are device arrays.
void mad_smallk_maps(std::uint32_t p, std::int64_t m, std::int64_t n, std::int64_t k,
                     const std::uint8_t* A, std::int64_t lda, const std::uint8_t* B, std::int64_t ldb,
                     const std::int32_t* brm, const std::uint8_t* Cin, std::int64_t ldc,
                     const std::int32_t* crm, std::uint8_t* D, std::int64_t ldd, const std::int32_t* drm,
                     cudaStream_t s);
constexpr int kSmallKMax = 32;

// Force a specific K1 implementation (tests / profiling).
void mad_simt(std::uint32_t p, std::int64_t m, std::int64_t n, std::int64_t k,
              const std::uint8_t* A, std::int64_t lda, const std::uint8_t* B,
              std::int64_t ldb, const std::uint8_t* Cin, std::int64_t ldc,
              std::uint8_t* D, std::int64_t ldd, cudaStream_t s);
// Returns false (launching nothing) when the operands are not TMA-legal.
bool mad_tc(std::uint32_t p, std::int64_t m, std::int64_t n, std::int64_t k,
            const std::uint8_t* A, std::int64_t lda, const std::uint8_t* B,
            std::int64_t ldb, const std::uint8_t* Cin, std::int64_t ldc,
            std::uint8_t* D, std::int64_t ldd, cudaStream_t s);

// K1f: the same contraction on the FP4 tensor cores (tcgen05.mma kind::mxf4,
// gf_mad_f4.cu) for p in {2, 3, 5, 7}: the residues as E2M1 values of their
// symmetric representatives, exact fp32 sums.  `scratch` holds the packed
// operands (mad_f4_scratch_bytes, 16-byte aligned, stream-ordered on s).
// Returns false (launching nothing) for other p or a k beyond the exact
// range.  use_f4 is the dispatch rule (policy, field, size).
bool f4_field(std::uint32_t p);
// SMs a persistent K1 / K1f launch on `s` may occupy: all of them, minus
// GFQ_K1_SM_RESERVE (default 0) on non-critical streams -- kept free for
// the critical path's kernels.  stream_is_critical: s has the device's
// greatest priority (the executor's Step-1 critical-path stream).
bool stream_is_critical(cudaStream_t s);
int k1_sms(cudaStream_t s);
// The critical-path partition (set per run by the Chief for large blocks):
// while on, persistent contractions from non-critical streams run one at a
// time on all but GFQ_K1_SM_RESERVE (16) SMs and the executor's bulk
// streams live in a green context without one SM group, so the diagonal
// ECH chain always finds SMs (cfg5s 157 -> 151 ms, cfg4 54 -> 53 ms; small
// blocks lose ~1.5% and keep it off).
void set_critical_partition(bool on);
bool critical_partition();
// Scope around a persistent contraction's launches (see kernels.cu).
class K1Lane {
 public:
  explicit K1Lane(cudaStream_t s);
  ~K1Lane();
  K1Lane(const K1Lane&) = delete;
  K1Lane& operator=(const K1Lane&) = delete;

 private:
  cudaStream_t s_;
  bool held_ = false;
  int* cur_ = nullptr;
};
bool use_f4(std::uint32_t p, std::int64_t m, std::int64_t n, std::int64_t k);
std::int64_t mad_f4_scratch_bytes(std::int64_t m, std::int64_t n, std::int64_t k);
bool mad_f4(std::uint32_t p, std::int64_t m, std::int64_t n, std::int64_t k, const std::uint8_t* A,
            std::int64_t lda, const std::uint8_t* B, std::int64_t ldb, const std::uint8_t* Cin, std::int64_t ldc,
            std::uint8_t* D, std::int64_t ldd, std::uint8_t* scratch, cudaStream_t s,
            const std::uint8_t* bt_packed = nullptr);
// The B operand's packing on its own (transposed E2M1 codes, mad_f4_bt_bytes
// bytes, 16-byte aligned): a B that several contractions share is packed
// once and handed to mad_f4 as bt_packed (jobs.cpp, ImmutableB).
std::int64_t mad_f4_bt_bytes(std::int64_t n, std::int64_t k);
void pack_b_f4(std::uint32_t p, std::int64_t n, std::int64_t k, const std::uint8_t* B, std::int64_t ldb,
               std::uint8_t* bt, cudaStream_t s);

// ---------------------------------------------------------------- accounting
// Every kernel launch of this library bumps a counter (bench.py's
// gpu_launches).  With profiling on, each K1 launch is bracketed by CUDA
// events on its own stream; profile_take() syncs them and returns, per path
// (0 = tcgen05, 1 = SIMT), launches, algorithmic int8 ops (2*m*n*k) and
// summed device milliseconds.
void count_launch(std::int64_t n = 1);
std::int64_t launch_count(bool reset);
void set_profile(bool on);
bool profile_on();
void profile_take(std::int64_t launches[2], double ops[2], double ms[2]);
// Kernel families timed by the profiler (bench.py's roofline lines): the
// work unit is int8 ops (2*m*n*k) for the contractions, algorithmic bytes
// (u8 payload read + written, +4 B per index) for the HBM-bound families.
enum ProfKind : int {
  kProfTc = 0,       // K1 tcgen05 contraction            (ops)
  kProfSimt = 1,     // K1 SIMT / small-K contraction     (ops)
  kProfEchGf2 = 2,   // GF(2) cluster / small ECH kernels (bytes)
  kProfEchPanel = 3, // general-p panel / step ECH kernels (bytes)
  kProfSelect = 4,   // row / column gathers, riffles      (bytes)
  kProfF4 = 5,       // K1f FP4 tcgen05 contraction        (ops)
  kProfKinds = 6
};
// Brackets the launches issued in its scope with CUDA events on `s` when
// profiling is on (a no-op otherwise).
class ProfScope {
 public:
  ProfScope(int kind, double work, cudaStream_t s);
  ~ProfScope();
  void set_kind(int kind) { kind_ = kind; }
  ProfScope(const ProfScope&) = delete;
  ProfScope& operator=(const ProfScope&) = delete;

 private:
  cudaEvent_t e0_ = nullptr, e1_ = nullptr;
  double work_ = 0;
  int kind_ = 0;
  cudaStream_t s_ = nullptr;
};
void profile_take_kinds(int n, std::int64_t* launches, double* work, double* ms, double* union_ms);

// Developer timing of K1 (env GFQ_TC_DEBUG): per-CTA globaltimer stamps of
// the last launch, 148 x 8 u64 (0 start, 1 setup done, 2 first stage
// landed, 3 MMAs issued, 4 first accumulator ready, 5 epilogue done, 6 exit).
void tc_debug_take(unsigned long long* host);

// Selects which path `mad` uses: 0 = auto, 1 = SIMT only, 2 = tcgen05 kind::i8
// whenever legal, 3 = the FP4 path (K1f) whenever legal (else as 2).
void set_mad_policy(int policy);
int mad_policy();
// Counters of K1 launches by path since the last reset (host-side).
void mad_counters(std::int64_t* simt, std::int64_t* tc);
void reset_mad_counters();

// ---------------------------------------------------------------- GF(p^k)
// Extension field GF(q), q = p^k <= 256, elements as encoded bytes
// (sum_i c_i p^i).  Tables live in device memory (FieldSpec::ext()).
struct ExtTables {
  std::uint32_t p, k, q;
  const std::uint8_t* mul;  // q x q products
  const std::uint8_t* add;  // q x q sums
  const std::uint8_t* neg;  // q
  const std::uint8_t* inv;  // q (inv[0] = 0)
  const std::uint8_t* dig;  // q x k base-p digits
  const std::uint8_t* red;  // (2k-1) x k digits of x^s mod the modulus
};
// D = (Cin ? Cin : 0) + A.B over GF(p^k) as ONE K1 contraction over GF(p):
// A (m x K) is split into its digit planes, interleaved (m x kK, column
// k.t + i = digit i of A[., t]); B (K x n) is expanded to the k x k blocks
// of the multiplication-by-element maps (kK x kn: row k.t + i, column
// k.j + u = sum_j' red[i + j'][u] . digit j' of B[t][j], mod p); the
// interleaved digits of Cin are the addend; the m x kn digit result is
// re-encoded into D.  scratch: mad_ext_scratch_bytes() bytes, 16-aligned.
std::int64_t mad_ext_scratch_bytes(std::uint32_t k, std::int64_t m, std::int64_t n, std::int64_t K);
void mad_ext(const ExtTables& f, std::int64_t m, std::int64_t n, std::int64_t K,
             const std::uint8_t* A, std::int64_t lda, const std::uint8_t* B, std::int64_t ldb,
             const std::uint8_t* Cin, std::int64_t ldc, std::uint8_t* D, std::int64_t ldd,
             std::uint8_t* scratch, cudaStream_t s);
// Base-case ECH of ech_base (rows, cols <= kEchBaseMax) over GF(p^k) with
// table arithmetic (mul / add tables staged in shared memory).
void ech_base_ext(const ExtTables& f, std::int64_t rows, std::int64_t cols, const std::uint8_t* H,
                  std::int64_t ldh, std::uint8_t* W, std::int64_t ldw, std::uint8_t* Tc,
                  std::int64_t ldt, std::int32_t* info, cudaStream_t s);

// ---------------------------------------------------------------- wide fields
// GF(p), 251 < p < 2^16, and GF(p^k), 256 < p^k < 2^20: u32 elements
// (wide.cu).  k == 1: prime-field arithmetic; else the log / antilog / Zech
// tables of FieldSpec::wide_dev (exp: q-1, log: q, zech: q-1 entries).
struct WideField {
  std::uint32_t p, k, q;
  const std::uint32_t* exp;
  const std::uint32_t* log;
  const std::int32_t* zech;
};
// D = (Cin ? Cin : 0) + A.B over a wide field (byte strides).
void mad_wide(const WideField& f, std::int64_t m, std::int64_t n, std::int64_t k, const std::uint8_t* A,
              std::int64_t lda, const std::uint8_t* B, std::int64_t ldb, const std::uint8_t* Cin, std::int64_t ldc,
              std::uint8_t* D, std::int64_t ldd, cudaStream_t s);
// ech_base over a wide field (rows, cols <= kEchBaseWideMax).
constexpr int kEchBaseWideMax = 64;
void ech_base_wide(const WideField& f, std::int64_t rows, std::int64_t cols, const std::uint8_t* H, std::int64_t ldh,
                   std::uint8_t* W, std::int64_t ldw, std::uint8_t* Tc, std::int64_t ldt, std::int32_t* info,
                   cudaStream_t s);
// dst (u32 elements)[pos[2q]][pos[2q+1]] = value for q < n.
void set_entries_u32(std::uint8_t* dst, std::int64_t ldd, const std::int32_t* pos, std::int64_t n,
                     std::uint32_t value, cudaStream_t s);
// dst[i][j] = (src[i][j] != 0) (u32 source, u8 mask).
void nonzero_mask_u32(std::int64_t rows, std::int64_t cols, const std::uint8_t* src, std::int64_t lds,
                      std::uint8_t* dst, std::int64_t ldd, cudaStream_t s);
// random_fill for a field of order q stored as u32.
void random_fill_wide(std::uint32_t q, std::int64_t rows, std::int64_t cols, std::uint64_t seed, std::uint64_t draw0,
                      std::int64_t draw_ld, std::uint8_t* dst, std::int64_t ldd, std::uint32_t* rejects,
                      cudaStream_t s);

// ---------------------------------------------------------------- K3/K4
// dst[i][j] = source element chosen by the row map and the column map:
//   rmap[i] >= 0 -> row rmap[i] of A;  rmap[i] <= -2 -> row (-rmap[i]-2) of B;
//   rmap[i] == -1 -> zero row.  rmap == nullptr -> row i of A.
//   cmap[j] likewise for columns (-1 = zero column, <= -2 = column of B).
// Maps are device arrays.  Used for take_rows/take_cols, cex/rex, rrf,
// crz, hcat/vcat and the column riffle.
void select2d(std::uint8_t* dst, std::int64_t ldd, std::int64_t rows,
              std::int64_t cols, const std::uint8_t* A, std::int64_t lda,
              const std::uint8_t* B, std::int64_t ldb, const std::int32_t* rmap,
              const std::int32_t* cmap, cudaStream_t s);

// select2d with HOST maps carried in the launch parameters (int16 entries,
// rows + cols <= 4096; no upload).  Returns false (nothing launched) when
// the maps do not fit or dst is not 16-byte aligned; the caller then
// uploads the maps and calls select2d.
template <int CAP>
struct InlineMaps {
  std::int32_t nr, nc;
  std::int16_t v[CAP];
};
bool select2d_inline(std::uint8_t* dst, std::int64_t ldd, std::int64_t rows, std::int64_t cols,
                     const std::uint8_t* A, std::int64_t lda, const std::uint8_t* B,
                     std::int64_t ldb, const std::int32_t* rmap, const std::int32_t* cmap,
                     cudaStream_t s);

// dst[pos[2q]][pos[2q+1]] = value for q < n  (identity planting, adi).
void set_entries(std::uint8_t* dst, std::int64_t ldd, const std::int32_t* pos,
                 std::int64_t n, std::uint8_t value, cudaStream_t s);

// ---------------------------------------------------------------- bits
// GF(2) transfers (bits.cu): rows x cols byte matrix <-> packed bit rows of
// ceil(cols / 8) bytes (element c at bit c % 8 of byte c / 8).
void pack_bits(const std::uint8_t* src, std::int64_t ld, std::int64_t rows, std::int64_t cols, std::uint8_t* dst,
               std::int64_t ldb, cudaStream_t s);
void unpack_bits(const std::uint8_t* src, std::int64_t ldb, std::int64_t rows, std::int64_t cols, std::uint8_t* dst,
                 std::int64_t ld, cudaStream_t s);

// ---------------------------------------------------------------- K2
// Base-case ECH of a small block (rows, cols <= kEchBaseMax) in one CTA:
// column-wise Gauss-Jordan with the reference's pivot rule (first
// non-pivotal row with a nonzero entry) and -1 pivots.  Writes the reduced
// block W (rows x cols), the compact transform Tc (rows x rank; column q =
// coefficient on the q-th pivot row in discovery order) and
// info = [rank, pivcol_0.., pivrow_0..] (2*min(rows,cols)+1 ints).
constexpr int kEchBaseMax = 128;
// ...and thin blocks (min(rows, cols) <= kEchThinMax, any length) whose
// rows x (cols + min) bytes fit kEchBaseSmem: the Chief's one-column /
// one-row ClearDowns, which the split recursion would cut into ~100 launches
constexpr int kEchThinMax = 32;
constexpr std::size_t kEchBaseSmem = 200 * 1024;
std::size_t ech_base_smem(std::int64_t rows, std::int64_t cols);
bool ech_base_fits(std::int64_t rows, std::int64_t cols);
void ech_base(std::uint32_t p, std::int64_t rows, std::int64_t cols,
              const std::uint8_t* H, std::int64_t ldh, std::uint8_t* W,
              std::int64_t ldw, std::uint8_t* Tc, std::int64_t ldt,
              std::int32_t* info, cudaStream_t s);

// Panel step of the device ECH (right-looking Gauss-Jordan on the augmented
// block Aug = [W | T], rows x (cols + rows), T starting at I).  One CTA:
// finds, among the rows not yet pivotal (flags[i] == 0), the pivots of
// panel columns [c0, c0+wc) with the column-wise rule, and writes
//   G (rows x 32): the panel multipliers, G = Ap.N2 with
//                  Ap = Aug[:, c0 + gamma2] (+ I on the new pivot rows) and
//                  N2 = -inv(Aug[rho2, c0 + gamma2]) (zero padded),
//   rho2 (32):     new pivot rows in discovery order (-1 padded),
// and appends (c0 + gamma2, rho2) to info = [rank, cols[cap], rows[cap]].
// The caller then applies Aug[:, c0:] += G.Aug[rho2, c0:].
// Requires w == 32 and rows * 33 <= kPanelSmem bytes.
constexpr int kPanelSmem = 200 * 1024;
// Bytes the caller allocates (and zeroes) for ech_panel's `flags`: one per
// row plus the persistent window state of the general-p panel kernel.
inline std::int64_t ech_panel_flag_bytes(std::int64_t rows) { return (rows + 15) / 16 * 16 + 16; }
void ech_panel(std::uint32_t p, std::int64_t rows, std::int64_t c0, std::int64_t wc,
               std::int64_t w, const std::uint8_t* Aug, std::int64_t ld, std::uint8_t* flags,
               std::int32_t* info, std::int64_t cap, std::uint8_t* G, std::int64_t ldg,
               std::int32_t* rho2, cudaStream_t s);

// Blocked (two-level) device ECH.  An outer panel of up to 256 columns is
// eliminated in a scratch Z = [X | Y] (X = the panel's columns of Aug, Y
// zero) by 32-wide ech_panel steps; after each step ech_panel_plant sets
// Y[rho2[q], slot] = 1 for the step's new pivots (slot = pivot number -
// *base), so the step's update carries Y along and Y ends as L.e_P for the
// outer panel's row operator L = I + Gout.S_P.  ech_outer_finish turns Y
// into Gout (subtracts the planted units), writes rmap[t] = the t-th new
// pivot row (-1 past the last) for kcols slots and advances *base to the
// rank (and shifts the panel's recorded pivot columns by col0, the outer
// panel's first column: the steps record scratch-local columns); the caller gathers Bt = Aug[rmap, right of the panel] and applies
// the trailing Aug[:, right] += Gout.Bt as ONE deep-K contraction on K1.
// One 32-wide step of an outer panel, as two launches: the pivot chain
// (one CTA; writes rho2 / info / flags, plants the step's Y units, and
// leaves NT, Gpiv and the transposed pivot rows BpT in step_scratch,
// ech_step_scratch_bytes) and the row-parallel update of Z columns
// [c0, c0 + n) (n a multiple of 16, <= 512; Z 16-byte aligned) with dp4a.
// Same result as ech_panel + ech_panel_plant + gather + K1 on those columns.
// chained_prev: the previous launch on s was the step before in the same
// outer panel; chained_next: the next one will be the step after.  Chained
// steps overlap the update of one with the chain of the next (two counters
// at the end of step_scratch, which must start zeroed; GFQ_STEP_OVERLAP=0
// serialises them at the grid boundary instead).  seq: 1, 2, ... over the
// steps that use one step_scratch (the chain's ready flag for its update);
// signalled: how many earlier steps on it had chained_next.
constexpr std::int64_t ech_step_scratch_bytes() { return 2 * 32 * 32 + 512 * 32 + 16; }
void ech_step(std::uint32_t p, std::int64_t rows, std::int64_t c0, std::int64_t wc, std::int64_t n,
              std::uint8_t* Z, std::int64_t ld, std::uint8_t* flags, std::int32_t* info,
              std::int64_t cap, std::int32_t* rho2, std::uint8_t* step_scratch, std::uint8_t* Y,
              const std::int32_t* base, bool chained_prev, bool chained_next, int seq, int signalled,
              cudaStream_t s);
void ech_panel_plant(std::uint8_t* Y, std::int64_t ldy, const std::int32_t* rho2,
                     const std::int32_t* info, const std::int32_t* base, cudaStream_t s);
void ech_outer_finish(std::uint32_t p, std::uint8_t* Y, std::int64_t ldy, std::int64_t kcols,
                      std::int32_t* info, std::int64_t cap, std::int32_t* base,
                      std::int32_t* rmap, std::int64_t col0, cudaStream_t s);
// dst[i][0:wd] = src[i][0:wd], dst[i][wd:width] = 0 (rows 16-byte aligned,
// width % 16 == 0); the two-level ECH's scratch copies, PDL-launched
void copy_cols(std::uint8_t* dst, std::int64_t ldd, const std::uint8_t* src, std::int64_t lds,
               std::int64_t rows, std::int64_t wd, std::int64_t width, cudaStream_t s);

// GF(2) block ECH in one launch (rows <= 1024, cols + rows <= 8192): the
// reduced [W | T] is written to Out (rows x (cols + rows) u8) and the pivots
// to info = [rank, cols[cap], rows[cap]].  scratch holds
// ech_gf2_scratch_words() 32-bit words.  Returns false (nothing launched)
// when the block is outside those limits.
bool ech_gf2_block(std::int64_t rows, std::int64_t cols, const std::uint8_t* H, std::int64_t ldh,
                   std::uint32_t* scratch, std::uint8_t* Out, std::int64_t ldo, std::int32_t* info,
                   std::int64_t cap, cudaStream_t s);
std::int64_t ech_gf2_scratch_words(std::int64_t rows, std::int64_t cols);
// Same contract, cluster-resident (one 8-CTA cluster, distributed shared
// memory): rows <= 1024 and cols + rows <= 8192, no scratch.  Returns false
// (nothing launched) outside those limits or with GFQ_NO_GF2_CLUSTER set.
// With ex (Out == nullptr) the kernel writes the reference's EchResult
// blocks directly: M (cap x cap: rows by pivot order, columns by sorted pivot
// row), K (rows x cap: non-pivot rows in order), R (cap x cols: non-pivot
// columns in order); the caller views the leading r x r / (rows-r) x r /
// r x (cols-r) corners once it has read the rank.
struct EchExtract {
  std::uint8_t *M, *K, *R;
  std::int64_t ldm, ldk, ldr;
  // scratch of the cluster path: packed rows (rows x Wd words) and index maps
  std::uint32_t* P;
  std::int16_t *RS, *QK, *GC;  // rows, rows, cols entries
};
bool ech_gf2_cluster(std::int64_t rows, std::int64_t cols, const std::uint8_t* H, std::int64_t ldh,
                     std::uint8_t* Out, std::int64_t ldo, std::int32_t* info, std::int64_t cap,
                     cudaStream_t s, const EchExtract* ex = nullptr);
// GF(2) ECH of a block with <= 32 rows (any width): one warp, extraction
// outputs as above.  Returns false (nothing launched) outside its limits.
bool ech_gf2_small(std::int64_t rows, std::int64_t cols, const std::uint8_t* H, std::int64_t ldh,
                   std::int32_t* info, std::int64_t cap, cudaStream_t s, const EchExtract& ex);

// One outer panel of the two-level GF(2) ECH in one 8-CTA cluster launch
// (ech_gf2_outer.cu): Z = [X | Y] (rows x 2 ow u8, X = Z[:, 0:wd], Y =
// Z[:, ow:2 ow] zero on entry), rows <= 8192, ow in {256, 512}; leaves Z,
// flags and info exactly as the 32-wide ech_step launches over the panel
// would (then ech_outer_finish).  Returns false (nothing launched) outside
// those limits or with GFQ_NO_GF2_OUTER set.
bool ech_gf2_outer(std::int64_t rows, std::int64_t wd, std::int64_t ow, std::uint8_t* Z, std::int64_t ldz,
                   std::uint8_t* flags, std::int32_t* info, std::int64_t cap, cudaStream_t s);

// dst[0:bytes] = src[0:bytes] by a kernel reading `src` (device address of
// pinned, mapped host memory) over the bus: a host-to-device upload that
// does not go through a copy engine (so it never waits behind a bulk copy).
// 16-byte aligned pointers, bytes a multiple of 4.
void copy_from_mapped(std::uint8_t* dst, const std::uint8_t* src, std::size_t bytes, cudaStream_t s);
// dst (device address of pinned, mapped host memory)[0:bytes] = src[0:bytes]
// by a kernel (a readback without a copy engine); bytes a multiple of 4.
void copy_to_mapped(std::uint8_t* dst, const std::uint8_t* src, std::size_t bytes, cudaStream_t s);
// dst[i][0:width] = value for i < rows, as a kernel (not a copy-engine memset).
void fill2d(std::uint8_t* dst, std::int64_t ldd, std::int64_t rows, std::int64_t width, std::uint8_t value,
            cudaStream_t s);

// dst[rmap[i]] = src[i] for rmap[i] >= 0 (row scatter).
void scatter_rows(std::uint8_t* dst, std::int64_t ldd, std::int64_t rows, std::int64_t cols,
                  const std::uint8_t* src, std::int64_t lds, const std::int32_t* rmap,
                  cudaStream_t s);

// ---------------------------------------------------------------- K6
// Counter-form SplitMix64: entry (r, c) takes draw index
// draw0 + r * draw_ld + c of the stream `seed` and is reduced mod p
// (draw_ld = the full matrix width, so a block column of random_matrix can
// be generated on its own).  Draws that the reference's rejection rule
// would reject are counted in *rejects so the caller can refuse them.
void random_fill(std::uint32_t p, std::int64_t rows, std::int64_t cols,
                 std::uint64_t seed, std::uint64_t draw0, std::int64_t draw_ld,
                 std::uint8_t* dst, std::int64_t ldd, std::uint32_t* rejects, cudaStream_t s);

// ---------------------------------------------------------------- verify
// count_first[0] += #mismatches, count_first[1] = min(first mismatch as
// row * cols + col) (caller initialises [0, ~0]).  mode 0: A == B;
// mode 1: A == 0; mode 2: A == value * I.
void compare(std::int64_t rows, std::int64_t cols, const std::uint8_t* A, std::int64_t lda,
             const std::uint8_t* B, std::int64_t ldb, int mode, std::uint8_t value,
             unsigned long long* count_first, cudaStream_t s);
// Echelon shape of the remnant R (rows x cols): R[r][c] must be 0 whenever
// restcol[c] < pivcol[r] (global column indices).
void echelon_check(std::int64_t rows, std::int64_t cols, const std::uint8_t* R, std::int64_t ldr,
                   const std::int32_t* pivcol, const std::int32_t* restcol,
                   unsigned long long* count_first, cudaStream_t s);

}  // namespace gfq::dev
