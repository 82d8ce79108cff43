/*
 * gfq.h -- C ABI of the B200-native GF(p) RREF + transformation library
 * (libgfq.so).  This is the drop-in boundary for the reference `gfrref`
 * block-elimination path (arXiv 1806.04211): each entry point names the
 * reference interface it replaces (file:line under
 * /root/reference/proj/include/gfrref/).  No torch types: plain pointers,
 * sizes and opaque handles.
 *
 * Conventions
 *  - Residues are uint8_t in 0..p-1, p prime <= 251.  Matrices are dense
 *    row-major with a row stride `ld` in bytes.
 *  - gfq_mat handles are DEVICE-resident (HBM) and immutable once returned;
 *    jobs/tasks return fresh handles the caller frees with gfq_mat_free.
 *    gfq_iset / gfq_bits are small host-side index sets / bit strings.
 *  - Every call is ordered on the calling thread's current CUDA stream
 *    (gfq_set_stream; default: the legacy default stream).  Calls that return
 *    data-dependent shapes (gfq_ech, gfq_clear_down, gfq_echelonize) block
 *    until those shapes are known.
 *  - Return value: GFQ_OK or an error code; gfq_last_error() gives the
 *    message (the reference's exception text for shape errors).  Error codes
 *    map onto the reference CLI exit codes (include/gfrref/cli.hpp:10-13):
 *    GFQ_ERR_INVALID -> 2 (unusable input), GFQ_ERR_RUNTIME -> 3 (task
 *    failed during execution).
 *  - No CPU fallback: without a usable sm_100a device every compute entry
 *    point fails with GFQ_ERR_CUDA.
 */
#ifndef GFQ_H
#define GFQ_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define GFQ_OK 0
#define GFQ_ERR_INVALID 1 /* std::invalid_argument (shape / universe / argument) */
#define GFQ_ERR_RUNTIME 2 /* std::runtime_error (task failure, cycle)           */
#define GFQ_ERR_CUDA 3    /* CUDA runtime / driver failure, no device           */
#define GFQ_ERR_LOGIC 4   /* std::logic_error (e.g. transform not computed)     */
#define GFQ_ERR_DOMAIN 5  /* std::domain_error (inverse of zero)                */

typedef struct gfq_mat gfq_mat;
typedef struct gfq_iset gfq_iset;
typedef struct gfq_bits gfq_bits;
typedef struct gfq_output gfq_output;

/* ------------------------------------------------------------ runtime */
const char* gfq_last_error(void);
int gfq_version(void);
/* Select and initialise a CUDA device (must be sm_100). */
int gfq_init(int device);
/* Order this thread's subsequent calls on `stream` (a cudaStream_t). */
int gfq_set_stream(void* stream);
int gfq_synchronize(void);

/* ------------------------------------------------------------ values */
/* Matrix (reference include/gfrref/matrix.hpp:15-43), device-resident. */
int gfq_mat_upload(int64_t rows, int64_t cols, const uint8_t* host, int64_t ld, gfq_mat** out);
/* Wide fields (GF(p), p > 251; GF(p^k), p^k > 256) store u32 elements:
 * gfq_mat_upload32 takes a host u32 array with row stride ld ELEMENTS (NULL:
 * zeros); gfq_mat_esize reports 1 (u8) or 4 (u32); gfq_mat_download and
 * gfq_mat_device_ptr strides are in bytes. */
int gfq_mat_upload32(int64_t rows, int64_t cols, const uint32_t* host, int64_t ld, gfq_mat** out);
int gfq_mat_esize(const gfq_mat* m, int* esize);
int gfq_mat_copy_device(int64_t rows, int64_t cols, const uint8_t* dev, int64_t ld,
                        gfq_mat** out);
int gfq_mat_shape(const gfq_mat* m, int64_t* rows, int64_t* cols);
int gfq_mat_download(const gfq_mat* m, uint8_t* host, int64_t ld);
int gfq_mat_device_ptr(const gfq_mat* m, uint8_t** ptr, int64_t* ld);
void gfq_mat_free(gfq_mat* m);
/* IndexSet (matrix.hpp:53-70) and BitString (matrix.hpp:75-87). */
int gfq_iset_create(uint64_t universe, const uint32_t* members, uint64_t n, gfq_iset** out);
int gfq_iset_get(const gfq_iset* s, uint64_t* universe, uint64_t* n, uint32_t* members);
void gfq_iset_free(gfq_iset* s);
int gfq_bits_create(const uint8_t* bits, uint64_t n, gfq_bits** out);
int gfq_bits_get(const gfq_bits* b, uint64_t* n, uint8_t* bits);
void gfq_bits_free(gfq_bits* b);

/* ------------------------------------------------------------ kernels */
/* K1: D = (Cin ? Cin : 0) + A.B mod p on raw device pointers
 * (replaces mul_add_kernel, src/matrix.cpp:81-133).  Cin may alias D. */
int gfq_mad_raw(uint32_t p, int64_t m, int64_t n, int64_t k, const uint8_t* A, int64_t lda,
                const uint8_t* B, int64_t ldb, const uint8_t* Cin, int64_t ldc, uint8_t* D,
                int64_t ldd);
/* K1 path policy: 0 auto, 1 SIMT only, 2 tcgen05 kind::i8 whenever TMA-legal,
 * 3 the FP4 tcgen05 path (kind::mxf4, p in {2,3,5,7}) whenever legal. */
int gfq_set_mad_policy(int policy);
int gfq_mad_counters(int64_t* simt_launches, int64_t* tc_launches, int reset);
/* K6: exact device replica of random_matrix / random_product_matrix
 * (include/gfrref/generate.hpp:33-39, src/generate.cpp:16-38). */
int gfq_random_matrix(uint32_t p, int64_t rows, int64_t cols, uint64_t seed, gfq_mat** out);
/* Fields.  Every entry point's `p` is a field code: a prime p < 2^16 is
 * GF(p) itself; gfq_field_register returns the code (>= 0x10000) of
 * GF(p^k), p^k < 2^20, with the given monic irreducible modulus c0..ck
 * (n_modulus = k + 1; NULL / 0: the reference's default modulus), the
 * reference's FieldSpec(p, k, modulus) (include/gfrref/field.hpp:24-30,
 * src/field.cpp:143-149).  Elements are encoded like the reference,
 * sum_i c_i p^i: one byte each for p <= 251 / p^k <= 256 (the tensor-core
 * path), u32 for the wider fields (gfq_mat_upload32 / gfq_mat_esize). */
int gfq_field_register(uint32_t p, uint32_t k, const uint32_t* modulus, int n_modulus,
                       uint32_t* code);
/* p, k, q = p^k and the modulus (k + 1 coefficients; {0, 1} for k = 1). */
int gfq_field_info(uint32_t code, uint32_t* p, uint32_t* k, uint32_t* q, uint32_t* modulus);
/* Host field arithmetic (reference FieldSpec add / mul / neg / inv,
 * include/gfrref/field.hpp:45-88): op 0 add, 1 mul, 2 neg(a), 3 inv(a). */
int gfq_field_op(uint32_t code, int op, uint32_t a, uint32_t b, uint32_t* out);
/* Reference default_modulus (include/gfrref/field.hpp:118): k + 1 coefficients. */
int gfq_default_modulus(uint32_t p, uint32_t k, uint32_t* modulus);
int gfq_random_product_matrix(uint32_t p, int64_t rows, int64_t cols, int64_t inner,
                              uint64_t seed, gfq_mat** out);
/* Reserve the stream-ordered device pool for an m x n echelonize (every
 * echelonize does this itself; calling it once up front keeps the one-time
 * mapping of physical memory out of the first call). */
int gfq_reserve_for(int64_t m, int64_t n, int with_transform);
/* Developer check (no reference counterpart): bit 0 fills every device
 * allocation with 0xA5, bit 1 every freed block with 0x5A, each on its
 * stream, so reads of never-written or released memory change results. */
int gfq_set_poison(int mode);
/* Base-case size of the device ECH recursion (<= 128; results unaffected). */
int gfq_set_ech_base(uint64_t n);
/* ECH algorithm: 0 = device ECH (default; GF(2) blocks beyond the whole-block
 * cluster kernel split by the reference's rule down to it), 1 = the
 * reference's split/combine recursion (src/jobs.cpp:202-225) over the small
 * base kernel, 2 = as 0 but tall GF(2) blocks on the two-level path with
 * single-CTA panel steps, 3 = as 0, 4 = as 0 but GF(2) blocks beyond the
 * whole-block cluster kernel (up to 8192 rows) on the two-level path with
 * one cluster launch per outer panel.  Same outputs. */
int gfq_set_ech_mode(int mode);
/* Outer panel width of the two-level device ECH: -1 = automatic (default),
 * 0 = one level (32-wide steps over all of [W | T]), else 32..256 (rounded
 * down to a multiple of 32).  Same outputs. */
int gfq_set_ech_outer(int width);
/* Accounting: kernel launches issued by this library (optionally reset),
 * and K1 per-launch device timing (CUDA events on the launch stream).
 * gfq_profile_take returns, for [0] = tcgen05 path and [1] = SIMT path,
 * launches, algorithmic int8 ops (2*m*n*k) and summed device ms. */
int gfq_launch_count(int reset, int64_t* launches);
int gfq_profile(int on);
int gfq_profile_take(int64_t* launches2, double* ops2, double* ms2);
/* HBM accounting: bytes held by live device matrices / scratch (the
 * library's own allocations), their high-water mark since the last reset,
 * and the stream-ordered pool's reserved high-water. */
int gfq_device_memory(int reset_peak, int64_t* live, int64_t* peak, int64_t* pool_reserved);
/* The same per kernel family (n <= 5): [0] K1 tcgen05, [1] K1 SIMT (work =
 * int8 ops), [2] GF(2) cluster ECH, [3] general-p panel/step ECH, [4]
 * gathers/riffles (work = algorithmic bytes read + written); ms = summed
 * per-launch event time, union_ms (may be NULL) = the time any launch of
 * the family was running (concurrent launches counted once). */
int gfq_profile_take_kinds(int n, int64_t* launches, double* work, double* ms, double* union_ms);
/* Developer timing of the last K1 tcgen05 launch when the process runs with
 * GFQ_TC_DEBUG set: 148 x 8 globaltimer stamps per CTA (0 start, 1 setup,
 * 2 first stage landed, 3 MMAs issued, 4 accumulator ready, 5 epilogue
 * done, 6 exit); zeros otherwise. */
int gfq_tc_debug_take(uint64_t* stamps);

/* ------------------------------------------------------------ jobs (jobs.hpp:37-82) */
int gfq_mul(uint32_t p, const gfq_mat* b, const gfq_mat* c, gfq_mat** out);            /* :40 */
int gfq_mad(uint32_t p, const gfq_mat* a, const gfq_mat* b, const gfq_mat* c,
            gfq_mat** out);                                                           /* :43 */
int gfq_ech(uint32_t p, const gfq_mat* h, uint64_t threshold, gfq_mat** M, gfq_mat** K,
            gfq_mat** R, gfq_iset** rho, gfq_iset** gamma);                           /* :50 */
int gfq_cex(const gfq_mat* h, const gfq_iset* gamma, gfq_mat** sel, gfq_mat** rest); /* :53 */
int gfq_rex(const gfq_mat* h, const gfq_iset* rho, gfq_mat** sel, gfq_mat** rest);   /* :56 */
int gfq_unh(const gfq_iset* rho1, const gfq_iset* rho2, gfq_iset** rho, gfq_bits** u); /* :61 */
int gfq_un0(const gfq_iset* rho2, gfq_iset** rho, gfq_bits** u);                     /* :64 */
int gfq_mkr(const gfq_iset* rho1, const gfq_iset* rho2, gfq_bits** out);             /* :68 */
int gfq_rrf(const gfq_bits* u, const gfq_mat* b, const gfq_mat* c, gfq_mat** out);   /* :72 */
int gfq_crz(const gfq_mat* m, const gfq_bits* lambda, uint64_t out_cols, gfq_mat** out); /* :77 */
int gfq_adi(const gfq_mat* k, const gfq_bits* delta, gfq_mat** out);                 /* :82 */

/* ------------------------------------------------------------ packages / tasks (tasks.hpp:19-59) */
/* PkgA (packages.hpp:17-26): A, E, lambda are NULL for a first-row package. */
typedef struct gfq_pkgA {
  gfq_mat* A;
  gfq_mat* M;
  gfq_mat* K;
  gfq_iset* rho_prime;
  gfq_mat* E;
  gfq_bits* lambda;
} gfq_pkgA;
/* PkgD (packages.hpp:30-36) */
typedef struct gfq_pkgD {
  gfq_mat* R;
  gfq_iset* gamma;
} gfq_pkgD;
/* PkgE (packages.hpp:40-45) */
typedef struct gfq_pkgE {
  gfq_iset* rho;
  gfq_bits* delta;
} gfq_pkgE;

int gfq_clear_down(uint32_t p, const gfq_mat* C, const gfq_pkgD* D, uint64_t i,
                   uint64_t ech_threshold, gfq_pkgD* D_out, gfq_pkgA* A_out); /* :19 */
int gfq_update_row(uint32_t p, const gfq_pkgA* A, const gfq_mat* C, const gfq_mat* B,
                   uint64_t i, gfq_mat** C_out, gfq_mat** B_out);            /* :26 (B NULL iff i==0) */
int gfq_update_row_trafo(uint32_t p, const gfq_pkgA* A, const gfq_mat* K, const gfq_mat* M,
                         const gfq_pkgE* E, uint64_t i, uint64_t h, uint64_t j,
                         gfq_mat** K_out, gfq_mat** M_out);                  /* :36 */
int gfq_extend(const gfq_pkgA* A, const gfq_pkgE* E, uint64_t j, gfq_pkgE* E_out); /* :44 */
int gfq_row_lengthen(const gfq_mat* M, const gfq_pkgE* E1, const gfq_pkgE* E2,
                     gfq_mat** out);                                         /* :48 */
int gfq_pre_clear_up(const gfq_mat* B, const gfq_pkgD* D, gfq_mat** X, gfq_mat** R); /* :52 */
int gfq_clear_up(uint32_t p, const gfq_mat* R, const gfq_mat* X, const gfq_mat* M,
                 gfq_mat** out);                                             /* :55 */
int gfq_copy_d(const gfq_pkgD* D, gfq_mat** out);                            /* :58 */
void gfq_pkgA_free(gfq_pkgA* a);
void gfq_pkgD_free(gfq_pkgD* d);
void gfq_pkgE_free(gfq_pkgE* e);

/* ------------------------------------------------------------ chief (chief.hpp:27-105) */
/* ChopMatrix (chief.hpp:27).  Either parts array may be NULL (query counts). */
int gfq_chop(uint64_t m, uint64_t n, uint64_t block, int remainder_first, uint64_t* row_parts,
             uint64_t* a, uint64_t* col_parts, uint64_t* b);

/* EchelonizeOptions (chief.hpp:76-84); `threads` = host workers, each
 * driving its own CUDA stream. */
typedef struct gfq_options {
  uint64_t block;
  int threads;
  int with_transform;
  uint64_t ech_threshold;
  int remainder_first;
  int collect_trace;
  int retain_all;
  int fuse;  /* 1 (default): wide UpdateRow / ClearUp jobs per panel (single GPU);
                0: the reference's per-block task grid */
} gfq_options;
void gfq_options_default(gfq_options* o);

/* RunReport (scheduler.hpp:100-107) */
typedef struct gfq_report {
  int64_t wall_ns;
  int64_t peak_live_bytes;
  int64_t initial_live_bytes;
  int64_t tasks;
  int workers;
} gfq_report;

/* echelonize (chief.hpp:88-90) on a device-resident input. */
int gfq_echelonize(uint32_t p, const gfq_mat* C, const gfq_options* opt, gfq_output** out);
/* Same, input in host memory (copied to HBM inside the call). */
int gfq_echelonize_host(uint32_t p, int64_t m, int64_t n, const uint8_t* C, int64_t ld,
                        const gfq_options* opt, gfq_output** out);
/* Same, and every output block also lands in host_out (gfq_output_download_blocks'
 * layout, cap bytes; pinned memory recommended): each block is copied as soon
 * as it is final, so the download overlaps the back-substitution (Step 3).
 * The buffer is complete when the call returns. */
int gfq_echelonize_host_into(uint32_t p, int64_t m, int64_t n, const uint8_t* C, int64_t ld,
                             const gfq_options* opt, uint8_t* host_out, uint64_t cap,
                             gfq_output** out);
/* Optional (off by default; GFQ_HOST_PACK=1 or gfq_set_host_pack(1)): GF(2)
 * host buffers cross PCIe packed 8:1 -- host threads pack C before its
 * upload and unpack the downloaded blocks into host_out.  Pays where host
 * memory bandwidth well exceeds PCIe's.  on = N >= 2 (GFQ_HOST_PACK=N) is the
 * hybrid: every N-th input block row and output block goes packed, the
 * others as byte copies, so the host's packing runs beside the PCIe copies
 * of the neighbours.  The bytes that crossed PCIe in the calling thread's
 * last gfq_echelonize_host / _host_into call: */
int gfq_set_host_pack(int on);
int gfq_last_transfer_bytes(int64_t* h2d, int64_t* d2h);

int gfq_output_rank(const gfq_output* o, uint64_t* rank);
int gfq_output_grid(const gfq_output* o, uint64_t* a, uint64_t* b);
/* which: 0 = upsilon[x] (pivot columns of block column x),
 *        1 = varrho[x]  (selected rows of block row x).  buf may be NULL. */
int gfq_output_select(const gfq_output* o, int which, uint64_t x, uint32_t* buf, uint64_t* count);
/* kind: 0 = R_blocks[x][y] (y >= x), 1 = T_M_blocks[x][y], 2 = T_K_blocks[x][y] (y <= x).
 * Returns a handle sharing the output's storage (free with gfq_mat_free). */
int gfq_output_block(const gfq_output* o, int kind, uint64_t x, uint64_t y, gfq_mat** blk);
/* EchelonOutput::assembled_R (chief.hpp:55) and materialize_transform (:100). */
int gfq_output_assembled_R(const gfq_output* o, gfq_mat** out);
int gfq_output_transform(const gfq_output* o, gfq_mat** out);
/* Bytes of all R / T_M / T_K blocks, and a D2H copy of them into one host
 * buffer, blocks packed row-major (ld = cols) in the order R[j][l>=j],
 * T_M[j][h], T_K[i][h<=i]. */
int gfq_output_block_bytes(const gfq_output* o, uint64_t* bytes);
int gfq_output_download_blocks(const gfq_output* o, uint8_t* host, uint64_t cap);
int gfq_output_report(const gfq_output* o, gfq_report* rep);
/* Trace: count, then arrays (each may be NULL) of kind, i, j, k, worker,
 * start_ns, end_ns, detail (ClearDown: r'). */
int gfq_output_trace(const gfq_output* o, uint64_t* n, int32_t* kind, int32_t* i, int32_t* j,
                     int32_t* k, int32_t* worker, int64_t* start_ns, int64_t* end_ns,
                     int32_t* detail);
/* Device window of each trace record (same order as gfq_output_trace): ns
 * from the run's start on the device to the task's stream reaching its
 * first kernel, and to its last kernel completing; -1 when unavailable. */
int gfq_output_trace_device(const gfq_output* o, uint64_t* n, int64_t* dev_start_ns,
                            int64_t* dev_end_ns);
/* Live package bytes right after each trace record's task (TraceRecord::
 * live_bytes, include/gfrref/scheduler.hpp:90), same order. */
int gfq_output_trace_live(const gfq_output* o, uint64_t* n, int64_t* live_bytes);
void gfq_output_free(gfq_output* o);

/* ------------------------------------------------------------ text I/O */
/* The reference's GFMAT v1 / SELECTS v1 / TRANSFORM v1 files, byte-identical
 * (include/gfrref/io.hpp:17-45; src/io.cpp:199-286), prime fields only.
 * Malformed input -> GFQ_ERR_INVALID with "file:line: message". */
int gfq_read_gfmat_file(const char* path, uint32_t* p, gfq_mat** out);
int gfq_write_gfmat_file(const char* path, uint32_t p, const gfq_mat* m);
int gfq_output_write_selects_file(const gfq_output* o, const char* path);
int gfq_output_write_transform_file(const gfq_output* o, const char* path);

/* gfrref::verify (src/chief.cpp:531-590) on the device, without the oracle
 * argument.  C is the device-resident input the output was computed from
 * (a sharded output must have been gathered).  method: 0 = auto (exact when
 * T, C and T.C fit in half the free HBM, else Freivalds), 1 = exact (T
 * materialised, T.C compared entry by entry), 2 = Freivalds (T.(C.X) vs
 * E.X for a seeded random n x 64 X, from T's blocks; false-accept
 * probability <= p^-64).  Without the transform the row-space containment
 * C[:,rest] + C[:,pivots].R == 0 is checked instead.  Always checks the
 * select sets against the rank and the echelon shape of R.  *ok = 1 when
 * every check passed; else diag (may be NULL) receives the first failure,
 * NUL-terminated and truncated to diag_len.  checked (may be NULL)
 * receives the check actually run ("exact" / "freivalds" / "row-space"). */
int gfq_verify(const gfq_output* o, const gfq_mat* C, int method, uint64_t seed, int* ok,
               char* diag, size_t diag_len, char* checked, size_t checked_len);

/* ------------------------------------------------------------ multi-GPU */
/* Block columns of C (and T) are sharded cyclically over the ranks; PkgA and
 * X packages are broadcast in one fixed order.  One process per GPU with an
 * NCCL communicator, or `world` in-process loopback ranks on one GPU. */
typedef struct gfq_comm gfq_comm;
int gfq_nccl_unique_id(uint8_t* out128);
int gfq_comm_nccl(int world, int rank, const uint8_t* id128, gfq_comm** out);
/* Fills comms[0..world-1]; each must be driven by its own host thread. */
int gfq_comm_loopback(int world, gfq_comm** comms);
void gfq_comm_free(gfq_comm* c);
/* C: the full device-resident input (only owned block columns are read) or
 * NULL to generate the owned columns of random_matrix(p, m, n, seed) on the
 * device.  gather != 0 makes the output complete on every rank. */
int gfq_echelonize_dist(gfq_comm* comm, uint32_t p, const gfq_mat* C, int64_t m, int64_t n,
                        uint64_t seed, const gfq_options* opt, int gather, gfq_output** out);
/* Host-only view of the sharded plan: per node (kind, i, j, k, owner; owner
 * -1 = every rank) and the broadcast schedule (is_a, i, j, k, root), in
 * order.  Either array may be NULL to query the counts. */
int gfq_dist_plan(uint64_t m, uint64_t n, uint64_t block, int with_transform, int world,
                  int32_t* nodes, uint64_t* n_nodes, int32_t* bcasts, uint64_t* n_bcast);

#ifdef __cplusplus
}
#endif
#endif /* GFQ_H */
