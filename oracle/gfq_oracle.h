/*
 * gfq_oracle.h -- TEST INFRASTRUCTURE ONLY.
 *
 * A plain-C CPU restatement of the reference algorithm for the GF(p)
 * elimination path (arXiv 1806.04211, reference `gfrref`).  It is the
 * *checker* for the B200 path: only tests/, __graft_entry__.smoke() and
 * bench.py's cpu_baseline leg may load it.  Nothing in the product library
 * (paper_1806_04211_b200/) links or calls it.
 *
 * Parity pin: tests/test_oracle.py checks every function here against the
 * reference's own golden vectors (tests/golden/, values from the reference
 * test suite) and against the reference library compiled from its sources
 * into oracle/_ref/ (oracle/Makefile).
 *
 * Elements are uint8_t residues 0..p-1 (p <= 251 prime); matrices are dense
 * row-major with the given row stride.
 */
#ifndef GFQ_ORACLE_H
#define GFQ_ORACLE_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* SplitMix64 step (reference include/gfrref/generate.hpp:16-21). */
uint64_t gfo_splitmix_next(uint64_t* state);
/* Rejection-sampled uniform draw in [0, bound) (reference src/generate.cpp:5-14). */
uint64_t gfo_below(uint64_t* state, uint64_t bound);

/* random_matrix (reference src/generate.cpp:16-24): one below(q) draw per
 * entry, row-major. */
void gfo_random_matrix(uint32_t p, size_t rows, size_t cols, uint64_t seed,
                       uint8_t* out, size_t ld);

/* random_product_matrix (reference src/generate.cpp:26-38): P (rows x inner)
 * then Q (inner x cols) from one stream, out = P.Q mod p. */
void gfo_random_product_matrix(uint32_t p, size_t rows, size_t cols,
                               size_t inner, uint64_t seed, uint8_t* out,
                               size_t ld);

/* D = (Cin ? Cin : 0) + A.B mod p (reference src/matrix.cpp:81-133, prime
 * path :91-114).  A is m x k, B is k x n, Cin/D are m x n.  D may alias Cin. */
void gfo_mad(uint32_t p, size_t m, size_t k, size_t n, const uint8_t* A,
             size_t lda, const uint8_t* B, size_t ldb, const uint8_t* Cin,
             size_t ldc, uint8_t* D, size_t ldd);

/* Sequential Gauss-Jordan with full transform tracking (reference
 * src/chief.cpp:427-487, `oracle_rref`).  Column-wise pivot rule: the pivot of
 * column c is the first not-yet-pivotal row with a nonzero entry.
 * Outputs (caller-allocated, capacities m for rho, n for gamma, m*m for M,
 * m*m for K, m*n for R; all dense with row stride = their column count):
 *   rho   ascending selected rows (size r)
 *   gamma pivot columns (ascending, size r)
 *   M     r x r      rows by pivot column, columns by ascending rho
 *   K     (m-r) x r  rows by ascending non-selected row
 *   R     r x (n-r)  columns by ascending non-pivot column
 * Returns the rank r (or -1 on allocation failure). */
int64_t gfo_oracle_rref(uint32_t p, size_t m, size_t n, const uint8_t* C,
                        size_t ldc, uint32_t* rho, uint32_t* gamma,
                        uint8_t* M, uint8_t* K, uint8_t* R);

/* Field helpers (reference include/gfrref/field.hpp:45-78, src/field.cpp:220-237). */
uint32_t gfo_inv(uint32_t p, uint32_t a);

/* Fields: every `p` above is a field code -- p for GF(p), or the code
 * gfo_field_ext returns for GF(p^k) (q = p^k <= 256, monic irreducible
 * modulus c0..ck; 0 on failure).  Elements are encoded sum_i c_i p^i. */
uint32_t gfo_field_ext(uint32_t p, uint32_t k, const uint32_t* modulus);
uint32_t gfo_order(uint32_t code);
uint32_t gfo_add(uint32_t code, uint32_t a, uint32_t b);
uint32_t gfo_mul(uint32_t code, uint32_t a, uint32_t b);
uint32_t gfo_neg(uint32_t code, uint32_t a);

#ifdef __cplusplus
}
#endif
#endif
