/*
 * gfq_oracle.c -- TEST INFRASTRUCTURE ONLY (see gfq_oracle.h).
 *
 * Plain-C restatement of the reference's GF(p) arithmetic, generators,
 * block multiply-accumulate and sequential RREF oracle.  Each function cites
 * the reference file:line it restates.  Not linked into the product.
 */
#include "gfq_oracle.h"

#include <stdlib.h>
#include <string.h>

/* ------------------------------------------------------------------ fields
 * A field "code" is p for GF(p) and GFO_EXT0 + i for the i-th extension
 * field registered with gfo_field_ext.  GF(p^k) (q = p^k <= 256) is held as
 * q x q add / mul tables over encoded elements sum_i c_i p^i, built by
 * polynomial arithmetic modulo the modulus (reference src/field.cpp:35-57,
 * 100-107: poly_mod, poly_mulmod, add_by_digits; the reference's log /
 * Zech tables give the same field operations). */
#define GFO_EXT0 0x10000u
#define GFO_MAXEXT 64
typedef struct {
  uint32_t p, k, q;
  uint32_t mod[9];
  uint8_t add[256 * 256], mul[256 * 256];
} gfo_ext;
static gfo_ext* g_ext[GFO_MAXEXT];
static int g_next = 0;

static void poly_mod_c(uint32_t* a, int na, const uint32_t* m, int k, uint32_t p) {
  /* a has na coefficients; reduce by the monic degree-k m in place */
  for (int i = na - 1; i >= k; --i) {
    const uint64_t c = a[i];
    if (!c) continue;
    for (int t = 0; t <= k; ++t) a[i - k + t] = (uint32_t)((a[i - k + t] + (p - m[t]) % p * c) % p);
  }
}

uint32_t gfo_field_ext(uint32_t p, uint32_t k, const uint32_t* mod) {
  for (int i = 0; i < g_next; ++i)
    if (g_ext[i]->p == p && g_ext[i]->k == k && !memcmp(g_ext[i]->mod, mod, (k + 1) * sizeof(uint32_t)))
      return GFO_EXT0 + (uint32_t)i;
  if (g_next >= GFO_MAXEXT || k < 2 || k > 8) return 0;
  gfo_ext* f = (gfo_ext*)calloc(1, sizeof(gfo_ext));
  f->p = p;
  f->k = k;
  f->q = 1;
  for (uint32_t i = 0; i < k; ++i) f->q *= p;
  if (f->q > 256) {
    free(f);
    return 0;
  }
  memcpy(f->mod, mod, (k + 1) * sizeof(uint32_t));
  for (uint32_t a = 0; a < f->q; ++a)
    for (uint32_t b = 0; b < f->q; ++b) {
      uint32_t da[8], db[8], prod[16] = {0};
      uint32_t x = a, y = b;
      for (uint32_t i = 0; i < k; ++i) {
        da[i] = x % p;
        x /= p;
        db[i] = y % p;
        y /= p;
      }
      uint32_t sum = 0, scale = 1;
      for (uint32_t i = 0; i < k; ++i) {
        sum += (da[i] + db[i]) % p * scale;
        scale *= p;
      }
      for (uint32_t i = 0; i < k; ++i)
        for (uint32_t j = 0; j < k; ++j) prod[i + j] = (prod[i + j] + da[i] * db[j]) % p;
      poly_mod_c(prod, (int)(2 * k - 1), f->mod, (int)k, p);
      uint32_t enc = 0;
      for (uint32_t i = k; i-- > 0;) enc = enc * p + prod[i];
      f->add[a * f->q + b] = (uint8_t)sum;
      f->mul[a * f->q + b] = (uint8_t)enc;
    }
  g_ext[g_next] = f;
  return GFO_EXT0 + (uint32_t)g_next++;
}

static const gfo_ext* ext_of(uint32_t code) {
  return code >= GFO_EXT0 ? g_ext[code - GFO_EXT0] : NULL;
}

uint32_t gfo_order(uint32_t code) {
  const gfo_ext* f = ext_of(code);
  return f ? f->q : code;
}

uint32_t gfo_add(uint32_t code, uint32_t a, uint32_t b) {
  const gfo_ext* f = ext_of(code);
  return f ? f->add[a * f->q + b] : (a + b) % code;
}

uint32_t gfo_mul(uint32_t code, uint32_t a, uint32_t b) {
  const gfo_ext* f = ext_of(code);
  return f ? f->mul[a * f->q + b] : (uint32_t)((uint64_t)a * b % code);
}

uint32_t gfo_neg(uint32_t code, uint32_t a) {
  const gfo_ext* f = ext_of(code);
  if (!f) return a == 0 ? 0 : code - a;
  for (uint32_t b = 0; b < f->q; ++b)
    if (f->add[a * f->q + b] == 0) return b;
  return 0;
}

/* reference include/gfrref/generate.hpp:16-21 */
uint64_t gfo_splitmix_next(uint64_t* state) {
  uint64_t z = (*state += 0x9e3779b97f4a7c15ULL);
  z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ULL;
  z = (z ^ (z >> 27)) * 0x94d049bb133111ebULL;
  return z ^ (z >> 31);
}

/* reference src/generate.cpp:5-14 */
uint64_t gfo_below(uint64_t* state, uint64_t bound) {
  if (bound <= 1) return 0;
  const uint64_t limit = UINT64_MAX - UINT64_MAX % bound;
  uint64_t v;
  do {
    v = gfo_splitmix_next(state);
  } while (v >= limit);
  return v % bound;
}

/* reference src/generate.cpp:16-24 */
void gfo_random_matrix(uint32_t p, size_t rows, size_t cols, uint64_t seed,
                       uint8_t* out, size_t ld) {
  uint64_t st = seed;
  const uint32_t q = gfo_order(p);
  for (size_t r = 0; r < rows; ++r)
    for (size_t c = 0; c < cols; ++c)
      out[r * ld + c] = (uint8_t)gfo_below(&st, q);
}

/* reference src/generate.cpp:26-38 */
void gfo_random_product_matrix(uint32_t p, size_t rows, size_t cols,
                               size_t inner, uint64_t seed, uint8_t* out,
                               size_t ld) {
  uint64_t st = seed;
  const uint32_t q = gfo_order(p);
  uint8_t* P = (uint8_t*)malloc(rows * inner + 1);
  uint8_t* Q = (uint8_t*)malloc(inner * cols + 1);
  for (size_t r = 0; r < rows; ++r)
    for (size_t c = 0; c < inner; ++c) P[r * inner + c] = (uint8_t)gfo_below(&st, q);
  for (size_t r = 0; r < inner; ++r)
    for (size_t c = 0; c < cols; ++c) Q[r * cols + c] = (uint8_t)gfo_below(&st, q);
  gfo_mad(p, rows, inner, cols, P, inner, Q, cols, NULL, 0, out, ld);
  free(P);
  free(Q);
}

/* reference src/matrix.cpp:81-133 (prime path :91-114): per output row a
 * 64-bit accumulator over `inner`, zero multipliers skipped, one % p at the
 * end. */
void gfo_mad(uint32_t p, size_t m, size_t k, size_t n, const uint8_t* A,
             size_t lda, const uint8_t* B, size_t ldb, const uint8_t* Cin,
             size_t ldc, uint8_t* D, size_t ldd) {
  if (m == 0 || n == 0) return;
  const gfo_ext* f = ext_of(p);
  if (f) {
    /* reference src/matrix.cpp:116-131: table-driven element operations */
    for (size_t i = 0; i < m; ++i) {
      uint8_t* orow = D + i * ldd;
      for (size_t j = 0; j < n; ++j) orow[j] = Cin ? Cin[i * ldc + j] : 0;
      for (size_t t = 0; t < k; ++t) {
        const uint32_t v = A[i * lda + t];
        if (v == 0) continue;
        const uint8_t* brow = B + t * ldb;
        const uint8_t* mv = f->mul + v * f->q;
        for (size_t j = 0; j < n; ++j) orow[j] = f->add[orow[j] * f->q + mv[brow[j]]];
      }
    }
    return;
  }
  uint64_t* acc = (uint64_t*)malloc(n * sizeof(uint64_t));
  for (size_t i = 0; i < m; ++i) {
    if (Cin)
      for (size_t j = 0; j < n; ++j) acc[j] = Cin[i * ldc + j];
    else
      memset(acc, 0, n * sizeof(uint64_t));
    for (size_t t = 0; t < k; ++t) {
      const uint64_t v = A[i * lda + t];
      if (v == 0) continue;
      const uint8_t* brow = B + t * ldb;
      for (size_t j = 0; j < n; ++j) acc[j] += v * brow[j];
    }
    for (size_t j = 0; j < n; ++j) D[i * ldd + j] = (uint8_t)(acc[j] % p);
  }
  free(acc);
}

/* reference src/field.cpp:220-237 (Fermat inverse a^(p-2)) */
uint32_t gfo_inv(uint32_t p, uint32_t a) {
  const gfo_ext* f = ext_of(p);
  if (f) {
    for (uint32_t b = 1; b < f->q && a; ++b)
      if (f->mul[a * f->q + b] == 1) return b;
    return 0;
  }
  uint64_t r = 1, b = a % p;
  uint32_t e = p - 2;
  while (e) {
    if (e & 1) r = r * b % p;
    b = b * b % p;
    e >>= 1;
  }
  return (uint32_t)r;
}

/* reference src/chief.cpp:427-487 (`oracle_rref`). */
int64_t gfo_oracle_rref(uint32_t p, size_t m, size_t n, const uint8_t* C,
                        size_t ldc, uint32_t* rho, uint32_t* gamma,
                        uint8_t* M, uint8_t* K, uint8_t* R) {
  uint8_t* w = (uint8_t*)malloc(m * n + 1);
  uint8_t* t = (uint8_t*)calloc(m * m + 1, 1);
  uint8_t* is_piv = (uint8_t*)calloc(m + 1, 1);
  uint32_t* prow = (uint32_t*)malloc((m + 1) * sizeof(uint32_t));
  uint32_t* pcol = (uint32_t*)malloc((n + 1) * sizeof(uint32_t));
  /* mul[a*q+b], add[a*q+b] over the field (GF(p) or a registered GF(p^k)) */
  const uint32_t q = gfo_order(p);
  uint8_t* mul = (uint8_t*)malloc((size_t)q * q);
  uint8_t* add = (uint8_t*)malloc((size_t)q * q);
  if (!w || !t || !is_piv || !prow || !pcol || !mul || !add) return -1;
  for (uint32_t a = 0; a < q; ++a)
    for (uint32_t b = 0; b < q; ++b) {
      mul[a * q + b] = (uint8_t)gfo_mul(p, a, b);
      add[a * q + b] = (uint8_t)gfo_add(p, a, b);
    }
  for (size_t i = 0; i < m; ++i) memcpy(w + i * n, C + i * ldc, n);
  for (size_t i = 0; i < m; ++i) t[i * m + i] = 1;

  size_t r = 0;
  for (size_t col = 0; col < n; ++col) {
    size_t sel = m;
    for (size_t row = 0; row < m; ++row)
      if (!is_piv[row] && w[row * n + col] != 0) {
        sel = row;
        break;
      }
    if (sel == m) continue;
    /* scale = -(inv(pivot)) so the pivot entry becomes -1 */
    const uint32_t scale = gfo_neg(p, gfo_inv(p, w[sel * n + col]));
    const uint8_t* ms = mul + (size_t)scale * q;
    uint8_t* ws = w + sel * n;
    uint8_t* ts = t + sel * m;
    for (size_t c = 0; c < n; ++c) ws[c] = ms[ws[c]];
    for (size_t c = 0; c < m; ++c) ts[c] = ms[ts[c]];
    for (size_t row = 0; row < m; ++row) {
      if (row == sel) continue;
      const uint32_t v = w[row * n + col];
      if (v == 0) continue;
      const uint8_t* mv = mul + (size_t)v * q;
      uint8_t* wr = w + row * n;
      uint8_t* tr = t + row * m;
      for (size_t c = 0; c < n; ++c) wr[c] = add[(size_t)wr[c] * q + mv[ws[c]]];
      for (size_t c = 0; c < m; ++c) tr[c] = add[(size_t)tr[c] * q + mv[ts[c]]];
    }
    is_piv[sel] = 1;
    prow[r] = (uint32_t)sel;
    pcol[r] = (uint32_t)col;
    ++r;
  }

  /* rho sorted ascending */
  size_t nr = 0;
  for (size_t row = 0; row < m; ++row)
    if (is_piv[row]) rho[nr++] = (uint32_t)row;
  for (size_t q = 0; q < r; ++q) gamma[q] = pcol[q];
  /* non-pivot columns ascending */
  uint8_t* is_pc = (uint8_t*)calloc(n + 1, 1);
  for (size_t q = 0; q < r; ++q) is_pc[pcol[q]] = 1;
  for (size_t q = 0; q < r; ++q) {
    const size_t row = prow[q];
    for (size_t s = 0; s < r; ++s) M[q * r + s] = t[row * m + rho[s]];
    size_t c2 = 0;
    for (size_t c = 0; c < n; ++c)
      if (!is_pc[c]) R[q * (n - r) + c2++] = w[row * n + c];
  }
  size_t u = 0;
  for (size_t row = 0; row < m; ++row) {
    if (is_piv[row]) continue;
    for (size_t s = 0; s < r; ++s) K[u * r + s] = t[row * m + rho[s]];
    ++u;
  }
  free(is_pc);
  free(w);
  free(t);
  free(is_piv);
  free(prow);
  free(pcol);
  free(mul);
  free(add);
  return (int64_t)r;
}
