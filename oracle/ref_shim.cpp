// ref_shim.cpp -- TEST INFRASTRUCTURE ONLY.
//
// A thin extern "C" shim over the *unmodified* reference library
// (/root/reference/proj/src/*.cpp, compiled where it lies by oracle/Makefile
// into oracle/_ref/libgfrref_ref.so).  It lets the Python tests and
// bench.py's reference arm call the reference's own entry points:
//   gfrref::random_matrix / random_product_matrix  (src/generate.cpp:16-38)
//   gfrref::mat_mul_add                             (src/matrix.cpp:137-144)
//   gfrref::ech                                     (src/jobs.cpp:202-225)
//   gfrref::oracle_rref                             (src/chief.cpp:427-487)
//   gfrref::echelonize                              (src/chief.cpp:322-386)
//   gfrref::materialize_transform / verify          (src/chief.cpp:489-590)
// No reference source is copied into this repository.
#include <chrono>
#include <cstdint>
#include <cstring>
#include <exception>
#include <string>
#include <thread>
#include <vector>

#include "gfrref/chief.hpp"
#include "gfrref/generate.hpp"
#include "gfrref/jobs.hpp"
#include "gfrref/matrix.hpp"

using namespace gfrref;

namespace {
thread_local std::string g_err;
// element width of every buffer crossing the shim: 1 (u8) or 4 (u32, the
// wide fields); leading dimensions stay in elements
int g_elem_bytes = 1;

Matrix from_u8(std::size_t rows, std::size_t cols, const std::uint8_t* src,
               std::size_t ld) {
  Matrix m(rows, cols);
  for (std::size_t r = 0; r < rows; ++r)
    for (std::size_t c = 0; c < cols; ++c)
      m.at(r, c) = g_elem_bytes == 4 ? reinterpret_cast<const std::uint32_t*>(src)[r * ld + c]
                                     : src[r * ld + c];
  return m;
}

void to_u8(const Matrix& m, std::uint8_t* dst, std::size_t ld) {
  for (std::size_t r = 0; r < m.rows(); ++r)
    for (std::size_t c = 0; c < m.cols(); ++c) {
      if (g_elem_bytes == 4)
        reinterpret_cast<std::uint32_t*>(dst)[r * ld + c] = static_cast<std::uint32_t>(m.at(r, c));
      else
        dst[r * ld + c] = static_cast<std::uint8_t>(m.at(r, c));
    }
}

// Field codes: p for GF(p); 0x10000 + i for the i-th field registered with
// ref_field_register (the reference's FieldSpec(p, k, modulus)).
std::vector<FieldSpec>& ext_fields() {
  static std::vector<FieldSpec> v;
  return v;
}
FieldSpec fs(std::uint32_t code) {
  if (code >= 0x10000u) return ext_fields().at(code - 0x10000u);
  return FieldSpec(code);
}

struct RefOut {
  EchelonOutput out;
  explicit RefOut(EchelonOutput o) : out(std::move(o)) {}
};
}  // namespace

extern "C" {

const char* ref_last_error() { return g_err.c_str(); }

// 1: u8 matrix buffers (default), 4: u32 (fields beyond u8 elements)
void ref_set_elem_bytes(int bytes) { g_elem_bytes = bytes == 4 ? 4 : 1; }

std::uint32_t ref_field_register(std::uint32_t p, std::uint32_t k, const std::uint32_t* mod,
                                 std::size_t n) {
  try {
    std::vector<std::uint32_t> m;
    if (mod) m.assign(mod, mod + n);
    FieldSpec f(p, k, m);
    auto& v = ext_fields();
    for (std::size_t i = 0; i < v.size(); ++i)
      if (v[i] == f) return std::uint32_t(0x10000u + i);
    v.push_back(f);
    return std::uint32_t(0x10000u + v.size() - 1);
  } catch (const std::exception& e) {
    g_err = e.what();
    return 0;
  }
}

std::uint32_t ref_field_op(std::uint32_t code, int op, std::uint32_t a, std::uint32_t b) {
  const FieldSpec f = fs(code);
  switch (op) {
    case 0: return f.add(a, b);
    case 1: return f.mul(a, b);
    case 2: return f.neg(a);
    default: return f.inv(a);
  }
}

void ref_default_modulus(std::uint32_t p, std::uint32_t k, std::uint32_t* out) {
  const auto m = default_modulus(p, k);
  for (std::size_t i = 0; i < m.size(); ++i) out[i] = m[i];
}

int ref_hardware_concurrency() {
  return static_cast<int>(std::thread::hardware_concurrency());
}

void ref_random_matrix(std::uint32_t p, std::size_t rows, std::size_t cols,
                       std::uint64_t seed, std::uint8_t* out, std::size_t ld) {
  to_u8(random_matrix(fs(p), rows, cols, seed), out, ld);
}

void ref_random_product_matrix(std::uint32_t p, std::size_t rows,
                               std::size_t cols, std::size_t inner,
                               std::uint64_t seed, std::uint8_t* out,
                               std::size_t ld) {
  to_u8(random_product_matrix(fs(p), rows, cols, inner, seed), out, ld);
}

int ref_mad(std::uint32_t p, std::size_t m, std::size_t k, std::size_t n,
            const std::uint8_t* A, std::size_t lda, const std::uint8_t* B,
            std::size_t ldb, const std::uint8_t* Cin, std::size_t ldc,
            std::uint8_t* D, std::size_t ldd) {
  try {
    const FieldSpec f = fs(p);
    const Matrix a = from_u8(m, k, A, lda), b = from_u8(k, n, B, ldb);
    const Matrix out = Cin ? mat_mul_add(f, from_u8(m, n, Cin, ldc), a, b)
                           : mat_mul(f, a, b);
    to_u8(out, D, ldd);
    return 0;
  } catch (const std::exception& e) {
    g_err = e.what();
    return 1;
  }
}

static std::int64_t put_ech(const EchResult& e, std::uint32_t* rho,
                            std::uint32_t* gamma, std::uint8_t* M,
                            std::uint8_t* K, std::uint8_t* R) {
  const std::size_t r = e.rank();
  for (std::size_t q = 0; q < r; ++q) rho[q] = e.rho.members[q];
  for (std::size_t q = 0; q < r; ++q) gamma[q] = e.gamma.members[q];
  to_u8(e.M, M, e.M.cols());
  to_u8(e.K, K, e.K.cols());
  to_u8(e.R, R, e.R.cols());
  return static_cast<std::int64_t>(r);
}

std::int64_t ref_ech(std::uint32_t p, std::size_t m, std::size_t n,
                     const std::uint8_t* H, std::size_t ld,
                     std::size_t threshold, std::uint32_t* rho,
                     std::uint32_t* gamma, std::uint8_t* M, std::uint8_t* K,
                     std::uint8_t* R) {
  try {
    return put_ech(ech(fs(p), from_u8(m, n, H, ld), threshold), rho,
                   gamma, M, K, R);
  } catch (const std::exception& e) {
    g_err = e.what();
    return -1;
  }
}

std::int64_t ref_oracle_rref(std::uint32_t p, std::size_t m, std::size_t n,
                             const std::uint8_t* C, std::size_t ld,
                             std::uint32_t* rho, std::uint32_t* gamma,
                             std::uint8_t* M, std::uint8_t* K,
                             std::uint8_t* R) {
  try {
    return put_ech(oracle_rref(fs(p), from_u8(m, n, C, ld)), rho, gamma,
                   M, K, R);
  } catch (const std::exception& e) {
    g_err = e.what();
    return -1;
  }
}

// Runs gfrref::echelonize; *wall_s receives the seconds spent inside the
// call (chop + plan + run + assembly), *run_s the scheduler's own wall_ns.
void* ref_echelonize(std::uint32_t p, std::size_t m, std::size_t n,
                     const std::uint8_t* C, std::size_t ld, std::size_t block,
                     int threads, int with_transform, std::size_t threshold,
                     double* wall_s, double* run_s) {
  try {
    const Matrix c = from_u8(m, n, C, ld);
    EchelonizeOptions o;
    o.block = block;
    o.threads = threads;
    o.with_transform = with_transform != 0;
    o.ech_threshold = threshold;
    RunReport rep;
    const auto t0 = std::chrono::steady_clock::now();
    EchelonOutput out = echelonize(c, fs(p), o, &rep);
    const auto t1 = std::chrono::steady_clock::now();
    if (wall_s) *wall_s = std::chrono::duration<double>(t1 - t0).count();
    if (run_s) *run_s = double(rep.wall_ns) * 1e-9;
    return new RefOut(std::move(out));
  } catch (const std::exception& e) {
    g_err = e.what();
    return nullptr;
  }
}

void ref_out_free(void* h) { delete static_cast<RefOut*>(h); }

std::int64_t ref_out_rank(void* h) {
  return static_cast<std::int64_t>(static_cast<RefOut*>(h)->out.rank);
}
std::int64_t ref_out_a(void* h) {
  return static_cast<std::int64_t>(static_cast<RefOut*>(h)->out.chop.a());
}
std::int64_t ref_out_b(void* h) {
  return static_cast<std::int64_t>(static_cast<RefOut*>(h)->out.chop.b());
}

// which: 0 = upsilon[x], 1 = varrho[x].  Returns the count, fills buf if
// non-null.
std::int64_t ref_out_select(void* h, int which, std::size_t x,
                            std::uint32_t* buf) {
  const EchelonOutput& o = static_cast<RefOut*>(h)->out;
  const IndexSet& s = which == 0 ? o.upsilon.at(x) : o.varrho.at(x);
  if (buf)
    for (std::size_t q = 0; q < s.size(); ++q) buf[q] = s.members[q];
  return static_cast<std::int64_t>(s.size());
}

// kind: 0 = R_blocks[x][y], 1 = T_M_blocks[x][y], 2 = T_K_blocks[x][y].
// Writes shape to rows/cols and, if buf is non-null, the dense data.
int ref_out_block(void* h, int kind, std::size_t x, std::size_t y,
                  std::int64_t* rows, std::int64_t* cols, std::uint8_t* buf) {
  try {
    const EchelonOutput& o = static_cast<RefOut*>(h)->out;
    const Matrix& m = kind == 0   ? o.R_blocks.at(x).at(y)
                      : kind == 1 ? o.T_M_blocks.at(x).at(y)
                                  : o.T_K_blocks.at(x).at(y);
    *rows = static_cast<std::int64_t>(m.rows());
    *cols = static_cast<std::int64_t>(m.cols());
    if (buf) to_u8(m, buf, m.cols());
    return 0;
  } catch (const std::exception& e) {
    g_err = e.what();
    return 1;
  }
}

int ref_out_materialize(void* h, std::uint8_t* buf) {
  try {
    const Matrix t = materialize_transform(static_cast<RefOut*>(h)->out);
    to_u8(t, buf, t.cols());
    return 0;
  } catch (const std::exception& e) {
    g_err = e.what();
    return 1;
  }
}

// Assembled remnant (rank x (n - rank)).
int ref_out_assembled_R(void* h, std::uint8_t* buf) {
  const Matrix r = static_cast<RefOut*>(h)->out.assembled_R();
  to_u8(r, buf, r.cols());
  return 0;
}

int ref_verify(void* h, std::uint32_t p, std::size_t m, std::size_t n,
               const std::uint8_t* C, std::size_t ld) {
  (void)p;
  std::string diag;
  const bool ok =
      verify(from_u8(m, n, C, ld), static_cast<RefOut*>(h)->out, &diag);
  g_err = diag;
  return ok ? 0 : 1;
}

}  // extern "C"
