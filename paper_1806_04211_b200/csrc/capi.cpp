// capi.cpp -- extern "C" boundary (include/gfq.h) over the C++ host layer.
#include <atomic>
#include <cstring>
#include <memory>
#include <string>

#include "../../include/gfq.h"
#include "host/chief.hpp"
#include "host/hostpack.hpp"
#include "host/dist.hpp"
#include "host/io.hpp"
#include "host/jobs.hpp"
#include "host/tasks.hpp"
#include "host/verify.hpp"
#include "kernels/kernels.hpp"

struct gfq_mat {
  gfq::Mat m;
};
struct gfq_iset {
  gfq::IndexSet s;
};
struct gfq_bits {
  gfq::BitString b;
};
struct gfq_output {
  gfq::EchelonOutput out;
  gfq::RunReport report;
  explicit gfq_output(gfq::EchelonOutput o) : out(std::move(o)) {}
};
struct gfq_comm {
  std::shared_ptr<gfq::Comm> c;
};

namespace {
thread_local std::string g_err;
// the device gfq_init chose; every host thread entering the ABI adopts it
// once (the CUDA runtime's current device is per thread)
std::atomic<int> g_device{-1};
thread_local int t_device = -1;

template <class F>
int guard(F&& f) {
  try {
    const int d = g_device.load(std::memory_order_relaxed);
    if (d >= 0 && t_device != d) {
      GFQ_CUDA(cudaSetDevice(d));
      t_device = d;
    }
    f();
    return GFQ_OK;
  } catch (const std::invalid_argument& e) {
    g_err = e.what();
    return GFQ_ERR_INVALID;
  } catch (const std::domain_error& e) {
    g_err = e.what();
    return GFQ_ERR_DOMAIN;
  } catch (const std::logic_error& e) {
    g_err = e.what();
    return GFQ_ERR_LOGIC;
  } catch (const gfq::CudaError& e) {
    g_err = e.what();
    return GFQ_ERR_CUDA;
  } catch (const std::exception& e) {
    g_err = e.what();
    return GFQ_ERR_RUNTIME;
  }
}

const gfq::Mat& M(const gfq_mat* h) {
  if (!h) throw std::invalid_argument("null matrix handle");
  return h->m;
}
const gfq::IndexSet& S(const gfq_iset* h) {
  if (!h) throw std::invalid_argument("null index-set handle");
  return h->s;
}
const gfq::BitString& B(const gfq_bits* h) {
  if (!h) throw std::invalid_argument("null bit-string handle");
  return h->b;
}
gfq_mat* wrap(gfq::Mat m) { return new gfq_mat{std::move(m)}; }
gfq_iset* wrap(gfq::IndexSet s) { return new gfq_iset{std::move(s)}; }
gfq_bits* wrap(gfq::BitString b) { return new gfq_bits{std::move(b)}; }

void require_device() {
  int n = 0;
  if (cudaGetDeviceCount(&n) != cudaSuccess || n == 0) {
    cudaGetLastError();
    throw gfq::CudaError("no CUDA device: the B200 path has no CPU fallback");
  }
}

gfq::PkgA unpack(const gfq_pkgA* a) {
  if (!a) throw std::invalid_argument("null package A");
  gfq::PkgA p;
  if (a->A) p.A = M(a->A);
  p.M = M(a->M);
  p.K = M(a->K);
  p.rho_prime = S(a->rho_prime);
  if (a->E) p.E = M(a->E);
  if (a->lambda) p.lambda = B(a->lambda);
  return p;
}
void pack(gfq::PkgA&& p, gfq_pkgA* a) {
  a->A = p.A ? wrap(std::move(*p.A)) : nullptr;
  a->M = wrap(std::move(p.M));
  a->K = wrap(std::move(p.K));
  a->rho_prime = wrap(std::move(p.rho_prime));
  a->E = p.E ? wrap(std::move(*p.E)) : nullptr;
  a->lambda = p.lambda ? wrap(std::move(*p.lambda)) : nullptr;
}
gfq::PkgD unpack(const gfq_pkgD* d) {
  if (!d) throw std::invalid_argument("null package D");
  return gfq::PkgD{M(d->R), S(d->gamma)};
}
void pack(gfq::PkgD&& p, gfq_pkgD* d) {
  d->R = wrap(std::move(p.R));
  d->gamma = wrap(std::move(p.gamma));
}
gfq::PkgE unpack(const gfq_pkgE* e) {
  if (!e) throw std::invalid_argument("null package E");
  return gfq::PkgE{S(e->rho), B(e->delta)};
}
void pack(gfq::PkgE&& p, gfq_pkgE* e) {
  e->rho = wrap(std::move(p.rho));
  e->delta = wrap(std::move(p.delta));
}
}  // namespace

extern "C" {

const char* gfq_last_error(void) { return g_err.c_str(); }
int gfq_version(void) { return 1; }

int gfq_init(int device) {
  return guard([&] {
    require_device();
    GFQ_CUDA(cudaSetDevice(device));
    g_device = device;
    t_device = device;
    cudaDeviceProp prop;
    GFQ_CUDA(cudaGetDeviceProperties(&prop, device));
    if (prop.major != 10)
      throw gfq::CudaError("device " + std::string(prop.name) + " is not sm_100 (B200)");
    GFQ_CUDA(cudaFree(nullptr));
    gfq::warm_runtime();
  });
}

int gfq_set_stream(void* stream) {
  return guard([&] { gfq::set_cur_stream(static_cast<cudaStream_t>(stream)); });
}
int gfq_synchronize(void) {
  return guard([&] { GFQ_CUDA(cudaStreamSynchronize(gfq::cur_stream())); });
}

// ---------------------------------------------------------------- values
int gfq_mat_upload(int64_t rows, int64_t cols, const uint8_t* host, int64_t ld, gfq_mat** out) {
  return guard([&] {
    require_device();
    *out = wrap(host ? gfq::Mat::from_host(rows, cols, host, ld) : gfq::Mat::zeros(rows, cols));
  });
}
int gfq_mat_upload32(int64_t rows, int64_t cols, const uint32_t* host, int64_t ld, gfq_mat** out) {
  return guard([&] {
    require_device();
    *out = wrap(host ? gfq::Mat::from_host(rows, cols, reinterpret_cast<const uint8_t*>(host), ld * 4, 4)
                     : gfq::Mat::zeros(rows, cols, 4));
  });
}
int gfq_set_host_pack(int on) {
  return guard([&] { gfq::hostpack::set_stride(on); });
}
int gfq_last_transfer_bytes(int64_t* h2d, int64_t* d2h) {
  return guard([&] {
    *h2d = gfq::hostpack::last_transfer().h2d;
    *d2h = gfq::hostpack::last_transfer().d2h;
  });
}
int gfq_mat_esize(const gfq_mat* m, int* esize) {
  return guard([&] { *esize = M(m).esize(); });
}
int gfq_mat_copy_device(int64_t rows, int64_t cols, const uint8_t* dev, int64_t ld, gfq_mat** out) {
  return guard([&] {
    gfq::Mat m(rows, cols);
    if (!m.empty())
      GFQ_CUDA(cudaMemcpy2DAsync(m.data(), size_t(m.ld()), dev, size_t(ld), size_t(cols),
                                 size_t(rows), cudaMemcpyDeviceToDevice, gfq::cur_stream()));
    *out = wrap(std::move(m));
  });
}
int gfq_mat_shape(const gfq_mat* m, int64_t* rows, int64_t* cols) {
  return guard([&] {
    *rows = M(m).rows();
    *cols = M(m).cols();
  });
}
int gfq_mat_download(const gfq_mat* m, uint8_t* host, int64_t ld) {
  return guard([&] { M(m).to_host(host, ld); });
}
int gfq_mat_device_ptr(const gfq_mat* m, uint8_t** ptr, int64_t* ld) {
  return guard([&] {
    *ptr = M(m).data();
    *ld = M(m).ld();
  });
}
void gfq_mat_free(gfq_mat* m) { delete m; }

int gfq_iset_create(uint64_t universe, const uint32_t* members, uint64_t n, gfq_iset** out) {
  return guard([&] {
    *out = wrap(gfq::IndexSet(size_t(universe), std::vector<uint32_t>(members, members + n)));
  });
}
int gfq_iset_get(const gfq_iset* s, uint64_t* universe, uint64_t* n, uint32_t* members) {
  return guard([&] {
    if (universe) *universe = S(s).universe;
    if (n) *n = S(s).size();
    if (members && S(s).size()) std::memcpy(members, S(s).members.data(), S(s).size() * 4);
  });
}
void gfq_iset_free(gfq_iset* s) { delete s; }
int gfq_bits_create(const uint8_t* bits, uint64_t n, gfq_bits** out) {
  return guard([&] {
    std::vector<uint8_t> v(bits, bits + n);
    for (auto& x : v) x = x ? 1 : 0;
    *out = wrap(gfq::BitString(std::move(v)));
  });
}
int gfq_bits_get(const gfq_bits* b, uint64_t* n, uint8_t* bits) {
  return guard([&] {
    if (n) *n = B(b).size();
    if (bits && B(b).size()) std::memcpy(bits, B(b).bits.data(), B(b).size());
  });
}
void gfq_bits_free(gfq_bits* b) { delete b; }

// ---------------------------------------------------------------- kernels
int gfq_mad_raw(uint32_t p, int64_t m, int64_t n, int64_t k, const uint8_t* A, int64_t lda,
                const uint8_t* Bm, int64_t ldb, const uint8_t* Cin, int64_t ldc, uint8_t* D,
                int64_t ldd) {
  return guard([&] {
    gfq::FieldSpec f(p);
    gfq::field_mad(f, m, n, k, A, lda, Bm, ldb, Cin, ldc, D, ldd, gfq::cur_stream());
  });
}
int gfq_set_mad_policy(int policy) { return guard([&] { gfq::dev::set_mad_policy(policy); }); }
int gfq_mad_counters(int64_t* simt, int64_t* tc, int reset) {
  return guard([&] {
    gfq::dev::mad_counters(simt, tc);
    if (reset) gfq::dev::reset_mad_counters();
  });
}

namespace {
// one below(q) draw per entry of the reference stream (src/generate.cpp:16-24);
// `p` is a field code, q its order
void fill_exact(uint32_t p, int64_t rows, int64_t cols, uint64_t seed, uint64_t draw0,
                uint8_t* dst, int64_t ld) {
  const gfq::FieldSpec f(p);
  gfq::random_fill_exact(f.order(), rows, cols, seed, draw0, cols, dst, ld, f.esize());
}
}  // namespace

// ---------------------------------------------------------------- fields
int gfq_field_register(uint32_t p, uint32_t k, const uint32_t* modulus, int n_modulus,
                       uint32_t* code) {
  return guard([&] {
    if (!code) throw std::invalid_argument("gfq_field_register: null output");
    std::vector<uint32_t> mod;
    if (modulus && n_modulus > 0) mod.assign(modulus, modulus + n_modulus);
    *code = gfq::FieldSpec(p, k, mod).code();
  });
}
int gfq_field_info(uint32_t code, uint32_t* p, uint32_t* k, uint32_t* q, uint32_t* modulus) {
  return guard([&] {
    const gfq::FieldSpec f(code);
    if (p) *p = f.p();
    if (k) *k = f.k();
    if (q) *q = f.order();
    if (modulus)
      for (std::size_t i = 0; i < f.modulus().size(); ++i) modulus[i] = f.modulus()[i];
  });
}
int gfq_field_op(uint32_t code, int op, uint32_t a, uint32_t b, uint32_t* out) {
  return guard([&] {
    const gfq::FieldSpec f(code);
    if (a >= f.order() || b >= f.order()) throw std::invalid_argument("field: element out of range");
    switch (op) {
      case 0: *out = f.add(a, b); break;
      case 1: *out = f.mul(a, b); break;
      case 2: *out = f.neg(a); break;
      case 3: *out = f.inv(a); break;
      default: throw std::invalid_argument("gfq_field_op: op must be 0..3");
    }
  });
}
int gfq_default_modulus(uint32_t p, uint32_t k, uint32_t* modulus) {
  return guard([&] {
    const auto m = gfq::default_modulus(p, k);
    for (std::size_t i = 0; i < m.size(); ++i) modulus[i] = m[i];
  });
}

int gfq_random_matrix(uint32_t p, int64_t rows, int64_t cols, uint64_t seed, gfq_mat** out) {
  return guard([&] {
    require_device();
    gfq::Mat m(rows, cols, gfq::FieldSpec(p).esize());
    if (!m.empty()) fill_exact(p, rows, cols, seed, 0, m.data(), m.ld());
    *out = wrap(std::move(m));
  });
}

int gfq_random_product_matrix(uint32_t p, int64_t rows, int64_t cols, int64_t inner,
                              uint64_t seed, gfq_mat** out) {
  return guard([&] {
    require_device();
    gfq::FieldSpec f(p);
    gfq::Mat P(rows, inner, f.esize()), Q(inner, cols, f.esize());
    if (!P.empty()) fill_exact(p, rows, inner, seed, 0, P.data(), P.ld());
    if (!Q.empty())
      fill_exact(p, inner, cols, seed, uint64_t(rows) * uint64_t(inner), Q.data(), Q.ld());
    *out = wrap(gfq::mat_mul(f, P, Q));
  });
}

int gfq_reserve_for(int64_t m, int64_t n, int with_transform) {
  return guard([&] {
    if (m < 0 || n < 0) throw std::invalid_argument("gfq_reserve_for: negative shape");
    gfq::reserve_for(std::size_t(m), std::size_t(n), with_transform != 0);
  });
}
int gfq_set_poison(int mode) {
  return guard([&] {
    if (mode < 0 || mode > 3) throw std::invalid_argument("poison mode must be 0..3");
    gfq::set_poison_mode(mode);
  });
}
int gfq_set_ech_base(uint64_t n) { return guard([&] { gfq::set_ech_base(size_t(n)); }); }
int gfq_set_ech_outer(int width) { return guard([&] { gfq::set_ech_outer(width); }); }
int gfq_set_ech_mode(int mode) {
  return guard([&] {
    if (mode < 0 || mode > 4) throw std::invalid_argument("ech mode must be 0..4");
    gfq::set_ech_mode(mode);
  });
}
int gfq_launch_count(int reset, int64_t* launches) {
  return guard([&] { *launches = gfq::dev::launch_count(reset != 0); });
}
int gfq_profile(int on) { return guard([&] { gfq::dev::set_profile(on != 0); }); }
int gfq_profile_take(int64_t* launches2, double* ops2, double* ms2) {
  return guard([&] { gfq::dev::profile_take(launches2, ops2, ms2); });
}
int gfq_device_memory(int reset_peak, int64_t* live, int64_t* peak, int64_t* pool_reserved) {
  return guard([&] {
    if (live) *live = gfq::live_device_bytes();
    if (peak) *peak = gfq::peak_device_bytes();
    if (pool_reserved) {
      int dev = 0;
      GFQ_CUDA(cudaGetDevice(&dev));
      cudaMemPool_t pool;
      GFQ_CUDA(cudaDeviceGetDefaultMemPool(&pool, dev));
      std::uint64_t v = 0;
      GFQ_CUDA(cudaMemPoolGetAttribute(pool, cudaMemPoolAttrReservedMemHigh, &v));
      *pool_reserved = int64_t(v);
    }
    if (reset_peak) gfq::reset_peak_device_bytes();
  });
}
int gfq_profile_take_kinds(int n, int64_t* launches, double* work, double* ms, double* union_ms) {
  return guard([&] {
    if (n < 0 || (n > 0 && (!launches || !work || !ms)))
      throw std::invalid_argument("gfq_profile_take_kinds: bad buffers");
    gfq::dev::profile_take_kinds(n, launches, work, ms, union_ms);
  });
}
int gfq_tc_debug_take(uint64_t* stamps) {
  return guard([&] {
    if (!stamps) throw std::invalid_argument("gfq_tc_debug_take: null buffer");
    gfq::dev::tc_debug_take(reinterpret_cast<unsigned long long*>(stamps));
  });
}

// ---------------------------------------------------------------- jobs
int gfq_mul(uint32_t p, const gfq_mat* b, const gfq_mat* c, gfq_mat** out) {
  return guard([&] { *out = wrap(gfq::mul(gfq::FieldSpec(p), M(b), M(c))); });
}
int gfq_mad(uint32_t p, const gfq_mat* a, const gfq_mat* b, const gfq_mat* c, gfq_mat** out) {
  return guard([&] { *out = wrap(gfq::mad(gfq::FieldSpec(p), M(a), M(b), M(c))); });
}
int gfq_ech(uint32_t p, const gfq_mat* h, uint64_t threshold, gfq_mat** Mo, gfq_mat** Ko,
            gfq_mat** Ro, gfq_iset** rho, gfq_iset** gamma) {
  return guard([&] {
    gfq::EchResult e = gfq::ech(gfq::FieldSpec(p), M(h), size_t(threshold));
    *Mo = wrap(std::move(e.M));
    *Ko = wrap(std::move(e.K));
    *Ro = wrap(std::move(e.R));
    *rho = wrap(std::move(e.rho));
    *gamma = wrap(std::move(e.gamma));
  });
}
int gfq_cex(const gfq_mat* h, const gfq_iset* gamma, gfq_mat** sel, gfq_mat** rest) {
  return guard([&] {
    auto [a, b] = gfq::cex(M(h), S(gamma));
    *sel = wrap(std::move(a));
    *rest = wrap(std::move(b));
  });
}
int gfq_rex(const gfq_mat* h, const gfq_iset* rho, gfq_mat** sel, gfq_mat** rest) {
  return guard([&] {
    auto [a, b] = gfq::rex(M(h), S(rho));
    *sel = wrap(std::move(a));
    *rest = wrap(std::move(b));
  });
}
int gfq_unh(const gfq_iset* rho1, const gfq_iset* rho2, gfq_iset** rho, gfq_bits** u) {
  return guard([&] {
    auto [r, b] = gfq::unh(S(rho1), S(rho2));
    *rho = wrap(std::move(r));
    *u = wrap(std::move(b));
  });
}
int gfq_un0(const gfq_iset* rho2, gfq_iset** rho, gfq_bits** u) {
  return guard([&] {
    auto [r, b] = gfq::un0(S(rho2));
    *rho = wrap(std::move(r));
    *u = wrap(std::move(b));
  });
}
int gfq_mkr(const gfq_iset* rho1, const gfq_iset* rho2, gfq_bits** out) {
  return guard([&] { *out = wrap(gfq::mkr(S(rho1), S(rho2))); });
}
int gfq_rrf(const gfq_bits* u, const gfq_mat* b, const gfq_mat* c, gfq_mat** out) {
  return guard([&] { *out = wrap(gfq::rrf(B(u), M(b), M(c))); });
}
int gfq_crz(const gfq_mat* m, const gfq_bits* lambda, uint64_t out_cols, gfq_mat** out) {
  return guard([&] { *out = wrap(gfq::crz(M(m), B(lambda), size_t(out_cols))); });
}
int gfq_adi(const gfq_mat* k, const gfq_bits* delta, gfq_mat** out) {
  return guard([&] { *out = wrap(gfq::adi(M(k), B(delta))); });
}

// ---------------------------------------------------------------- tasks
int gfq_clear_down(uint32_t p, const gfq_mat* C, const gfq_pkgD* D, uint64_t i,
                   uint64_t ech_threshold, gfq_pkgD* D_out, gfq_pkgA* A_out) {
  return guard([&] {
    const gfq::PkgD d = D ? unpack(D) : gfq::PkgD{};
    auto [d2, a2] = gfq::clear_down(gfq::FieldSpec(p), M(C), d, size_t(i), size_t(ech_threshold));
    pack(std::move(d2), D_out);
    pack(std::move(a2), A_out);
  });
}
int gfq_update_row(uint32_t p, const gfq_pkgA* A, const gfq_mat* C, const gfq_mat* Bm, uint64_t i,
                   gfq_mat** C_out, gfq_mat** B_out) {
  return guard([&] {
    std::optional<gfq::Mat> b;
    if (Bm) b = M(Bm);
    auto [c2, b2] = gfq::update_row(gfq::FieldSpec(p), unpack(A), M(C), b, size_t(i));
    *C_out = wrap(std::move(c2));
    *B_out = wrap(std::move(b2));
  });
}
int gfq_update_row_trafo(uint32_t p, const gfq_pkgA* A, const gfq_mat* K, const gfq_mat* Mm,
                         const gfq_pkgE* E, uint64_t i, uint64_t h, uint64_t j, gfq_mat** K_out,
                         gfq_mat** M_out) {
  return guard([&] {
    std::optional<gfq::Mat> k, m;
    if (K) k = M(K);
    if (Mm) m = M(Mm);
    auto [k2, m2] = gfq::update_row_trafo(gfq::FieldSpec(p), unpack(A), k, m, unpack(E), size_t(i),
                                          size_t(h), size_t(j));
    *K_out = wrap(std::move(k2));
    *M_out = wrap(std::move(m2));
  });
}
int gfq_extend(const gfq_pkgA* A, const gfq_pkgE* E, uint64_t j, gfq_pkgE* E_out) {
  return guard([&] {
    std::optional<gfq::PkgE> e;
    if (E) e = unpack(E);
    pack(gfq::extend(unpack(A), e, size_t(j)), E_out);
  });
}
int gfq_row_lengthen(const gfq_mat* Mm, const gfq_pkgE* E1, const gfq_pkgE* E2, gfq_mat** out) {
  return guard([&] { *out = wrap(gfq::row_lengthen(M(Mm), unpack(E1), unpack(E2))); });
}
int gfq_pre_clear_up(const gfq_mat* Bm, const gfq_pkgD* D, gfq_mat** X, gfq_mat** R) {
  return guard([&] {
    auto [x, r] = gfq::pre_clear_up(M(Bm), unpack(D));
    *X = wrap(std::move(x));
    *R = wrap(std::move(r));
  });
}
int gfq_clear_up(uint32_t p, const gfq_mat* R, const gfq_mat* X, const gfq_mat* Mm, gfq_mat** out) {
  return guard([&] { *out = wrap(gfq::clear_up(gfq::FieldSpec(p), M(R), M(X), M(Mm))); });
}
int gfq_copy_d(const gfq_pkgD* D, gfq_mat** out) {
  return guard([&] { *out = wrap(gfq::copy_d(unpack(D))); });
}
void gfq_pkgA_free(gfq_pkgA* a) {
  if (!a) return;
  gfq_mat_free(a->A);
  gfq_mat_free(a->M);
  gfq_mat_free(a->K);
  gfq_iset_free(a->rho_prime);
  gfq_mat_free(a->E);
  gfq_bits_free(a->lambda);
  *a = gfq_pkgA{};
}
void gfq_pkgD_free(gfq_pkgD* d) {
  if (!d) return;
  gfq_mat_free(d->R);
  gfq_iset_free(d->gamma);
  *d = gfq_pkgD{};
}
void gfq_pkgE_free(gfq_pkgE* e) {
  if (!e) return;
  gfq_iset_free(e->rho);
  gfq_bits_free(e->delta);
  *e = gfq_pkgE{};
}

// ---------------------------------------------------------------- chief
int gfq_chop(uint64_t m, uint64_t n, uint64_t block, int remainder_first, uint64_t* row_parts,
             uint64_t* a, uint64_t* col_parts, uint64_t* b) {
  return guard([&] {
    const gfq::ChopSpec cs = gfq::chop(size_t(m), size_t(n), size_t(block), remainder_first != 0);
    if (a) *a = cs.a();
    if (b) *b = cs.b();
    if (row_parts)
      for (size_t i = 0; i < cs.a(); ++i) row_parts[i] = cs.row_parts[i];
    if (col_parts)
      for (size_t j = 0; j < cs.b(); ++j) col_parts[j] = cs.col_parts[j];
  });
}

void gfq_options_default(gfq_options* o) {
  o->block = 256;
  o->threads = 1;
  o->with_transform = 1;
  o->ech_threshold = 256;
  o->remainder_first = 0;
  o->collect_trace = 0;
  o->retain_all = 0;
  o->fuse = 1;
}

namespace {
gfq::EchelonizeOptions to_opts(const gfq_options* o) {
  gfq_options d;
  gfq_options_default(&d);
  if (!o) o = &d;
  gfq::EchelonizeOptions e;
  e.block = size_t(o->block);
  e.threads = o->threads;
  e.with_transform = o->with_transform != 0;
  e.ech_threshold = size_t(o->ech_threshold);
  e.remainder_first = o->remainder_first != 0;
  e.collect_trace = o->collect_trace != 0;
  e.retain_all = o->retain_all != 0;
  e.fuse = o->fuse != 0;
  return e;
}
const gfq_output& O(const gfq_output* o) {
  if (!o) throw std::invalid_argument("null output handle");
  return *o;
}
}  // namespace

int gfq_echelonize(uint32_t p, const gfq_mat* C, const gfq_options* opt, gfq_output** out) {
  return guard([&] {
    gfq::RunReport rep;
    auto res = std::make_unique<gfq_output>(
        gfq::echelonize(M(C), gfq::FieldSpec(p), to_opts(opt), &rep));
    res->report = std::move(rep);
    *out = res.release();
  });
}

int gfq_echelonize_host(uint32_t p, int64_t m, int64_t n, const uint8_t* C, int64_t ld,
                        const gfq_options* opt, gfq_output** out) {
  return guard([&] {
    require_device();
    const gfq::FieldSpec f(p);
    if (m < 0 || n < 0 || (m > 0 && n > 0 && (!C || ld < n)))
      throw std::invalid_argument("echelonize_host: bad matrix arguments");
    gfq::RunReport rep;
    auto res = std::make_unique<gfq_output>(gfq::echelonize_host(C, m, n, ld, f, to_opts(opt), &rep));
    res->report = std::move(rep);
    *out = res.release();
  });
}

int gfq_echelonize_host_into(uint32_t p, int64_t m, int64_t n, const uint8_t* C, int64_t ld,
                             const gfq_options* opt, uint8_t* host_out, uint64_t cap,
                             gfq_output** out) {
  return guard([&] {
    require_device();
    const gfq::FieldSpec f(p);
    if (m < 0 || n < 0 || (m > 0 && n > 0 && (!C || ld < n)))
      throw std::invalid_argument("echelonize_host: bad matrix arguments");
    if (!host_out) throw std::invalid_argument("echelonize_host_into: null output buffer");
    gfq::EchelonizeOptions o = to_opts(opt);
    o.host_out = host_out;
    o.host_out_cap = cap;
    gfq::RunReport rep;
    auto res = std::make_unique<gfq_output>(gfq::echelonize_host(C, m, n, ld, f, o, &rep));
    res->report = std::move(rep);
    *out = res.release();
  });
}

int gfq_output_rank(const gfq_output* o, uint64_t* rank) {
  return guard([&] { *rank = O(o).out.rank; });
}
int gfq_output_grid(const gfq_output* o, uint64_t* a, uint64_t* b) {
  return guard([&] {
    *a = O(o).out.chop.a();
    *b = O(o).out.chop.b();
  });
}
int gfq_output_select(const gfq_output* o, int which, uint64_t x, uint32_t* buf, uint64_t* count) {
  return guard([&] {
    const auto& v = which == 0 ? O(o).out.upsilon : O(o).out.varrho;
    const gfq::IndexSet& s = v.at(size_t(x));
    if (count) *count = s.size();
    if (buf && s.size()) std::memcpy(buf, s.members.data(), s.size() * 4);
  });
}
int gfq_output_block(const gfq_output* o, int kind, uint64_t x, uint64_t y, gfq_mat** blk) {
  return guard([&] {
    const auto& out = O(o).out;
    if (kind != 0 && !out.with_transform) throw std::logic_error("transformation was not computed");
    const auto& grid = kind == 0 ? out.R_blocks : kind == 1 ? out.T_M_blocks : out.T_K_blocks;
    if (kind == 0 && y < x) throw std::invalid_argument("R_blocks[j][l] requires l >= j");
    *blk = wrap(grid.at(size_t(x)).at(size_t(y)));
  });
}
int gfq_output_assembled_R(const gfq_output* o, gfq_mat** out) {
  return guard([&] { *out = wrap(O(o).out.assembled_R()); });
}
int gfq_output_transform(const gfq_output* o, gfq_mat** out) {
  return guard([&] { *out = wrap(gfq::materialize_transform(O(o).out)); });
}

}  // extern "C"
namespace {
template <class F>
void for_each_block(const gfq::EchelonOutput& out, F&& f) {
  for (size_t j = 0; j < out.R_blocks.size(); ++j)
    for (size_t l = j; l < out.R_blocks.size(); ++l) f(out.R_blocks[j][l]);
  for (const auto& row : out.T_M_blocks)
    for (const auto& m : row) f(m);
  for (const auto& row : out.T_K_blocks)
    for (const auto& m : row) f(m);
}
}  // namespace
extern "C" {

int gfq_output_block_bytes(const gfq_output* o, uint64_t* bytes) {
  return guard([&] {
    uint64_t n = 0;
    for_each_block(O(o).out, [&](const gfq::Mat& m) { n += uint64_t(m.rows()) * uint64_t(m.row_bytes()); });
    *bytes = n;
  });
}
int gfq_output_download_blocks(const gfq_output* o, uint8_t* host, uint64_t cap) {
  return guard([&] {
    uint64_t off = 0;
    for_each_block(O(o).out, [&](const gfq::Mat& m) {
      const uint64_t sz = uint64_t(m.rows()) * uint64_t(m.row_bytes());
      if (off + sz > cap) throw std::invalid_argument("download_blocks: buffer too small");
      if (sz)
        GFQ_CUDA(cudaMemcpy2DAsync(host + off, size_t(m.row_bytes()), m.data(), size_t(m.ld()),
                                   size_t(m.row_bytes()), size_t(m.rows()), cudaMemcpyDeviceToHost,
                                   gfq::cur_stream()));
      off += sz;
    });
    GFQ_CUDA(cudaStreamSynchronize(gfq::cur_stream()));
  });
}
int gfq_output_report(const gfq_output* o, gfq_report* rep) {
  return guard([&] {
    const auto& r = O(o).report;
    rep->wall_ns = r.wall_ns;
    rep->peak_live_bytes = r.peak_live_bytes;
    rep->initial_live_bytes = r.initial_live_bytes;
    rep->tasks = int64_t(r.trace.size());
    rep->workers = r.workers;
  });
}
int gfq_output_trace(const gfq_output* o, uint64_t* n, int32_t* kind, int32_t* i, int32_t* j,
                     int32_t* k, int32_t* worker, int64_t* start_ns, int64_t* end_ns,
                     int32_t* detail) {
  return guard([&] {
    const auto& tr = O(o).report.trace;
    if (n) *n = tr.size();
    for (size_t q = 0; q < tr.size(); ++q) {
      if (kind) kind[q] = int32_t(tr[q].kind);
      if (i) i[q] = tr[q].c0;
      if (j) j[q] = tr[q].c1;
      if (k) k[q] = tr[q].c2;
      if (worker) worker[q] = tr[q].worker;
      if (start_ns) start_ns[q] = tr[q].start_ns;
      if (end_ns) end_ns[q] = tr[q].end_ns;
      if (detail) detail[q] = tr[q].detail;
    }
  });
}
int gfq_output_trace_device(const gfq_output* o, uint64_t* n, int64_t* dev_start_ns,
                            int64_t* dev_end_ns) {
  return guard([&] {
    const auto& tr = O(o).report.trace;
    if (n) *n = tr.size();
    for (size_t q = 0; q < tr.size(); ++q) {
      if (dev_start_ns) dev_start_ns[q] = tr[q].dev_start_ns;
      if (dev_end_ns) dev_end_ns[q] = tr[q].dev_end_ns;
    }
  });
}
int gfq_output_trace_live(const gfq_output* o, uint64_t* n, int64_t* live_bytes) {
  return guard([&] {
    const auto& tr = O(o).report.trace;
    if (n) *n = tr.size();
    if (live_bytes)
      for (size_t q = 0; q < tr.size(); ++q) live_bytes[q] = tr[q].live_bytes;
  });
}
void gfq_output_free(gfq_output* o) { delete o; }

int gfq_read_gfmat_file(const char* path, uint32_t* p, gfq_mat** out) {
  return guard([&] {
    if (!path || !p || !out) throw std::invalid_argument("gfq_read_gfmat_file: null argument");
    const gfq::GfMatHost h = gfq::read_gfmat_file(path);
    *p = h.p;
    *out = wrap(gfq::Mat::from_host(h.rows, h.cols, h.data.data(), h.cols > 0 ? h.cols * h.esize : 1, h.esize));
  });
}
int gfq_write_gfmat_file(const char* path, uint32_t p, const gfq_mat* m) {
  return guard([&] {
    if (!path) throw std::invalid_argument("gfq_write_gfmat_file: null path");
    gfq::write_gfmat_file(path, p, M(m));
  });
}
int gfq_output_write_selects_file(const gfq_output* o, const char* path) {
  return guard([&] {
    if (!o || !path) throw std::invalid_argument("gfq_output_write_selects_file: null argument");
    gfq::write_selects_file(path, O(o).out);
  });
}
int gfq_output_write_transform_file(const gfq_output* o, const char* path) {
  return guard([&] {
    if (!o || !path) throw std::invalid_argument("gfq_output_write_transform_file: null argument");
    gfq::write_transform_file(path, O(o).out);
  });
}

int gfq_verify(const gfq_output* o, const gfq_mat* C, int method, uint64_t seed, int* ok,
               char* diag, size_t diag_len, char* checked, size_t checked_len) {
  return guard([&] {
    if (!o || !C || !ok) throw std::invalid_argument("gfq_verify: null argument");
    if (method < 0 || method > 2) throw std::invalid_argument("gfq_verify: method must be 0, 1 or 2");
    const gfq::VerifyResult r =
        gfq::verify(M(C), O(o).out, static_cast<gfq::VerifyMethod>(method), seed);
    *ok = r.ok ? 1 : 0;
    auto put = [](char* dst, size_t len, const std::string& v) {
      if (!dst || len == 0) return;
      const size_t k = v.size() < len - 1 ? v.size() : len - 1;
      std::memcpy(dst, v.data(), k);
      dst[k] = 0;
    };
    put(diag, diag_len, r.diag);
    put(checked, checked_len, r.method);
  });
}

// ---------------------------------------------------------------- multi-GPU
int gfq_nccl_unique_id(uint8_t* out128) {
  return guard([&] { gfq::nccl_unique_id(out128); });
}
int gfq_comm_nccl(int world, int rank, const uint8_t* id128, gfq_comm** out) {
  return guard([&] {
    require_device();
    if (world < 1 || rank < 0 || rank >= world) throw std::invalid_argument("bad rank / world");
    *out = new gfq_comm{gfq::make_nccl_comm(world, rank, id128)};
  });
}
int gfq_comm_loopback(int world, gfq_comm** comms) {
  return guard([&] {
    if (world < 1) throw std::invalid_argument("bad world size");
    auto v = gfq::make_loopback_comms(world);
    for (int r = 0; r < world; ++r) comms[r] = new gfq_comm{v[std::size_t(r)]};
  });
}
void gfq_comm_free(gfq_comm* c) { delete c; }

int gfq_echelonize_dist(gfq_comm* comm, uint32_t p, const gfq_mat* C, int64_t m, int64_t n,
                        uint64_t seed, const gfq_options* opt, int gather, gfq_output** out) {
  return guard([&] {
    require_device();
    if (!comm) throw std::invalid_argument("null communicator");
    gfq::RunReport rep;
    auto res = std::make_unique<gfq_output>(gfq::echelonize_dist(
        C ? &M(C) : nullptr, m, n, seed, gfq::FieldSpec(p), to_opts(opt), *comm->c, &rep,
        gather != 0));
    res->report = std::move(rep);
    *out = res.release();
  });
}

int gfq_dist_plan(uint64_t m, uint64_t n, uint64_t block, int with_transform, int world,
                  int32_t* nodes, uint64_t* n_nodes, int32_t* bcasts, uint64_t* n_bcast) {
  return guard([&] {
    if (world < 1) throw std::invalid_argument("bad world size");
    const gfq::ChopSpec cs = gfq::chop(size_t(m), size_t(n), size_t(block));
    if (cs.a() == 0 || cs.b() == 0) {
      if (n_nodes) *n_nodes = 0;
      if (n_bcast) *n_bcast = 0;
      return;
    }
    gfq::TaskGraph g;
    const gfq::PlanHandles h = gfq::build_plan(
        g, [](size_t, size_t) -> std::optional<gfq::Mat> { return std::nullopt; },
        gfq::FieldSpec(2), cs, with_transform != 0);
    const gfq::Sharding sh{world, 0};
    if (n_nodes) *n_nodes = g.node_count();
    if (nodes)
      for (size_t q = 0; q < g.node_count(); ++q) {
        const gfq::TaskNode& nd = g.node(int32_t(q));
        int o = sh.owner(nd);
        if (o == -2)
          o = g.slot(nd.out[0]).key.kind == gfq::PkgKind::R ? sh.owner_col(size_t(nd.c2))
                                                            : sh.owner_trow(size_t(nd.c2));
        nodes[5 * q + 0] = int32_t(nd.kind);
        nodes[5 * q + 1] = nd.c0;
        nodes[5 * q + 2] = nd.c1;
        nodes[5 * q + 3] = nd.c2;
        nodes[5 * q + 4] = o;
      }
    const auto sched = gfq::bcast_schedule(cs, h, g, sh);
    if (n_bcast) *n_bcast = sched.size();
    if (bcasts)
      for (size_t q = 0; q < sched.size(); ++q) {
        bcasts[5 * q + 0] = sched[q].is_a ? 1 : 0;
        bcasts[5 * q + 1] = int32_t(sched[q].i);
        bcasts[5 * q + 2] = int32_t(sched[q].j);
        bcasts[5 * q + 3] = int32_t(sched[q].k);
        bcasts[5 * q + 4] = sched[q].root;
      }
  });
}

}  // extern "C"
