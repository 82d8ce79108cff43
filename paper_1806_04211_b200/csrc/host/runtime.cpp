// runtime.cpp -- device memory, streams, staging and the value types.
#include <algorithm>
#include <atomic>
#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <mutex>
#include <unordered_map>
#include <vector>
#include <stdexcept>

#include "types.hpp"
#include "../kernels/kernels.hpp"

namespace gfq {

[[noreturn]] void throw_cuda(cudaError_t e, const char* what, const char* file, int line) {
  throw CudaError(std::string("CUDA error ") + cudaGetErrorName(e) + " (" +
                  cudaGetErrorString(e) + ") in " + what + " at " + file + ":" +
                  std::to_string(line));
}

namespace {
thread_local cudaStream_t t_stream = nullptr;
std::atomic<std::int64_t> g_live{0}, g_peak{0};
std::atomic<std::int64_t> g_cached{0};  // bytes parked in the block cache's lists
std::once_flag g_pool_once;

void init_pool() {
  std::call_once(g_pool_once, [] {
    int dev = 0;
    GFQ_CUDA(cudaGetDevice(&dev));
    cudaMemPool_t pool;
    GFQ_CUDA(cudaDeviceGetDefaultMemPool(&pool, dev));
    std::uint64_t thr = ~0ULL;  // keep freed blocks cached in the pool
    GFQ_CUDA(cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &thr));
  });
}
}  // namespace

namespace {
thread_local cudaEvent_t t_waits[80];
thread_local int t_n_waits = 0;
thread_local bool t_touched = false;
}  // namespace

cudaStream_t cur_stream() {
  if (t_n_waits) {
    const int n = t_n_waits;
    t_n_waits = 0;
    hprof::Scope hp(hprof::kEvent);
    for (int q = 0; q < n; ++q) GFQ_CUDA(cudaStreamWaitEvent(t_stream, t_waits[q], 0));
  }
  t_touched = true;
  return t_stream;
}
cudaStream_t cur_stream_raw() { return t_stream; }
void set_cur_stream(cudaStream_t s) { t_stream = s; }
void set_pending_waits(const cudaEvent_t* evs, int n) {
  if (n > 80) throw std::logic_error("set_pending_waits: too many events");
  for (int q = 0; q < n; ++q) t_waits[q] = evs[q];
  t_n_waits = n;
  t_touched = false;
  static const bool eager = std::getenv("GFQ_NO_LAZY_WAITS") != nullptr;
  if (eager) cur_stream();
}
bool stream_touched() { return t_touched; }
void end_pending_waits() {
  t_n_waits = 0;
  t_touched = false;
}

int sm_count() {
  static int n = 0;
  if (n == 0) {
    int dev = 0;
    GFQ_CUDA(cudaGetDevice(&dev));
    GFQ_CUDA(cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev));
  }
  return n;
}

// ---------------------------------------------------------------- FieldSpec
// ---------------------------------------------------------------- fields
namespace {
using Poly = std::vector<std::uint32_t>;
bool is_prime(std::uint32_t p) {
  if (p < 2) return false;
  for (std::uint32_t d = 2; d * d <= p; ++d)
    if (p % d == 0) return false;
  return true;
}
int deg(const Poly& a) {
  for (int i = int(a.size()) - 1; i >= 0; --i)
    if (a[std::size_t(i)] != 0) return i;
  return -1;
}
// a mod m over GF(p), m monic (reference src/field.cpp:35-46)
Poly poly_mod(Poly a, const Poly& m, std::uint32_t p) {
  const int dm = deg(m);
  for (int i = deg(a); dm >= 0 && i >= dm; i = deg(a)) {
    const std::uint64_t c = a[std::size_t(i)];
    for (int t = 0; t <= dm; ++t) {
      const std::uint64_t v = a[std::size_t(i - dm + t)] + (p - m[std::size_t(t)]) % p * c;
      a[std::size_t(i - dm + t)] = std::uint32_t(v % p);
    }
  }
  return a;
}
// no monic divisor of degree 1..k/2 (reference src/field.cpp:59-78)
bool poly_irreducible(const Poly& m, std::uint32_t p) {
  const int k = deg(m);
  if (k < 1) return false;
  for (int d = 1; 2 * d <= k; ++d) {
    std::uint64_t count = 1;
    for (int i = 0; i < d; ++i) count *= p;
    for (std::uint64_t c = 0; c < count; ++c) {
      Poly div(std::size_t(d) + 1, 0);
      std::uint64_t t = c;
      for (int i = 0; i < d; ++i) {
        div[std::size_t(i)] = std::uint32_t(t % p);
        t /= p;
      }
      div[std::size_t(d)] = 1;
      if (deg(poly_mod(m, div, p)) < 0) return false;
    }
  }
  return true;
}
}  // namespace

std::vector<std::uint32_t> default_modulus(std::uint32_t p, std::uint32_t k) {
  if (!is_prime(p)) throw std::invalid_argument("field: p must be prime");
  if (k == 1) return {0, 1};
  std::uint64_t count = 1;
  for (std::uint32_t i = 0; i < k; ++i) count *= p;
  for (std::uint64_t c = 0; c < count; ++c) {
    Poly m(k + 1, 0);
    std::uint64_t t = c;
    for (std::uint32_t i = 0; i < k; ++i) {
      m[i] = std::uint32_t(t % p);
      t /= p;
    }
    m[k] = 1;
    if (poly_irreducible(m, p)) return m;
  }
  throw std::logic_error("field: no irreducible modulus found");
}

/// Host + device tables of GF(p^k) (q <= 256): the arithmetic is table
/// lookups on encoded elements (the reference uses log / antilog / Zech
/// tables, src/field.cpp:180-212; products of polynomials mod the modulus
/// give the same field, so the tables hold identical values).
struct ExtTablesHost {
  std::uint32_t p = 0, k = 1, q = 0;
  std::vector<std::uint32_t> modulus;
  std::vector<std::uint8_t> mul, add, neg, inv, dig, red;
  std::uint32_t code = 0;
  mutable std::once_flag dev_once;
  mutable std::uint8_t* dev = nullptr;
  mutable dev::ExtTables view{};
  // wide extension fields (q > 256): log / antilog / Zech tables of a
  // generator g of GF(q)* (the reference's own representation,
  // src/field.cpp:180-212); zech[n] = log(1 + g^n), -1 where 1 + g^n = 0
  bool wide = false;
  std::vector<std::uint32_t> wexp, wlog;
  std::vector<std::int32_t> wzech;
  mutable std::uint32_t* wdev = nullptr;
};

namespace {
std::mutex g_field_mtx;
std::vector<std::shared_ptr<const ExtTablesHost>>* g_fields =
    new std::vector<std::shared_ptr<const ExtTablesHost>>();  // process lifetime
constexpr std::uint32_t kFieldCode0 = 0x10000;

std::shared_ptr<const ExtTablesHost> make_ext(std::uint32_t p, std::uint32_t k, Poly mod) {
  auto t = std::make_shared<ExtTablesHost>();
  std::uint32_t q = 1;
  for (std::uint32_t i = 0; i < k; ++i) q *= p;
  t->p = p;
  t->k = k;
  t->q = q;
  t->modulus = mod;
  const auto decode = [&](std::uint32_t e) {
    Poly d(k, 0);
    for (std::uint32_t i = 0; i < k; ++i) {
      d[i] = e % p;
      e /= p;
    }
    return d;
  };
  const auto encode = [&](const Poly& d) {
    std::uint32_t v = 0;
    for (std::uint32_t i = k; i-- > 0;) v = v * p + (i < d.size() ? d[i] : 0);
    return v;
  };
  t->dig.resize(std::size_t(q) * k);
  for (std::uint32_t e = 0; e < q; ++e) {
    const Poly d = decode(e);
    for (std::uint32_t i = 0; i < k; ++i) t->dig[std::size_t(e) * k + i] = std::uint8_t(d[i]);
  }
  t->red.resize(std::size_t(2 * k - 1) * k);
  for (std::uint32_t sdeg = 0; sdeg < 2 * k - 1; ++sdeg) {
    Poly x(sdeg + 1, 0);
    x[sdeg] = 1;
    const Poly r = poly_mod(x, mod, p);
    for (std::uint32_t u = 0; u < k; ++u)
      t->red[std::size_t(sdeg) * k + u] = std::uint8_t(u < r.size() ? r[u] : 0);
  }
  t->mul.resize(std::size_t(q) * q);
  t->add.resize(std::size_t(q) * q);
  for (std::uint32_t a = 0; a < q; ++a)
    for (std::uint32_t b = 0; b < q; ++b) {
      const Poly da = decode(a), db = decode(b);
      Poly sum(k), prod(2 * k - 1, 0);
      for (std::uint32_t i = 0; i < k; ++i) sum[i] = (da[i] + db[i]) % p;
      for (std::uint32_t i = 0; i < k; ++i)
        for (std::uint32_t j = 0; j < k; ++j) prod[i + j] = (prod[i + j] + da[i] * db[j]) % p;
      t->add[std::size_t(a) * q + b] = std::uint8_t(encode(sum));
      t->mul[std::size_t(a) * q + b] = std::uint8_t(encode(poly_mod(prod, mod, p)));
    }
  t->neg.resize(q);
  t->inv.assign(q, 0);
  for (std::uint32_t a = 0; a < q; ++a) {
    const Poly d = decode(a);
    Poly n(k);
    for (std::uint32_t i = 0; i < k; ++i) n[i] = (p - d[i]) % p;
    t->neg[a] = std::uint8_t(encode(n));
    for (std::uint32_t b = 1; b < q && a; ++b)
      if (t->mul[std::size_t(a) * q + b] == 1) {
        t->inv[a] = std::uint8_t(b);
        break;
      }
  }
  return t;
}

// Wide GF(p^k) (256 < q < 2^20): the tables above would be q x q, so the
// field is held as log / antilog / Zech tables built from polynomial
// products mod the modulus.
std::shared_ptr<const ExtTablesHost> make_ext_wide(std::uint32_t p, std::uint32_t k, Poly mod) {
  auto t = std::make_shared<ExtTablesHost>();
  std::uint32_t q = 1;
  for (std::uint32_t i = 0; i < k; ++i) q *= p;
  t->p = p;
  t->k = k;
  t->q = q;
  t->modulus = mod;
  t->wide = true;
  const auto decode = [&](std::uint32_t e) {
    Poly d(k, 0);
    for (std::uint32_t i = 0; i < k; ++i) {
      d[i] = e % p;
      e /= p;
    }
    return d;
  };
  const auto encode = [&](const Poly& d) {
    std::uint32_t v = 0;
    for (std::uint32_t i = k; i-- > 0;) v = v * p + (i < d.size() ? d[i] : 0);
    return v;
  };
  const auto mulenc = [&](std::uint32_t a, std::uint32_t b) {
    const Poly da = decode(a), db = decode(b);
    Poly prod(2 * k - 1, 0);
    for (std::uint32_t i = 0; i < k; ++i)
      for (std::uint32_t j = 0; j < k; ++j)
        prod[i + j] = std::uint32_t((prod[i + j] + std::uint64_t(da[i]) * db[j]) % p);
    return encode(poly_mod(prod, mod, p));
  };
  const auto powenc = [&](std::uint32_t a, std::uint64_t e) {
    std::uint32_t r = 1;
    while (e) {
      if (e & 1) r = mulenc(r, a);
      a = mulenc(a, a);
      e >>= 1;
    }
    return r;
  };
  // the prime factors of q - 1 and the smallest generator
  std::vector<std::uint32_t> fac;
  {
    std::uint32_t n = q - 1;
    for (std::uint32_t d = 2; d * d <= n; ++d)
      if (n % d == 0) {
        fac.push_back(d);
        while (n % d == 0) n /= d;
      }
    if (n > 1) fac.push_back(n);
  }
  std::uint32_t g = 0;
  for (std::uint32_t c = 2; c < q && !g; ++c) {
    bool ok = true;
    for (std::uint32_t r : fac)
      if (powenc(c, (q - 1) / r) == 1) {
        ok = false;
        break;
      }
    if (ok) g = c;
  }
  if (!g) throw std::logic_error("field: no generator found");
  t->wexp.resize(q - 1);
  t->wlog.assign(q, 0);
  std::uint32_t x = 1;
  for (std::uint32_t i = 0; i + 1 < q; ++i) {
    t->wexp[i] = x;
    t->wlog[x] = i;
    x = mulenc(x, g);
  }
  t->wzech.resize(q - 1);
  for (std::uint32_t n = 0; n + 1 < q; ++n) {
    const Poly d = decode(t->wexp[n]);
    Poly e = d;
    e[0] = (e[0] + 1) % p;  // 1 + g^n
    const std::uint32_t v = encode(e);
    t->wzech[n] = v == 0 ? -1 : std::int32_t(t->wlog[v]);
  }
  return t;
}
}  // namespace

FieldSpec::FieldSpec(std::uint32_t p) {
  if (p >= kFieldCode0) {
    std::lock_guard<std::mutex> lk(g_field_mtx);
    const std::size_t idx = p - kFieldCode0;
    if (idx >= g_fields->size()) throw std::invalid_argument("field: unknown field code");
    ext_ = (*g_fields)[idx];
    p_ = ext_->p;
    k_ = ext_->k;
    q_ = ext_->q;
    return;
  }
  if (!is_prime(p)) throw std::invalid_argument("field: p must be prime");
  if (p >= (1u << 16)) throw std::invalid_argument("field: p must be < 2^16");
  p_ = q_ = p;
}

FieldSpec::FieldSpec(std::uint32_t p, std::uint32_t k, std::vector<std::uint32_t> modulus) {
  // reference src/field.cpp:143-169 validation order and messages
  if (!is_prime(p)) throw std::invalid_argument("field: p must be prime");
  if (p >= (1u << 16)) throw std::invalid_argument("field: p must be < 2^16");
  if (k < 1) throw std::invalid_argument("field: k must be >= 1");
  std::uint64_t q = 1;
  for (std::uint32_t i = 0; i < k; ++i) {
    q *= p;
    if (q >= (1u << 20)) throw std::invalid_argument("field: p^k must be < 2^20");
  }
  if (k == 1) {
    *this = FieldSpec(p);
    return;
  }
  if (modulus.empty()) modulus = default_modulus(p, k);
  if (modulus.size() != std::size_t(k) + 1 || modulus[k] != 1)
    throw std::invalid_argument("field: modulus must be monic of degree k");
  for (std::uint32_t c : modulus)
    if (c >= p) throw std::invalid_argument("field: modulus coefficient >= p");
  if (!poly_irreducible(modulus, p)) throw std::invalid_argument("field: modulus is not irreducible");
  p_ = p;
  k_ = k;
  q_ = std::uint32_t(q);
  std::lock_guard<std::mutex> lk(g_field_mtx);
  for (const auto& e : *g_fields)
    if (e->p == p && e->k == k && e->modulus == modulus) {
      ext_ = e;
      return;
    }
  auto t = q > 256 ? make_ext_wide(p, k, modulus) : make_ext(p, k, modulus);
  const_cast<ExtTablesHost&>(*t).code = kFieldCode0 + std::uint32_t(g_fields->size());
  g_fields->push_back(t);
  ext_ = t;
}

std::uint32_t FieldSpec::code() const { return ext_ ? ext_->code : p_; }

const std::vector<std::uint32_t>& FieldSpec::modulus() const {
  static const std::vector<std::uint32_t> prime_mod{0, 1};
  return ext_ ? ext_->modulus : prime_mod;
}

namespace {
// base-p digit-wise a + s.b of two encoded GF(p^k) elements (s = 1 or p-1)
Elem digit_axpy(Elem a, Elem b, std::uint32_t s, std::uint32_t p, std::uint32_t k) {
  Elem r = 0, m = 1;
  for (std::uint32_t i = 0; i < k; ++i) {
    r += Elem((a % p + std::uint64_t(s) * (b % p)) % p) * m;
    a /= p;
    b /= p;
    m *= p;
  }
  return r;
}
}  // namespace

Elem FieldSpec::add(Elem a, Elem b) const {
  if (ext_ && ext_->wide) return digit_axpy(a, b, 1, p_, k_);
  return ext_ ? ext_->add[std::size_t(a) * q_ + b] : (a + b) % p_;
}
Elem FieldSpec::neg(Elem a) const {
  if (ext_ && ext_->wide) return digit_axpy(0, a, p_ - 1, p_, k_);
  return ext_ ? ext_->neg[a] : (a == 0 ? 0 : p_ - a);
}
Elem FieldSpec::mul(Elem a, Elem b) const {
  if (ext_ && ext_->wide)
    return (a == 0 || b == 0) ? 0 : ext_->wexp[(std::uint64_t(ext_->wlog[a]) + ext_->wlog[b]) % (q_ - 1)];
  return ext_ ? ext_->mul[std::size_t(a) * q_ + b] : Elem(std::uint64_t(a) * b % p_);
}

Elem FieldSpec::inv(Elem a) const {
  if (a % q_ == 0) throw std::domain_error("field: inverse of zero");
  if (ext_ && ext_->wide) return ext_->wexp[(q_ - 1 - ext_->wlog[a] % (q_ - 1)) % (q_ - 1)];
  if (ext_) return ext_->inv[a];
  std::uint64_t r = 1, b = a % p_;
  std::uint32_t e = p_ - 2;
  while (e) {
    if (e & 1) r = r * b % p_;
    b = b * b % p_;
    e >>= 1;
  }
  return Elem(r);
}

dev::WideField FieldSpec::wide_dev() const {
  dev::WideField w{p_, k_, q_, nullptr, nullptr, nullptr};
  if (!ext_) return w;
  const ExtTablesHost& t = *ext_;
  if (!t.wide) throw std::logic_error("FieldSpec::wide_dev on a u8 extension field");
  std::call_once(t.dev_once, [&] {
    const std::size_t n = (t.q - 1) + t.q + (t.q - 1);
    GFQ_CUDA(cudaMalloc(&t.wdev, n * 4));  // process lifetime, like the field registry
    std::vector<std::uint32_t> all;
    all.reserve(n);
    all.insert(all.end(), t.wexp.begin(), t.wexp.end());
    all.insert(all.end(), t.wlog.begin(), t.wlog.end());
    for (std::int32_t z : t.wzech) all.push_back(std::uint32_t(z));
    GFQ_CUDA(cudaMemcpy(t.wdev, all.data(), n * 4, cudaMemcpyHostToDevice));
  });
  w.exp = t.wdev;
  w.log = t.wdev + (t.q - 1);
  w.zech = reinterpret_cast<const std::int32_t*>(t.wdev + (t.q - 1) + t.q);
  return w;
}

const dev::ExtTables& FieldSpec::ext_dev() const {
  if (!ext_) throw std::logic_error("FieldSpec::ext_dev on a prime field");
  if (ext_->wide) throw std::logic_error("FieldSpec::ext_dev on a wide extension field");
  const ExtTablesHost& t = *ext_;
  std::call_once(t.dev_once, [&] {
    const std::size_t q = t.q, k = t.k;
    const std::size_t n = 2 * q * q + 2 * q + q * k + (2 * k - 1) * k;
    GFQ_CUDA(cudaMalloc(&t.dev, n));  // process lifetime, like the field registry
    std::vector<std::uint8_t> all;
    all.reserve(n);
    all.insert(all.end(), t.mul.begin(), t.mul.end());
    all.insert(all.end(), t.add.begin(), t.add.end());
    all.insert(all.end(), t.neg.begin(), t.neg.end());
    all.insert(all.end(), t.inv.begin(), t.inv.end());
    all.insert(all.end(), t.dig.begin(), t.dig.end());
    all.insert(all.end(), t.red.begin(), t.red.end());
    GFQ_CUDA(cudaMemcpy(t.dev, all.data(), n, cudaMemcpyHostToDevice));
    std::uint8_t* d = t.dev;
    t.view = dev::ExtTables{t.p, t.k, t.q, d, d + q * q, d + 2 * q * q, d + 2 * q * q + q,
                            d + 2 * q * q + 2 * q, d + 2 * q * q + 2 * q + q * k};
  });
  return t.view;
}

// ---------------------------------------------------------------- host profile
namespace hprof {
const bool on = std::getenv("GFQ_HOSTPROF") != nullptr;
thread_local const char* t_task_name = "-";
namespace {
std::atomic<std::int64_t> g_ns[kSlots];
std::atomic<std::int64_t> g_cnt[kSlots];
struct Printer {
  ~Printer() {
    if (!on) return;
    static const char* names[kSlots] = {
        "malloc", "free",  "upload", "mad", "select", "event", "memset", "alloc_miss", "sync",
        "other_launch", "task", "ClearDown", "UpdateRow", "UpdateRowTrafo", "Extend", "RowLengthen",
        "PreClearUp", "ClearUp", "Copy", "UpdateRowW", "ClearUpRW", "ClearUpMW", "UpdateRowTrafoW"};
    for (int q = 0; q < kSlots; ++q)
      std::fprintf(stderr, "hostprof %-12s %10.3f ms %8lld calls %8.2f us/call\n", names[q],
                   double(g_ns[q]) / 1e6, static_cast<long long>(g_cnt[q].load()),
                   g_cnt[q] ? double(g_ns[q]) / 1e3 / double(g_cnt[q]) : 0.0);
  }
} g_printer;
}  // namespace
void add(Slot s, std::int64_t ns, std::int64_t count) {
  g_ns[s] += ns;
  g_cnt[s] += count;
}
std::int64_t now() {
  return std::chrono::duration_cast<std::chrono::nanoseconds>(
             std::chrono::steady_clock::now().time_since_epoch())
      .count();
}
}  // namespace hprof

// ---------------------------------------------------------------- DevBuf / Mat
// Caching block allocator over the stream-ordered pool.  A block freed
// while the current stream is s goes back to s's free list and is reused
// by the next allocation on s at once (stream order makes that safe, the
// same contract as cudaFreeAsync); release_stream(s) -- called once s has
// drained -- moves s's blocks to the idle list any stream may take.  Hits
// cost a mutex instead of a CUDA API call; sizes are rounded to classes of
// 1/8 of a power of two (<= 12.5% slack).
namespace {
struct BlockCache {
  std::mutex mtx;
  std::unordered_map<cudaStream_t, std::unordered_map<std::size_t, std::vector<void*>>> by_stream;
  std::unordered_map<std::size_t, std::vector<void*>> idle;
  std::unordered_map<void*, std::size_t> cls_of;
};
BlockCache& cache() {
  static BlockCache* c = new BlockCache();  // process lifetime
  return *c;
}
std::size_t size_class(std::size_t n) {
  if (n <= 4096) return (n + 511) / 512 * 512;
  std::size_t p2 = std::size_t(1) << (63 - __builtin_clzll(n));
  const std::size_t step = p2 / 8;
  return (n + step - 1) / step * step;
}
void* take(std::unordered_map<std::size_t, std::vector<void*>>& lists, std::size_t cls) {
  auto it = lists.find(cls);
  if (it == lists.end() || it->second.empty()) return nullptr;
  void* p = it->second.back();
  it->second.pop_back();
  g_cached -= std::int64_t(cls);
  return p;
}
}  // namespace

namespace {
std::atomic<int> g_poison{[] {
  const char* e = std::getenv("GFQ_POISON");
  return e ? std::atoi(e) : 0;
}()};
}  // namespace
int poison_mode() { return g_poison.load(std::memory_order_relaxed); }
void set_poison_mode(int mode) { g_poison = mode; }

// Grow the stream-ordered pool in ONE step to hold `bytes` more than it
// uses now: hundreds of block-cache misses that each grow the pool by a
// mapping cost milliseconds apiece (cfg5s: ~500 misses, first steps up to
// 1.6x slower); one big reservation up front makes them cheap carve-outs.
void reserve_pool(std::size_t bytes) {
  init_pool();
  int dev = 0;
  GFQ_CUDA(cudaGetDevice(&dev));
  cudaMemPool_t pool;
  GFQ_CUDA(cudaDeviceGetDefaultMemPool(&pool, dev));
  std::uint64_t reserved = 0, used = 0;
  GFQ_CUDA(cudaMemPoolGetAttribute(pool, cudaMemPoolAttrReservedMemCurrent, &reserved));
  GFQ_CUDA(cudaMemPoolGetAttribute(pool, cudaMemPoolAttrUsedMemCurrent, &used));
  // blocks parked in the cache are "used" to the pool but free to us
  const std::int64_t parked = g_cached.load();
  if (parked > 0) used = used > std::uint64_t(parked) ? used - std::uint64_t(parked) : 0;
  if (reserved >= used + bytes) return;
  std::size_t free_b = 0, total_b = 0;
  GFQ_CUDA(cudaMemGetInfo(&free_b, &total_b));
  std::size_t want = used + bytes - reserved;
  const std::size_t cap = free_b > (std::size_t(2) << 30) ? free_b - (std::size_t(2) << 30) : 0;
  if (want > cap) want = cap;
  if (want < (std::size_t(64) << 20)) return;
  void* p = nullptr;
  const cudaStream_t s = cur_stream_raw();
  if (cudaMallocAsync(&p, want, s) == cudaSuccess) {
    GFQ_CUDA(cudaFreeAsync(p, s));
    GFQ_CUDA(cudaStreamSynchronize(s));
  } else {
    cudaGetLastError();
  }
}

void release_stream(cudaStream_t s) {
  BlockCache& c = cache();
  std::lock_guard<std::mutex> lk(c.mtx);
  auto it = c.by_stream.find(s);
  if (it == c.by_stream.end()) return;
  for (auto& [cls, v] : it->second) {
    auto& dst = c.idle[cls];
    dst.insert(dst.end(), v.begin(), v.end());
  }
  c.by_stream.erase(it);
}

DevBuf::DevBuf(std::size_t n) : bytes(n) {
  if (n == 0) return;
  init_pool();
  hprof::Scope hp(hprof::kMalloc);
  const cudaStream_t s = cur_stream_raw();
  const std::size_t cls = size_class(n);
  BlockCache& c = cache();
  void* p = nullptr;
  static const bool nocache = std::getenv("GFQ_NO_BLOCK_CACHE") != nullptr;
  if (!nocache) {
    std::lock_guard<std::mutex> lk(c.mtx);
    auto it = c.by_stream.find(s);
    if (it != c.by_stream.end()) p = take(it->second, cls);
    if (!p) p = take(c.idle, cls);
  }
  if (!p) {
    hprof::Scope hm(hprof::kMiss);
    cudaError_t e = cudaMallocAsync(&p, cls, s);
    if (e == cudaErrorMemoryAllocation) {
      // return every idle cached block to the pool and retry once
      cudaGetLastError();
      std::vector<void*> drop;
      {
        std::lock_guard<std::mutex> lk(c.mtx);
        for (auto& [k, v] : c.idle)
          for (void* q : v) {
            drop.push_back(q);
            c.cls_of.erase(q);
            g_cached -= std::int64_t(k);
          }
        c.idle.clear();
      }
      for (void* q : drop) cudaFreeAsync(q, s);
      e = cudaMallocAsync(&p, cls, s);
    }
    GFQ_CUDA(e);
    std::lock_guard<std::mutex> lk(c.mtx);
    c.cls_of[p] = cls;
  }
  ptr = static_cast<std::uint8_t*>(p);
  // Developer check (GFQ_POISON bit 0): fill every allocation with 0xA5 on
  // its stream, so a read of memory the code never wrote shows up as a
  // wrong result instead of silently seeing zeros or a recycled block.
  if (poison_mode() & 1) GFQ_CUDA(cudaMemsetAsync(p, 0xA5, cls, s));
  const std::int64_t now = (g_live += std::int64_t(n));
  std::int64_t prev = g_peak.load();
  while (now > prev && !g_peak.compare_exchange_weak(prev, now)) {
  }
}

DevBuf::~DevBuf() {
  if (ptr) {
    // Stream-ordered release: every job on this value was issued on the
    // current stream (or joined into it by the executor) before release.
    hprof::Scope hp(hprof::kFree);
    // GFQ_POISON bit 1: overwrite the block on the freeing stream, so a
    // kernel on another stream that still reads it (a missing dependency)
    // sees garbage.
    if (poison_mode() & 2) cudaMemsetAsync(ptr, 0x5A, bytes, cur_stream_raw());
    BlockCache& c = cache();
    std::lock_guard<std::mutex> lk(c.mtx);
    auto it = c.cls_of.find(ptr);
    static const bool nocache = std::getenv("GFQ_NO_BLOCK_CACHE") != nullptr;
    if (it != c.cls_of.end() && !nocache) {
      c.by_stream[cur_stream_raw()][it->second].push_back(ptr);
      g_cached += std::int64_t(it->second);
    }
    else {
      if (it != c.cls_of.end()) c.cls_of.erase(it);
      cudaFreeAsync(ptr, cur_stream_raw());
    }
    g_live -= std::int64_t(bytes);
  }
}

std::int64_t live_device_bytes() { return g_live; }
std::int64_t peak_device_bytes() { return g_peak; }
void reset_peak_device_bytes() { g_peak = g_live.load(); }

Mat::Mat(std::int64_t rows, std::int64_t cols, int esize) : rows_(rows), cols_(cols), esize_(esize) {
  if (rows < 0 || cols < 0) throw std::invalid_argument("matrix: negative shape");
  if (esize != 1 && esize != 4) throw std::invalid_argument("matrix: element size must be 1 or 4");
  ld_ = round_up(cols > 0 ? cols * esize : 1, 16);
  if (rows > 0 && cols > 0) {
    buf_ = std::make_shared<DevBuf>(std::size_t(rows) * std::size_t(ld_));
    data_ = buf_->ptr;
  }
}

Mat Mat::zeros(std::int64_t rows, std::int64_t cols, int esize) {
  Mat m(rows, cols, esize);
  if (!m.empty()) {
    hprof::Scope hp(hprof::kMemset);
    dev::fill2d(m.data_, m.ld_, rows, m.ld_, 0, cur_stream());
  }
  return m;
}

Mat Mat::from_host(std::int64_t rows, std::int64_t cols, const std::uint8_t* src,
                   std::int64_t ld, int esize) {
  Mat m(rows, cols, esize);
  if (!m.empty()) {
    GFQ_CUDA(cudaMemcpy2DAsync(m.data_, std::size_t(m.ld_), src, std::size_t(ld),
                               std::size_t(cols * esize), std::size_t(rows), cudaMemcpyHostToDevice,
                               cur_stream()));
    // pageable source: make the copy complete before the caller may reuse it
    GFQ_CUDA(cudaStreamSynchronize(cur_stream()));
  }
  return m;
}

Mat Mat::view_of(std::shared_ptr<DevBuf> buf, std::size_t offset, std::int64_t rows,
                 std::int64_t cols, std::int64_t ld, int esize) {
  Mat v;
  v.rows_ = rows;
  v.cols_ = cols;
  v.ld_ = ld;
  v.esize_ = esize;
  if (rows > 0 && cols > 0) {
    if (!buf || offset + std::size_t((rows - 1) * ld + cols * esize) > buf->bytes)
      throw std::invalid_argument("matrix: view outside its allocation");
    v.data_ = buf->ptr + offset;
  }
  v.buf_ = std::move(buf);
  return v;
}

Mat Mat::with_capacity(std::int64_t rows, std::int64_t cols, std::int64_t cap_cols, int esize) {
  if (cap_cols <= cols || rows <= 0 || cols <= 0) return Mat(rows, cols, esize);
  Mat full(rows, cap_cols, esize);
  return full.col_view(0, cols);
}

Mat Mat::widened(std::int64_t cols) const {
  if (cols < cols_ || !buf_ || !data_ || rows_ <= 0) return Mat();
  const std::int64_t in_row = std::int64_t(data_ - buf_->ptr) % ld_;
  if (in_row + cols * esize_ > ld_) return Mat();
  if (std::size_t(data_ - buf_->ptr) + std::size_t((rows_ - 1) * ld_ + cols * esize_) > buf_->bytes) return Mat();
  Mat v = *this;
  v.cols_ = cols;
  return v;
}

Mat Mat::row_view(std::int64_t r0, std::int64_t n) const {
  if (r0 < 0 || n < 0 || r0 + n > rows_) throw std::invalid_argument("matrix: row view out of range");
  Mat v;
  v.buf_ = buf_;
  v.rows_ = n;
  v.cols_ = cols_;
  v.ld_ = ld_;
  v.esize_ = esize_;
  v.data_ = (data_ && n > 0 && cols_ > 0) ? data_ + r0 * ld_ : nullptr;
  return v;
}

Mat Mat::col_view(std::int64_t c0, std::int64_t n) const {
  if (c0 < 0 || n < 0 || c0 + n > cols_) throw std::invalid_argument("matrix: column view out of range");
  Mat v;
  v.buf_ = buf_;
  v.rows_ = rows_;
  v.cols_ = n;
  v.ld_ = ld_;
  v.esize_ = esize_;
  v.data_ = (data_ && n > 0 && rows_ > 0) ? data_ + c0 * esize_ : nullptr;
  return v;
}

void Mat::to_host(std::uint8_t* dst, std::int64_t ld) const {
  if (empty()) return;
  GFQ_CUDA(cudaMemcpy2DAsync(dst, std::size_t(ld), data_, std::size_t(ld_), std::size_t(cols_ * esize_),
                             std::size_t(rows_), cudaMemcpyDeviceToHost, cur_stream()));
  GFQ_CUDA(cudaStreamSynchronize(cur_stream()));
}

std::vector<std::uint8_t> Mat::to_host() const {
  std::vector<std::uint8_t> out(std::size_t(rows_) * std::size_t(cols_) * std::size_t(esize_));
  to_host(out.data(), cols_ > 0 ? cols_ * esize_ : 1);
  return out;
}

// ---------------------------------------------------------------- index types
IndexSet::IndexSet(std::size_t universe, std::vector<std::uint32_t> members)
    : universe(universe), members(std::move(members)) {
  for (std::size_t i = 0; i < this->members.size(); ++i) {
    if (this->members[i] >= universe)
      throw std::invalid_argument("index set: member out of universe");
    if (i > 0 && this->members[i] <= this->members[i - 1])
      throw std::invalid_argument("index set: members must be increasing");
  }
}

IndexSet index_set_complement(const IndexSet& s) {
  IndexSet out;
  out.universe = s.universe;
  out.members.reserve(s.universe - s.members.size());
  std::size_t next = 0;
  for (std::uint32_t v = 0; v < s.universe; ++v) {
    if (next < s.members.size() && s.members[next] == v)
      ++next;
    else
      out.members.push_back(v);
  }
  return out;
}

std::size_t BitString::count_ones() const {
  std::size_t n = 0;
  for (auto b : bits) n += b ? 1 : 0;
  return n;
}

std::size_t PkgA::byte_size() const {
  std::size_t n = M.byte_size() + K.byte_size() + rho_prime.byte_size();
  if (A) n += A->byte_size();
  if (E) n += E->byte_size();
  if (lambda) n += lambda->byte_size();
  return n;
}

// ---------------------------------------------------------------- staging
namespace {
// One process-wide pinned, device-mapped staging ring for small index
// uploads (pinning is expensive: it is done once, not per executor thread or
// per call).  An upload is a memcpy into the ring and a tiny kernel that
// reads the ring over the bus into the device buffer -- not a copy-engine
// transfer, so it never queues behind a bulk host-to-device copy (the
// streamed input of gfq_echelonize_host: 4.3 GB at cfg5s held every index
// upload of the first ECH for ~70 ms).  Reuse of a ring region waits for
// the copy kernels that read it (events recorded after each one).
struct Staging {
  std::mutex mtx;
  std::uint8_t* host = nullptr;
  std::uint8_t* dev = nullptr;  // the ring's device-side address (mapped)
  std::size_t cap = 0, off = 0;
  std::vector<cudaEvent_t> inflight, spare;  // copy kernels since the last wrap
  void ensure() {
    if (host) return;
    cap = std::size_t(64) << 20;
    GFQ_CUDA(cudaHostAlloc(reinterpret_cast<void**>(&host), cap, cudaHostAllocMapped | cudaHostAllocPortable));
    GFQ_CUDA(cudaHostGetDevicePointer(reinterpret_cast<void**>(&dev), host, 0));
  }
  cudaEvent_t event() {
    if (spare.empty()) {
      cudaEvent_t e;
      GFQ_CUDA(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
      return e;
    }
    cudaEvent_t e = spare.back();
    spare.pop_back();
    return e;
  }
  void drain() {
    for (cudaEvent_t e : inflight) {
      GFQ_CUDA(cudaEventSynchronize(e));
      spare.push_back(e);
    }
    inflight.clear();
  }
};
Staging& staging() {
  static Staging* st = new Staging();  // intentionally leaked (process lifetime)
  return *st;
}
}  // namespace

void warm_runtime() {
  init_pool();
  // Map pool memory once up front (release threshold is infinite, so it
  // stays mapped): later cache misses carve from it instead of growing the
  // pool by a few hundred microseconds each.
  static std::once_flag reserve_once;
  std::call_once(reserve_once, [] {
    const char* e = std::getenv("GFQ_POOL_RESERVE_MB");
    const std::size_t mb = e ? std::size_t(std::atoll(e)) : 4096;
    if (mb == 0) return;
    void* p = nullptr;
    if (cudaMallocAsync(&p, mb << 20, cur_stream_raw()) == cudaSuccess) {
      GFQ_CUDA(cudaFreeAsync(p, cur_stream_raw()));
      GFQ_CUDA(cudaStreamSynchronize(cur_stream_raw()));
    } else {
      cudaGetLastError();
    }
  });
  Staging& st = staging();
  std::lock_guard<std::mutex> lk(st.mtx);
  st.ensure();
}

std::shared_ptr<DevBuf> upload_i32(const std::vector<std::int32_t>& v) {
  hprof::Scope hp(hprof::kUpload);
  const std::size_t bytes = v.size() * sizeof(std::int32_t);
  auto buf = std::make_shared<DevBuf>(bytes > 0 ? bytes : 4);
  if (bytes == 0) return buf;
  Staging& st = staging();
  const std::size_t need = (bytes + 255) / 256 * 256;
  std::lock_guard<std::mutex> lk(st.mtx);
  st.ensure();
  if (need > st.cap) {
    // oversized: synchronous copy through pageable memory
    GFQ_CUDA(cudaMemcpyAsync(buf->ptr, v.data(), bytes, cudaMemcpyHostToDevice, cur_stream()));
    GFQ_CUDA(cudaStreamSynchronize(cur_stream()));
    return buf;
  }
  if (st.off + need > st.cap) {
    // wrap: the copy kernels that read the ring since the last wrap must be done
    st.drain();
    st.off = 0;
  }
  std::memcpy(st.host + st.off, v.data(), bytes);
  const cudaStream_t s = cur_stream();
  dev::copy_from_mapped(buf->ptr, st.dev + st.off, bytes, s);
  cudaEvent_t e = st.event();
  GFQ_CUDA(cudaEventRecord(e, s));
  st.inflight.push_back(e);
  st.off += need;
  return buf;
}

void download_i32(const std::int32_t* dev, std::int32_t* host, std::size_t n) {
  if (n == 0) return;
  hprof::Scope hp(hprof::kSync);
  // through a per-thread pinned, device-mapped buffer written by a kernel:
  // no copy-engine transfer, so a readback never queues behind a bulk
  // host copy (the streamed input of gfq_echelonize_host)
  struct Mapped {
    std::uint8_t* host = nullptr;
    std::uint8_t* dev = nullptr;
    std::size_t cap = 0;
    ~Mapped() {
      if (host) cudaFreeHost(host);
    }
  };
  thread_local Mapped mb;
  const std::size_t bytes = n * sizeof(std::int32_t);
  if (bytes > mb.cap) {
    if (mb.host) GFQ_CUDA(cudaFreeHost(mb.host));
    mb.cap = std::max<std::size_t>(bytes, std::size_t(1) << 16);
    GFQ_CUDA(cudaHostAlloc(reinterpret_cast<void**>(&mb.host), mb.cap, cudaHostAllocMapped | cudaHostAllocPortable));
    GFQ_CUDA(cudaHostGetDevicePointer(reinterpret_cast<void**>(&mb.dev), mb.host, 0));
  }
  const cudaStream_t s = cur_stream();
  dev::copy_to_mapped(mb.dev, reinterpret_cast<const std::uint8_t*>(dev), bytes, s);
  GFQ_CUDA(cudaStreamSynchronize(s));
  std::memcpy(host, mb.host, bytes);
}

}  // namespace gfq
