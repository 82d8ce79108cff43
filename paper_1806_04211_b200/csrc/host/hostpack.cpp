// hostpack.cpp -- see hostpack.hpp.
#include "hostpack.hpp"

#include <cuda_runtime.h>
#include <immintrin.h>

#include <algorithm>
#include <atomic>
#include <cstdlib>
#include <cstring>
#include <deque>
#include <thread>
#include <vector>

#include "../common.hpp"

namespace gfq::hostpack {

namespace {
std::atomic<int> g_enabled{[] {
  const char* e = std::getenv("GFQ_HOST_PACK");
  const int v = e ? std::atoi(e) : 0;
  return v >= 0 && v <= 64 ? v : 0;
}()};
}  // namespace
bool enabled() { return g_enabled.load() != 0; }
void set_enabled(bool on) { g_enabled.store(on ? 1 : 0); }
int stride() { return g_enabled.load(); }
void set_stride(int n) { g_enabled.store(n >= 0 && n <= 64 ? n : 0); }
bool packs(std::size_t index) {
  const int n = g_enabled.load();
  return n > 0 && index % std::size_t(n) == std::size_t(n - 1);
}

namespace {

bool have_avx512bw() {
  static const bool yes = __builtin_cpu_supports("avx512bw") && __builtin_cpu_supports("avx512f");
  return yes;
}

// 64 elements -> 8 bytes per step: a byte is 1 iff it is odd (GF(2) values)
__attribute__((target("avx512f,avx512bw"))) void pack_row_avx512(const std::uint8_t* s, std::int64_t cols,
                                                                   std::uint8_t* d) {
  const __m512i one = _mm512_set1_epi8(1);
  std::int64_t c = 0;
  for (; c + 64 <= cols; c += 64) {
    const __m512i v = _mm512_loadu_si512(reinterpret_cast<const void*>(s + c));
    const std::uint64_t m = _mm512_test_epi8_mask(v, one);
    std::memcpy(d + c / 8, &m, 8);
  }
  for (; c < cols; c += 8) {
    std::uint32_t byte = 0;
    for (int k = 0; k < 8 && c + k < cols; ++k) byte |= std::uint32_t(s[c + k] & 1u) << k;
    d[c / 8] = static_cast<std::uint8_t>(byte);
  }
}

__attribute__((target("avx512f,avx512bw"))) void unpack_row_avx512(const std::uint8_t* s, std::int64_t cols,
                                                                     std::uint8_t* d) {
  const __m512i one = _mm512_set1_epi8(1);
  std::int64_t c = 0;
  for (; c + 64 <= cols; c += 64) {
    std::uint64_t m;
    std::memcpy(&m, s + c / 8, 8);
    _mm512_storeu_si512(reinterpret_cast<void*>(d + c), _mm512_maskz_mov_epi8(m, one));
  }
  for (; c < cols; ++c) d[c] = static_cast<std::uint8_t>((s[c / 8] >> (c % 8)) & 1u);
}

void pack_row_scalar(const std::uint8_t* s, std::int64_t cols, std::uint8_t* d) {
  for (std::int64_t c = 0; c < cols; c += 8) {
    std::uint32_t byte = 0;
    for (int k = 0; k < 8 && c + k < cols; ++k) byte |= std::uint32_t(s[c + k] & 1u) << k;
    d[c / 8] = static_cast<std::uint8_t>(byte);
  }
}

void unpack_row_scalar(const std::uint8_t* s, std::int64_t cols, std::uint8_t* d) {
  for (std::int64_t c = 0; c < cols; ++c) d[c] = static_cast<std::uint8_t>((s[c / 8] >> (c % 8)) & 1u);
}

class Pool {
 public:
  explicit Pool(int n) {
    for (int i = 0; i < n; ++i)
      threads_.emplace_back([this] {
        for (;;) {
          std::function<void()> fn;
          {
            std::unique_lock<std::mutex> lk(m_);
            cv_.wait(lk, [&] { return !q_.empty(); });
            fn = std::move(q_.front());
            q_.pop_front();
          }
          fn();
        }
      });
    for (auto& t : threads_) t.detach();  // process lifetime
  }
  void submit(std::function<void()> fn) {
    {
      std::lock_guard<std::mutex> lk(m_);
      q_.push_back(std::move(fn));
    }
    cv_.notify_one();
  }
  int size() const { return int(threads_.size()); }

 private:
  std::mutex m_;
  std::condition_variable cv_;
  std::deque<std::function<void()>> q_;
  std::vector<std::thread> threads_;
};

Pool& pool() {
  static Pool* p = [] {
    const char* e = std::getenv("GFQ_HOST_THREADS");
    const int hw = int(std::thread::hardware_concurrency());
    const int n = e ? std::max(1, std::atoi(e)) : std::max(1, std::min(8, hw / 2));
    return new Pool(n);
  }();
  return *p;
}

}  // namespace

void pack_rows(const std::uint8_t* src, std::int64_t ld, std::int64_t rows, std::int64_t cols, std::uint8_t* dst,
               std::int64_t ldb) {
  const bool v = have_avx512bw();
  for (std::int64_t r = 0; r < rows; ++r)
    v ? pack_row_avx512(src + r * ld, cols, dst + r * ldb) : pack_row_scalar(src + r * ld, cols, dst + r * ldb);
}

void unpack_rows(const std::uint8_t* src, std::int64_t ldb, std::int64_t rows, std::int64_t cols, std::uint8_t* dst,
                 std::int64_t ld) {
  const bool v = have_avx512bw();
  for (std::int64_t r = 0; r < rows; ++r)
    v ? unpack_row_avx512(src + r * ldb, cols, dst + r * ld) : unpack_row_scalar(src + r * ldb, cols, dst + r * ld);
}

void Latch::add(std::int64_t k) {
  std::lock_guard<std::mutex> lk(m_);
  n_ += k;
}
void Latch::done() {
  std::lock_guard<std::mutex> lk(m_);
  if (--n_ <= 0) cv_.notify_all();
}
void Latch::wait() {
  std::unique_lock<std::mutex> lk(m_);
  cv_.wait(lk, [&] { return n_ <= 0; });
}

void submit(std::function<void()> fn) { pool().submit(std::move(fn)); }
int pool_threads() { return pool().size(); }

namespace {
std::mutex g_pin_m;
std::vector<std::pair<std::size_t, std::uint8_t*>>* g_pin_free = new std::vector<std::pair<std::size_t, std::uint8_t*>>();
}  // namespace

PinnedLease::PinnedLease(std::size_t bytes) {
  {
    std::lock_guard<std::mutex> lk(g_pin_m);
    auto& v = *g_pin_free;
    // the smallest free buffer that fits
    std::size_t best = v.size();
    for (std::size_t i = 0; i < v.size(); ++i)
      if (v[i].first >= bytes && (best == v.size() || v[i].first < v[best].first)) best = i;
    if (best < v.size()) {
      cap_ = v[best].first;
      p_ = v[best].second;
      v.erase(v.begin() + std::ptrdiff_t(best));
      return;
    }
  }
  cap_ = std::max<std::size_t>(bytes, 1);
  GFQ_CUDA(cudaHostAlloc(reinterpret_cast<void**>(&p_), cap_, cudaHostAllocPortable));
}

PinnedLease::~PinnedLease() {
  if (!p_) return;
  std::lock_guard<std::mutex> lk(g_pin_m);
  g_pin_free->emplace_back(cap_, p_);
}

TransferBytes& last_transfer() {
  thread_local TransferBytes t;
  return t;
}

}  // namespace gfq::hostpack
