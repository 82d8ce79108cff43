// runtime.cpp -- device memory, streams, staging and the value types.
#include <algorithm>
#include <atomic>
#include <cstring>
#include <mutex>
#include <stdexcept>

#include "types.hpp"

namespace gfq {

[[noreturn]] void throw_cuda(cudaError_t e, const char* what, const char* file, int line) {
  throw CudaError(std::string("CUDA error ") + cudaGetErrorName(e) + " (" +
                  cudaGetErrorString(e) + ") in " + what + " at " + file + ":" +
                  std::to_string(line));
}

namespace {
thread_local cudaStream_t t_stream = nullptr;
std::atomic<std::int64_t> g_live{0}, g_peak{0};
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

cudaStream_t cur_stream() { return t_stream; }
void set_cur_stream(cudaStream_t s) { t_stream = s; }

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
FieldSpec::FieldSpec(std::uint32_t p) : p_(p) {
  bool prime = p >= 2;
  for (std::uint32_t d = 2; prime && d * d <= p; ++d)
    if (p % d == 0) prime = false;
  if (!prime) throw std::invalid_argument("field: p must be prime");
  if (p > 251)
    throw std::invalid_argument("field: the B200 path stores residues as u8 (p <= 251)");
}

Elem FieldSpec::inv(Elem a) const {
  if (a % p_ == 0) throw std::domain_error("field: inverse of zero");
  std::uint64_t r = 1, b = a % p_;
  std::uint32_t e = p_ - 2;
  while (e) {
    if (e & 1) r = r * b % p_;
    b = b * b % p_;
    e >>= 1;
  }
  return Elem(r);
}

// ---------------------------------------------------------------- DevBuf / Mat
DevBuf::DevBuf(std::size_t n) : bytes(n) {
  if (n == 0) return;
  init_pool();
  void* p = nullptr;
  GFQ_CUDA(cudaMallocAsync(&p, n, cur_stream()));
  ptr = static_cast<std::uint8_t*>(p);
  const std::int64_t now = (g_live += std::int64_t(n));
  std::int64_t prev = g_peak.load();
  while (now > prev && !g_peak.compare_exchange_weak(prev, now)) {
  }
}

DevBuf::~DevBuf() {
  if (ptr) {
    // Stream-ordered free: every job on this value was issued on the
    // current stream (or joined into it by the executor) before release.
    cudaFreeAsync(ptr, cur_stream());
    g_live -= std::int64_t(bytes);
  }
}

std::int64_t live_device_bytes() { return g_live; }
std::int64_t peak_device_bytes() { return g_peak; }
void reset_peak_device_bytes() { g_peak = g_live.load(); }

Mat::Mat(std::int64_t rows, std::int64_t cols) : rows_(rows), cols_(cols) {
  if (rows < 0 || cols < 0) throw std::invalid_argument("matrix: negative shape");
  ld_ = round_up(cols > 0 ? cols : 1, 16);
  if (rows > 0 && cols > 0) {
    buf_ = std::make_shared<DevBuf>(std::size_t(rows) * std::size_t(ld_));
    data_ = buf_->ptr;
  }
}

Mat Mat::zeros(std::int64_t rows, std::int64_t cols) {
  Mat m(rows, cols);
  if (!m.empty())
    GFQ_CUDA(cudaMemsetAsync(m.data_, 0, std::size_t(rows) * std::size_t(m.ld_), cur_stream()));
  return m;
}

Mat Mat::from_host(std::int64_t rows, std::int64_t cols, const std::uint8_t* src,
                   std::int64_t ld) {
  Mat m(rows, cols);
  if (!m.empty()) {
    GFQ_CUDA(cudaMemcpy2DAsync(m.data_, std::size_t(m.ld_), src, std::size_t(ld),
                               std::size_t(cols), std::size_t(rows), cudaMemcpyHostToDevice,
                               cur_stream()));
    // pageable source: make the copy complete before the caller may reuse it
    GFQ_CUDA(cudaStreamSynchronize(cur_stream()));
  }
  return m;
}

Mat Mat::view_of(std::shared_ptr<DevBuf> buf, std::size_t offset, std::int64_t rows,
                 std::int64_t cols, std::int64_t ld) {
  Mat v;
  v.rows_ = rows;
  v.cols_ = cols;
  v.ld_ = ld;
  if (rows > 0 && cols > 0) {
    if (!buf || offset + std::size_t((rows - 1) * ld + cols) > buf->bytes)
      throw std::invalid_argument("matrix: view outside its allocation");
    v.data_ = buf->ptr + offset;
  }
  v.buf_ = std::move(buf);
  return v;
}

Mat Mat::row_view(std::int64_t r0, std::int64_t n) const {
  if (r0 < 0 || n < 0 || r0 + n > rows_) throw std::invalid_argument("matrix: row view out of range");
  Mat v;
  v.buf_ = buf_;
  v.rows_ = n;
  v.cols_ = cols_;
  v.ld_ = ld_;
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
  v.data_ = (data_ && n > 0 && rows_ > 0) ? data_ + c0 : nullptr;
  return v;
}

void Mat::to_host(std::uint8_t* dst, std::int64_t ld) const {
  if (empty()) return;
  GFQ_CUDA(cudaMemcpy2DAsync(dst, std::size_t(ld), data_, std::size_t(ld_), std::size_t(cols_),
                             std::size_t(rows_), cudaMemcpyDeviceToHost, cur_stream()));
  GFQ_CUDA(cudaStreamSynchronize(cur_stream()));
}

std::vector<std::uint8_t> Mat::to_host() const {
  std::vector<std::uint8_t> out(std::size_t(rows_) * std::size_t(cols_));
  to_host(out.data(), cols_ > 0 ? cols_ : 1);
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
// One process-wide pinned staging ring for small index uploads (pinning is
// expensive: it is done once, not per executor thread or per call).
struct Staging {
  std::mutex mtx;
  std::uint8_t* host = nullptr;
  std::size_t cap = 0, off = 0;
};
Staging& staging() {
  static Staging* st = new Staging();  // intentionally leaked (process lifetime)
  return *st;
}
}  // namespace

std::shared_ptr<DevBuf> upload_i32(const std::vector<std::int32_t>& v) {
  const std::size_t bytes = v.size() * sizeof(std::int32_t);
  auto buf = std::make_shared<DevBuf>(bytes > 0 ? bytes : 4);
  if (bytes == 0) return buf;
  Staging& st = staging();
  const std::size_t need = (bytes + 255) / 256 * 256;
  std::lock_guard<std::mutex> lk(st.mtx);
  if (!st.host) {
    st.cap = std::size_t(64) << 20;
    GFQ_CUDA(cudaMallocHost(reinterpret_cast<void**>(&st.host), st.cap));
  }
  if (need > st.cap) {
    // oversized: synchronous copy through pageable memory
    GFQ_CUDA(cudaMemcpyAsync(buf->ptr, v.data(), bytes, cudaMemcpyHostToDevice, cur_stream()));
    GFQ_CUDA(cudaStreamSynchronize(cur_stream()));
    return buf;
  }
  if (st.off + need > st.cap) {
    // wrap: earlier copies out of the ring (on any stream) must have landed
    GFQ_CUDA(cudaDeviceSynchronize());
    st.off = 0;
  }
  std::memcpy(st.host + st.off, v.data(), bytes);
  GFQ_CUDA(cudaMemcpyAsync(buf->ptr, st.host + st.off, bytes, cudaMemcpyHostToDevice,
                           cur_stream()));
  st.off += need;
  return buf;
}

void download_i32(const std::int32_t* dev, std::int32_t* host, std::size_t n) {
  if (n == 0) return;
  GFQ_CUDA(cudaMemcpyAsync(host, dev, n * sizeof(std::int32_t), cudaMemcpyDeviceToHost,
                           cur_stream()));
  GFQ_CUDA(cudaStreamSynchronize(cur_stream()));
}

}  // namespace gfq
