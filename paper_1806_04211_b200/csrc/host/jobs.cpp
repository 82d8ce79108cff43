// jobs.cpp -- block jobs on device (see jobs.hpp).
#include "jobs.hpp"

#include <algorithm>
#include <cstdlib>
#include <string>
#include <atomic>
#include <memory>
#include <mutex>
#include <vector>
#include <stdexcept>

#include "../kernels/kernels.hpp"

namespace gfq {

bool runs_of(const std::vector<std::int32_t>& map, std::vector<Run>& out, std::size_t cap) {
  out.clear();
  for (std::size_t t = 0; t < map.size();) {
    const std::int32_t v = map[t];
    const int from = v >= 0 ? 0 : (v == -1 ? -1 : 1);
    const std::int64_t src = v >= 0 ? v : (v == -1 ? 0 : -std::int64_t(v) - 2);
    std::size_t e = t + 1;
    while (e < map.size()) {
      const std::int32_t w = map[e];
      const std::int64_t d = std::int64_t(e - t);
      const bool cont = from == 0 ? w == v + d : (from == -1 ? w == -1 : w == v - d);
      if (!cont) break;
      ++e;
    }
    out.push_back(Run{std::int64_t(t), std::int64_t(e - t), src, from});
    if (out.size() > cap) return false;
    t = e;
  }
  return true;
}
namespace {
std::atomic<std::size_t> g_ech_base{64};

const std::int32_t* dptr(const std::shared_ptr<DevBuf>& b) {
  return b ? reinterpret_cast<const std::int32_t*>(b->ptr) : nullptr;
}

// out = select(A | B) by optional row/column maps (kernels.hpp select2d).
Mat select(std::int64_t rows, std::int64_t cols, const Mat& A, const Mat* B,
           const std::vector<std::int32_t>* rmap, const std::vector<std::int32_t>* cmap) {
  // element size of the result: the sources' (an empty source carries no
  // storage and may have been made without one)
  int es = A.esize();
  if (B && B->esize() != es) {
    if (A.empty())
      es = B->esize();
    else if (!B->empty())
      throw std::invalid_argument("select: element sizes of the sources disagree");
  }
  Mat out(rows, cols, es);
  if (out.empty()) return out;
  // wide elements: the byte-level kernels get byte columns and a byte map
  std::vector<std::int32_t> bmap;
  if (es != 1 && cmap) {
    bmap.resize(cmap->size() * std::size_t(es));
    for (std::size_t j = 0; j < cmap->size(); ++j) {
      const std::int32_t v = (*cmap)[j];
      for (int b = 0; b < es; ++b)
        bmap[j * std::size_t(es) + std::size_t(b)] =
            v >= 0 ? v * es + b : (v == -1 ? -1 : -((-v - 2) * es + b) - 2);
    }
    cmap = &bmap;
  }
  const std::int64_t bcols = cols * es;
  // small maps ride in the launch parameters (no upload call)
  static const bool inline_maps = std::getenv("GFQ_NO_INLINE_MAPS") == nullptr;
  if (inline_maps &&
      dev::select2d_inline(out.data(), out.ld(), rows, bcols, A.data(), A.ld(), B ? B->data() : nullptr,
                           B ? B->ld() : 0, rmap ? rmap->data() : nullptr,
                           cmap ? cmap->data() : nullptr, cur_stream()))
    return out;
  auto rb = rmap ? upload_i32(*rmap) : nullptr;
  auto cb = cmap ? upload_i32(*cmap) : nullptr;
  dev::select2d(out.data(), out.ld(), rows, bcols, A.data(), A.ld(), B ? B->data() : nullptr,
                B ? B->ld() : 0, dptr(rb), dptr(cb), cur_stream());
  return out;
}

std::vector<std::int32_t> as_i32(const std::vector<std::uint32_t>& v) {
  return std::vector<std::int32_t>(v.begin(), v.end());
}
}  // namespace

namespace {
std::atomic<int> g_ech_mode{0};
}
void set_ech_mode(int mode) { g_ech_mode = mode; }
int ech_mode() { return g_ech_mode; }

void random_fill_exact(std::uint32_t p, std::int64_t rows, std::int64_t cols, std::uint64_t seed,
                       std::uint64_t draw0, std::int64_t draw_ld, std::uint8_t* dst,
                       std::int64_t ld, int esize) {
  if (rows == 0 || cols == 0) return;
  DevBuf rej{4};
  dev::fill2d(rej.ptr, 4, 1, 4, 0, cur_stream());
  if (esize == 4)
    dev::random_fill_wide(p, rows, cols, seed, draw0, draw_ld, dst, ld,
                          reinterpret_cast<std::uint32_t*>(rej.ptr), cur_stream());
  else
    dev::random_fill(p, rows, cols, seed, draw0, draw_ld, dst, ld,
                     reinterpret_cast<std::uint32_t*>(rej.ptr), cur_stream());
  std::int32_t nrej = 0;
  download_i32(reinterpret_cast<const std::int32_t*>(rej.ptr), &nrej, 1);
  if (nrej != 0)
    throw std::runtime_error(
        "random_matrix: a SplitMix64 draw hit the rejection band; exact replay not supported");
}

void set_ech_base(std::size_t n) {
  g_ech_base = std::max<std::size_t>(1, std::min<std::size_t>(n, dev::kEchBaseMax));
}
std::size_t ech_base() { return g_ech_base; }

// ---------------------------------------------------------------- packed B cache
namespace {
thread_local DevBuf* t_b_owner = nullptr;
struct PackedB {
  const std::uint8_t* src;
  std::int64_t n, k, ldb;
  std::uint32_t p;
  cudaStream_t stream;
  cudaEvent_t ev = nullptr;
  std::unique_ptr<DevBuf> buf;
};
struct PackedBCache {
  std::mutex mtx;
  std::vector<PackedB> items;
  ~PackedBCache() {
    for (auto& it : items)
      if (it.ev) cudaEventDestroy(it.ev);
  }
};
std::mutex g_packed_create_mtx;
// The packing of B (k x n at ldb) held with its storage, made on `s` if this
// is the first contraction to need it; nullptr when B is not inside the
// thread's ImmutableB scope.  The returned block is ordered before s.
const std::uint8_t* packed_b_for(std::uint32_t p, std::int64_t n, std::int64_t k, const std::uint8_t* B,
                                 std::int64_t ldb, cudaStream_t s) {
  static const bool off = std::getenv("GFQ_NO_BPACK_CACHE") != nullptr;
  DevBuf* owner = t_b_owner;
  if (off || !owner || !owner->ptr || B < owner->ptr || B >= owner->ptr + owner->bytes) return nullptr;
  PackedBCache* cache;
  {
    std::lock_guard<std::mutex> lk(g_packed_create_mtx);
    if (!owner->packed_b) owner->packed_b = std::make_shared<PackedBCache>();
    cache = static_cast<PackedBCache*>(owner->packed_b.get());
  }
  std::lock_guard<std::mutex> lk(cache->mtx);
  for (const PackedB& it : cache->items)
    if (it.src == B && it.n == n && it.k == k && it.ldb == ldb && it.p == p) {
      if (it.stream != s) GFQ_CUDA(cudaStreamWaitEvent(s, it.ev, 0));
      return it.buf->ptr;
    }
  PackedB it{B, n, k, ldb, p, s, nullptr, nullptr};
  it.buf = std::make_unique<DevBuf>(static_cast<std::size_t>(dev::mad_f4_bt_bytes(n, k)));
  GFQ_CUDA(cudaEventCreateWithFlags(&it.ev, cudaEventDisableTiming));
  dev::pack_b_f4(p, n, k, B, ldb, it.buf->ptr, s);
  GFQ_CUDA(cudaEventRecord(it.ev, s));
  cache->items.push_back(std::move(it));
  return cache->items.back().buf->ptr;
}
}  // namespace
ImmutableB::ImmutableB(const Mat& b) : prev_(t_b_owner) { t_b_owner = b.buf().get(); }
ImmutableB::~ImmutableB() { t_b_owner = prev_; }

// ---------------------------------------------------------------- products
// D = (Cin ? Cin : 0) + A.B over the field: K1 for GF(p), the digit-plane
// contraction (dev::mad_ext, one K1 launch over GF(p)) for GF(p^k).
void field_mad(const FieldSpec& f, std::int64_t m, std::int64_t n, std::int64_t k,
               const std::uint8_t* A, std::int64_t lda, const std::uint8_t* B, std::int64_t ldb,
               const std::uint8_t* Cin, std::int64_t ldc, std::uint8_t* D, std::int64_t ldd,
               cudaStream_t s) {
  if (f.wide()) {
    dev::mad_wide(f.wide_dev(), m, n, k, A, lda, B, ldb, Cin, ldc, D, ldd, s);
    return;
  }
  if (!f.is_ext()) {
    // K1f (FP4 tensor cores) for the small fields: its packed operands live
    // in a stream-ordered scratch block on this (the current) stream
    if (s == cur_stream_raw() && dev::use_f4(f.p(), m, n, k)) {
      if (const std::uint8_t* bt = packed_b_for(f.p(), n, k, B, ldb, s)) {
        DevBuf scratch{static_cast<std::size_t>(dev::mad_f4_scratch_bytes(m, 0, k))};
        if (dev::mad_f4(f.p(), m, n, k, A, lda, B, ldb, Cin, ldc, D, ldd, scratch.ptr, s, bt)) return;
      } else {
        DevBuf scratch{static_cast<std::size_t>(dev::mad_f4_scratch_bytes(m, n, k))};
        if (dev::mad_f4(f.p(), m, n, k, A, lda, B, ldb, Cin, ldc, D, ldd, scratch.ptr, s)) return;
      }
    }
    dev::mad(f.p(), m, n, k, A, lda, B, ldb, Cin, ldc, D, ldd, s);
    return;
  }
  if (m == 0 || n == 0) return;
  DevBuf scratch{static_cast<std::size_t>(dev::mad_ext_scratch_bytes(f.k(), m, n, k))};
  dev::mad_ext(f.ext_dev(), m, n, k, A, lda, B, ldb, Cin, ldc, D, ldd, scratch.ptr, s);
}

static Mat mul_add_kernel(const FieldSpec& f, const Mat* addend, const Mat& b, const Mat& c) {
  // reference src/matrix.cpp:81-89 shape contract
  if (b.cols() != c.rows()) throw std::invalid_argument("mul: inner dimensions disagree");
  if (addend && (addend->rows() != b.rows() || addend->cols() != c.cols()))
    throw std::invalid_argument("mad: addend shape mismatch");
  const std::int64_t m = b.rows(), inner = b.cols(), n = c.cols();
  Mat out(m, n, f.esize());
  if (m == 0 || n == 0) return out;
  field_mad(f, m, n, inner, b.data(), b.ld(), c.data(), c.ld(),
            addend ? addend->data() : nullptr, addend ? addend->ld() : 0, out.data(), out.ld(),
            cur_stream());
  return out;
}

Mat mat_mul(const FieldSpec& f, const Mat& b, const Mat& c) {
  return mul_add_kernel(f, nullptr, b, c);
}

void col_gather_into(const Mat& dst, const Mat& a, const Mat* b, const std::vector<std::int32_t>* cmap) {
  if (dst.empty()) return;
  if (dst.esize() != 1 || a.esize() != 1 || (b && b->esize() != 1))
    throw std::invalid_argument("col_gather_into: byte elements only");
  if (a.rows() != dst.rows() || (b && b->rows() != dst.rows()) ||
      (cmap ? std::int64_t(cmap->size()) != dst.cols() : a.cols() != dst.cols()))
    throw std::invalid_argument("col_gather_into: shape mismatch");
  auto cb = cmap ? upload_i32(*cmap) : nullptr;
  dev::select2d(dst.data(), dst.ld(), dst.rows(), dst.cols(), a.data(), a.ld(), b ? b->data() : nullptr,
                b ? b->ld() : 0, nullptr, dptr(cb), cur_stream());
}

Mat col_gather(const Mat& m, std::int64_t out_cols, const std::vector<std::int32_t>& cmap) {
  return select(m.rows(), out_cols, m, nullptr, nullptr, &cmap);
}
Mat col_gather2(const Mat& a, const Mat* b, std::int64_t out_cols, const std::vector<std::int32_t>& cmap) {
  return select(a.rows(), out_cols, a, b, nullptr, &cmap);
}

void mad_into(const FieldSpec& f, const Mat& d, const Mat* addend, const Mat& b, const Mat& c) {
  if (b.cols() != c.rows()) throw std::invalid_argument("mul: inner dimensions disagree");
  if (d.rows() != b.rows() || d.cols() != c.cols())
    throw std::invalid_argument("mad_into: destination shape mismatch");
  if (addend && (addend->rows() != b.rows() || addend->cols() != c.cols()))
    throw std::invalid_argument("mad_into: addend shape mismatch (" + std::to_string(addend->rows()) +
                                "x" + std::to_string(addend->cols()) + " vs " +
                                std::to_string(b.rows()) + "x" + std::to_string(c.cols()) + ")");
  if (d.empty()) return;
  field_mad(f, d.rows(), d.cols(), b.cols(), b.data(), b.ld(), c.data(), c.ld(),
            addend ? addend->data() : nullptr, addend ? addend->ld() : 0, d.data(), d.ld(),
            cur_stream());
}
Mat mat_mul_add(const FieldSpec& f, const Mat& a, const Mat& b, const Mat& c) {
  return mul_add_kernel(f, &a, b, c);
}
Mat mul(const FieldSpec& f, const Mat& b, const Mat& c) { return mat_mul(f, b, c); }
Mat mad(const FieldSpec& f, const Mat& a, const Mat& b, const Mat& c) {
  return mat_mul_add(f, a, b, c);
}

Mat cpy(const Mat& a) { return select(a.rows(), a.cols(), a, nullptr, nullptr, nullptr); }

// ---------------------------------------------------------------- gathers
Mat take_rows(const Mat& m, const std::vector<std::uint32_t>& rows) {
  for (auto r : rows)
    if (std::int64_t(r) >= m.rows()) throw std::invalid_argument("take_rows: index out of range");
  const auto map = as_i32(rows);
  return select(std::int64_t(rows.size()), m.cols(), m, nullptr, &map, nullptr);
}

Mat take_cols(const Mat& m, const std::vector<std::uint32_t>& cols) {
  for (auto c : cols)
    if (std::int64_t(c) >= m.cols()) throw std::invalid_argument("take_cols: index out of range");
  const auto map = as_i32(cols);
  return select(m.rows(), std::int64_t(cols.size()), m, nullptr, nullptr, &map);
}

Mat vcat(const Mat& a, const Mat& b) {
  if (a.cols() != b.cols()) throw std::invalid_argument("vcat: column counts disagree");
  std::vector<std::int32_t> map(std::size_t(a.rows() + b.rows()));
  for (std::int64_t i = 0; i < a.rows(); ++i) map[i] = std::int32_t(i);
  for (std::int64_t i = 0; i < b.rows(); ++i) map[a.rows() + i] = -std::int32_t(i) - 2;
  return select(a.rows() + b.rows(), a.cols(), a, &b, &map, nullptr);
}

Mat hcat(const Mat& a, const Mat& b) {
  if (a.rows() != b.rows()) throw std::invalid_argument("hcat: row counts disagree");
  std::vector<std::int32_t> map(std::size_t(a.cols() + b.cols()));
  for (std::int64_t j = 0; j < a.cols(); ++j) map[j] = std::int32_t(j);
  for (std::int64_t j = 0; j < b.cols(); ++j) map[a.cols() + j] = -std::int32_t(j) - 2;
  return select(a.rows(), a.cols() + b.cols(), a, &b, nullptr, &map);
}

// Column riffle of two matrices (reference src/jobs.cpp:13-28).
static Mat col_riffle(const BitString& u, const Mat& zeros_side, const Mat& ones_side) {
  if (zeros_side.rows() != ones_side.rows())
    throw std::invalid_argument("col_riffle: row counts disagree");
  if (std::int64_t(u.count_zeros()) != zeros_side.cols() ||
      std::int64_t(u.count_ones()) != ones_side.cols())
    throw std::invalid_argument("col_riffle: bit counts disagree");
  std::vector<std::int32_t> map(u.size());
  std::int32_t zc = 0, oc = 0;
  for (std::size_t l = 0; l < u.size(); ++l) map[l] = u.bits[l] ? -(oc++) - 2 : zc++;
  return select(zeros_side.rows(), std::int64_t(u.size()), zeros_side, &ones_side, nullptr, &map);
}

std::pair<Mat, Mat> cex(const Mat& h, const IndexSet& gamma) {
  if (std::int64_t(gamma.universe) != h.cols()) throw std::invalid_argument("cex: universe mismatch");
  const IndexSet rest = index_set_complement(gamma);
  return {take_cols(h, gamma.members), take_cols(h, rest.members)};
}

std::pair<Mat, Mat> rex(const Mat& h, const IndexSet& rho) {
  if (std::int64_t(rho.universe) != h.rows()) throw std::invalid_argument("rex: universe mismatch");
  const IndexSet rest = index_set_complement(rho);
  return {take_rows(h, rho.members), take_rows(h, rest.members)};
}

// ---------------------------------------------------------------- index jobs (host)
std::pair<IndexSet, BitString> unh(const IndexSet& rho1, const IndexSet& rho2) {
  const IndexSet comp = index_set_complement(rho1);
  if (rho2.universe != comp.size())
    throw std::invalid_argument("unh: universe of rho2 must be the complement size");
  std::vector<std::uint32_t> merged;
  merged.reserve(rho1.size() + rho2.size());
  BitString u;
  u.bits.reserve(rho1.size() + rho2.size());
  std::size_t i = 0, j = 0;
  while (i < rho1.size() || j < rho2.size()) {
    const std::uint32_t e = j < rho2.size() ? comp.members[rho2.members[j]] : 0;
    if (j >= rho2.size() || (i < rho1.size() && rho1.members[i] < e)) {
      merged.push_back(rho1.members[i++]);
      u.bits.push_back(0);
    } else {
      merged.push_back(e);
      ++j;
      u.bits.push_back(1);
    }
  }
  return {IndexSet(rho1.universe, std::move(merged)), std::move(u)};
}

std::pair<IndexSet, BitString> un0(const IndexSet& rho2) {
  BitString u;
  u.bits.assign(rho2.size(), 1);
  return {rho2, std::move(u)};
}

BitString mkr(const IndexSet& rho1, const IndexSet& rho2) {
  BitString out;
  out.bits.assign(rho2.size(), 0);
  std::size_t i = 0;
  for (std::size_t l = 0; l < rho2.members.size(); ++l)
    if (i < rho1.members.size() && rho1.members[i] == rho2.members[l]) {
      out.bits[l] = 1;
      ++i;
    }
  if (i != rho1.members.size()) throw std::invalid_argument("mkr: rho1 must be a subset of rho2");
  return out;
}

// ---------------------------------------------------------------- riffles
Mat rrf(const BitString& u, const Mat& b, const Mat& c) {
  if (std::int64_t(u.count_zeros()) != b.rows() || std::int64_t(u.count_ones()) != c.rows())
    throw std::invalid_argument("rrf: bit counts do not match row counts");
  if (b.cols() != c.cols() && b.rows() != 0 && c.rows() != 0)
    throw std::invalid_argument("rrf: column counts disagree");
  const std::int64_t cols = (b.rows() != 0 || c.rows() == 0) ? b.cols() : c.cols();
  // one side empty: the riffle is the other input (values are immutable,
  // so the result may share its storage -- no copy)
  if (b.rows() == 0 && c.cols() == cols) return c;
  if (c.rows() == 0 && b.cols() == cols) return b;
  std::vector<std::int32_t> map(u.size());
  std::int32_t bi = 0, ci = 0;
  for (std::size_t l = 0; l < u.size(); ++l) map[l] = u.bits[l] ? -(ci++) - 2 : bi++;
  return select(std::int64_t(u.size()), cols, b, &c, &map, nullptr);
}

Mat crz(const Mat& m, const BitString& lambda, std::size_t out_cols) {
  if (lambda.size() != out_cols) throw std::invalid_argument("crz: lambda length must equal out_cols");
  if (std::int64_t(lambda.count_ones()) != m.cols())
    throw std::invalid_argument("crz: ones count must equal input columns");
  if (std::int64_t(out_cols) == m.cols()) return m;  // no zero column to insert
  std::vector<std::int32_t> map(out_cols);
  std::int32_t src = 0;
  for (std::size_t l = 0; l < out_cols; ++l) map[l] = lambda.bits[l] ? src++ : -1;
  return select(m.rows(), std::int64_t(out_cols), m, nullptr, nullptr, &map);
}

Mat adi(const Mat& k, const BitString& delta) {
  if (std::int64_t(delta.size()) != k.cols())
    throw std::invalid_argument("adi: delta length must equal columns");
  if (std::int64_t(delta.count_ones()) > k.rows())
    throw std::invalid_argument("adi: more marked positions than rows");
  Mat out = cpy(k);
  std::vector<std::int32_t> pos;
  std::int32_t i = 0;
  for (std::size_t l = 0; l < delta.size(); ++l)
    if (delta.bits[l]) {
      pos.push_back(i++);
      pos.push_back(std::int32_t(l));
    }
  if (!pos.empty()) {
    auto pb = upload_i32(pos);
    if (out.esize() == 4)
      dev::set_entries_u32(out.data(), out.ld(), dptr(pb), std::int64_t(pos.size() / 2), 1, cur_stream());
    else
      dev::set_entries(out.data(), out.ld(), dptr(pb), std::int64_t(pos.size() / 2), 1, cur_stream());
  }
  return out;
}

// ---------------------------------------------------------------- ECH
namespace {

// Base case: K2 kernel, then gather M/K/R in the reference's conventions
// (rows of M and R by ascending pivot column, columns of M/K by ascending
// selected row, rows of K by ascending non-selected row; jobs.cpp:85-120).
EchResult direct_ech(const FieldSpec& f, const Mat& h) {
  const std::int64_t a = h.rows(), b = h.cols();
  const std::int64_t rmax = std::min(a, b);
  Mat W(a, b, f.esize()), Tc(a, rmax > 0 ? rmax : 1, f.esize());
  auto info = std::make_shared<DevBuf>(std::size_t(4 * (2 * rmax + 1)));
  if (f.wide())
    dev::ech_base_wide(f.wide_dev(), a, b, h.data(), h.ld(), W.data(), W.ld(), Tc.data(), Tc.ld(),
                       reinterpret_cast<std::int32_t*>(info->ptr), cur_stream());
  else if (f.is_ext())
    dev::ech_base_ext(f.ext_dev(), a, b, h.data(), h.ld(), W.data(), W.ld(), Tc.data(), Tc.ld(),
                      reinterpret_cast<std::int32_t*>(info->ptr), cur_stream());
  else
    dev::ech_base(f.p(), a, b, h.data(), h.ld(), W.data(), W.ld(), Tc.data(), Tc.ld(),
                  reinterpret_cast<std::int32_t*>(info->ptr), cur_stream());
  std::vector<std::int32_t> hi(std::size_t(2 * rmax + 1));
  download_i32(reinterpret_cast<const std::int32_t*>(info->ptr), hi.data(), hi.size());
  const std::int64_t r = hi[0];
  std::vector<std::int32_t> pcol(hi.begin() + 1, hi.begin() + 1 + r);
  std::vector<std::int32_t> prow(hi.begin() + 1 + rmax, hi.begin() + 1 + rmax + r);

  EchResult out;
  std::vector<std::uint32_t> rho(prow.begin(), prow.end());
  std::sort(rho.begin(), rho.end());
  out.rho = IndexSet(std::size_t(a), rho);
  out.gamma = IndexSet(std::size_t(b), std::vector<std::uint32_t>(pcol.begin(), pcol.end()));
  // discovery position of each pivot row
  std::vector<std::int32_t> pos_of(std::size_t(a), -1);
  for (std::int64_t q = 0; q < r; ++q) pos_of[prow[q]] = std::int32_t(q);
  std::vector<std::int32_t> tcols(static_cast<std::size_t>(r));
  for (std::int64_t s = 0; s < r; ++s) tcols[s] = pos_of[rho[s]];
  const IndexSet grest = index_set_complement(out.gamma);
  const IndexSet nonsel = index_set_complement(out.rho);
  const auto gcols = as_i32(grest.members);
  const auto krows = as_i32(nonsel.members);
  out.M = select(r, r, Tc, nullptr, &prow, &tcols);
  out.K = select(a - r, r, Tc, nullptr, &krows, &tcols);
  out.R = select(r, b - r, W, nullptr, &prow, &gcols);
  return out;
}

// Read back the pivots (the one host round trip of a device ECH) and gather
// M, K, R from the reduced Aug = [W | T] (T uncompacted: column t = original
// row t) in the reference's conventions.
EchResult extract_ech(std::int64_t a, std::int64_t b, const Mat& aug, const std::int32_t* inf,
                      std::int64_t cap, std::int64_t toff) {
  std::vector<std::int32_t> hi(std::size_t(1 + 2 * cap));
  download_i32(inf, hi.data(), hi.size());
  const std::int64_t r = hi[0];
  std::vector<std::int32_t> pcol(hi.begin() + 1, hi.begin() + 1 + r);
  std::vector<std::int32_t> prow(hi.begin() + 1 + cap, hi.begin() + 1 + cap + r);
  EchResult out;
  std::vector<std::uint32_t> rho(prow.begin(), prow.end());
  std::sort(rho.begin(), rho.end());
  out.rho = IndexSet(std::size_t(a), rho);
  out.gamma = IndexSet(std::size_t(b), std::vector<std::uint32_t>(pcol.begin(), pcol.end()));
  const auto tcols = as_i32(rho);
  const auto krows = as_i32(index_set_complement(out.rho).members);
  const auto gcols = as_i32(index_set_complement(out.gamma).members);
  const Mat W = aug.col_view(0, b), T = aug.col_view(toff, a);
  out.M = select(r, r, T, nullptr, &prow, &tcols);
  out.K = select(a - r, r, T, nullptr, &krows, &tcols);
  out.R = select(r, b - r, W, nullptr, &prow, &gcols);
  return out;
}

// Outer panel width of the two-level device ECH (0 = one level).  Every
// block wider than one step takes 256-wide outer panels: the 32-wide steps
// then only sweep an L2-resident rows x 512 scratch (two fused launches a
// step), and the rest of [W | T] sees one K = 256 contraction per outer
// panel instead of eight K = 32 ones (cfg1's 500-blocks: 11.7 -> 5.5 ms a
// step).  GFQ_ECH_OUTER / set_ech_outer override (0 = one level).
constexpr std::int64_t kEchOuterMax = 256;
std::atomic<int> g_ech_outer{[] {
  const char* e = std::getenv("GFQ_ECH_OUTER");
  return e ? std::atoi(e) : -1;
}()};
std::int64_t ech_outer_width(std::int64_t b) {
  const std::int64_t forced = g_ech_outer;
  if (forced >= 0) return forced == 0 ? 0 : std::min<std::int64_t>(kEchOuterMax, std::max<std::int64_t>(32, forced / 32 * 32));
  return b > 32 ? kEchOuterMax : 0;
}

// Device ECH: right-looking panel Gauss-Jordan on Aug = [W | T] (T = I), one
// K2 panel launch + a row gather + two K1 launches per 32-column panel, no
// host round trip until the pivots are read back at the end.  Outputs in the
// reference's conventions (same extraction as direct_ech, T uncompacted).
// GF(2) blocks beyond the whole-block cluster kernel's fast path may take
// the two-level path with each outer panel factorized by ONE cluster launch
// (dev::ech_gf2_outer, rows <= 8192; ech mode 4 or GFQ_GF2_OUTER=1): no host
// round trip until the end, but on 8192^2 blocks it measured slower than the
// split (10.4 vs 8.7 ms alone, cfg5s 197 vs 174 ms), so the split stays the
// default.
bool gf2_outer_enabled() {
  static const bool env = [] {
    const char* e = std::getenv("GFQ_GF2_OUTER");
    return e && e[0] == '1';
  }();
  return ech_mode() == 4 || (env && ech_mode() == 0);
}
constexpr std::int64_t kGf2OuterRows = 8192;
std::int64_t gf2_outer_width() {
  static const std::int64_t w = [] {
    const char* e = std::getenv("GFQ_GF2_OUTER_W");
    const std::int64_t v = e ? std::atoll(e) : 256;
    return v == 512 ? std::int64_t(512) : std::int64_t(256);
  }();
  return w;
}

EchResult panel_ech(const FieldSpec& f, const Mat& h, bool block_cluster = true) {
  const std::int64_t a = h.rows(), b = h.cols(), w = 32;
  const std::int64_t cap = std::min(a, b);
  const cudaStream_t s = cur_stream();
  if (block_cluster && f.p() == 2 && a <= 1024 && (a + b + 31) / 32 <= 256) {
    DevBuf info{static_cast<std::size_t>(4 * (1 + 2 * cap))};
    auto* inf = reinterpret_cast<std::int32_t*>(info.ptr);
    {
      // GF(2), one 8-CTA cluster: the kernel writes M / K / R itself (no
      // unpacked [W | T] and no gathers on the host's critical path)
      Mat mb(cap, cap), kb(a, cap), rb(cap, b);
      const std::int64_t wd = (a + b + 31) / 32;
      DevBuf scratch{static_cast<std::size_t>(4 * a * wd + 2 * (2 * a + b) + 64)};
      auto* pk = reinterpret_cast<std::uint32_t*>(scratch.ptr);
      auto* maps = reinterpret_cast<std::int16_t*>(pk + a * wd);
      const dev::EchExtract ex{mb.data(), kb.data(), rb.data(), mb.ld(), kb.ld(), rb.ld(),
                               pk, maps, maps + a, maps + 2 * a};
      if (dev::ech_gf2_small(a, b, h.data(), h.ld(), inf, cap, s, ex) ||
          dev::ech_gf2_cluster(a, b, h.data(), h.ld(), nullptr, 0, inf, cap, s, &ex)) {
        std::vector<std::int32_t> hi(std::size_t(1 + 2 * cap));
        download_i32(inf, hi.data(), hi.size());
        const std::int64_t r = hi[0];
        EchResult out;
        std::vector<std::uint32_t> rho(hi.begin() + 1 + cap, hi.begin() + 1 + cap + r);
        std::sort(rho.begin(), rho.end());
        out.rho = IndexSet(std::size_t(a), std::move(rho));
        out.gamma = IndexSet(std::size_t(b), std::vector<std::uint32_t>(hi.begin() + 1, hi.begin() + 1 + r));
        out.M = mb.row_view(0, r).col_view(0, r);
        out.K = kb.row_view(0, a - r).col_view(0, r);
        out.R = rb.row_view(0, r).col_view(0, b - r);
        return out;
      }
    }
    Mat aug(a, b + a);
    {
      DevBuf scratch{static_cast<std::size_t>(4 * dev::ech_gf2_scratch_words(a, b))};
      dev::ech_gf2_block(a, b, h.data(), h.ld(), reinterpret_cast<std::uint32_t*>(scratch.ptr),
                         aug.data(), aug.ld(), inf, cap, s);
    }
    return extract_ech(a, b, aug, inf, cap, b);
  }
  // Aug = [W | 0 | T]: T starts at the 16-aligned column tb so every
  // trailing update below is a TMA-legal view
  const std::int64_t tb = (b + 15) / 16 * 16;
  Mat aug = Mat::zeros(a, tb + a);
  dev::select2d(aug.data(), aug.ld(), a, b, h.data(), h.ld(), nullptr, 0, nullptr, nullptr, s);
  {
    std::vector<std::int32_t> diag(std::size_t(2 * a));
    for (std::int64_t i = 0; i < a; ++i) {
      diag[2 * i] = std::int32_t(i);
      diag[2 * i + 1] = std::int32_t(tb + i);
    }
    auto db = upload_i32(diag);
    dev::set_entries(aug.data(), aug.ld(), dptr(db), a, 1, s);
  }
  DevBuf flags{static_cast<std::size_t>(dev::ech_panel_flag_bytes(a))};
  DevBuf info{static_cast<std::size_t>(4 * (1 + 2 * cap) + 4 * (2 + 512))};  // + base, rmap (<= 512 slots)
  DevBuf rho2{static_cast<std::size_t>(4 * w)};
  dev::fill2d(flags.ptr, std::int64_t(flags.bytes), 1, std::int64_t(flags.bytes), 0, s);
  dev::fill2d(info.ptr, std::int64_t(info.bytes), 1, std::int64_t(info.bytes), 0, s);
  auto* inf = reinterpret_cast<std::int32_t*>(info.ptr);
  auto* r2 = reinterpret_cast<std::int32_t*>(rho2.ptr);
  const std::int64_t ow = (f.p() == 2 && !block_cluster && a <= kGf2OuterRows && b > 256)
                             ? gf2_outer_width()
                             : ech_outer_width(b);
  if (ow == 0) {
    Mat G(a, w), Bp(w, tb + a);
    for (std::int64_t c0 = 0; c0 < b; c0 += w) {
      const std::int64_t wc = std::min(w, b - c0), n = tb + a - c0;
      dev::ech_panel(f.p(), a, c0, wc, w, aug.data(), aug.ld(), flags.ptr, inf, cap, G.data(),
                     G.ld(), r2, s);
      dev::select2d(Bp.data(), Bp.ld(), w, n, aug.data() + c0, aug.ld(), nullptr, 0, r2, nullptr, s);
      dev::mad(f.p(), a, n, w, G.data(), G.ld(), Bp.data(), Bp.ld(), aug.data() + c0, aug.ld(),
               aug.data() + c0, aug.ld(), s);
    }
    return extract_ech(a, b, aug, inf, cap, tb);
  }
  // Two-level: each outer panel of `ow` columns is eliminated in Z = [X | Y]
  // by 32-wide steps (their updates stay inside Z, L2-resident), then ONE
  // deep-K contraction Aug[:, right] += Gout.Aug[P, right] applies the
  // panel's row operator to everything right of it (W and T) on K1.
  auto* base = inf + 1 + 2 * cap;  // rank at the start of the outer panel
  auto* rmap = base + 1;           // the outer panel's pivot rows (ow slots)
  const bool gf2o = f.p() == 2 && !block_cluster && a <= kGf2OuterRows;
  Mat Z(a, 2 * ow), Bt(ow, tb + a);
  DevBuf step{static_cast<std::size_t>(dev::ech_step_scratch_bytes())};
  dev::fill2d(step.ptr, std::int64_t(step.bytes), 1, std::int64_t(step.bytes), 0, s);
  std::int64_t step_seq = 0, signalled = 0;
  const bool fused = a * 33 <= dev::kPanelSmem;
  Mat G(fused ? 0 : a, w), Bp(fused ? 0 : w, 2 * ow);
  for (std::int64_t C0 = 0; C0 < b; C0 += ow) {
    const std::int64_t wd = std::min(ow, b - C0), kc = std::min(wd, a);
    // Z[:, 0:wd] = Aug[:, C0:C0+wd], Z[:, ow:] = 0
    dev::copy_cols(Z.data(), Z.ld(), aug.data() + C0, aug.ld(), a, wd, 2 * ow, s);
    std::uint8_t* Y = Z.data() + ow;
    const bool done_outer = gf2o && dev::ech_gf2_outer(a, wd, ow, Z.data(), Z.ld(), flags.ptr, inf, cap, s);
    for (std::int64_t c0 = done_outer ? wd : 0; c0 < wd; c0 += w) {
      const std::int64_t wc = std::min(w, wd - c0);
      // the step updates Z columns from c0 through Y's used slots
      const std::int64_t n = (ow + std::min(kc, c0 + w) - c0 + 15) / 16 * 16;
      if (fused) {
        dev::ech_step(f.p(), a, c0, wc, n, Z.data(), Z.ld(), flags.ptr, inf, cap, r2, step.ptr, Y,
                      base, c0 > 0, c0 + w < wd, int(++step_seq), int(signalled), s);
        if (c0 + w < wd) ++signalled;
        continue;
      }
      // GF(2) blocks too tall for the fused step's fallback: the panel
      // kernel's G for every row, then the gather and the K1 update
      dev::ech_panel(f.p(), a, c0, wc, w, Z.data(), Z.ld(), flags.ptr, inf, cap, G.data(), G.ld(),
                     r2, s);
      dev::ech_panel_plant(Y, Z.ld(), r2, inf, base, s);
      dev::select2d(Bp.data(), Bp.ld(), w, n, Z.data() + c0, Z.ld(), nullptr, 0, r2, nullptr, s);
      dev::mad(f.p(), a, n, w, G.data(), G.ld(), Bp.data(), Bp.ld(), Z.data() + c0, Z.ld(),
               Z.data() + c0, Z.ld(), s);
    }
    dev::ech_outer_finish(f.p(), Y, Z.ld(), kc, inf, cap, base, rmap, C0, s);
    // (columns [wd, round16(wd)) of the last panel are the zero gap before T)
    dev::copy_cols(aug.data() + C0, aug.ld(), Z.data(), Z.ld(), a, wd, (wd + 15) / 16 * 16, s);
    const std::int64_t r0 = C0 + wd, n = tb + a - r0;
    dev::select2d(Bt.data(), Bt.ld(), kc, n, aug.data() + r0, aug.ld(), nullptr, 0, rmap, nullptr, s);
    dev::mad(f.p(), a, n, kc, Y, Z.ld(), Bt.data(), Bt.ld(), aug.data() + r0, aug.ld(),
             aug.data() + r0, aug.ld(), s);
  }
  return extract_ech(a, b, aug, inf, cap, tb);
}

// GF(2) blocks the cluster kernel (ech_gf2_cluster) eliminates in one
// launch on its fast path: <= 1024 rows and a packed [W | T] row of <= 96
// words (its nibble-table update; wider rows take a bit-serial update
// several times slower than splitting).
constexpr std::int64_t kGf2ClusterRows = 1024;
bool gf2_cluster_fits(std::int64_t a, std::int64_t b) {
  return a <= kGf2ClusterRows && (a + b + 31) / 32 <= 96;
}
// ech mode 2 (or GFQ_GF2_SPLIT=0) keeps tall GF(2) blocks on the
// two-level panel path
bool gf2_split_enabled() {
  static const bool on = [] {
    const char* e = std::getenv("GFQ_GF2_SPLIT");
    return !(e && e[0] == '0');
  }();
  return on && ech_mode() != 2;
}

// Split point: half, rounded to a multiple of 16 so column views keep the
// 16-byte alignment the TMA path needs (outputs do not depend on it).
std::int64_t split_of(std::int64_t n) {
  const std::int64_t h = n / 2;
  return (n >= 64 && h >= 16) ? h / 16 * 16 : h;
}

IndexSet shifted_union(const IndexSet& a, const IndexSet& b, std::size_t off, std::size_t universe) {
  std::vector<std::uint32_t> mem = a.members;
  for (auto v : b.members) mem.push_back(std::uint32_t(off + v));
  return IndexSet(universe, std::move(mem));
}

// reference src/jobs.cpp:125-156
EchResult combine_horizontal(const FieldSpec& f, const Mat& h2, const EchResult& e1,
                             std::int64_t alpha1, std::size_t thr) {
  auto [a_cols, h2_rest] = cex(h2, e1.gamma);
  const Mat h2_clean = mad(f, h2_rest, a_cols, e1.R);
  const EchResult e2 = ech(f, h2_clean, thr);
  auto [a_sel, a_rest] = rex(a_cols, e2.rho);
  auto [e_mid, r1_rest] = cex(e1.R, e2.gamma);
  auto [gamma, lam] = unh(e1.gamma, e2.gamma);
  const Mat mc = mul(f, mul(f, e2.M, a_sel), e1.M);
  const Mat ma = mad(f, e1.M, e_mid, mc);
  const Mat mb = mul(f, e_mid, e2.M);
  EchResult out;
  out.gamma = std::move(gamma);
  out.M = rrf(lam, hcat(ma, mb), hcat(mc, e2.M));
  out.R = rrf(lam, mad(f, r1_rest, e_mid, e2.R), e2.R);
  const Mat k_bottom_left = mul(f, mad(f, a_rest, e2.K, a_sel), e1.M);
  out.K = vcat(hcat(e1.K, Mat::zeros(e1.K.rows(), std::int64_t(e2.rho.size()), f.esize())),
               hcat(k_bottom_left, e2.K));
  out.rho = shifted_union(e1.rho, e2.rho, std::size_t(alpha1), std::size_t(alpha1 + h2.rows()));
  return out;
}

// reference src/jobs.cpp:160-187
EchResult combine_vertical(const FieldSpec& f, const Mat& h2, const EchResult& e1,
                           std::int64_t beta1, std::size_t thr) {
  auto [h2_sel, h2_rest] = rex(h2, e1.rho);
  const Mat x = mul(f, e1.M, h2_sel);
  const Mat h2_clean = mad(f, h2_rest, e1.K, h2_sel);
  const EchResult e2 = ech(f, h2_clean, thr);
  auto [rho, u] = unh(e1.rho, e2.rho);
  auto [k1_sel, k1_rest] = rex(e1.K, e2.rho);
  const Mat g = mul(f, e2.M, k1_sel);
  auto [x_piv, x_rest] = cex(x, e2.gamma);
  EchResult out;
  out.rho = std::move(rho);
  out.gamma = shifted_union(e1.gamma, e2.gamma, std::size_t(beta1), std::size_t(beta1 + h2.cols()));
  out.M = col_riffle(u, vcat(mad(f, e1.M, x_piv, g), g), vcat(mul(f, x_piv, e2.M), e2.M));
  out.R = vcat(hcat(e1.R, mad(f, x_rest, x_piv, e2.R)),
               hcat(Mat::zeros(std::int64_t(e2.rho.size()), e1.R.cols(), f.esize()), e2.R));
  out.K = col_riffle(u, mad(f, k1_rest, e2.K, k1_sel), e2.K);
  return out;
}

}  // namespace

void set_ech_outer(int width) {
  if (width < -1 || width > kEchOuterMax) throw std::invalid_argument("ech outer width must be -1..256");
  g_ech_outer = width;
}

EchResult ech(const FieldSpec& f, const Mat& h, std::size_t threshold) {
  if (threshold < 1) threshold = 1;
  const std::int64_t alpha = h.rows(), beta = h.cols();
  if (alpha == 0 || beta == 0) {
    EchResult e;
    e.M = Mat(0, 0, f.esize());
    e.K = Mat(alpha, 0, f.esize());
    e.R = Mat(0, beta, f.esize());
    e.rho = IndexSet(std::size_t(alpha), {});
    e.gamma = IndexSet(std::size_t(beta), {});
    return e;
  }
  // GF(p^k): the reference's split/combine recursion (its products are
  // digit-plane K1 contractions) over the table-driven base case
  if (ech_mode() != 1 && !f.is_ext() && !f.wide()) {
    // thin blocks (rank <= 32: the Chief's one-column / one-row ClearDowns)
    // in one base-case launch
    if (std::min(alpha, beta) <= dev::kEchThinMax && dev::ech_base_fits(alpha, beta)) return direct_ech(f, h);
    // GF(2): the 8-CTA cluster kernel takes blocks of <= 1024 rows with
    // rows + cols <= 8192; anything larger follows the reference's own
    // split rule (src/jobs.cpp:202-225: rows when alpha >= beta, else
    // columns) down to it, so a tall 8192^2 ECH is eight cluster ECHs plus
    // K1 combines instead of 256 single-CTA panel steps.
    if (f.p() == 2 && !gf2_cluster_fits(alpha, beta) && alpha > 32 && alpha <= kGf2OuterRows &&
        gf2_outer_enabled())
      return panel_ech(f, h, false);
    if (f.p() == 2 && gf2_split_enabled() && !gf2_cluster_fits(alpha, beta)) {
      if (alpha >= beta) {
        const std::int64_t alpha1 = split_of(alpha);
        const EchResult e1 = ech(f, h.row_view(0, alpha1), threshold);
        return combine_horizontal(f, h.row_view(alpha1, alpha - alpha1), e1, alpha1, threshold);
      }
      const std::int64_t beta1 = split_of(beta);
      const EchResult e1 = ech(f, h.col_view(0, beta1), threshold);
      return combine_vertical(f, h.col_view(beta1, beta - beta1), e1, beta1, threshold);
    }
    // panel ECH whenever the panel fits one CTA's shared memory; taller
    // blocks split their rows (reference combine_horizontal) first
    if (alpha * (f.p() == 2 ? 5 : 33) <= dev::kPanelSmem) return panel_ech(f, h);
    const std::int64_t alpha1 = split_of(alpha);
    const EchResult e1 = ech(f, h.row_view(0, alpha1), threshold);
    return combine_horizontal(f, h.row_view(alpha1, alpha - alpha1), e1, alpha1, threshold);
  }
  std::int64_t base = std::int64_t(std::min(threshold, ech_base()));
  if (f.wide()) base = std::min<std::int64_t>(base, dev::kEchBaseWideMax);
  if (alpha <= base && beta <= base) return direct_ech(f, h);
  if (alpha >= beta) {
    const std::int64_t alpha1 = split_of(alpha);
    const EchResult e1 = ech(f, h.row_view(0, alpha1), threshold);
    return combine_horizontal(f, h.row_view(alpha1, alpha - alpha1), e1, alpha1, threshold);
  }
  const std::int64_t beta1 = split_of(beta);
  const EchResult e1 = ech(f, h.col_view(0, beta1), threshold);
  return combine_vertical(f, h.col_view(beta1, beta - beta1), e1, beta1, threshold);
}

}  // namespace gfq
