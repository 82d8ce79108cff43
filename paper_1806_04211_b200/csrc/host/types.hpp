// types.hpp -- value types of the B200 GF(p) elimination path.
//
// Mirrors the reference's value types (include/gfrref/field.hpp,
// matrix.hpp, jobs.hpp, packages.hpp) with one change of storage: a matrix
// is a *device-resident* u8 block (one byte per residue, row-major, 16-byte
// aligned rows) instead of a host std::vector<uint32_t>.  Index sets and bit
// strings are small host vectors (they steer the gathers and are needed on
// the host to size the data-dependent shapes).
#pragma once

#include <cstddef>
#include <cstdint>
#include <memory>
#include <optional>
#include <string>
#include <utility>
#include <vector>

#include "../common.hpp"

namespace gfq {

using Elem = std::uint32_t;

/// Tables of an extension field GF(p^k), q = p^k <= 256 (runtime.cpp):
/// mul / add are q x q, neg / inv q entries, dig the k base-p digits of
/// every element, red the digits of x^s mod the modulus for s < 2k - 1;
/// a device copy (kernels.hpp dev::ExtTables) is uploaded on first use.
struct ExtTablesHost;
namespace dev {
struct ExtTables;
struct WideField;
}

/// GF(q), q = p^k, elements encoded like the reference
/// (include/gfrref/field.hpp:12-14: sum_i c_i p^i).  Mirrors reference
/// FieldSpec (include/gfrref/field.hpp:20-110, src/field.cpp:143-237):
/// FieldSpec(p) is the prime field (p < 2^16), FieldSpec(p, k, modulus) the
/// extension with a monic irreducible modulus (empty: the lexicographically
/// first one, constant coefficient varying fastest), p^k < 2^20.  Storage:
/// one byte per element when p <= 251 (prime) or q <= 256 (extension), the
/// tensor-core path; four bytes (u32) otherwise ("wide" fields: SIMT
/// contraction, the reference's split/combine ECH over a one-CTA base case).
/// code(): the integer the C ABI passes as "p" -- p itself for a prime
/// field, a registered id >= 0x10000 for an extension field (FieldSpec(code)
/// resolves either).
class FieldSpec {
 public:
  explicit FieldSpec(std::uint32_t p_or_code);
  FieldSpec(std::uint32_t p, std::uint32_t k, std::vector<std::uint32_t> modulus = {});
  std::uint32_t p() const { return p_; }
  std::uint32_t k() const { return k_; }
  std::uint32_t order() const { return q_; }
  bool is_ext() const { return k_ > 1; }
  /// u32 storage (p > 251 or q > 256)
  bool wide() const { return k_ > 1 ? q_ > 256 : p_ > 251; }
  /// bytes per stored element
  int esize() const { return wide() ? 4 : 1; }
  std::uint32_t code() const;
  const std::vector<std::uint32_t>& modulus() const;
  Elem add(Elem a, Elem b) const;
  Elem neg(Elem a) const;
  Elem mul(Elem a, Elem b) const;
  Elem inv(Elem a) const;
  bool operator==(const FieldSpec& o) const {
    return p_ == o.p_ && k_ == o.k_ && modulus() == o.modulus();
  }
  std::string name() const {
    return k_ == 1 ? "GF(" + std::to_string(p_) + ")"
                   : "GF(" + std::to_string(p_) + "^" + std::to_string(k_) + ")";
  }
  /// Device tables (extension fields only; uploaded on first use).
  const dev::ExtTables& ext_dev() const;
  /// Device view of a wide field (log / antilog / Zech tables for wide
  /// extension fields, uploaded on first use).
  dev::WideField wide_dev() const;

 private:
  std::uint32_t p_ = 0, k_ = 1, q_ = 0;
  std::shared_ptr<const ExtTablesHost> ext_;
};
/// Reference default_modulus (src/field.cpp:125-138).
std::vector<std::uint32_t> default_modulus(std::uint32_t p, std::uint32_t k);

/// A stream-ordered device allocation (cudaMallocAsync pool).
struct DevBuf {
  std::uint8_t* ptr = nullptr;
  std::size_t bytes = 0;
  DevBuf() = default;
  explicit DevBuf(std::size_t n);
  ~DevBuf();
  DevBuf(const DevBuf&) = delete;
  DevBuf& operator=(const DevBuf&) = delete;
  /// K1f packings of B operands that live in this block (jobs.cpp,
  /// ImmutableB): created by the first contraction that needs one, shared
  /// by the later ones, released with the block.
  std::shared_ptr<void> packed_b;
};

/// The stream `s` has drained (synchronised): blocks released on it become
/// reusable from any stream.
void release_stream(cudaStream_t s);
/// Developer check: bit 0 fills every allocation with 0xA5, bit 1 every
/// freed block with 0x5A (on its stream); GFQ_POISON sets the start value.
int poison_mode();
void set_poison_mode(int mode);
/// Make the stream-ordered pool hold `bytes` beyond its current use (one
/// growth step instead of many small ones).
void reserve_pool(std::size_t bytes);
/// One-time runtime setup (memory pool attributes, pinned staging ring).
void warm_runtime();

/// Live device bytes held by DevBufs (for RunReport accounting).
std::int64_t live_device_bytes();
std::int64_t peak_device_bytes();
void reset_peak_device_bytes();

/// Device-resident dense matrix of u8 (esize 1) or u32 (esize 4, wide
/// fields) elements.  Zero-dimensional shapes carry no storage.  Values are
/// immutable once published (jobs return fresh matrices); row/column views
/// share the parent's storage.  cols() counts elements, ld() bytes.
class Mat {
 public:
  Mat() = default;
  Mat(std::int64_t rows, std::int64_t cols, int esize = 1);  // uninitialised storage
  static Mat zeros(std::int64_t rows, std::int64_t cols, int esize = 1);
  static Mat from_host(std::int64_t rows, std::int64_t cols, const std::uint8_t* src,
                       std::int64_t ld, int esize = 1);

  std::int64_t rows() const { return rows_; }
  std::int64_t cols() const { return cols_; }
  std::int64_t ld() const { return ld_; }
  int esize() const { return esize_; }
  /// bytes of one row's elements
  std::int64_t row_bytes() const { return cols_ * esize_; }
  std::uint8_t* data() const { return data_; }
  const std::shared_ptr<DevBuf>& buf() const { return buf_; }
  bool empty() const { return rows_ == 0 || cols_ == 0; }

  /// A matrix living inside an existing allocation (e.g. a received
  /// broadcast payload): rows x cols at byte `offset`, row stride ld.
  static Mat view_of(std::shared_ptr<DevBuf> buf, std::size_t offset, std::int64_t rows,
                     std::int64_t cols, std::int64_t ld, int esize = 1);
  /// Uninitialised rows x cols whose row stride has room for cap_cols
  /// columns: `widened` can later append columns in place.
  static Mat with_capacity(std::int64_t rows, std::int64_t cols, std::int64_t cap_cols, int esize = 1);
  /// The same rows with `cols` >= cols() columns, the new ones being the
  /// storage to the right of this view -- an empty Mat when the row stride
  /// has no room for them.  The new columns are uninitialised.
  Mat widened(std::int64_t cols) const;
  /// Rows [r0, r0+n) as a view (no copy).
  Mat row_view(std::int64_t r0, std::int64_t n) const;
  /// Columns [c0, c0+n) as a view (no copy; may lose 16-byte alignment).
  Mat col_view(std::int64_t c0, std::int64_t n) const;

  void to_host(std::uint8_t* dst, std::int64_t ld) const;  // synchronous
  std::vector<std::uint8_t> to_host() const;

  /// Bytes accounted to this value (reference Matrix::byte_size analogue).
  std::size_t byte_size() const { return std::size_t(rows_) * std::size_t(cols_) * std::size_t(esize_) + 48; }

 private:
  std::shared_ptr<DevBuf> buf_;
  std::uint8_t* data_ = nullptr;
  std::int64_t rows_ = 0, cols_ = 0, ld_ = 0;
  int esize_ = 1;
};

/// A sorted subset of {0, ..., universe-1} (reference include/gfrref/matrix.hpp:53-70).
struct IndexSet {
  std::size_t universe = 0;
  std::vector<std::uint32_t> members;
  IndexSet() = default;
  IndexSet(std::size_t universe, std::vector<std::uint32_t> members);
  std::size_t size() const { return members.size(); }
  bool operator==(const IndexSet& o) const {
    return universe == o.universe && members == o.members;
  }
  std::size_t byte_size() const { return members.size() * 4 + 32; }
};
IndexSet index_set_complement(const IndexSet& s);

/// reference include/gfrref/matrix.hpp:75-87
struct BitString {
  std::vector<std::uint8_t> bits;
  BitString() = default;
  explicit BitString(std::vector<std::uint8_t> b) : bits(std::move(b)) {}
  std::size_t size() const { return bits.size(); }
  std::size_t count_ones() const;
  std::size_t count_zeros() const { return size() - count_ones(); }
  bool operator==(const BitString& o) const { return bits == o.bits; }
  std::size_t byte_size() const { return bits.size() + 32; }
};

/// reference include/gfrref/jobs.hpp:20-32
struct EchResult {
  Mat M, K, R;
  IndexSet rho, gamma;
  std::size_t rank() const { return gamma.size(); }
};

/// reference include/gfrref/packages.hpp:17-26
struct PkgA {
  std::optional<Mat> A;
  Mat M;
  Mat K;
  IndexSet rho_prime;
  std::optional<Mat> E;
  std::optional<BitString> lambda;
  std::size_t byte_size() const;
};

/// reference include/gfrref/packages.hpp:30-36
struct PkgD {
  Mat R;
  IndexSet gamma;
  std::size_t rank() const { return gamma.size(); }
  std::size_t byte_size() const { return R.byte_size() + gamma.byte_size(); }
};

/// reference include/gfrref/packages.hpp:40-45
struct PkgE {
  IndexSet rho;
  BitString delta;
  std::size_t byte_size() const { return rho.byte_size() + delta.byte_size(); }
};

/// A block-row (or block-column-set) panel stored as ONE device matrix: part
/// p is columns [off[p], off[p] + w[p]) of m.  Part starts are 16-column
/// aligned (TMA-legal views); padding columns hold don't-care residues.  The
/// fused single-GPU plan uses it to run one wide job instead of one per block.
struct MatParts {
  Mat m;
  std::vector<std::int64_t> off, w;
  std::size_t parts() const { return w.size(); }
  Mat part(std::size_t p) const { return m.col_view(off[p], w[p]); }
  /// parts [p, end) as one view (their padded span)
  Mat tail(std::size_t p) const {
    return p == 0 ? m : m.col_view(off[p], m.cols() - off[p]);
  }
  MatParts tail_parts(std::size_t p) const;
  std::size_t byte_size() const { return m.byte_size(); }
};
/// Padded layout for part widths: starts rounded up to 16 columns.
MatParts layout_parts(std::int64_t rows, const std::vector<std::int64_t>& widths);

// ---------------------------------------------------------------- staging
/// Upload a small host int32 array to a fresh device buffer on the current
/// stream (through a pinned staging ring).
std::shared_ptr<DevBuf> upload_i32(const std::vector<std::int32_t>& v);
/// Synchronous download of a small device int32 array.
void download_i32(const std::int32_t* dev, std::int32_t* host, std::size_t n);

}  // namespace gfq
