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

/// GF(p), p prime <= 251 (one residue per byte).  Mirrors the prime-field
/// half of reference FieldSpec (include/gfrref/field.hpp:20-110); extension
/// fields are out of scope for the B200 path.
class FieldSpec {
 public:
  explicit FieldSpec(std::uint32_t p);
  std::uint32_t p() const { return p_; }
  std::uint32_t order() const { return p_; }
  Elem add(Elem a, Elem b) const { return (a + b) % p_; }
  Elem neg(Elem a) const { return a == 0 ? 0 : p_ - a; }
  Elem mul(Elem a, Elem b) const { return Elem(std::uint64_t(a) * b % p_); }
  Elem inv(Elem a) const;
  bool operator==(const FieldSpec& o) const { return p_ == o.p_; }
  std::string name() const { return "GF(" + std::to_string(p_) + ")"; }

 private:
  std::uint32_t p_;
};

/// A stream-ordered device allocation (cudaMallocAsync pool).
struct DevBuf {
  std::uint8_t* ptr = nullptr;
  std::size_t bytes = 0;
  DevBuf() = default;
  explicit DevBuf(std::size_t n);
  ~DevBuf();
  DevBuf(const DevBuf&) = delete;
  DevBuf& operator=(const DevBuf&) = delete;
};

/// The stream `s` has drained (synchronised): blocks released on it become
/// reusable from any stream.
void release_stream(cudaStream_t s);
/// One-time runtime setup (memory pool attributes, pinned staging ring).
void warm_runtime();

/// Live device bytes held by DevBufs (for RunReport accounting).
std::int64_t live_device_bytes();
std::int64_t peak_device_bytes();
void reset_peak_device_bytes();

/// Device-resident dense u8 matrix.  Zero-dimensional shapes carry no
/// storage.  Values are immutable once published (jobs return fresh
/// matrices); row/column views share the parent's storage.
class Mat {
 public:
  Mat() = default;
  Mat(std::int64_t rows, std::int64_t cols);  // uninitialised storage
  static Mat zeros(std::int64_t rows, std::int64_t cols);
  static Mat from_host(std::int64_t rows, std::int64_t cols, const std::uint8_t* src,
                       std::int64_t ld);

  std::int64_t rows() const { return rows_; }
  std::int64_t cols() const { return cols_; }
  std::int64_t ld() const { return ld_; }
  std::uint8_t* data() const { return data_; }
  bool empty() const { return rows_ == 0 || cols_ == 0; }

  /// A matrix living inside an existing allocation (e.g. a received
  /// broadcast payload): rows x cols at byte `offset`, row stride ld.
  static Mat view_of(std::shared_ptr<DevBuf> buf, std::size_t offset, std::int64_t rows,
                     std::int64_t cols, std::int64_t ld);
  /// Rows [r0, r0+n) as a view (no copy).
  Mat row_view(std::int64_t r0, std::int64_t n) const;
  /// Columns [c0, c0+n) as a view (no copy; may lose 16-byte alignment).
  Mat col_view(std::int64_t c0, std::int64_t n) const;

  void to_host(std::uint8_t* dst, std::int64_t ld) const;  // synchronous
  std::vector<std::uint8_t> to_host() const;

  /// Bytes accounted to this value (reference Matrix::byte_size analogue).
  std::size_t byte_size() const { return std::size_t(rows_) * std::size_t(cols_) + 48; }

 private:
  std::shared_ptr<DevBuf> buf_;
  std::uint8_t* data_ = nullptr;
  std::int64_t rows_ = 0, cols_ = 0, ld_ = 0;
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
