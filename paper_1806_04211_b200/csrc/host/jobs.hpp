// jobs.hpp -- the atomic block jobs of the Chief (reference
// include/gfrref/jobs.hpp:37-82 and the matrix helpers of
// include/gfrref/matrix.hpp:90-109), on device-resident u8 blocks.
//
// Every job takes const& inputs and returns fresh values (reference
// SPEC.md:130); work is enqueued on gfq::cur_stream().  Shape errors throw
// std::invalid_argument with the reference's messages.
#pragma once

#include <utility>

#include "types.hpp"

namespace gfq {

/// D = (Cin ? Cin : 0) + A.B over the field f (K1 for GF(p), the digit-plane
/// contraction for GF(p^k)); raw device operands, stream-ordered.
void field_mad(const FieldSpec& f, std::int64_t m, std::int64_t n, std::int64_t k,
               const std::uint8_t* A, std::int64_t lda, const std::uint8_t* B, std::int64_t ldb,
               const std::uint8_t* Cin, std::int64_t ldc, std::uint8_t* D, std::int64_t ldd,
               cudaStream_t s);
Mat cpy(const Mat& a);                                             // jobs.hpp:37
Mat mul(const FieldSpec& f, const Mat& b, const Mat& c);           // jobs.hpp:40
Mat mad(const FieldSpec& f, const Mat& a, const Mat& b, const Mat& c);  // jobs.hpp:43
Mat mat_mul(const FieldSpec& f, const Mat& b, const Mat& c);       // matrix.hpp:90
Mat mat_mul_add(const FieldSpec& f, const Mat& a, const Mat& b, const Mat& c);  // matrix.hpp:93
/// d = (addend ? addend : 0) + b.c written into an existing matrix or view
/// (the fused plan's wide outputs); addend may alias d.
void mad_into(const FieldSpec& f, const Mat& d, const Mat* addend, const Mat& b, const Mat& c);
/// While alive on this thread, contractions whose B operand lies inside
/// `b`'s storage may keep (and reuse) its K1f packing with that storage.
/// For published, immutable packages only: the pivot rows B(j, k) / the
/// T_M(j, .) panels that every block row below multiplies by, and Step 3's
/// final rows -- the packing (a transpose to K-major E2M1 codes) is then
/// done once per package instead of once per product.  GFQ_NO_BPACK_CACHE=1
/// turns it off.
class ImmutableB {
 public:
  explicit ImmutableB(const Mat& b);
  ~ImmutableB();
  ImmutableB(const ImmutableB&) = delete;
  ImmutableB& operator=(const ImmutableB&) = delete;

 private:
  DevBuf* prev_;
};
/// out[:, c] = m[:, cmap[c]] (cmap[c] = -1: zero column), one K3 launch.
Mat col_gather(const Mat& m, std::int64_t out_cols, const std::vector<std::int32_t>& cmap);
/// out[:, c] = a[:, cmap[c]] (>= 0), b[:, -cmap[c]-2] (<= -2) or 0 (-1); one K3 launch.
Mat col_gather2(const Mat& a, const Mat* b, std::int64_t out_cols, const std::vector<std::int32_t>& cmap);
/// The same gather (cmap null: a plain copy of a) into an existing matrix or
/// view; u8 elements.
void col_gather_into(const Mat& dst, const Mat& a, const Mat* b, const std::vector<std::int32_t>* cmap);

/// Negative reduced echelonisation of one block (jobs.hpp:50).  Same
/// recursion as the reference (split the longer dimension, combine), base
/// case = the single-CTA K2 kernel.  The outputs are canonical,
/// so `threshold` only moves the recursion/base boundary.
EchResult ech(const FieldSpec& f, const Mat& h, std::size_t threshold = 256);

std::pair<Mat, Mat> cex(const Mat& h, const IndexSet& gamma);      // jobs.hpp:53
std::pair<Mat, Mat> rex(const Mat& h, const IndexSet& rho);        // jobs.hpp:56
std::pair<IndexSet, BitString> unh(const IndexSet& rho1, const IndexSet& rho2);  // :61
std::pair<IndexSet, BitString> un0(const IndexSet& rho2);          // :64
BitString mkr(const IndexSet& rho1, const IndexSet& rho2);         // :68
Mat rrf(const BitString& u, const Mat& b, const Mat& c);           // :72
Mat crz(const Mat& m, const BitString& lambda, std::size_t out_cols);  // :77
Mat adi(const Mat& k, const BitString& delta);                     // :82

Mat take_rows(const Mat& m, const std::vector<std::uint32_t>& rows);  // matrix.hpp:100
Mat take_cols(const Mat& m, const std::vector<std::uint32_t>& cols);  // matrix.hpp:103
Mat vcat(const Mat& a, const Mat& b);                                 // matrix.hpp:106
Mat hcat(const Mat& a, const Mat& b);                                 // matrix.hpp:109

/// K6: rows x cols of reference random_matrix (src/generate.cpp:16-24) whose
/// entry (r, c) takes draw draw0 + r * draw_ld + c.  A draw in the
/// rejection band (probability < 2^-56 per draw) would shift the reference's
/// stream; that case is reported (std::runtime_error), never silently wrong.
/// esize 4: u32 elements (wide fields; p is then the field order).
void random_fill_exact(std::uint32_t p, std::int64_t rows, std::int64_t cols, std::uint64_t seed,
                       std::uint64_t draw0, std::int64_t draw_ld, std::uint8_t* dst,
                       std::int64_t ld, int esize = 1);

/// Tunable: largest block the K2 base-case kernel takes (<= kEchBaseMax).
void set_ech_base(std::size_t n);
std::size_t ech_base();
/// ECH algorithm: 0 = device panel Gauss-Jordan (default), 1 = the
/// reference's split/combine recursion down to the K2 base case.  Both give
/// the same (canonical) outputs.
/// A gather map as runs: output [t, t+len) from consecutive source indices
/// src.. of operand `from` (0: A, 1: B; codes v >= 0 / v <= -2 of the
/// select maps) or zeros (from = -1, code -1).  False when more than `cap`.
struct Run {
  std::int64_t t, len, src;
  int from;
};
bool runs_of(const std::vector<std::int32_t>& map, std::vector<Run>& out, std::size_t cap);

void set_ech_mode(int mode);
/// Outer panel width of the two-level device ECH: -1 = automatic, 0 = one
/// level, else 32..256 (multiple of 32).  Outputs do not depend on it.
void set_ech_outer(int width);
int ech_mode();

}  // namespace gfq
