// tasks.hpp -- the Chief's composite tasks (reference include/gfrref/tasks.hpp:19-59)
// over device-resident packages.  Same signatures, argument meaning and
// error behaviour as the reference; the block contractions inside run on the
// K1 tensor-core kernel, the gathers/riffles on K3/K4, ECH on K2 + K1.
#pragma once

#include <optional>
#include <utility>

#include "types.hpp"

namespace gfq {

std::pair<PkgD, PkgA> clear_down(const FieldSpec& f, const Mat& C, const PkgD& D,
                                 std::size_t i, std::size_t ech_threshold = 256);
std::pair<Mat, Mat> update_row(const FieldSpec& f, const PkgA& A, const Mat& C,
                               const std::optional<Mat>& B, std::size_t i);
/// UpdateRowTrafo(i, j, h) for every h < i at once (fused plan).  Kw: the
/// K(i, h, j-1) panel (j > 0); Mw: M(j, h, i-1-h) for h < i-1 as a panel
/// (i >= 2), Md: M(j, i-1, 0); deltas[h] = E(h, j).delta.  Returns the
/// K(i, h, j) and M(j, h, i-h) panels in the padded layout of the widths
/// |delta_h|.  m_capacity > 0: new M panels get a row stride of that many
/// columns, and a block row that adds no pivot appends Md to Mw's storage in
/// place (the returned panel is then a wider view of Mw's).
std::pair<MatParts, MatParts> update_row_trafo_off(const FieldSpec& f, const PkgA& A,
                                                   const MatParts* Kw, const MatParts* Mw,
                                                   const Mat& Md,
                                                   const std::vector<const BitString*>& deltas,
                                                   std::size_t i, std::size_t j,
                                                   std::int64_t m_capacity = 0);

std::pair<Mat, Mat> update_row_trafo(const FieldSpec& f, const PkgA& A,
                                     const std::optional<Mat>& K,
                                     const std::optional<Mat>& M, const PkgE& E,
                                     std::size_t i, std::size_t h, std::size_t j);
PkgE extend(const PkgA& A, const std::optional<PkgE>& E, std::size_t j);
Mat row_lengthen(const Mat& M, const PkgE& E1, const PkgE& E2);
std::pair<Mat, Mat> pre_clear_up(const Mat& B, const PkgD& D);
Mat clear_up(const FieldSpec& f, const Mat& R, const Mat& X, const Mat& M);
Mat copy_d(const PkgD& D);

}  // namespace gfq
