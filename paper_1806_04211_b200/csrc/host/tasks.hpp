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
