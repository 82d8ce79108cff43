// verify.hpp -- on-device certificate of an EchelonOutput (reference
// gfrref::verify, src/chief.cpp:531-590, without the oracle argument: the
// product never runs a CPU elimination).
#pragma once

#include <cstdint>
#include <string>

#include "chief.hpp"

namespace gfq {

enum class VerifyMethod : int {
  Auto = 0,       // Exact when T, C and T.C fit comfortably in free HBM, else Freivalds
  Exact = 1,      // materialise T (m x m) and compare T.C entry by entry
  Freivalds = 2,  // T.(C.X) == E.X for a random n x 64 X, block by block (no T)
};

struct VerifyResult {
  bool ok = false;
  std::string diag;    // empty when ok
  std::string method;  // what was actually checked
};

/// Checks, for the device-resident input C (m x n) and a complete
/// (gathered) output:
///  1. the select sets agree with the rank (reference :539-543);
///  2. the remnant is in echelon shape: a pivot row has no nonzero entry in
///     a non-pivot column left of its pivot -- with 3 this pins the unique
///     RREF, which the reference proves by comparing with its oracle;
///  3. with the transform, the defining identity T.C = E where row r of E
///     has -1 at the r-th pivot column and R's row r on the non-pivot
///     columns, and the non-pivot rows of E are zero (reference :565-588);
///     without the transform, that every row of C lies in the row space of
///     E: C[:, rest] + C[:, pivots] . R == 0.
VerifyResult verify(const Mat& C, const EchelonOutput& out, VerifyMethod method,
                    std::uint64_t seed);

}  // namespace gfq
