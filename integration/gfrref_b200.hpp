// gfrref_b200.hpp -- the reference-side drop-in: gfrref::echelonize's
// signature (/root/reference/proj/include/gfrref/chief.hpp:88-90) over the
// B200 library's C ABI (include/gfq.h).  A gfrref maintainer adds this file
// and gfrref_b200.cpp next to src/chief.cpp and links libgfq.so; callers
// switch `gfrref::echelonize(...)` to `gfrref_b200::echelonize(...)` and get
// the same EchelonOutput (bit-exact, tests/test_gpu_dropin.py).
#pragma once

#include "gfrref/chief.hpp"

namespace gfrref_b200 {

/// gfrref::echelonize on one B200 (chop -> Steps 1-3 -> EchelonOutput with
/// every R / T_M / T_K block copied back into reference Matrix values).
/// Same exceptions as the reference: std::invalid_argument for unusable
/// input, std::runtime_error("Kind(i,j,k): msg") for a failed task; a
/// field the B200 path cannot store (p > 251, p^k > 256) or a missing
/// device raises instead of falling back to the CPU.
gfrref::EchelonOutput echelonize(const gfrref::Matrix& C, const gfrref::FieldSpec& field,
                                 const gfrref::EchelonizeOptions& options,
                                 gfrref::RunReport* report = nullptr);

}  // namespace gfrref_b200
