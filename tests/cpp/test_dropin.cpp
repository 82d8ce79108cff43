// test_dropin.cpp -- TEST INFRASTRUCTURE: the reference-side drop-in
// (integration/gfrref_b200.cpp) against the reference library itself
// (oracle/_ref/libgfrref_ref.so, compiled from /root/reference).
//
// For every case: gfrref::echelonize (the reference, src/chief.cpp:322-386)
// and gfrref_b200::echelonize on the same gfrref::Matrix must return equal
// EchelonOutput fields (rank, upsilon, varrho, every R / T_M / T_K block),
// and the reference's own gfrref::verify (src/chief.cpp:531-590) must
// accept the B200 output.  Prints one PASS/FAIL line per case; exit 1 on
// any failure.   Usage: test_dropin [quick|full]
#include <cstdio>
#include <cstring>
#include <exception>
#include <stdexcept>
#include <string>

#include "gfrref/chief.hpp"
#include "gfrref/generate.hpp"
#include "gfrref_b200.hpp"

using namespace gfrref;

namespace {
int failures = 0;

bool same(const EchelonOutput& a, const EchelonOutput& b, std::string* why) {
  if (a.rank != b.rank) return *why = "rank", false;
  if (a.upsilon != b.upsilon) return *why = "upsilon", false;
  if (a.varrho != b.varrho) return *why = "varrho", false;
  if (a.R_blocks != b.R_blocks) return *why = "R_blocks", false;
  if (a.T_M_blocks != b.T_M_blocks) return *why = "T_M_blocks", false;
  if (a.T_K_blocks != b.T_K_blocks) return *why = "T_K_blocks", false;
  if (a.with_transform != b.with_transform) return *why = "with_transform", false;
  return true;
}

void run_case(const char* name, const Matrix& C, const FieldSpec& f, std::size_t block,
              bool with_transform = true) {
  EchelonizeOptions o;
  o.block = block;
  o.threads = 4;
  o.with_transform = with_transform;
  std::string why = "-";
  bool ok = false;
  try {
    const EchelonOutput ref = echelonize(C, f, o);
    const EchelonOutput got = gfrref_b200::echelonize(C, f, o);
    ok = same(ref, got, &why);
    if (ok && with_transform) {
      std::string diag;
      ok = verify(C, got, &diag);
      if (!ok) why = "gfrref::verify: " + diag;
    }
  } catch (const std::exception& e) {
    why = std::string("exception: ") + e.what();
  }
  std::printf("%s %s (%zux%zu GF(%u^%u) block %zu%s)%s%s\n", ok ? "PASS" : "FAIL", name, C.rows(),
              C.cols(), f.p(), f.k(), block, with_transform ? "" : " no-transform", ok ? "" : ": ",
              ok ? "" : why.c_str());
  failures += ok ? 0 : 1;
}

template <class E, class F>
void expect_throw(const char* name, F fn) {
  bool ok = false;
  std::string what = "no exception";
  try {
    fn();
  } catch (const E& e) {
    ok = true;
    what = e.what();
  } catch (const std::exception& e) {
    what = std::string("wrong exception: ") + e.what();
  }
  std::printf("%s %s: %s\n", ok ? "PASS" : "FAIL", name, what.c_str());
  failures += ok ? 0 : 1;
}
}  // namespace

int main(int argc, char** argv) {
  const bool full = argc > 1 && std::strcmp(argv[1], "full") == 0;
  // the paper's 6x6 GF(3) example (tests/test_chief.cpp:22-28 values)
  {
    const FieldSpec f(3);
    const Matrix C6 = mat_build(6, 6, {{0, 2, 2, 0, 1, 0}, {0, 2, 2, 1, 2, 2}, {1, 0, 1, 0, 2, 1},
                                       {2, 0, 1, 0, 2, 2}, {0, 1, 1, 2, 1, 1}, {1, 2, 2, 2, 0, 0}});
    run_case("paper-6x6", C6, f, 3);
    run_case("paper-6x6", C6, f, 3, false);
  }
  for (std::uint32_t p : {2u, 3u, 7u, 251u}) {
    const FieldSpec f(p);
    run_case("random", random_matrix(f, 300, 260, 11 + p), f, 64);
    run_case("random-ragged", random_matrix(f, 257, 333, 12 + p), f, 100);
    run_case("low-rank", random_product_matrix(f, 240, 200, 90, 13 + p), f, 48);
    run_case("low-rank", random_product_matrix(f, 240, 200, 90, 13 + p), f, 48, false);
    run_case("zero", Matrix(70, 50), f, 32);
  }
  {
    const FieldSpec f(3, 2);   // GF(9), default modulus
    run_case("ext-field", random_matrix(f, 150, 130, 21), f, 40);
    const FieldSpec f16(2, 4);
    run_case("ext-field", random_product_matrix(f16, 120, 140, 60, 22), f16, 32);
  }
  if (full) {
    const FieldSpec f(3);
    run_case("cfg1", random_matrix(f, 2000, 2000, 1), f, 500);    // BASELINE configs[0]
    const FieldSpec f2(2);
    run_case("gf2-2048", random_matrix(f2, 2048, 2048, 5), f2, 256);
  }
  {
    // wide fields (u32 elements): GF(257), GF(65521) and the reference's own
    // chief-test field GF(11^3) (tests/test_chief.cpp:371)
    const FieldSpec f(257);
    run_case("wide-prime", random_matrix(f, 90, 70, 31), f, 20);
    const FieldSpec f2(65521);
    run_case("wide-prime", random_product_matrix(f2, 60, 75, 30, 32), f2, 16);
    const FieldSpec f3(11, 3);
    run_case("wide-ext", random_matrix(f3, 9, 7, 33), f3, 3);
    run_case("wide-ext", random_matrix(f3, 50, 40, 34), f3, 12, false);
  }
  // error behaviour: invalid inputs raise, never fall back
  expect_throw<std::invalid_argument>("entry outside the field", [] {
    const FieldSpec f(3);
    gfrref_b200::echelonize(mat_build(1, 2, {{1, 5}}), f, EchelonizeOptions{});
  });
  std::printf("%s: %d failure(s)\n", failures ? "FAILED" : "OK", failures);
  return failures ? 1 : 0;
}
