// verify.cpp -- on-device certificate of an EchelonOutput (reference
// src/chief.cpp:531-590).  Every product / comparison runs on the device
// (K1 contractions, K3 gathers, the compare / echelon_check reductions);
// only mismatch counters come back to the host.
#include "verify.hpp"

#include <algorithm>
#include <sstream>

#include "../kernels/kernels.hpp"
#include "jobs.hpp"

namespace gfq {
namespace {

struct Mismatch {
  DevBuf buf{16};
  int es = 1;  // element bytes of the compared matrices (positions come back in bytes)
  Mismatch() {
    const unsigned long long init[2] = {0ull, ~0ull};
    GFQ_CUDA(cudaMemcpyAsync(buf.ptr, init, sizeof init, cudaMemcpyHostToDevice, cur_stream()));
    GFQ_CUDA(cudaStreamSynchronize(cur_stream()));
  }
  unsigned long long* dev() { return reinterpret_cast<unsigned long long*>(buf.ptr); }
  // (count, first) after the queued checks
  std::pair<unsigned long long, unsigned long long> take() {
    unsigned long long h[2];
    GFQ_CUDA(cudaMemcpyAsync(h, buf.ptr, sizeof h, cudaMemcpyDeviceToHost, cur_stream()));
    GFQ_CUDA(cudaStreamSynchronize(cur_stream()));
    // (the count is of bytes for wide elements: a differing element counts
    // once per differing byte; the first position is returned in elements)
    return {h[0], es == 1 || h[0] == 0 ? h[1] : h[1] / std::uint64_t(es)};
  }
};

// a == b (mode 0), a == 0 (mode 1), a == value.I (mode 2), on u8 or u32
// elements (wide fields: byte-level compares; value.I as an explicit matrix)
void cmp(const Mat& a, const Mat* b, int mode, std::uint32_t value, Mismatch& mm) {
  if (a.esize() == 1) {
    dev::compare(a.rows(), a.cols(), a.data(), a.ld(), b ? b->data() : nullptr, b ? b->ld() : 0, mode,
                 std::uint8_t(value), mm.dev(), cur_stream());
    return;
  }
  mm.es = a.esize();
  Mat vi;
  if (mode == 2) {
    vi = Mat::zeros(a.rows(), a.cols(), a.esize());
    std::vector<std::int32_t> pos;
    for (std::int64_t i = 0; i < std::min(a.rows(), a.cols()); ++i) {
      pos.push_back(std::int32_t(i));
      pos.push_back(std::int32_t(i));
    }
    if (!pos.empty()) {
      auto pb = upload_i32(pos);
      dev::set_entries_u32(vi.data(), vi.ld(), reinterpret_cast<const std::int32_t*>(pb->ptr),
                           std::int64_t(pos.size() / 2), value, cur_stream());
    }
    b = &vi;
    mode = 0;
  }
  dev::compare(a.rows(), a.row_bytes(), a.data(), a.ld(), b ? b->data() : nullptr, b ? b->ld() : 0, mode, 0,
               mm.dev(), cur_stream());
  if (mode == 0 && b == &vi) GFQ_CUDA(cudaStreamSynchronize(cur_stream()));  // vi dies on return
}

// u8 mask (1 where the u32 element is nonzero) of a wide matrix
Mat nonzero_mask(const Mat& a) {
  Mat out(a.rows(), a.cols(), 1);
  if (!out.empty()) dev::nonzero_mask_u32(a.rows(), a.cols(), a.data(), a.ld(), out.data(), out.ld(), cur_stream());
  return out;
}

std::vector<std::uint32_t> complement(std::size_t universe, const std::vector<std::uint32_t>& s) {
  std::vector<std::uint32_t> out;
  out.reserve(universe - s.size());
  std::size_t q = 0;
  for (std::uint32_t c = 0; c < universe; ++c) {
    if (q < s.size() && s[q] == c) {
      ++q;
      continue;
    }
    out.push_back(c);
  }
  return out;
}

std::vector<std::uint32_t> shifted(const IndexSet& s, std::size_t off) {
  std::vector<std::uint32_t> v(s.members.size());
  for (std::size_t q = 0; q < v.size(); ++q) v[q] = std::uint32_t(off + s.members[q]);
  return v;
}

std::string where(const char* what, unsigned long long count, unsigned long long first,
                  std::int64_t cols) {
  std::ostringstream os;
  os << what << " (" << count << " entries, first at row " << (first / std::uint64_t(cols))
     << ", column " << (first % std::uint64_t(cols)) << ")";
  return os.str();
}

// The output must carry every block (a sharded run must be gathered).
bool complete(const EchelonOutput& out) {
  const std::size_t a = out.chop.a(), b = out.chop.b();
  if (out.upsilon.size() != b || out.varrho.size() != a || out.R_blocks.size() != b) return false;
  for (std::size_t j = 0; j < b; ++j)
    for (std::size_t l = j; l < b; ++l) {
      const Mat& m = out.R_blocks[j][l];
      const std::int64_t w = std::int64_t(out.chop.col_parts[l] - out.upsilon[l].size());
      const std::int64_t r = std::int64_t(out.upsilon[j].size());
      if (r > 0 && w > 0 && (m.rows() != r || m.cols() < w)) return false;
    }
  if (!out.with_transform) return true;
  for (std::size_t j = 0; j < b; ++j)
    for (std::size_t h = 0; h < a; ++h) {
      const Mat& m = out.T_M_blocks[j][h];
      const std::int64_t r = std::int64_t(out.upsilon[j].size()),
                         c = std::int64_t(out.varrho[h].size());
      if (r > 0 && c > 0 && (m.rows() != r || m.cols() != c)) return false;
    }
  for (std::size_t i = 0; i < a; ++i)
    for (std::size_t h = 0; h <= i; ++h) {
      const Mat& m = out.T_K_blocks[i][h];
      const std::int64_t r = std::int64_t(out.chop.row_parts[i] - out.varrho[i].size()),
                         c = std::int64_t(out.varrho[h].size());
      if (r > 0 && c > 0 && (m.rows() != r || m.cols() != c)) return false;
    }
  return true;
}

// T.C == E, T materialised (reference :565-588 verbatim in meaning).
std::string check_exact(const Mat& C, const EchelonOutput& out, const Mat& Rasm,
                        const std::vector<std::uint32_t>& gups,
                        const std::vector<std::uint32_t>& grest) {
  const FieldSpec& f = out.field;
  const std::int64_t m = C.rows(), r = std::int64_t(out.rank);
  const Mat P = mat_mul(f, materialize_transform(out), C);
  Mismatch top_piv, top_rest, bottom;
  if (r > 0) {
    const Mat top = P.row_view(0, r);
    cmp(take_cols(top, gups), nullptr, 2, f.neg(1), top_piv);
    if (!grest.empty()) {
      const Mat tr = take_cols(top, grest);
      cmp(tr, &Rasm, 0, 0, top_rest);
    }
  }
  if (m > r) cmp(P.row_view(r, m - r), nullptr, 1, 0, bottom);
  if (auto [c, first] = top_piv.take(); c)
    return where("T.C differs from -1 on the pivot columns", c, first, r);
  if (auto [c, first] = top_rest.take(); c)
    return where("T.C differs from the remnant R on the non-pivot columns", c, first,
                 std::int64_t(grest.size()));
  if (auto [c, first] = bottom.take(); c)
    return where("T.C is not zero on the non-pivot rows", c, first, C.cols());
  return {};
}

// Freivalds: T.(C.X) == E.X for X uniform n x s over GF(p), evaluated block
// by block from T's stored blocks (never materialised).  A wrong T.C
// passes with probability <= p^-s.
std::string check_freivalds(const Mat& C, const EchelonOutput& out, std::uint64_t seed,
                            std::int64_t s) {
  const FieldSpec& f = out.field;
  const ChopSpec& ch = out.chop;
  const std::size_t a = ch.a(), b = ch.b();
  const std::int64_t n = C.cols();
  Mat X(n, s, f.esize());
  if (f.wide())
    dev::random_fill_wide(f.order(), n, s, seed, 0, s, X.data(), X.ld(), nullptr, cur_stream());
  else
    dev::random_fill(f.p(), n, s, seed, 0, s, X.data(), X.ld(), nullptr, cur_stream());
  const Mat Y = mat_mul(f, C, X);  // m x s
  // Y restricted to the pivot rows of each block row (the columns of T_M / T_K).
  std::vector<Mat> Yv(a);
  for (std::size_t h = 0; h < a; ++h)
    if (!out.varrho[h].members.empty()) Yv[h] = take_rows(Y, shifted(out.varrho[h], ch.row_offset(h)));
  Mismatch piv, rest;
  std::vector<Mat> keep;  // results stay alive until the counters are read
  for (std::size_t j = 0; j < b; ++j) {
    const std::int64_t rj = std::int64_t(out.upsilon[j].size());
    if (rj == 0) continue;
    // lhs = X[pivot cols of j] + sum_h T_M(j,h) . Yv_h   ( = T.Y + X_piv on these rows)
    Mat lhs = take_rows(X, shifted(out.upsilon[j], ch.col_offset(j)));
    for (std::size_t h = 0; h < a; ++h)
      if (!Yv[h].empty()) lhs = mat_mul_add(f, lhs, out.T_M_blocks[j][h], Yv[h]);
    // rhs = sum_{l >= j} R(j,l) . X[non-pivot cols of l]   ( = E.X + X_piv)
    Mat rhs = Mat::zeros(rj, s, f.esize());
    for (std::size_t l = j; l < b; ++l) {
      const std::size_t w = ch.col_parts[l] - out.upsilon[l].size();
      if (w == 0) continue;
      const auto restl = complement(ch.col_parts[l], out.upsilon[l].members);
      std::vector<std::uint32_t> g(restl.size());
      for (std::size_t q = 0; q < g.size(); ++q) g[q] = std::uint32_t(ch.col_offset(l) + restl[q]);
      const Mat& Rjl = out.R_blocks[j][l];
      rhs = mat_mul_add(f, rhs, Rjl.cols() == std::int64_t(w) ? Rjl : Rjl.col_view(0, std::int64_t(w)),
                        take_rows(X, g));
    }
    cmp(lhs, &rhs, 0, 0, piv);
    keep.push_back(lhs);
    keep.push_back(rhs);
  }
  for (std::size_t i = 0; i < a; ++i) {
    const auto resti = complement(ch.row_parts[i], out.varrho[i].members);
    if (resti.empty()) continue;
    std::vector<std::uint32_t> g(resti.size());
    for (std::size_t q = 0; q < g.size(); ++q) g[q] = std::uint32_t(ch.row_offset(i) + resti[q]);
    Mat z = take_rows(Y, g);
    for (std::size_t h = 0; h <= i; ++h)
      if (!Yv[h].empty()) z = mat_mul_add(f, z, out.T_K_blocks[i][h], Yv[h]);
    cmp(z, nullptr, 1, 0, rest);
    keep.push_back(z);
  }
  if (auto [c, first] = piv.take(); c)
    return where("Freivalds: T.C.X differs from E.X on the pivot rows", c, first, s);
  if (auto [c, first] = rest.take(); c)
    return where("Freivalds: T.C.X is not zero on the non-pivot rows", c, first, s);
  (void)n;
  return {};
}

// Without T: every row of C lies in the row space of E.
std::string check_row_space(const Mat& C, const EchelonOutput& out, const Mat& Rasm,
                            const std::vector<std::uint32_t>& gups,
                            const std::vector<std::uint32_t>& grest) {
  if (grest.empty()) return {};
  Mismatch mm;
  const Mat rest = take_cols(C, grest);
  const Mat z = gups.empty() ? rest : mat_mul_add(out.field, rest, take_cols(C, gups), Rasm);
  cmp(z, nullptr, 1, 0, mm);
  if (auto [c, first] = mm.take(); c)
    return where("a row of C is outside the row space of the echelon form "
                 "(C[:, rest] + C[:, pivots].R != 0)",
                 c, first, std::int64_t(grest.size()));
  return {};
}

}  // namespace

VerifyResult verify(const Mat& C, const EchelonOutput& out, VerifyMethod method,
                    std::uint64_t seed) {
  VerifyResult res;
  auto fail = [&](std::string d) {
    res.ok = false;
    res.diag = std::move(d);
    return res;
  };
  const ChopSpec& ch = out.chop;
  if (std::int64_t(ch.rows()) != C.rows() || std::int64_t(ch.cols()) != C.cols())
    return fail("partition does not match the input matrix");
  if (!complete(out))
    return fail("output blocks are missing or misshapen (gather a sharded run first)");
  std::size_t rc = 0, rr = 0;
  for (const auto& g : out.upsilon) rc += g.members.size();
  for (const auto& r : out.varrho) rr += r.members.size();
  if (rc != out.rank || rr != out.rank)
    return fail("select sets disagree with the reported rank");

  const std::vector<std::uint32_t> gups = out.global_upsilon();
  const std::vector<std::uint32_t> grest = complement(ch.cols(), gups);
  const Mat Rasm = out.assembled_R();
  if (!Rasm.empty()) {
    std::vector<std::int32_t> pc(gups.begin(), gups.end()), rcv(grest.begin(), grest.end());
    auto dpc = upload_i32(pc), drc = upload_i32(rcv);
    Mismatch mm;
    // wide elements: the check reads a nonzero mask (one byte per element)
    const Mat Rchk = Rasm.esize() == 1 ? Rasm : nonzero_mask(Rasm);
    dev::echelon_check(Rchk.rows(), Rchk.cols(), Rchk.data(), Rchk.ld(),
                       reinterpret_cast<const std::int32_t*>(dpc->ptr),
                       reinterpret_cast<const std::int32_t*>(drc->ptr), mm.dev(), cur_stream());
    if (auto [c, first] = mm.take(); c)
      return fail(where("remnant is not in echelon shape (nonzero left of a pivot)", c, first,
                        Rasm.cols()));
  }

  std::string d;
  if (!out.with_transform) {
    res.method = "row-space";
    d = check_row_space(C, out, Rasm, gups, grest);
  } else {
    if (method == VerifyMethod::Auto) {
      std::size_t free_b = 0, total_b = 0;
      GFQ_CUDA(cudaMemGetInfo(&free_b, &total_b));
      const double need = double(C.rows()) * double(C.rows()) + 2.0 * double(C.rows()) * double(C.cols());
      method = need < 0.5 * double(free_b) ? VerifyMethod::Exact : VerifyMethod::Freivalds;
    }
    if (method == VerifyMethod::Exact) {
      res.method = "exact";
      d = check_exact(C, out, Rasm, gups, grest);
    } else {
      res.method = "freivalds";
      d = check_freivalds(C, out, seed, 64);
    }
  }
  if (!d.empty()) return fail(d);
  res.ok = true;
  return res;
}

}  // namespace gfq
