// gfrref_b200.cpp -- see gfrref_b200.hpp.  Pure host glue: field code,
// u32 -> u8 input, one gfq_echelonize_host_into call (H2D inside, every
// output block streamed D2H as it becomes final), then the blocks are
// sliced out of the packed download (R[j][l>=j], T_M[j][h], T_K[i][h<=i],
// shapes from |upsilon_j| and |varrho_i|, include/gfrref/chief.hpp:41-50).
// Wide fields (p > 251, p^k > 256: u32 elements on the device) take
// gfq_mat_upload32 + gfq_echelonize + gfq_output_download_blocks instead.
#include "gfrref_b200.hpp"

#include <cstdint>
#include <cstring>
#include <stdexcept>
#include <string>
#include <vector>

#include "gfq.h"

namespace gfrref_b200 {
namespace {

[[noreturn]] void raise(int rc) {
  const std::string msg = gfq_last_error();
  switch (rc) {
    case GFQ_ERR_INVALID: throw std::invalid_argument(msg);
    case GFQ_ERR_LOGIC: throw std::logic_error(msg);
    case GFQ_ERR_DOMAIN: throw std::domain_error(msg);
    default: throw std::runtime_error(msg);
  }
}
void check(int rc) {
  if (rc != GFQ_OK) raise(rc);
}

struct Out {
  gfq_output* h = nullptr;
  ~Out() { gfq_output_free(h); }
};

std::uint32_t field_code(const gfrref::FieldSpec& f) {
  if (f.k() == 1) return f.p();
  std::uint32_t code = 0;
  const auto& mod = f.modulus();
  check(gfq_field_register(f.p(), f.k(), mod.data(), int(mod.size()), &code));
  return code;
}

// the next rows x cols block of the packed download (es bytes an element)
gfrref::Matrix take(const std::uint8_t*& at, std::size_t rows, std::size_t cols, int es) {
  gfrref::Matrix m(rows, cols);
  for (std::size_t r = 0; r < rows; ++r)
    for (std::size_t c = 0; c < cols; ++c) {
      if (es == 4) {
        std::uint32_t v;
        std::memcpy(&v, at, 4);
        m.at(r, c) = v;
      } else {
        m.at(r, c) = *at;
      }
      at += es;
    }
  return m;
}

struct MatH {
  gfq_mat* h = nullptr;
  ~MatH() { gfq_mat_free(h); }
};

}  // namespace

gfrref::EchelonOutput echelonize(const gfrref::Matrix& C, const gfrref::FieldSpec& field,
                                 const gfrref::EchelonizeOptions& options,
                                 gfrref::RunReport* report) {
  const std::uint32_t code = field_code(field);
  const std::size_t m = C.rows(), n = C.cols();
  const bool wide = field.k() == 1 ? field.p() > 251 : field.order() > 256;
  const int es = wide ? 4 : 1;
  std::vector<std::uint8_t> c8(wide ? 0 : m * n);
  for (std::size_t t = 0; t < m * n; ++t) {
    const gfrref::Elem v = C.data()[t];
    if (!field.valid(v)) throw std::invalid_argument("echelonize: matrix entry outside the field");
    if (!wide) c8[t] = std::uint8_t(v);
  }
  gfq_options o;
  gfq_options_default(&o);
  o.block = options.block;
  o.threads = options.threads;
  o.with_transform = options.with_transform ? 1 : 0;
  o.ech_threshold = options.ech_threshold;
  o.remainder_first = options.remainder_first ? 1 : 0;
  o.collect_trace = options.collect_trace ? 1 : 0;
  o.retain_all = options.retain_all ? 1 : 0;

  gfrref::EchelonOutput r(field);
  r.chop = gfrref::chop(m, n, options.block, options.remainder_first);
  r.with_transform = options.with_transform;
  // upper bound of the packed block bytes: R <= r x n, T <= m x m
  const std::uint64_t cap = (std::uint64_t(m) * (n + (options.with_transform ? m : 0)) + 16) * std::uint64_t(es);
  std::vector<std::uint8_t> blocks(cap);
  Out out;
  if (wide) {
    MatH dev;
    const std::vector<std::uint32_t> c32(C.data().begin(), C.data().end());
    check(gfq_mat_upload32(std::int64_t(m), std::int64_t(n), c32.empty() ? nullptr : c32.data(),
                           std::int64_t(n > 0 ? n : 1), &dev.h));
    check(gfq_echelonize(code, dev.h, &o, &out.h));
    check(gfq_output_download_blocks(out.h, blocks.data(), cap));
  } else {
    check(gfq_echelonize_host_into(code, std::int64_t(m), std::int64_t(n), c8.empty() ? nullptr : c8.data(),
                                   std::int64_t(n > 0 ? n : 1), &o, blocks.data(), cap, &out.h));
  }
  std::uint64_t rank = 0, a = 0, b = 0;
  check(gfq_output_rank(out.h, &rank));
  check(gfq_output_grid(out.h, &a, &b));
  if (a != r.chop.a() || b != r.chop.b()) throw std::logic_error("echelonize_b200: block grid mismatch");
  r.rank = rank;
  const auto select = [&](int which, std::size_t x, std::size_t universe) {
    std::uint64_t cnt = 0;
    check(gfq_output_select(out.h, which, x, nullptr, &cnt));
    std::vector<std::uint32_t> mem(cnt);
    if (cnt) check(gfq_output_select(out.h, which, x, mem.data(), &cnt));
    return gfrref::IndexSet(universe, std::move(mem));
  };
  for (std::size_t j = 0; j < b; ++j) r.upsilon.push_back(select(0, j, r.chop.col_parts[j]));
  for (std::size_t i = 0; i < a; ++i) r.varrho.push_back(select(1, i, r.chop.row_parts[i]));
  const std::uint8_t* at = blocks.data();
  r.R_blocks.assign(b, std::vector<gfrref::Matrix>(b));
  for (std::size_t j = 0; j < b; ++j)
    for (std::size_t l = j; l < b; ++l)
      r.R_blocks[j][l] = take(at, r.upsilon[j].size(), r.chop.col_parts[l] - r.upsilon[l].size(), es);
  if (options.with_transform) {
    r.T_M_blocks.assign(b, std::vector<gfrref::Matrix>(a));
    for (std::size_t j = 0; j < b; ++j)
      for (std::size_t h = 0; h < a; ++h) r.T_M_blocks[j][h] = take(at, r.upsilon[j].size(), r.varrho[h].size(), es);
    r.T_K_blocks.resize(a);
    for (std::size_t i = 0; i < a; ++i)
      for (std::size_t h = 0; h <= i; ++h)
        r.T_K_blocks[i].push_back(take(at, r.chop.row_parts[i] - r.varrho[i].size(), r.varrho[h].size(), es));
  }
  if (report) {
    gfq_report rep{};
    check(gfq_output_report(out.h, &rep));
    report->wall_ns = rep.wall_ns;
    report->peak_live_bytes = rep.peak_live_bytes;
    report->initial_live_bytes = rep.initial_live_bytes;
    report->workers = rep.workers;
    report->trace.clear();
  }
  return r;
}

}  // namespace gfrref_b200
