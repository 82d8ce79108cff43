// io.cpp -- GFMAT / SELECTS / TRANSFORM text formats (reference
// src/io.cpp:143-286, byte-identical output for prime fields).
#include "io.hpp"

#include <charconv>
#include <cstring>
#include <fstream>
#include <istream>
#include <ostream>

namespace gfq {
namespace {

// One matrix row as "v v v\n": a matrix body line (reference :175-186).
void put_rows(std::ostream& out, const std::uint8_t* data, std::int64_t rows, std::int64_t cols,
              std::int64_t ld, int esize) {
  std::string line;
  char buf[12];
  for (std::int64_t r = 0; r < rows; ++r) {
    line.clear();
    const std::uint8_t* row = data + r * ld;
    for (std::int64_t c = 0; c < cols; ++c) {
      if (c) line.push_back(' ');
      unsigned v = row[c];
      if (esize == 4) std::memcpy(&v, row + 4 * c, 4);
      const auto res = std::to_chars(buf, buf + sizeof buf, v);
      line.append(buf, res.ptr);
    }
    line.push_back('\n');
    out << line;
  }
}

void put_matrix(std::ostream& out, const Mat& m) {
  if (m.empty()) {
    // zero columns still print one (empty) line per row, like the reference
    for (std::int64_t r = 0; r < m.rows(); ++r) out << '\n';
    return;
  }
  const std::vector<std::uint8_t> h = m.to_host();
  put_rows(out, h.data(), m.rows(), m.cols(), m.row_bytes(), m.esize());
}

// reference src/io.cpp:143-153 (write_field_line); `code` is a field code
void put_field(std::ostream& out, std::uint32_t code) {
  const FieldSpec f(code);
  out << "field p=" << f.p() << " k=" << f.k();
  if (f.k() > 1) {
    out << " modulus=";
    const std::vector<std::uint32_t>& mod = f.modulus();
    for (std::size_t t = 0; t < mod.size(); ++t) out << (t ? "," : "") << mod[t];
  }
  out << "\n";
}


std::ofstream open_out(const std::string& path) {
  std::ofstream out(path, std::ios::binary);
  if (!out) throw ParseError(path + ": cannot open for writing");
  return out;
}
void finish(std::ofstream& out, const std::string& path) {
  out.flush();
  if (!out) throw ParseError(path + ": write failed");
}

// Line-oriented strict reader.
struct Lines {
  std::istream& in;
  std::string name;
  std::size_t lineno = 0;

  [[noreturn]] void fail(const std::string& msg) const {
    throw ParseError(name + ":" + std::to_string(lineno) + ": " + msg);
  }
  bool next(std::string& s) {
    if (!std::getline(in, s)) return false;
    ++lineno;
    if (!s.empty() && s.back() == '\r') s.pop_back();
    return true;
  }
  std::string expect(const std::string& what) {
    std::string s;
    if (!next(s)) fail("unexpected end of file, expected " + what);
    return s;
  }
};

std::vector<std::string> tokens(const std::string& s) {
  std::vector<std::string> out;
  std::size_t i = 0;
  while (i < s.size()) {
    while (i < s.size() && (s[i] == ' ' || s[i] == '\t')) ++i;
    std::size_t j = i;
    while (j < s.size() && s[j] != ' ' && s[j] != '\t') ++j;
    if (j > i) out.push_back(s.substr(i, j - i));
    i = j;
  }
  return out;
}

bool to_u64(const std::string& s, std::uint64_t& v) {
  if (s.empty()) return false;
  const auto r = std::from_chars(s.data(), s.data() + s.size(), v);
  return r.ec == std::errc() && r.ptr == s.data() + s.size();
}

std::uint64_t key_u64(const Lines& lr, const std::vector<std::string>& t, std::size_t idx,
                      const std::string& key) {
  if (idx >= t.size()) lr.fail("missing " + key + "=...");
  const std::string& tok = t[idx];
  if (tok.size() <= key.size() || tok.compare(0, key.size(), key) != 0 || tok[key.size()] != '=')
    lr.fail("expected " + key + "=..., got '" + tok + "'");
  std::uint64_t v = 0;
  if (!to_u64(tok.substr(key.size() + 1), v)) lr.fail("invalid number in " + tok);
  return v;
}

}  // namespace

// reference src/io.cpp:527-543
std::vector<std::uint32_t> parse_modulus(const std::string& text) {
  std::vector<std::uint32_t> out;
  std::size_t pos = 0;
  while (true) {
    const std::size_t comma = text.find(',', pos);
    const std::string tok = comma == std::string::npos ? text.substr(pos) : text.substr(pos, comma - pos);
    std::uint64_t v = 0;
    if (!to_u64(tok, v) || v >= (1u << 16)) throw ParseError("invalid modulus coefficient: '" + tok + "'");
    out.push_back(std::uint32_t(v));
    if (comma == std::string::npos) break;
    pos = comma + 1;
  }
  return out;
}

// reference src/io.cpp:199-213
GfMatHost read_gfmat(std::istream& in, const std::string& name) {
  Lines lr{in, name};
  if (lr.expect("'GFMAT v1'") != "GFMAT v1") lr.fail("expected 'GFMAT v1'");
  const std::vector<std::string> ft = tokens(lr.expect("field header"));
  if (ft.empty() || ft[0] != "field") lr.fail("expected a field header");
  const std::uint64_t p = key_u64(lr, ft, 1, "p");
  const std::uint64_t k = key_u64(lr, ft, 2, "k");
  // reference src/io.cpp:115-140 (parse_field_line)
  if (p < 2 || p >= (1u << 16)) lr.fail("field characteristic out of range");
  if (k < 1) lr.fail("field degree must be at least 1");
  std::uint32_t code = 0, q = 0;
  if (k == 1) {
    if (ft.size() != 3) lr.fail("prime fields take no modulus");
    try {
      const FieldSpec f{std::uint32_t(p)};
      code = f.code();
      q = f.order();
    } catch (const std::exception& e) {
      lr.fail(e.what());
    }
  } else {
    if (ft.size() != 4) lr.fail("extension fields need modulus=c0,...,ck");
    const std::string& mt = ft[3];
    if (mt.rfind("modulus=", 0) != 0) lr.fail("expected modulus=...");
    try {
      const FieldSpec f(std::uint32_t(p), std::uint32_t(k), parse_modulus(mt.substr(8)));
      code = f.code();
      q = f.order();
    } catch (const ParseError&) {
      throw;
    } catch (const std::exception& e) {
      lr.fail(e.what());
    }
  }
  const std::vector<std::string> dt = tokens(lr.expect("rows=... cols=..."));
  const std::uint64_t rows = key_u64(lr, dt, 0, "rows");
  const std::uint64_t cols = key_u64(lr, dt, 1, "cols");
  if (dt.size() != 2) lr.fail("unexpected tokens after cols=...");
  if (rows > (1u << 24) || cols > (1u << 24)) lr.fail("dimensions out of range");
  GfMatHost m;
  m.p = code;
  m.rows = std::int64_t(rows);
  m.cols = std::int64_t(cols);
  m.esize = FieldSpec(code).esize();
  m.data.resize(std::size_t(rows * cols) * std::size_t(m.esize));
  for (std::uint64_t r = 0; r < rows; ++r) {
    const std::string line = lr.expect("a matrix row");
    const char* s = line.data();
    const char* e = s + line.size();
    std::uint64_t c = 0;
    while (true) {
      while (s < e && (*s == ' ' || *s == '\t')) ++s;
      if (s == e) break;
      unsigned v = 0;
      const auto res = std::from_chars(s, e, v);
      if (res.ec != std::errc() || (res.ptr < e && *res.ptr != ' ' && *res.ptr != '\t'))
        lr.fail("invalid entry");
      if (v >= q) lr.fail("entry '" + std::to_string(v) + "' is not an element encoding");
      if (c >= cols) lr.fail("too many entries in row");
      if (m.esize == 4)
        std::memcpy(&m.data[std::size_t(r * cols + c) * 4], &v, 4);
      else
        m.data[std::size_t(r * cols + c)] = std::uint8_t(v);
      ++c;
      s = res.ptr;
    }
    if (c != cols)
      lr.fail("expected " + std::to_string(cols) + " entries, got " + std::to_string(c));
  }
  std::string rest;
  while (lr.next(rest))
    if (!tokens(rest).empty()) lr.fail("unexpected trailing content");
  return m;
}

GfMatHost read_gfmat_file(const std::string& path) {
  std::ifstream in(path, std::ios::binary);
  if (!in) throw ParseError(path + ": cannot open");
  return read_gfmat(in, path);
}

// reference src/io.cpp:221-226
void write_gfmat(std::ostream& out, std::uint32_t p, const Mat& m) {
  out << "GFMAT v1\n";
  put_field(out, p);
  out << "rows=" << m.rows() << " cols=" << m.cols() << "\n";
  put_matrix(out, m);
}

void write_gfmat_file(const std::string& path, std::uint32_t p, const Mat& m) {
  std::ofstream out = open_out(path);
  write_gfmat(out, p, m);
  finish(out, path);
}

// reference src/io.cpp:235-259
void write_selects(std::ostream& out, const EchelonOutput& res) {
  out << "SELECTS v1\n";
  out << "rank=" << res.rank << " block_rows=" << res.chop.a() << " block_cols=" << res.chop.b()
      << "\n";
  const auto put_set = [&](const char* tag, const char* var, std::size_t x, std::size_t off,
                           const IndexSet& s) {
    out << tag << ' ' << var << '=' << x << " offset=" << off << " size=" << s.universe
        << " count=" << s.members.size();
    for (auto v : s.members) out << ' ' << v;
    out << '\n';
  };
  for (std::size_t i = 0; i < res.chop.a(); ++i)
    put_set("row", "i", i, res.chop.row_offset(i), res.varrho[i]);
  for (std::size_t j = 0; j < res.chop.b(); ++j)
    put_set("col", "j", j, res.chop.col_offset(j), res.upsilon[j]);
  out << "global_rows count=" << res.rank;
  for (auto v : res.global_varrho()) out << ' ' << v;
  out << '\n';
  out << "global_cols count=" << res.rank;
  for (auto v : res.global_upsilon()) out << ' ' << v;
  out << '\n';
}

void write_selects_file(const std::string& path, const EchelonOutput& res) {
  std::ofstream out = open_out(path);
  write_selects(out, res);
  finish(out, path);
}

// reference src/io.cpp:267-286
void write_transform(std::ostream& out, const EchelonOutput& res) {
  if (!res.with_transform) throw std::logic_error("transformation was not computed");
  out << "TRANSFORM v1\n";
  put_field(out, res.field.code());
  out << "block_rows=" << res.chop.a() << " block_cols=" << res.chop.b() << "\n";
  for (std::size_t j = 0; j < res.chop.b(); ++j)
    for (std::size_t h = 0; h < res.chop.a(); ++h) {
      const Mat& m = res.T_M_blocks[j][h];
      out << "M j=" << j << " h=" << h << " rows=" << m.rows() << " cols=" << m.cols() << "\n";
      put_matrix(out, m);
    }
  for (std::size_t i = 0; i < res.chop.a(); ++i)
    for (std::size_t h = 0; h <= i; ++h) {
      const Mat& m = res.T_K_blocks[i][h];
      out << "K i=" << i << " h=" << h << " rows=" << m.rows() << " cols=" << m.cols() << "\n";
      put_matrix(out, m);
    }
}

void write_transform_file(const std::string& path, const EchelonOutput& res) {
  std::ofstream out = open_out(path);
  write_transform(out, res);
  finish(out, path);
}

}  // namespace gfq
