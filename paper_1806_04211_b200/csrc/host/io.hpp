// io.hpp -- the reference's text formats for the cmd_ech drop-in (SURVEY
// §8f item 3): GFMAT v1 matrices, SELECTS v1 and TRANSFORM v1 files
// (reference include/gfrref/io.hpp:17-45, src/io.cpp:143-286), written
// byte-identically from device-resident outputs.  Every field of the
// reference (u32 elements for p > 251 / p^k > 256).
#pragma once

#include <cstdint>
#include <iosfwd>
#include <stdexcept>
#include <string>
#include <vector>

#include "chief.hpp"

namespace gfq {

/// A malformed input file; the message names the file and line.  Maps to
/// GFQ_ERR_INVALID (the reference CLI's "bad input", exit 2).
struct ParseError : std::invalid_argument {
  using std::invalid_argument::invalid_argument;
};

struct GfMatHost {
  std::uint32_t p = 2;
  std::int64_t rows = 0, cols = 0;
  int esize = 1;                   // bytes per element (4: wide field)
  std::vector<std::uint8_t> data;  // row-major, ld = cols * esize
};

GfMatHost read_gfmat(std::istream& in, const std::string& name);
GfMatHost read_gfmat_file(const std::string& path);
void write_gfmat(std::ostream& out, std::uint32_t p, const Mat& m);
void write_gfmat_file(const std::string& path, std::uint32_t p, const Mat& m);
void write_selects(std::ostream& out, const EchelonOutput& res);
void write_selects_file(const std::string& path, const EchelonOutput& res);
void write_transform(std::ostream& out, const EchelonOutput& res);
void write_transform_file(const std::string& path, const EchelonOutput& res);

}  // namespace gfq
