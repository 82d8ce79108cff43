// ref_ech_main.cpp -- TEST INFRASTRUCTURE ONLY.
//
// A small driver over the *unmodified* reference library (linked against
// oracle/_ref/libgfrref_ref.so) that does what the reference's `gfrref ech`
// command does (src/cli.cpp:67-104) without its CLI11 front end:
//   ref_ech gfmat <p> <m> <n> <raw_u8_file> <out.gfmat>
//       write a row-major u8 matrix with gfrref::write_gfmat_file
//   ref_ech ech <in.gfmat> <block> <threads> <with_transform 0|1> <out_r> <out_selects> <out_t|->
//       read_gfmat_file -> echelonize -> write_gfmat_file(assembled_R) /
//       write_selects_file / write_transform_file; prints "rank r"
// Run as a separate process by tests/test_gpu_io.py.
#include <cstdio>
#include <cstdlib>
#include <fstream>
#include <string>
#include <vector>

#include "gfrref/chief.hpp"
#include "gfrref/io.hpp"

using namespace gfrref;

int main(int argc, char** argv) {
  try {
    const std::string cmd = argc > 1 ? argv[1] : "";
    if (cmd == "gfmat" && argc == 7) {
      const auto p = std::uint32_t(std::atoi(argv[2]));
      const std::size_t m = std::strtoull(argv[3], nullptr, 10), n = std::strtoull(argv[4], nullptr, 10);
      std::ifstream in(argv[5], std::ios::binary);
      std::vector<char> raw(m * n);
      if (m * n) in.read(raw.data(), std::streamsize(raw.size()));
      Matrix a(m, n);
      for (std::size_t r = 0; r < m; ++r)
        for (std::size_t c = 0; c < n; ++c) a.at(r, c) = std::uint8_t(raw[r * n + c]);
      write_gfmat_file(argv[6], FieldSpec(p), a);
      return 0;
    }
    if (cmd == "ech" && argc == 9) {
      const GfMat in = read_gfmat_file(argv[2]);
      EchelonizeOptions o;
      o.block = std::strtoull(argv[3], nullptr, 10);
      o.threads = std::atoi(argv[4]);
      o.with_transform = std::atoi(argv[5]) != 0;
      const EchelonOutput out = echelonize(in.matrix, in.field, o);
      write_gfmat_file(argv[6], out.field, out.assembled_R());
      write_selects_file(argv[7], out);
      if (std::string(argv[8]) != "-") write_transform_file(argv[8], out);
      std::printf("rank %zu\n", out.rank);
      return 0;
    }
    std::fprintf(stderr, "usage: ref_ech gfmat|ech ...\n");
    return 2;
  } catch (const std::exception& e) {
    std::fprintf(stderr, "%s\n", e.what());
    return 3;
  }
}
