// chief.hpp -- ChopMatrix, the Chief's plan and the echelonize entry point
// (reference include/gfrref/chief.hpp:27-105), B200 edition.
#pragma once

#include <cstddef>
#include <functional>
#include <optional>
#include <string>
#include <vector>

#include "scheduler.hpp"

namespace gfq {

/// reference include/gfrref/chief.hpp:15-25
struct ChopSpec {
  std::vector<std::size_t> row_parts;
  std::vector<std::size_t> col_parts;
  std::size_t a() const { return row_parts.size(); }
  std::size_t b() const { return col_parts.size(); }
  std::size_t rows() const;
  std::size_t cols() const;
  std::size_t row_offset(std::size_t i) const;
  std::size_t col_offset(std::size_t j) const;
};

/// reference include/gfrref/chief.hpp:27-28
ChopSpec chop(std::size_t m, std::size_t n, std::size_t block, bool remainder_first = false);

/// reference include/gfrref/chief.hpp:33-59, blocks device-resident.
struct EchelonOutput {
  FieldSpec field;
  ChopSpec chop;
  bool with_transform = false;
  std::size_t rank = 0;
  explicit EchelonOutput(FieldSpec f) : field(f) {}
  std::vector<std::vector<Mat>> R_blocks;    // [j][l], l >= j
  std::vector<std::vector<Mat>> T_M_blocks;  // [j][h]
  std::vector<std::vector<Mat>> T_K_blocks;  // [i][h], h <= i
  std::vector<IndexSet> varrho;              // per block row
  std::vector<IndexSet> upsilon;             // per block column
  std::vector<std::uint32_t> global_upsilon() const;
  std::vector<std::uint32_t> global_varrho() const;
  /// rank x (n - rank) remnant, assembled on the device.
  Mat assembled_R() const;
};

struct PlanHandles {
  std::vector<std::int32_t> d_final, e_final;
  std::vector<std::vector<std::int32_t>> r_final, m_final, k_final;
  // fused plan: the block is part r_part / m_part of a MatParts slot (-1: plain)
  std::vector<std::vector<std::int32_t>> r_part, m_part, k_part;
};

/// reference include/gfrref/chief.hpp:72: Steps 1-3 into a fresh graph.
/// Input blocks are views of the device-resident C (no copy).
PlanHandles build_plan(TaskGraph& graph, const Mat& C, const FieldSpec& field,
                       const ChopSpec& chop, bool with_transform);
/// Same plan; input block (i, k) is `input(i, k)` when it returns a value
/// (a sharded rank only holds its own block columns).
PlanHandles build_plan(TaskGraph& graph, const std::function<std::optional<Mat>(std::size_t, std::size_t)>& input,
                       const FieldSpec& field, const ChopSpec& chop, bool with_transform);

/// reference include/gfrref/chief.hpp:76-84 (+ `workers`: host threads,
/// one CUDA stream each; the reference's `threads`).
struct EchelonizeOptions {
  std::size_t block = 256;
  int threads = 1;
  bool with_transform = true;
  std::size_t ech_threshold = 256;
  bool remainder_first = false;
  bool collect_trace = false;
  bool retain_all = false;
  bool fuse = true;  // wide UpdateRow / ClearUp jobs (single GPU); false = the reference's task grid
  // Optional pinned host buffer receiving every output block in
  // gfq_output_download_blocks' layout, each block copied (on its own copy
  // stream) as soon as it is final -- the download overlaps Step 3.
  std::uint8_t* host_out = nullptr;
  std::uint64_t host_out_cap = 0;
};

/// The fused single-GPU plan (same values, wide jobs per panel).  With
/// row_ready, block row i of C is valid once row_ready[2i] (its block
/// column 0) and row_ready[2i + 1] (the rest of the row) have fired.
PlanHandles build_plan_fused(TaskGraph& graph, const Mat& C, const FieldSpec& field,
                             const ChopSpec& chop, bool with_transform,
                             const std::vector<std::shared_ptr<EventBox>>* row_ready = nullptr);

/// echelonize from host memory: block rows are copied to HBM on a copy
/// stream in the order Step 1 needs them, and each block row's tasks start
/// as soon as its copy lands (the fused plan; otherwise one upload first).
EchelonOutput echelonize_host(const std::uint8_t* host, std::int64_t m, std::int64_t n,
                              std::int64_t ld, const FieldSpec& field,
                              const EchelonizeOptions& options, RunReport* report = nullptr);

/// reference include/gfrref/chief.hpp:88-90.  C is device-resident.
EchelonOutput echelonize(const Mat& C, const FieldSpec& field, const EchelonizeOptions& options,
                         RunReport* report = nullptr);
/// Reserve the device pool for an m x n echelonize up front (every call
/// does it too; doing it once before timing keeps the one-time mapping of
/// physical memory out of the first step).
void reserve_for(std::size_t m, std::size_t n, bool with_transform);

/// reference include/gfrref/chief.hpp:100: the m x m transformation,
/// materialised on the device.
Mat materialize_transform(const EchelonOutput& out);

}  // namespace gfq
