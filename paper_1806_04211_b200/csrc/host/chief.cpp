// chief.cpp -- chop, plan, run, assemble (see chief.hpp).
#include "chief.hpp"

#include <algorithm>
#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <condition_variable>
#include <deque>
#include <memory>
#include <mutex>
#include <thread>
#include <unordered_map>
#include <unordered_set>
#include <numeric>
#include <string>
#include <stdexcept>

#include "../kernels/kernels.hpp"
#include "hostpack.hpp"
#include "jobs.hpp"

namespace gfq {

std::size_t ChopSpec::rows() const {
  return std::accumulate(row_parts.begin(), row_parts.end(), std::size_t(0));
}
std::size_t ChopSpec::cols() const {
  return std::accumulate(col_parts.begin(), col_parts.end(), std::size_t(0));
}
std::size_t ChopSpec::row_offset(std::size_t i) const {
  return std::accumulate(row_parts.begin(), row_parts.begin() + std::ptrdiff_t(i), std::size_t(0));
}
std::size_t ChopSpec::col_offset(std::size_t j) const {
  return std::accumulate(col_parts.begin(), col_parts.begin() + std::ptrdiff_t(j), std::size_t(0));
}

// reference src/chief.cpp:33-53
static std::vector<std::size_t> chop_axis(std::size_t total, std::size_t block, bool rem_first) {
  std::vector<std::size_t> parts;
  const std::size_t full = total / block, rem = total % block;
  if (rem && rem_first) parts.push_back(rem);
  parts.insert(parts.end(), full, block);
  if (rem && !rem_first) parts.push_back(rem);
  return parts;
}

ChopSpec chop(std::size_t m, std::size_t n, std::size_t block, bool remainder_first) {
  if (block < 1) throw std::invalid_argument("chop: block must be >= 1");
  return ChopSpec{chop_axis(m, block, remainder_first), chop_axis(n, block, remainder_first)};
}

// ---------------------------------------------------------------- plan
namespace {
struct Emitter {
  TaskGraph& g;
  std::int32_t slot(PkgKind k, std::size_t c0, std::size_t c1, std::size_t c2, std::size_t v) {
    return g.require_slot({k, std::uint16_t(c0), std::uint16_t(c1), std::uint16_t(c2),
                           std::uint16_t(v)});
  }
  void node(TaskKind kind, std::int32_t c0, std::int32_t c1, std::int32_t c2, std::int32_t pri,
            std::initializer_list<std::int32_t> in, std::initializer_list<std::int32_t> out) {
    TaskNode nd;
    nd.kind = kind;
    nd.c0 = c0;
    nd.c1 = c1;
    nd.c2 = c2;
    nd.priority = pri;
    for (auto s : in) nd.in[nd.n_in++] = s;
    for (auto s : out) nd.out[nd.n_out++] = s;
    g.plan_add(nd);
  }
  void node(TaskKind kind, std::int32_t c0, std::int32_t c1, std::int32_t c2, std::int32_t pri,
            const std::vector<std::int32_t>& in, std::initializer_list<std::int32_t> out) {
    TaskNode nd;
    nd.kind = kind;
    nd.c0 = c0;
    nd.c1 = c1;
    nd.c2 = c2;
    nd.priority = pri;
    for (auto s : in) nd.in[nd.n_in++] = s;
    for (auto s : out) nd.out[nd.n_out++] = s;
    g.plan_add(nd);
  }
};
}  // namespace

// The slot/version scheme and loop order of reference src/chief.cpp:67-287
// (SURVEY Appendix A): Step 1 j-outer/i-inner, Step 2 RowLengthen, Step 3
// descending rounds k = b-1..1.
PlanHandles build_plan(TaskGraph& graph, const Mat& C, const FieldSpec& field,
                       const ChopSpec& cs, bool with_transform) {
  if (std::int64_t(cs.rows()) != C.rows() || std::int64_t(cs.cols()) != C.cols())
    throw std::invalid_argument("build_plan: partition does not match matrix");
  return build_plan(
      graph,
      [&](std::size_t i, std::size_t k) -> std::optional<Mat> {
        return C.row_view(std::int64_t(cs.row_offset(i)), std::int64_t(cs.row_parts[i]))
            .col_view(std::int64_t(cs.col_offset(k)), std::int64_t(cs.col_parts[k]));
      },
      field, cs, with_transform);
}

PlanHandles build_plan(TaskGraph& graph,
                       const std::function<std::optional<Mat>(std::size_t, std::size_t)>& input,
                       const FieldSpec& field, const ChopSpec& cs, bool with_transform) {
  const std::size_t a = cs.a(), b = cs.b();
  if (a == 0 || b == 0) throw std::invalid_argument("build_plan: empty partition");
  if (a >= (1u << 14) || b >= (1u << 14))
    throw std::invalid_argument("build_plan: block grid exceeds slot coordinates");
  graph.set_field(field);
  Emitter e{graph};
  using K = PkgKind;
  using T = TaskKind;

  for (std::size_t i = 0; i < a; ++i)
    for (std::size_t k = 0; k < b; ++k) {
      std::optional<Mat> blk = input(i, k);
      if (blk)
        graph.add_input({K::C, std::uint16_t(i), std::uint16_t(k), 0, 0}, std::move(*blk));
      else
        graph.require_slot({K::C, std::uint16_t(i), std::uint16_t(k), 0, 0});
    }

  // Step 1
  for (std::size_t j = 0; j < b; ++j) {
    for (std::size_t i = 0; i < a; ++i) {
      const std::int32_t pri = std::int32_t(i + j);
      const auto sD = [&](std::size_t v) { return e.slot(K::D, j, 0, 0, v); };
      const std::int32_t sA = e.slot(K::A, i, j, 0, 0);
      if (i > 0)
        e.node(T::ClearDown, std::int32_t(i), std::int32_t(j), -1, pri,
               {e.slot(K::C, i, j, 0, j), sD(i - 1)}, {sD(i), sA});
      else
        e.node(T::ClearDown, std::int32_t(i), std::int32_t(j), -1, pri, {e.slot(K::C, i, j, 0, j)},
               {sD(i), sA});
      if (j > 0)
        e.node(T::Extend, std::int32_t(i), std::int32_t(j), -1, pri,
               {sA, e.slot(K::E, i, 0, 0, j - 1)}, {e.slot(K::E, i, 0, 0, j)});
      else
        e.node(T::Extend, std::int32_t(i), std::int32_t(j), -1, pri, {sA},
               {e.slot(K::E, i, 0, 0, j)});
      for (std::size_t k = j + 1; k < b; ++k) {
        const std::int32_t cin = e.slot(K::C, i, k, 0, j), cout = e.slot(K::C, i, k, 0, j + 1);
        const std::int32_t bout = e.slot(K::B, j, k, 0, i);
        if (i > 0)
          e.node(T::UpdateRow, std::int32_t(i), std::int32_t(j), std::int32_t(k), pri,
                 {sA, cin, e.slot(K::B, j, k, 0, i - 1)}, {cout, bout});
        else
          e.node(T::UpdateRow, std::int32_t(i), std::int32_t(j), std::int32_t(k), pri, {sA, cin},
                 {cout, bout});
      }
      if (with_transform) {
        for (std::size_t h = 0; h <= i; ++h) {
          TaskNode tr;
          tr.kind = T::UpdateRowTrafo;
          tr.c0 = std::int32_t(i);
          tr.c1 = std::int32_t(j);
          tr.c2 = std::int32_t(h);
          tr.priority = pri;
          tr.in[tr.n_in++] = sA;
          tr.in[tr.n_in++] = e.slot(K::E, h, 0, 0, j);
          if (j > 0) tr.in[tr.n_in++] = e.slot(K::K, i, h, 0, j - 1);
          if (h < i) tr.in[tr.n_in++] = e.slot(K::M, j, h, 0, i - 1 - h);
          tr.out[tr.n_out++] = e.slot(K::K, i, h, 0, j);
          tr.out[tr.n_out++] = e.slot(K::M, j, h, 0, i - h);
          graph.plan_add(tr);
        }
      }
    }
  }
  // Step 2
  if (with_transform)
    for (std::size_t j = 0; j < b; ++j)
      for (std::size_t h = 0; h < a; ++h)
        e.node(T::RowLengthen, -1, std::int32_t(j), std::int32_t(h), std::int32_t(a + b - 1),
               {e.slot(K::M, j, h, 0, a - 1 - h), e.slot(K::E, h, 0, 0, j),
                e.slot(K::E, h, 0, 0, b - 1)},
               {e.slot(K::M, j, h, 0, a - h)});
  // Step 3
  for (std::size_t k = 0; k < b; ++k)
    e.node(T::Copy, -1, std::int32_t(k), -1, std::int32_t(a + b + (b - 1 - k)),
           {e.slot(K::D, k, 0, 0, a - 1)}, {e.slot(K::R, k, k, 0, 0)});
  for (std::size_t k = b; k-- > 1;) {
    const std::int32_t pri = std::int32_t(a + b + (b - 1 - k));
    for (std::size_t j = 0; j < k; ++j) {
      const std::int32_t sX = e.slot(K::X, j, k, 0, 0);
      e.node(T::PreClearUp, -1, std::int32_t(j), std::int32_t(k), pri,
             {e.slot(K::B, j, k, 0, a - 1), e.slot(K::D, k, 0, 0, a - 1)},
             {sX, e.slot(K::R, j, k, 0, 0)});
      for (std::size_t l = k; l < b; ++l)
        e.node(T::ClearUp, std::int32_t(k), std::int32_t(j), std::int32_t(l), pri,
               {e.slot(K::R, j, l, 0, l - k), sX, e.slot(K::R, k, l, 0, l - k)},
               {e.slot(K::R, j, l, 0, l - k + 1)});
      if (with_transform)
        for (std::size_t h = 0; h < a; ++h)
          e.node(T::ClearUp, std::int32_t(k), std::int32_t(j), std::int32_t(h), pri,
                 {e.slot(K::M, j, h, 0, a - h + (b - 1 - k)), sX,
                  e.slot(K::M, k, h, 0, a - h + (b - 1 - k))},
                 {e.slot(K::M, j, h, 0, a - h + (b - k))});
    }
  }

  PlanHandles hd;
  for (std::size_t j = 0; j < b; ++j) hd.d_final.push_back(e.slot(K::D, j, 0, 0, a - 1));
  for (std::size_t i = 0; i < a; ++i) hd.e_final.push_back(e.slot(K::E, i, 0, 0, b - 1));
  hd.r_final.assign(b, std::vector<std::int32_t>(b, -1));
  for (std::size_t j = 0; j < b; ++j)
    for (std::size_t l = j; l < b; ++l) hd.r_final[j][l] = e.slot(K::R, j, l, 0, l - j);
  if (with_transform) {
    hd.m_final.assign(b, std::vector<std::int32_t>(a, -1));
    for (std::size_t j = 0; j < b; ++j)
      for (std::size_t h = 0; h < a; ++h)
        hd.m_final[j][h] = e.slot(K::M, j, h, 0, a - h + (b - 1 - j));
    hd.k_final.resize(a);
    for (std::size_t i = 0; i < a; ++i)
      for (std::size_t h = 0; h <= i; ++h) hd.k_final[i].push_back(e.slot(K::K, i, h, 0, b - 1));
  }
  graph.drop_key_index_if_large();
  return hd;
}

// Fused single-GPU plan: the same Steps 1-3 and slot versions, but the jobs
// that apply one package to every block of a panel run as ONE wide job:
//   UpdateRow(i, j, k): k = j+1 (on the Step-1 critical path) alone, k > j+1
//     together on the row panel (UpdateRowW); C and B row panels stay one
//     matrix (MatParts) from the input view onwards;
//   ClearUp(k, j, l) for all l (ClearUpRW) and ClearUp(k, j, h) for all h
//     (ClearUpMW), on padded panels.
// Every value is the one the reference plan computes (the jobs are
// column-separable); only the task granularity changes.
PlanHandles build_plan_fused(TaskGraph& graph, const Mat& C, const FieldSpec& field,
                             const ChopSpec& cs, bool with_transform,
                             const std::vector<std::shared_ptr<EventBox>>* row_ready) {
  const std::size_t a = cs.a(), b = cs.b();
  if (a == 0 || b == 0) throw std::invalid_argument("build_plan: empty partition");
  if (2 * a + 1 > std::size_t(TaskNode::kMaxIn))
    throw std::invalid_argument("build_plan_fused: block grid too tall for the fused plan");
  if (std::int64_t(cs.rows()) != C.rows() || std::int64_t(cs.cols()) != C.cols())
    throw std::invalid_argument("build_plan: partition does not match matrix");
  graph.set_field(field);
  {
    // the widest a T_M(j, .) panel gets: every row block's part, 16-aligned
    std::int64_t cap = 0;
    for (std::size_t h = 0; h < a; ++h) cap += (std::int64_t(cs.row_parts[h]) + 15) / 16 * 16;
    graph.set_trafo_capacity(cap);
  }
  Emitter e{graph};
  using K = PkgKind;
  using T = TaskKind;
  const auto blk = [&](std::size_t i, std::size_t k) {
    return C.row_view(std::int64_t(cs.row_offset(i)), std::int64_t(cs.row_parts[i]))
        .col_view(std::int64_t(cs.col_offset(k)), std::int64_t(cs.col_parts[k]));
  };
  // row_ready holds two events a block row: [2i] block column 0 landed
  // (all ClearDown(i, 0) needs), [2i + 1] the rest of the row
  const auto ready = [&](std::size_t i, std::size_t part = 1) {
    return row_ready ? (*row_ready)[2 * i + part] : std::shared_ptr<EventBox>();
  };
  for (std::size_t i = 0; i < a; ++i) {
    graph.add_input({K::C, std::uint16_t(i), 0, 0, 0}, blk(i, 0), ready(i, 0), true);
    if (b > 1) {
      MatParts panel;
      const std::int64_t o1 = std::int64_t(cs.col_offset(1));
      panel.m = C.row_view(std::int64_t(cs.row_offset(i)), std::int64_t(cs.row_parts[i]))
                    .col_view(o1, C.cols() - o1);
      for (std::size_t k = 1; k < b; ++k) {
        panel.off.push_back(std::int64_t(cs.col_offset(k)) - o1);
        panel.w.push_back(std::int64_t(cs.col_parts[k]));
      }
      graph.add_input({K::CW, std::uint16_t(i), 1, 0, 0}, std::move(panel), ready(i), true);
    }
  }

  // Task priorities (lower first; only the GPU schedule depends on them).
  // The reference keys Step 1 by i + j (src/chief.cpp:116): a wavefront
  // over anti-diagonals.  On the GPU the diagonal ClearDowns (the block
  // ECHs) cost several times a below- or above-diagonal step, so a task's
  // deadline is the diagonal step d = max(i, j) it feeds minus the chain of
  // cheap steps still between it and that ECH: key = w.max(i, j) +
  // min(i, j) (w = GFQ_PRIORITY_W, default 3; w = 1 is the reference's
  // i + j).  UpdateRow(i, j, k) takes the key of the ClearDown(i, k) it
  // feeds, the wide UpdateRow k = j + 2; the transform tasks (consumed only
  // by Steps 2-3) follow the chain tasks of the same key; Steps 2-3 last.
  static const int w_pri = [] {
    const char* v = std::getenv("GFQ_PRIORITY_W");
    const int w = v ? std::atoi(v) : 3;
    return w >= 1 && w <= 16 ? w : 3;
  }();
  const auto key = [&](std::size_t i, std::size_t j) {
    return std::int32_t(std::size_t(w_pri) * std::max(i, j) + std::min(i, j));
  };
  const auto pchain = [&](std::size_t i, std::size_t j, std::size_t kt) {
    return w_pri == 1 ? std::int32_t(i + j) : key(i, kt) * 4;
  };
  const auto ptrafo = [&](std::size_t i, std::size_t j) {
    return w_pri == 1 ? std::int32_t(i + j) : key(i, j) * 4 + 2;
  };
  const auto plate = [&](std::size_t v) {
    return w_pri == 1 ? std::int32_t(v) : std::int32_t((1 << 20) + v);
  };
  // Step 1
  for (std::size_t j = 0; j < b; ++j) {
    for (std::size_t i = 0; i < a; ++i) {
      const std::int32_t pri = pchain(i, j, j), pri_t = ptrafo(i, j);
      const std::int32_t pri_u = pchain(i, j, j + 1), pri_w = pchain(i, j, j + 2);
      const auto sD = [&](std::size_t v) { return e.slot(K::D, j, 0, 0, v); };
      const std::int32_t sA = e.slot(K::A, i, j, 0, 0);
      const std::int32_t sC = e.slot(K::C, i, j, 0, j);
      if (i > 0)
        e.node(T::ClearDown, std::int32_t(i), std::int32_t(j), -1, pri, {sC, sD(i - 1)}, {sD(i), sA});
      else
        e.node(T::ClearDown, std::int32_t(i), std::int32_t(j), -1, pri, {sC}, {sD(i), sA});
      if (j > 0)
        e.node(T::Extend, std::int32_t(i), std::int32_t(j), -1, pri_t,
               {sA, e.slot(K::E, i, 0, 0, j - 1)}, {e.slot(K::E, i, 0, 0, j)});
      else
        e.node(T::Extend, std::int32_t(i), std::int32_t(j), -1, pri_t, {sA},
               {e.slot(K::E, i, 0, 0, j)});
      if (j + 1 < b) {
        const std::int32_t panel = e.slot(K::CW, i, j + 1, 0, j);
        const std::int32_t cout = e.slot(K::C, i, j + 1, 0, j + 1);
        const std::int32_t bout = e.slot(K::B, j, j + 1, 0, i);
        if (i > 0)
          e.node(T::UpdateRow, std::int32_t(i), std::int32_t(j), std::int32_t(j + 1), pri_u,
                 {sA, panel, e.slot(K::B, j, j + 1, 0, i - 1)}, {cout, bout});
        else
          e.node(T::UpdateRow, std::int32_t(i), std::int32_t(j), std::int32_t(j + 1), pri_u,
                 {sA, panel}, {cout, bout});
        if (j + 2 < b) {
          const std::int32_t pout = e.slot(K::CW, i, j + 2, 0, j + 1);
          const std::int32_t bwout = e.slot(K::BW, j, j + 2, 0, i);
          if (i > 0)
            e.node(T::UpdateRowW, std::int32_t(i), std::int32_t(j), std::int32_t(j + 2), pri_w,
                   {sA, panel, e.slot(K::BW, j, j + 2, 0, i - 1)}, {pout, bwout});
          else
            e.node(T::UpdateRowW, std::int32_t(i), std::int32_t(j), std::int32_t(j + 2), pri_w,
                   {sA, panel}, {pout, bwout});
        }
      }
      if (with_transform) {
        // h = i: the reference task (K(i,i,.) and M(j,i,0) stay blocks)
        {
          TaskNode tr;
          tr.kind = T::UpdateRowTrafo;
          tr.c0 = std::int32_t(i);
          tr.c1 = std::int32_t(j);
          tr.c2 = std::int32_t(i);
          tr.priority = pri_t;
          tr.in[tr.n_in++] = sA;
          tr.in[tr.n_in++] = e.slot(K::E, i, 0, 0, j);
          if (j > 0) tr.in[tr.n_in++] = e.slot(K::K, i, i, 0, j - 1);
          tr.out[tr.n_out++] = e.slot(K::K, i, i, 0, j);
          tr.out[tr.n_out++] = e.slot(K::M, j, i, 0, 0);
          graph.plan_add(tr);
        }
        // h < i: one wide task on the K(i, ., .) and T_M(j, ., .) panels
        if (i > 0) {
          std::vector<std::int32_t> in{sA};
          for (std::size_t h = 0; h < i; ++h) in.push_back(e.slot(K::E, h, 0, 0, j));
          if (j > 0) in.push_back(e.slot(K::KW, i, 0, 0, j - 1));
          if (i >= 2) in.push_back(e.slot(K::MT, j, 0, 0, i - 1));
          in.push_back(e.slot(K::M, j, i - 1, 0, 0));
          e.node(T::UpdateRowTrafoW, std::int32_t(i), std::int32_t(j), -1, pri_t, in,
                 {e.slot(K::KW, i, 0, 0, j), e.slot(K::MT, j, 0, 0, i)});
        }
      }
    }
  }
  // Step 2: one wide RowLengthen per j (c0 = -2) widening every part h of
  // row j's T_M panel (row block a-1's panel + the M(j, a-1) block) into
  // the panel MW(j, b)
  static const bool rl_narrow = std::getenv("GFQ_RL_NARROW") != nullptr;  // A/B: per-h tasks
  if (with_transform && rl_narrow)
    for (std::size_t j = 0; j < b; ++j)
      for (std::size_t h = 0; h < a; ++h) {
        const bool part = h + 1 < a;
        e.node(T::RowLengthen, part ? std::int32_t(h) : -1, std::int32_t(j), std::int32_t(h),
               plate(a + b - 1),
               {part ? e.slot(K::MT, j, 0, 0, a - 1) : e.slot(K::M, j, a - 1, 0, 0),
                e.slot(K::E, h, 0, 0, j), e.slot(K::E, h, 0, 0, b - 1)},
               {e.slot(K::M, j, h, 0, a - h)});
      }
  // GFQ_RL_SPLIT=1 (read per plan): RowLengthen in two halves, below.  Off by
  // default: it lowers the HBM high-water (cfg5s 33.6 -> 29.9 GB) but not
  // the step time -- the one-piece copy already hides behind
  // UpdateRowTrafoW(a-1, b-1)
  const bool rl_split = [] {
    const char* v = std::getenv("GFQ_RL_SPLIT");
    return v && v[0] == '1';
  }();
  if (with_transform && !rl_narrow)
    for (std::size_t j = 0; j < b; ++j) {
      if (rl_split && a > 1) {
        // two halves (scheduler.cpp RowLengthen c0 = -3 / -4): parts h < a-1
        // need nothing from block row a-1, so for j < b-1 they are widened
        // while the last diagonal ClearDown still runs; part a-1 is appended
        // in place once E(a-1, b-1) exists
        std::vector<std::int32_t> in1{e.slot(K::MT, j, 0, 0, a - 1)};
        for (std::size_t h = 0; h + 1 < a; ++h) in1.push_back(e.slot(K::E, h, 0, 0, j));
        for (std::size_t h = 0; h + 1 < a; ++h) in1.push_back(e.slot(K::E, h, 0, 0, b - 1));
        const std::int32_t half = e.slot(K::MW, j, b + 1, 0, 0);
        e.node(T::RowLengthen, -3, std::int32_t(j), -1, plate(a + b - 1), in1, {half});
        e.node(T::RowLengthen, -4, std::int32_t(j), -1, plate(a + b - 1),
               {half, e.slot(K::M, j, a - 1, 0, 0), e.slot(K::E, a - 1, 0, 0, j),
                e.slot(K::E, a - 1, 0, 0, b - 1)},
               {e.slot(K::MW, j, b, 0, 0)});
        continue;
      }
      std::vector<std::int32_t> in;
      if (a > 1) in.push_back(e.slot(K::MT, j, 0, 0, a - 1));
      in.push_back(e.slot(K::M, j, a - 1, 0, 0));
      for (std::size_t h = 0; h < a; ++h) in.push_back(e.slot(K::E, h, 0, 0, j));
      for (std::size_t h = 0; h < a; ++h) in.push_back(e.slot(K::E, h, 0, 0, b - 1));
      e.node(T::RowLengthen, -2, std::int32_t(j), -1, plate(a + b - 1), in,
             {e.slot(K::MW, j, b, 0, 0)});
    }
  // Step 3
  for (std::size_t k = 0; k < b; ++k)
    e.node(T::Copy, -1, std::int32_t(k), -1, plate(a + b + (b - 1 - k)),
           {e.slot(K::D, k, 0, 0, a - 1)}, {e.slot(K::R, k, k, 0, 0)});
  // Step-3 order.  ClearUp(k, j) needs row k final and row j's ClearUp(k+1, j):
  // the reference walks k outermost (every row finishes in the last few
  // steps).  Row-major order (default; GFQ_STEP3_ORDER=0 restores k
  // outermost) is another topological order of the same DAG: row j gets all
  // its updates k = b-1 .. j+1 before row j-1 does, so rows become final
  // one by one from the bottom and the host-buffer path downloads row j
  // while rows < j are still being cleared.
  static const bool row_major = [] {
    const char* v = std::getenv("GFQ_STEP3_ORDER");
    return !v || std::atoi(v) != 0;
  }();
  for (std::size_t k = b; k-- > 1;) {
    for (std::size_t j = 0; j < k; ++j) {
      const std::int32_t pri = row_major && w_pri != 1
                                   ? plate(a + b + b + (b - 1 - j) * b + (b - 1 - k))
                                   : plate(a + b + (b - 1 - k));
      const std::int32_t sX = e.slot(K::X, j, k, 0, 0);
      if (k == j + 1)
        e.node(T::PreClearUp, -1, std::int32_t(j), std::int32_t(k), pri,
               {e.slot(K::B, j, k, 0, a - 1), e.slot(K::D, k, 0, 0, a - 1)},
               {sX, e.slot(K::R, j, k, 0, 0)});
      else
        e.node(T::PreClearUp, std::int32_t(k - (j + 2)), std::int32_t(j), std::int32_t(k), pri,
               {e.slot(K::BW, j, j + 2, 0, a - 1), e.slot(K::D, k, 0, 0, a - 1)},
               {sX, e.slot(K::R, j, k, 0, 0)});
      std::vector<std::int32_t> rin{sX, e.slot(K::R, j, k, 0, 0), e.slot(K::R, k, k, 0, 0)};
      if (k + 1 < b) {
        rin.push_back(e.slot(K::RW, j, k + 1, 0, 0));
        rin.push_back(e.slot(K::RW, k, k + 1, 0, 0));
      }
      e.node(T::ClearUpRW, std::int32_t(k), std::int32_t(j), -1, pri, rin,
             {e.slot(K::RW, j, k, 0, 0)});
      if (with_transform) {
        std::vector<std::int32_t> min{sX};
        if (k + 1 == b && rl_narrow) {
          for (std::size_t h = 0; h < a; ++h) min.push_back(e.slot(K::M, j, h, 0, a - h));
          for (std::size_t h = 0; h < a; ++h) min.push_back(e.slot(K::M, k, h, 0, a - h));
        } else if (k + 1 == b) {
          min.push_back(e.slot(K::MW, j, b, 0, 0));
          min.push_back(e.slot(K::MW, k, b, 0, 0));
        } else {
          min.push_back(e.slot(K::MW, j, k + 1, 0, 0));
          min.push_back(e.slot(K::MW, k, k + 1, 0, 0));
        }
        e.node(T::ClearUpMW, std::int32_t(k), std::int32_t(j), -1, pri, min,
               {e.slot(K::MW, j, k, 0, 0)});
      }
    }
  }

  PlanHandles hd;
  for (std::size_t j = 0; j < b; ++j) hd.d_final.push_back(e.slot(K::D, j, 0, 0, a - 1));
  for (std::size_t i = 0; i < a; ++i) hd.e_final.push_back(e.slot(K::E, i, 0, 0, b - 1));
  hd.r_final.assign(b, std::vector<std::int32_t>(b, -1));
  hd.r_part.assign(b, std::vector<std::int32_t>(b, -1));
  for (std::size_t j = 0; j < b; ++j)
    for (std::size_t l = j; l < b; ++l) {
      if (l == j) {
        hd.r_final[j][l] = e.slot(K::R, j, j, 0, 0);
      } else {
        hd.r_final[j][l] = e.slot(K::RW, j, j + 1, 0, 0);
        hd.r_part[j][l] = std::int32_t(l - (j + 1));
      }
    }
  if (with_transform) {
    hd.m_final.assign(b, std::vector<std::int32_t>(a, -1));
    hd.m_part.assign(b, std::vector<std::int32_t>(a, -1));
    for (std::size_t j = 0; j < b; ++j)
      for (std::size_t h = 0; h < a; ++h) {
        if (j + 1 == b && rl_narrow) {
          hd.m_final[j][h] = e.slot(K::M, j, h, 0, a - h);
        } else {
          hd.m_final[j][h] = e.slot(K::MW, j, j + 1, 0, 0);  // j = b-1: the RowLengthen panel
          hd.m_part[j][h] = std::int32_t(h);
        }
      }
    hd.k_final.resize(a);
    hd.k_part.resize(a);
    for (std::size_t i = 0; i < a; ++i)
      for (std::size_t h = 0; h <= i; ++h) {
        hd.k_final[i].push_back(h == i ? e.slot(K::K, i, i, 0, b - 1) : e.slot(K::KW, i, 0, 0, b - 1));
        hd.k_part[i].push_back(h == i ? -1 : std::int32_t(h));
      }
  }
  graph.drop_key_index_if_large();
  return hd;
}

// ---------------------------------------------------------------- echelonize
namespace {
// Early output download (EchelonizeOptions::host_out): every final block is
// copied D2H, in gfq_output_download_blocks' layout (R_blocks[j][l >= j],
// T_M_blocks[j][h], T_K_blocks[i][h <= i]), the moment its slot is
// published.  Block shapes follow from the final D (|gamma_j|) and E
// (|rho_i|) packages, so copies start once the last of those is published
// (end of Step 1) and the Step-3 blocks stream out as their rounds finish.
// Developer timeline of the host-buffer path (GFQ_E2E_DEBUG): device times
// of each input row's arrival and each output block's download, from the
// start of the upload.
bool e2e_debug() {
  static const bool on = std::getenv("GFQ_E2E_DEBUG") != nullptr;
  return on;
}
cudaEvent_t g_e2e_t0 = nullptr;

class EarlyDownload {
 public:
  // packed: GF(2) blocks leave HBM as bit rows (dev::pack_bits), cross PCIe
  // into a pinned staging buffer and are unpacked into `host` by the host
  // pool (hostpack) -- an eighth of the PCIe bytes
  EarlyDownload(const PlanHandles& h, const ChopSpec& cs, bool with_transform, std::uint8_t* host,
                std::uint64_t cap, bool packed)
      : h_(h), cs_(cs), host_(host), cap_(cap), packed_(packed) {
    const std::size_t a = cs.a(), b = cs.b();
    for (std::size_t j = 0; j < b; ++j)
      for (std::size_t l = j; l < b; ++l)
        add(0, j, l, h.r_final[j][l], h.r_part.empty() ? -1 : h.r_part[j][l]);
    if (with_transform) {
      for (std::size_t j = 0; j < b; ++j)
        for (std::size_t hh = 0; hh < a; ++hh)
          add(1, j, hh, h.m_final[j][hh], h.m_part.empty() ? -1 : h.m_part[j][hh]);
      for (std::size_t i = 0; i < a; ++i)
        for (std::size_t hh = 0; hh <= i; ++hh)
          add(2, i, hh, h.k_final[i][hh], h.k_part.empty() ? -1 : h.k_part[i][hh]);
    }
    for (auto sid : h.d_final) interest_.insert(sid);
    for (auto sid : h.e_final) interest_.insert(sid);
    GFQ_CUDA(cudaGetDevice(&device_));
    GFQ_CUDA(cudaStreamCreateWithFlags(&stream_, cudaStreamNonBlocking));
    thread_ = std::thread([this] { loop(); });
  }
  ~EarlyDownload() {
    try {
      finish();
    } catch (...) {
      // an error was already reported (or the run itself failed)
    }
    if (e2e_debug() && g_e2e_t0) {
      for (const auto& [label, ev] : dbg_) {
        float ms = 0;
        if (cudaEventElapsedTime(&ms, g_e2e_t0, ev) == cudaSuccess)
          std::fprintf(stderr, "e2e download %s done at %.2f ms\n", label.c_str(), double(ms));
        cudaEventDestroy(ev);
      }
      cudaGetLastError();
    }
    cudaStreamDestroy(stream_);
  }
  // RunOptions::on_publish (executor lock held): queue interesting slots
  void publish(std::int32_t sid, const std::shared_ptr<Published>& pub) {
    if (!interest_.count(sid)) return;
    std::lock_guard<std::mutex> lk(mtx_);
    q_.emplace_back(sid, pub);
    cv_.notify_one();
  }
  // after run(): drain, wait for the copies, rethrow a failure
  void finish() {
    if (thread_.joinable()) {
      {
        std::lock_guard<std::mutex> lk(mtx_);
        done_ = true;
        cv_.notify_one();
      }
      thread_.join();
      GFQ_CUDA(cudaStreamSynchronize(stream_));
      unpacked_.wait();  // the host unpacks of the last blocks
    }
    if (!error_.empty()) throw std::runtime_error("early download: " + error_);
  }
  std::int64_t d2h_bytes() const { return d2h_; }

 private:
  struct Blk {
    int kind;
    std::size_t x, y;
    std::int32_t slot, part;
    std::uint64_t off = 0, rows = 0, cols = 0, poff = 0;
  };
  struct Unpack {
    EarlyDownload* self;
    const std::uint8_t* src;
    std::int64_t ldb, rows, cols;
    std::uint8_t* dst;
  };
  // stream callback once a packed block landed in the staging buffer: the
  // unpack goes to the host pool in row chunks (no CUDA calls here)
  static void CUDART_CB on_landed(void* p) {
    auto* u = static_cast<Unpack*>(p);
    const std::int64_t chunk = 512;
    const std::int64_t n = (u->rows + chunk - 1) / chunk;
    u->self->unpacked_.add(n);
    for (std::int64_t r = 0; r < u->rows; r += chunk) {
      const std::int64_t nr = std::min(chunk, u->rows - r);
      hostpack::submit([u, r, nr] {
        hostpack::unpack_rows(u->src + r * u->ldb, u->ldb, nr, u->cols, u->dst + r * u->cols, u->cols);
        u->self->unpacked_.done();
      });
    }
    u->self->unpacked_.done();  // the block's own count (issue)
  }
  void add(int kind, std::size_t x, std::size_t y, std::int32_t slot, std::int32_t part) {
    by_slot_[slot].push_back(blocks_.size());
    blocks_.push_back(Blk{kind, x, y, slot, part});
    interest_.insert(slot);
  }
  void loop() {
    cudaSetDevice(device_);
    set_cur_stream(stream_);
    try {
      for (;;) {
        std::pair<std::int32_t, std::shared_ptr<Published>> item;
        {
          std::unique_lock<std::mutex> lk(mtx_);
          cv_.wait(lk, [&] { return done_ || !q_.empty(); });
          if (q_.empty()) return;
          item = std::move(q_.front());
          q_.pop_front();
        }
        pubs_[item.first] = item.second;
        if (!layout_) {
          bool all = true;
          for (auto sid : h_.d_final) all = all && pubs_.count(sid);
          for (auto sid : h_.e_final) all = all && pubs_.count(sid);
          if (!all) continue;
          make_layout();
          for (const auto& kv : pubs_) issue(kv.first, *kv.second);
        } else {
          issue(item.first, *item.second);
        }
      }
    } catch (const std::exception& e) {
      error_ = e.what();
    }
  }
  void make_layout() {
    const auto gam = [&](std::size_t j) { return std::get<PkgD>(pubs_[h_.d_final[j]]->value).gamma.size(); };
    const auto rho = [&](std::size_t i) { return std::get<PkgE>(pubs_[h_.e_final[i]]->value).rho.size(); };
    std::uint64_t off = 0, poff = 0;
    for (auto& bk : blocks_) {
      if (bk.kind == 0) {
        bk.rows = gam(bk.x);
        bk.cols = cs_.col_parts[bk.y] - gam(bk.y);
      } else if (bk.kind == 1) {
        bk.rows = gam(bk.x);
        bk.cols = rho(bk.y);
      } else {
        bk.rows = cs_.row_parts[bk.x] - rho(bk.x);
        bk.cols = rho(bk.y);
      }
      bk.off = off;
      off += bk.rows * bk.cols;
      bk.poff = poff;
      poff += bk.rows * ((bk.cols + 63) / 64 * 8);  // 8-byte aligned packed rows
    }
    if (off > cap_) throw std::invalid_argument("host_out buffer too small");
    if (packed_) {
      dstage_ = std::make_unique<DevBuf>(std::size_t(poff));
      hstage_ = std::make_unique<hostpack::PinnedLease>(std::size_t(poff));
    }
    layout_ = true;
  }
  void issue(std::int32_t sid, const Published& pub) {
    auto it = by_slot_.find(sid);
    if (it == by_slot_.end()) return;
    bool waited = false;
    for (std::size_t bi : it->second) {
      const Blk& bk = blocks_[bi];
      if (!bk.rows || !bk.cols) continue;
      const Mat m = bk.part < 0 ? std::get<Mat>(pub.value)
                                : std::get<MatParts>(pub.value).part(std::size_t(bk.part));
      if (std::uint64_t(m.rows()) != bk.rows || std::uint64_t(m.cols()) != bk.cols)
        throw std::logic_error("output block shape disagrees with the layout");
      if (!waited && pub.ready) GFQ_CUDA(cudaStreamWaitEvent(stream_, pub.ready->ev, 0));
      if (!waited && e2e_debug()) {
        // when the block's data was final (a timing event behind the publish event)
        if (!dbg_stream_) GFQ_CUDA(cudaStreamCreateWithFlags(&dbg_stream_, cudaStreamNonBlocking));
        if (pub.ready) GFQ_CUDA(cudaStreamWaitEvent(dbg_stream_, pub.ready->ev, 0));
        cudaEvent_t ev;
        GFQ_CUDA(cudaEventCreate(&ev));
        GFQ_CUDA(cudaEventRecord(ev, dbg_stream_));
        dbg_.emplace_back(std::string("  READY slot ") + std::to_string(sid) + " kind" + std::to_string(bk.kind) +
                              " [" + std::to_string(bk.x) + "][" + std::to_string(bk.y) + "]",
                          ev);
      }
      waited = true;
      if (packed_ && hostpack::packs(n_issued_++)) {
        const std::int64_t ldb = std::int64_t((bk.cols + 63) / 64 * 8);
        const std::int64_t rows = std::int64_t(bk.rows), cols = std::int64_t(bk.cols);
        dev::pack_bits(m.data(), m.ld(), rows, cols, dstage_->ptr + bk.poff, ldb, stream_);
        GFQ_CUDA(cudaMemcpyAsync(hstage_->data() + bk.poff, dstage_->ptr + bk.poff, std::size_t(rows * ldb),
                                 cudaMemcpyDeviceToHost, stream_));
        d2h_ += rows * ldb;
        jobs_.push_back(std::make_unique<Unpack>(Unpack{this, hstage_->data() + bk.poff, ldb, rows, cols,
                                                        host_ + bk.off}));
        unpacked_.add(1);
        GFQ_CUDA(cudaLaunchHostFunc(stream_, &EarlyDownload::on_landed, jobs_.back().get()));
      } else {
        GFQ_CUDA(cudaMemcpy2DAsync(host_ + bk.off, std::size_t(bk.cols), m.data(), std::size_t(m.ld()),
                                   std::size_t(bk.cols), std::size_t(bk.rows), cudaMemcpyDeviceToHost,
                                   stream_));
        d2h_ += std::int64_t(bk.rows * bk.cols);
      }
      if (e2e_debug()) {
        cudaEvent_t ev;
        GFQ_CUDA(cudaEventCreate(&ev));
        GFQ_CUDA(cudaEventRecord(ev, stream_));
        dbg_.emplace_back(std::string("kind") + std::to_string(bk.kind) + " [" + std::to_string(bk.x) + "][" +
                              std::to_string(bk.y) + "] " + std::to_string(bk.rows) + "x" + std::to_string(bk.cols),
                          ev);
      }
    }
  }

  const PlanHandles& h_;
  const ChopSpec& cs_;
  std::uint8_t* host_;
  std::uint64_t cap_;
  bool packed_;
  std::size_t n_issued_ = 0;  // blocks issued so far (hybrid: every N-th goes packed)
  std::unique_ptr<DevBuf> dstage_;
  std::unique_ptr<hostpack::PinnedLease> hstage_;
  std::vector<std::unique_ptr<Unpack>> jobs_;
  hostpack::Latch unpacked_;
  std::int64_t d2h_ = 0;
  std::vector<Blk> blocks_;
  std::unordered_map<std::int32_t, std::vector<std::size_t>> by_slot_;
  std::unordered_set<std::int32_t> interest_;
  std::unordered_map<std::int32_t, std::shared_ptr<Published>> pubs_;
  bool layout_ = false;
  int device_ = 0;
  cudaStream_t stream_ = nullptr;
  std::mutex mtx_;
  std::condition_variable cv_;
  std::deque<std::pair<std::int32_t, std::shared_ptr<Published>>> q_;
  bool done_ = false;
  std::string error_;
  std::thread thread_;
  std::vector<std::pair<std::string, cudaEvent_t>> dbg_;
  cudaStream_t dbg_stream_ = nullptr;
};

EchelonOutput echelonize_impl(const Mat& C, const FieldSpec& field, const EchelonizeOptions& options,
                              RunReport* report,
                              const std::vector<std::shared_ptr<EventBox>>* row_ready);
}  // namespace

void reserve_for(std::size_t m, std::size_t n, bool with_transform) {
  // live high-water ~6.8x the input at cfg5s (input, T, panels in flight,
  // ECH scratch); the block cache's size-class lists hold about 2.5x that
  // in the pool (cfg5s: ~90 GB reserved for a 33 GB live peak): with less
  // reserved, each new size class maps memory (~0.3-1 ms a miss).  Mapping
  // is a one-time cost (cfg5s: ~3.5 s), so callers may pay it up front.
  reserve_pool(10 * m * n + (with_transform ? 10 * m * m : 0));
}

EchelonOutput echelonize(const Mat& C, const FieldSpec& field, const EchelonizeOptions& options,
                         RunReport* report) {
  return echelonize_impl(C, field, options, report, nullptr);
}

EchelonOutput echelonize_host(const std::uint8_t* host, std::int64_t m, std::int64_t n,
                              std::int64_t ld, const FieldSpec& field,
                              const EchelonizeOptions& options, RunReport* report) {
  const auto h0 = std::chrono::steady_clock::now();
  const auto hms = [&h0] {
    return std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - h0).count();
  };
  Mat C(m, n);
  if (e2e_debug()) std::fprintf(stderr, "e2e host: input allocated at %.2f ms\n", hms());
  const ChopSpec cs = chop(std::size_t(m), std::size_t(n), options.block, options.remainder_first);
  if (field.wide())
    throw std::invalid_argument("echelonize_host: wide fields (u32 elements) take a device matrix");
  const bool streamed = options.fuse && !C.empty() && cs.a() > 0 && cs.b() > 0 &&
                        2 * cs.a() + 1 <= std::size_t(TaskNode::kMaxIn);
  if (!streamed) {
    if (!C.empty()) {
      GFQ_CUDA(cudaMemcpy2DAsync(C.data(), std::size_t(C.ld()), host, std::size_t(ld), std::size_t(n),
                                 std::size_t(m), cudaMemcpyHostToDevice, cur_stream()));
    }
    return echelonize_impl(C, field, options, report, nullptr);
  }
  // copy stream ordered after the allocation, one event per block row
  cudaStream_t cs_stream;
  GFQ_CUDA(cudaStreamCreateWithFlags(&cs_stream, cudaStreamNonBlocking));
  std::vector<std::shared_ptr<EventBox>> row_ready;
  // (outside the try: the copy stream and the pool may still use them when
  // an exception unwinds)
  const bool packed = field.p() == 2 && !field.is_ext() && hostpack::enabled();
  const std::int64_t ldb = (n + 63) / 64 * 8;
  std::unique_ptr<hostpack::PinnedLease> stage;
  std::unique_ptr<DevBuf> dpk;
  std::vector<std::unique_ptr<hostpack::Latch>> packed_rows;
  try {
    auto alloc_done = std::make_shared<EventBox>();
    GFQ_CUDA(cudaEventRecord(alloc_done->ev, cur_stream()));
    GFQ_CUDA(cudaStreamWaitEvent(cs_stream, alloc_done->ev, 0));
    std::vector<cudaEvent_t> dbg_rows;
    if (e2e_debug()) {
      if (!g_e2e_t0) GFQ_CUDA(cudaEventCreate(&g_e2e_t0));
      GFQ_CUDA(cudaEventRecord(g_e2e_t0, cs_stream));
    }
    // GF(2): the pool packs each block row to bits in a pinned staging
    // buffer (row order, so block row 0 is ready first); the copy stream
    // waits for a block row's packing (a host function blocking the stream),
    // copies an eighth of the bytes and unpacks them in HBM
    if (packed) {
      stage = std::make_unique<hostpack::PinnedLease>(std::size_t(m * ldb));
      dpk = std::make_unique<DevBuf>(std::size_t(m * ldb));
      const std::int64_t chunk = 256;
      for (std::size_t i = 0; i < cs.a(); ++i) {
        const std::int64_t nr = std::int64_t(cs.row_parts[i]);
        packed_rows.push_back(std::make_unique<hostpack::Latch>((nr + chunk - 1) / chunk));
      }
      for (std::size_t i = 0; i < cs.a(); ++i) {
        if (!hostpack::packs(i)) continue;
        const std::int64_t r0 = std::int64_t(cs.row_offset(i)), nr = std::int64_t(cs.row_parts[i]);
        hostpack::Latch* l = packed_rows[i].get();
        std::uint8_t* st = stage->data();
        for (std::int64_t r = 0; r < nr; r += chunk) {
          const std::int64_t k = std::min(chunk, nr - r);
          hostpack::submit([=] {
            hostpack::pack_rows(host + (r0 + r) * ld, ld, k, n, st + (r0 + r) * ldb, ldb);
            l->done();
          });
        }
      }
      std::int64_t bytes = 0;
      for (std::size_t i = 0; i < cs.a(); ++i)
        bytes += std::int64_t(cs.row_parts[i]) * (hostpack::packs(i) ? ldb : n);
      hostpack::last_transfer().h2d = bytes;
    } else {
      hostpack::last_transfer().h2d = m * n;
    }
    for (std::size_t i = 0; i < cs.a(); ++i) {
      const std::int64_t r0 = std::int64_t(cs.row_offset(i)), nr = std::int64_t(cs.row_parts[i]);
      if (packed && hostpack::packs(i)) {
        GFQ_CUDA(cudaLaunchHostFunc(
            cs_stream, [](void* p) { static_cast<hostpack::Latch*>(p)->wait(); }, packed_rows[i].get()));
        GFQ_CUDA(cudaMemcpyAsync(dpk->ptr + r0 * ldb, stage->data() + r0 * ldb, std::size_t(nr * ldb),
                                 cudaMemcpyHostToDevice, cs_stream));
        dev::unpack_bits(dpk->ptr + r0 * ldb, ldb, nr, n, C.data() + r0 * C.ld(), C.ld(), cs_stream);
        auto ev0 = std::make_shared<EventBox>();
        GFQ_CUDA(cudaEventRecord(ev0->ev, cs_stream));
        row_ready.push_back(ev0);
      } else {
        // block column 0 first: the row's ClearDown(i, 0) -- for i = 0 the
        // first diagonal ECH -- starts while the rest of the row is in flight
        const std::int64_t c0 = cs.b() > 1 ? std::int64_t(cs.col_parts[0]) : n;
        GFQ_CUDA(cudaMemcpy2DAsync(C.data() + r0 * C.ld(), std::size_t(C.ld()), host + r0 * ld,
                                   std::size_t(ld), std::size_t(c0), std::size_t(nr),
                                   cudaMemcpyHostToDevice, cs_stream));
        auto ev0 = std::make_shared<EventBox>();
        GFQ_CUDA(cudaEventRecord(ev0->ev, cs_stream));
        row_ready.push_back(std::move(ev0));
        if (c0 < n)
          GFQ_CUDA(cudaMemcpy2DAsync(C.data() + r0 * C.ld() + c0, std::size_t(C.ld()),
                                     host + r0 * ld + c0, std::size_t(ld), std::size_t(n - c0),
                                     std::size_t(nr), cudaMemcpyHostToDevice, cs_stream));
      }
      auto ev = std::make_shared<EventBox>();
      GFQ_CUDA(cudaEventRecord(ev->ev, cs_stream));
      row_ready.push_back(std::move(ev));
      if (e2e_debug()) {
        cudaEvent_t t;
        GFQ_CUDA(cudaEventCreate(&t));
        GFQ_CUDA(cudaEventRecord(t, cs_stream));
        dbg_rows.push_back(t);
      }
    }
    if (e2e_debug()) std::fprintf(stderr, "e2e host: uploads enqueued at %.2f ms\n", hms());
    EchelonOutput out = echelonize_impl(C, field, options, report, &row_ready);
    if (e2e_debug()) std::fprintf(stderr, "e2e host: run + downloads done at %.2f ms\n", hms());
    GFQ_CUDA(cudaStreamSynchronize(cs_stream));  // the host buffer may be reused on return
    if (e2e_debug()) std::fprintf(stderr, "e2e host: upload stream synchronized at %.2f ms\n", hms());
    for (std::size_t i = 0; i < dbg_rows.size(); ++i) {
      float ms = 0;
      GFQ_CUDA(cudaEventElapsedTime(&ms, g_e2e_t0, dbg_rows[i]));
      std::fprintf(stderr, "e2e upload row %zu landed at %.2f ms\n", i, double(ms));
      cudaEventDestroy(dbg_rows[i]);
    }
    cudaStreamDestroy(cs_stream);
    if (e2e_debug()) std::fprintf(stderr, "e2e host: return at %.2f ms\n", hms());
    return out;
  } catch (...) {
    for (std::size_t i = 0; i < packed_rows.size(); ++i)
      if (hostpack::packs(i)) packed_rows[i]->wait();
    cudaStreamSynchronize(cs_stream);
    cudaStreamDestroy(cs_stream);
    throw;
  }
}

namespace {
EchelonOutput echelonize_impl(const Mat& C, const FieldSpec& field, const EchelonizeOptions& options,
                              RunReport* report,
                              const std::vector<std::shared_ptr<EventBox>>* row_ready) {
  const ChopSpec cs = chop(std::size_t(C.rows()), std::size_t(C.cols()), options.block,
                           options.remainder_first);
  const std::size_t a = cs.a(), b = cs.b();
  EchelonOutput out{field};
  out.chop = cs;
  out.with_transform = options.with_transform;
  if (a == 0 || b == 0) {
    // reference src/chief.cpp:289-320 (empty_output)
    if (report) *report = RunReport{};
    for (std::size_t j = 0; j < b; ++j) out.upsilon.emplace_back(cs.col_parts[j], std::vector<std::uint32_t>{});
    for (std::size_t i = 0; i < a; ++i) out.varrho.emplace_back(cs.row_parts[i], std::vector<std::uint32_t>{});
    out.R_blocks.assign(b, std::vector<Mat>(b));
    for (std::size_t j = 0; j < b; ++j)
      for (std::size_t l = j; l < b; ++l) out.R_blocks[j][l] = Mat(0, std::int64_t(cs.col_parts[l]), field.esize());
    if (options.with_transform) {
      out.T_M_blocks.assign(b, std::vector<Mat>(a));
      out.T_K_blocks.resize(a);
      for (std::size_t i = 0; i < a; ++i)
        for (std::size_t h = 0; h <= i; ++h)
          out.T_K_blocks[i].push_back(Mat(std::int64_t(cs.row_parts[i]), 0, field.esize()));
    }
    return out;
  }

  // the run's working set (input-sized panels, the transformation, ECH
  // scratch) in one pool growth step, not hundreds of cache misses
  reserve_for(std::size_t(C.rows()), std::size_t(C.cols()), options.with_transform);
  TaskGraph graph;
  graph.ech_threshold = options.ech_threshold;
  // wide fields (u32 storage) run the reference's per-block task grid
  const bool fused = options.fuse && !field.wide() && 2 * a + 1 <= std::size_t(TaskNode::kMaxIn);
  // the critical-path SM partition pays off once blocks are large
  // (kernels.hpp set_critical_partition); GFQ_PARTITION=0/1 forces it
  {
    static const int forced = [] {
      const char* e = std::getenv("GFQ_PARTITION");
      return e ? std::atoi(e) : -1;
    }();
    dev::set_critical_partition(forced >= 0 ? forced != 0 : (fused && options.block >= 4096));
  }
  const PlanHandles h = fused ? build_plan_fused(graph, C, field, cs, options.with_transform, row_ready)
                              : build_plan(graph, C, field, cs, options.with_transform);
  for (auto id : h.d_final) graph.retain(id);
  for (auto id : h.e_final) graph.retain(id);
  for (const auto& row : h.r_final)
    for (auto id : row)
      if (id >= 0) graph.retain(id);
  for (const auto& row : h.m_final)
    for (auto id : row) graph.retain(id);
  for (const auto& row : h.k_final)
    for (auto id : row) graph.retain(id);

  RunOptions ro;
  ro.workers = options.threads;
  ro.collect_trace = options.collect_trace;
  ro.retain_all = options.retain_all;
  std::unique_ptr<EarlyDownload> early;
  if (options.host_out) {
    early = std::make_unique<EarlyDownload>(h, cs, options.with_transform, options.host_out,
                                            options.host_out_cap,
                                            field.p() == 2 && !field.is_ext() && hostpack::enabled());
    ro.on_publish = [&early](std::int32_t sid, const std::shared_ptr<Published>& pub) {
      early->publish(sid, pub);
    };
  }
  RunReport rep = run(graph, ro);
  if (early) {
    early->finish();
    hostpack::last_transfer().d2h = early->d2h_bytes();
  }
  if (report) *report = std::move(rep);

  for (std::size_t j = 0; j < b; ++j) {
    const PkgD& d = std::get<PkgD>(*graph.payload(h.d_final[j]));
    out.rank += d.gamma.size();
    out.upsilon.push_back(d.gamma);
  }
  for (std::size_t i = 0; i < a; ++i)
    out.varrho.push_back(std::get<PkgE>(*graph.payload(h.e_final[i])).rho);
  out.R_blocks.assign(b, std::vector<Mat>(b));
  const auto value_of = [&](std::int32_t slot, std::int32_t part) {
    const PackageValue& v = *graph.payload(slot);
    return part < 0 ? std::get<Mat>(v) : std::get<MatParts>(v).part(std::size_t(part));
  };
  for (std::size_t j = 0; j < b; ++j)
    for (std::size_t l = j; l < b; ++l)
      out.R_blocks[j][l] = value_of(h.r_final[j][l], h.r_part.empty() ? -1 : h.r_part[j][l]);
  if (options.with_transform) {
    out.T_M_blocks.assign(b, std::vector<Mat>(a));
    for (std::size_t j = 0; j < b; ++j)
      for (std::size_t hh = 0; hh < a; ++hh)
        out.T_M_blocks[j][hh] = value_of(h.m_final[j][hh], h.m_part.empty() ? -1 : h.m_part[j][hh]);
    out.T_K_blocks.resize(a);
    for (std::size_t i = 0; i < a; ++i)
      for (std::size_t hh = 0; hh <= i; ++hh)
        out.T_K_blocks[i].push_back(value_of(h.k_final[i][hh], h.k_part.empty() ? -1 : h.k_part[i][hh]));
  }
  return out;
}

}  // namespace

// ---------------------------------------------------------------- assembly
std::vector<std::uint32_t> EchelonOutput::global_upsilon() const {
  std::vector<std::uint32_t> v;
  for (std::size_t j = 0; j < upsilon.size(); ++j)
    for (auto x : upsilon[j].members) v.push_back(std::uint32_t(chop.col_offset(j) + x));
  return v;
}

std::vector<std::uint32_t> EchelonOutput::global_varrho() const {
  std::vector<std::uint32_t> v;
  for (std::size_t i = 0; i < varrho.size(); ++i)
    for (auto x : varrho[i].members) v.push_back(std::uint32_t(chop.row_offset(i) + x));
  return v;
}

// reference src/chief.cpp:408-425, as device-to-device block copies.
Mat EchelonOutput::assembled_R() const {
  const std::int64_t n = std::int64_t(chop.cols());
  const int es = field.esize();
  Mat out = Mat::zeros(std::int64_t(rank), n - std::int64_t(rank), es);
  if (out.empty()) return out;
  std::int64_t row = 0;
  for (std::size_t j = 0; j < upsilon.size(); ++j) {
    std::int64_t col = 0;
    for (std::size_t l = 0; l < upsilon.size(); ++l) {
      const std::int64_t width = std::int64_t(chop.col_parts[l] - upsilon[l].size());
      if (l >= j && width > 0 && upsilon[j].size() > 0) {
        const Mat& blk = R_blocks[j][l];
        GFQ_CUDA(cudaMemcpy2DAsync(out.data() + row * out.ld() + col * es, std::size_t(out.ld()),
                                   blk.data(), std::size_t(blk.ld()), std::size_t(width * es),
                                   std::size_t(blk.rows()), cudaMemcpyDeviceToDevice,
                                   cur_stream()));
      }
      col += width;
    }
    row += std::int64_t(upsilon[j].size());
  }
  return out;
}

// reference src/chief.cpp:489-520: T rows = pivot rows by (j, q), then
// non-pivot rows by block row; columns = original rows.  Built as column
// scatters of the M / K blocks into zero-initialised stripes.
Mat materialize_transform(const EchelonOutput& out) {
  if (!out.with_transform) throw std::logic_error("transformation was not computed");
  const std::int64_t m = std::int64_t(out.chop.rows());
  const std::size_t a = out.chop.a(), b = out.chop.b();
  const int es = out.field.esize();
  Mat t = Mat::zeros(m, m, es);
  if (t.empty()) return t;
  // per block row h: column map of its stripe (selected row -> position),
  // byte-level for wide elements
  std::vector<std::shared_ptr<DevBuf>> cmaps(a);
  for (std::size_t h = 0; h < a; ++h) {
    std::vector<std::int32_t> map(out.chop.row_parts[h] * std::size_t(es), -1);
    for (std::size_t s = 0; s < out.varrho[h].size(); ++s)
      for (int q = 0; q < es; ++q)
        map[std::size_t(out.varrho[h].members[s]) * std::size_t(es) + std::size_t(q)] =
            std::int32_t(s) * es + q;
    cmaps[h] = upload_i32(map);
  }
  std::int64_t row = 0;
  for (std::size_t j = 0; j < b; ++j) {
    const std::int64_t nr = std::int64_t(out.upsilon[j].size());
    for (std::size_t h = 0; h < a && nr > 0; ++h) {
      const Mat& mjh = out.T_M_blocks[j][h];
      if (out.varrho[h].size() == 0) continue;
      dev::select2d(t.data() + row * t.ld() + std::int64_t(out.chop.row_offset(h)) * es, t.ld(), nr,
                    std::int64_t(out.chop.row_parts[h]) * es, mjh.data(), mjh.ld(), nullptr, 0,
                    nullptr, reinterpret_cast<const std::int32_t*>(cmaps[h]->ptr), cur_stream());
    }
    row += nr;
  }
  std::vector<std::int32_t> ones;
  for (std::size_t i = 0; i < a; ++i) {
    const IndexSet rest = index_set_complement(out.varrho[i]);
    const std::int64_t nr = std::int64_t(rest.size());
    for (std::size_t h = 0; h <= i && nr > 0; ++h) {
      const Mat& kih = out.T_K_blocks[i][h];
      if (out.varrho[h].size() == 0) continue;
      dev::select2d(t.data() + row * t.ld() + std::int64_t(out.chop.row_offset(h)) * es, t.ld(), nr,
                    std::int64_t(out.chop.row_parts[h]) * es, kih.data(), kih.ld(), nullptr, 0,
                    nullptr, reinterpret_cast<const std::int32_t*>(cmaps[h]->ptr), cur_stream());
    }
    // identity at the row's own column (written after the stripe scatter,
    // which puts 0 at non-selected columns)
    for (std::size_t u = 0; u < rest.size(); ++u) {
      ones.push_back(std::int32_t(row + std::int64_t(u)));
      ones.push_back(std::int32_t(out.chop.row_offset(i) + rest.members[u]));
    }
    row += nr;
  }
  if (!ones.empty()) {
    auto pb = upload_i32(ones);
    if (es == 4)
      dev::set_entries_u32(t.data(), t.ld(), reinterpret_cast<const std::int32_t*>(pb->ptr),
                           std::int64_t(ones.size() / 2), 1, cur_stream());
    else
      dev::set_entries(t.data(), t.ld(), reinterpret_cast<const std::int32_t*>(pb->ptr),
                       std::int64_t(ones.size() / 2), 1, cur_stream());
  }
  return t;
}

}  // namespace gfq
