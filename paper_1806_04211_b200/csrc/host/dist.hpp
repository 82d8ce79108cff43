// dist.hpp -- the block-column sharded Chief over several B200s.
//
// Ownership: block column k of C and transform block column h (= original
// block row h) live on rank k % world / h % world.  Every task runs on the
// owner of the column it writes:
//   ClearDown(i,j), Copy(j)              -> owner of column j
//   UpdateRow(i,j,k), PreClearUp(j,k)    -> owner of column k
//   ClearUp-R(k; j, l)                   -> owner of column l
//   UpdateRowTrafo(i,j,h), RowLengthen(j,h), ClearUp-M(k; j, h) -> owner of T column h
//   Extend(i,j)                          -> every rank (host-only index merge)
// The only packages that cross ranks are PkgA(i,j) (root: owner of column
// j) and X(j,k) (root: owner of column k).  They are broadcast in one fixed
// global order -- A by anti-diagonal i + j then column (the Step-1
// wavefront), then X in Step-3 order -- which is a topological order of the
// plan (A(i,j) depends only on A(i',j') with i' <= i, j' < j; X only on
// Step-1 outputs), so every rank can issue the collectives in the same
// sequence without deadlock.
#pragma once

#include <cstdint>
#include <memory>
#include <vector>

#include "chief.hpp"

namespace gfq {

struct Sharding {
  int world = 1, rank = 0;
  int owner_col(std::size_t k) const { return int(k % std::size_t(world)); }
  int owner_trow(std::size_t h) const { return int(h % std::size_t(world)); }
  /// Rank that executes `nd` (-1: every rank).
  int owner(const TaskNode& nd) const;
};

/// A broadcast communicator over device buffers.  Every rank calls bcast
/// with the same sequence of (bytes, root).
class Comm {
 public:
  virtual ~Comm() = default;
  virtual int rank() const = 0;
  virtual int world() const = 0;
  /// Broadcast `bytes` from `root`'s `buf` into every rank's `buf`, ordered
  /// on `s`.  May block the calling (communication) thread.
  virtual void bcast(void* buf, std::size_t bytes, int root, cudaStream_t s) = 0;
  /// A second, independent channel over the same ranks (every rank calls it
  /// at the same point): its broadcasts order only against each other.
  virtual std::shared_ptr<Comm> split_channel() = 0;
};

/// NCCL communicator (libnccl.so.2 opened at run time).
std::shared_ptr<Comm> make_nccl_comm(int world, int rank, const void* unique_id128);
void nccl_unique_id(void* out128);

/// `world` ranks as threads of one process on the current device: bcast is a
/// device-to-device copy from the root's buffer (no kernels that wait on one
/// another), so the sharded executor can be validated on a single GPU.
std::vector<std::shared_ptr<Comm>> make_loopback_comms(int world);

/// The broadcast schedule of a plan (slot ids in order, with roots).
struct BcastItem {
  std::int32_t slot;
  int root;
  bool is_a;  // PkgA (else X)
  std::size_t i, j, k;
};
std::vector<BcastItem> bcast_schedule(const ChopSpec& cs, const PlanHandles& h, TaskGraph& g,
                                      const Sharding& sh);

/// Sharded echelonize.  Each rank passes either the full device-resident C
/// (only its owned block columns are read) or nullptr and a seed, in which
/// case it generates its owned block columns of random_matrix(p, m, n, seed)
/// with K6.  The returned output is complete on every rank (owned blocks are
/// gathered by broadcast after the run).
EchelonOutput echelonize_dist(const Mat* C, std::int64_t m, std::int64_t n, std::uint64_t seed,
                              const FieldSpec& field, const EchelonizeOptions& options, Comm& comm,
                              RunReport* report = nullptr, bool gather = true);

}  // namespace gfq
