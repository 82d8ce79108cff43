// hostpack.hpp -- the host half of the packed GF(2) transfers of the
// host-buffer entry point (gfq_echelonize_host*): a persistent pool of host
// threads that pack input rows to bits before their upload and unpack
// downloaded output blocks into the caller's byte buffer, and grow-only
// pinned staging buffers for both directions.  Layout as dev::pack_bits
// (kernels/bits.cu): element c of a row at bit c % 8 of byte c / 8.
#pragma once

#include <atomic>
#include <condition_variable>
#include <cstddef>
#include <cstdint>
#include <functional>
#include <mutex>

namespace gfq::hostpack {

// Off by default (GFQ_HOST_PACK=1 / gfq_set_host_pack): it pays only where
// the host's memory bandwidth well exceeds PCIe's -- on the measured B200
// VM (16 cores) packing 4.3 GB and unpacking 4.3 GB ran no faster than the
// byte copies and its threads slowed the executor's launches (e2e 253 vs
// 245 ms).
bool enabled();
void set_enabled(bool on);
// Hybrid transfers (GFQ_HOST_PACK=N / gfq_set_host_pack(N), N >= 2): only
// every N-th input block row and every N-th output block goes packed, the
// others as plain byte copies -- the pool's packing / unpacking of one piece
// then runs while the copy engine moves its neighbours, so the host's memory
// bandwidth and PCIe add up instead of replacing one another.  N = 1 packs
// everything; packs(i) says whether piece i is a packed one.
int stride();
void set_stride(int n);
bool packs(std::size_t index);

void pack_rows(const std::uint8_t* src, std::int64_t ld, std::int64_t rows, std::int64_t cols, std::uint8_t* dst,
               std::int64_t ldb);
void unpack_rows(const std::uint8_t* src, std::int64_t ldb, std::int64_t rows, std::int64_t cols, std::uint8_t* dst,
                 std::int64_t ld);

// A count of outstanding pool jobs that can be waited for.
class Latch {
 public:
  explicit Latch(std::int64_t n = 0) : n_(n) {}
  void add(std::int64_t k);
  void done();
  void wait();

 private:
  std::mutex m_;
  std::condition_variable cv_;
  std::int64_t n_;
};

// Run fn on a pool thread (GFQ_HOST_THREADS, default min(8, cores / 2)).
void submit(std::function<void()> fn);
int pool_threads();

// An exclusively held pinned host buffer of at least `bytes`; buffers go
// back to a process-wide free list (cudaHostAlloc of 0.5 GB costs ~0.1 s,
// so a run reuses the previous run's).
class PinnedLease {
 public:
  explicit PinnedLease(std::size_t bytes);
  ~PinnedLease();
  PinnedLease(const PinnedLease&) = delete;
  PinnedLease& operator=(const PinnedLease&) = delete;
  std::uint8_t* data() const { return p_; }

 private:
  std::uint8_t* p_ = nullptr;
  std::size_t cap_ = 0;
};

// bytes that crossed PCIe in the calling thread's last host-buffer run
struct TransferBytes {
  std::int64_t h2d = 0, d2h = 0;
};
TransferBytes& last_transfer();

}  // namespace gfq::hostpack
