// common.hpp -- shared plumbing for the B200 GF(p) elimination library.
#pragma once

#include <cuda_runtime.h>

#include <cstdint>
#include <stdexcept>
#include <string>

namespace gfq {

/// A CUDA runtime failure; mapped to status GFQ_ERR_CUDA at the C ABI.
struct CudaError : std::runtime_error {
  using std::runtime_error::runtime_error;
};

[[noreturn]] void throw_cuda(cudaError_t e, const char* what, const char* file,
                             int line);

#define GFQ_CUDA(call)                                                     \
  do {                                                                     \
    cudaError_t _e = (call);                                               \
    if (_e != cudaSuccess) ::gfq::throw_cuda(_e, #call, __FILE__, __LINE__); \
  } while (0)

/// The stream every device job of the calling host thread is ordered on.
/// Set by the executor (one stream per worker) or by gfq_set_stream().
/// The first call after set_pending_waits() enqueues those event waits on
/// the stream first (so a task that never touches the device issues no
/// waits), and every call marks the thread's stream as touched.
cudaStream_t cur_stream();
void set_cur_stream(cudaStream_t s);
/// The stream without flushing waits or marking it touched (allocator).
cudaStream_t cur_stream_raw();
/// Executor hooks: events the next device operation on this thread's
/// stream must wait for (the caller keeps them alive until
/// end_pending_waits()), whether the device was touched since, and the
/// end of the task (unflushed waits are dropped: nothing needed them).
void set_pending_waits(const cudaEvent_t* evs, int n);
bool stream_touched();
void end_pending_waits();

/// Number of SMs of the current device (cached).
int sm_count();

/// Developer host-cost profile (env GFQ_HOSTPROF): wall ns spent in the
/// CUDA API / host work of each category, summed over threads, printed to
/// stderr at exit.
namespace hprof {
enum Slot { kMalloc, kFree, kUpload, kMad, kSelect, kEvent, kMemset, kMiss, kSync, kOtherLaunch, kTask,
            kTaskKind0, kSlots = kTaskKind0 + 12 };
extern const bool on;
void add(Slot s, std::int64_t ns, std::int64_t count = 1);
std::int64_t now();
struct Scope {
  Slot slot;
  std::int64_t t0;
  explicit Scope(Slot s) : slot(s), t0(on ? now() : 0) {}
  ~Scope() {
    if (on) add(slot, now() - t0);
  }
};
// Name of the task the calling thread executes (developer shape logs).
extern thread_local const char* t_task_name;
}  // namespace hprof

inline std::int64_t round_up(std::int64_t v, std::int64_t m) {
  return (v + m - 1) / m * m;
}

}  // namespace gfq
