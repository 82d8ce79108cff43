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
cudaStream_t cur_stream();
void set_cur_stream(cudaStream_t s);

/// Number of SMs of the current device (cached).
int sm_count();

inline std::int64_t round_up(std::int64_t v, std::int64_t m) {
  return (v + m - 1) / m * m;
}

}  // namespace gfq
