// Shared helpers for the TT B200 library: status codes, error capture, launch
// accounting.  No exception crosses the C ABI: every extern "C" entry point is
// wrapped in TTB_TRY_BEGIN / TTB_TRY_END and returns an int status, with the
// message retrievable through ttb_last_error().
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include <cstdio>
#include <stdexcept>
#include <string>

#include "../../include/ttb.h"

namespace ttb {

struct Error : public std::runtime_error {
  int code;
  Error(int c, const std::string& m) : std::runtime_error(m), code(c) {}
};

void set_last_error(const std::string& msg);
void count_launch(int n = 1);
// raise a kernel's dynamic shared-memory limit on the CURRENT device, once per
// (kernel, device, size): the attribute is per device, and the bookkeeping is
// shared by every context / host thread of the process (mutex-guarded)
void smem_attr(const void* fn, size_t bytes);

#define TTB_THROW(code, msg) throw ::ttb::Error((code), (msg))

#define TTB_CHECK(cond, code, msg)          \
  do {                                      \
    if (!(cond)) TTB_THROW((code), (msg));  \
  } while (0)

#define TTB_CUDA(call)                                                            \
  do {                                                                            \
    cudaError_t _e = (call);                                                      \
    if (_e != cudaSuccess)                                                        \
      TTB_THROW(TTB_ERR_CUDA, std::string(#call " failed: ") + cudaGetErrorString(_e)); \
  } while (0)

#define TTB_LAUNCHED()                                                            \
  do {                                                                            \
    cudaError_t _e = cudaGetLastError();                                          \
    if (_e != cudaSuccess)                                                        \
      TTB_THROW(TTB_ERR_CUDA, std::string("kernel launch failed (") + __FILE__ + ":" + std::to_string(__LINE__) + \
                                  "): " + cudaGetErrorString(_e));                                      \
    ::ttb::count_launch();                                                        \
  } while (0)

#define TTB_TRY_BEGIN try {
#define TTB_TRY_END                                      \
  }                                                      \
  catch (const ::ttb::Error& e) {                        \
    ::ttb::set_last_error(e.what());                     \
    return e.code;                                       \
  }                                                      \
  catch (const std::exception& e) {                      \
    ::ttb::set_last_error(e.what());                     \
    return TTB_ERR_CUDA;                                 \
  }                                                      \
  return TTB_OK;

inline int ceil_div(int64_t a, int64_t b) { return (int)((a + b - 1) / b); }
__host__ __device__ __forceinline__ int64_t min64(int64_t a, int64_t b) { return a < b ? a : b; }
__host__ __device__ __forceinline__ int64_t max64(int64_t a, int64_t b) { return a > b ? a : b; }

}  // namespace ttb
