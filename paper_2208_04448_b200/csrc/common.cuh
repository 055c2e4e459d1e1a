// Host-side helpers shared by the C-ABI translation units: thread-local error
// reporting and CUDA error checks.  No C++ exception crosses the ABI.
#pragma once
#include <cuda_runtime.h>

#include <atomic>
#include <cstdarg>
#include <cstdio>
#include <string>

#include "../../include/nvdb_b200.h"

namespace nvdb {

inline std::string& last_error_slot() {
  static thread_local std::string msg;
  return msg;
}

inline int fail(int code, const char* fmt, ...) {
  char buf[512];
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(buf, sizeof(buf), fmt, ap);
  va_end(ap);
  last_error_slot() = buf;
  return code;
}

#define NVDB_CUDA_TRY(expr)                                                                          \
  do {                                                                                               \
    cudaError_t _e = (expr);                                                                         \
    if (_e != cudaSuccess)                                                                           \
      return ::nvdb::fail(NVDB_ECUDA, "%s failed: %s (%s:%d)", #expr, cudaGetErrorString(_e), __FILE__, \
                          __LINE__);                                                                 \
  } while (0)

// every kernel launch of this library is followed by NVDB_CHECK_LAUNCH, which
// also counts it (nvdb_launch_count; reported by bench.py as gpu_launches)
inline std::atomic<long long>& launch_counter() {
  static std::atomic<long long> n{0};
  return n;
}

#define NVDB_CHECK_LAUNCH()                                                                 \
  do {                                                                                      \
    ::nvdb::launch_counter().fetch_add(1, std::memory_order_relaxed);                       \
    cudaError_t _e = cudaGetLastError();                                                    \
    if (_e != cudaSuccess)                                                                  \
      return ::nvdb::fail(NVDB_ECUDA, "kernel launch failed: %s (%s:%d)", cudaGetErrorString(_e), \
                          __FILE__, __LINE__);                                              \
  } while (0)

inline int num_sms() {
  static int n = 0;
  if (n == 0) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev);
    if (n <= 0) n = 148;
  }
  return n;
}

inline size_t align_up(size_t v, size_t a) { return (v + a - 1) / a * a; }

// Opt a kernel into the largest dynamic shared memory the device allows and
// return that limit (bytes), or -1 on failure.
template <class K>
inline long long enable_max_smem(K kernel) {
  int dev = 0, optin = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev);
  cudaFuncAttributes fa{};
  if (cudaFuncGetAttributes(&fa, kernel) != cudaSuccess) return -1;
  const long long lim = (long long)optin - (long long)fa.sharedSizeBytes;
  if (cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)lim) != cudaSuccess) return -1;
  return lim;
}

}  // namespace nvdb
