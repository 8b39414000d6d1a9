// Status/error plumbing for the C ABI (codes in include/salr_b200.h).
#pragma once
#include <cstdarg>
#include <cstdio>
#include <cuda_runtime.h>

#include "../../include/salr_b200.h"

namespace salr {

int set_error(int code, const char* fmt, ...);

#define SALR_CHECK_ARG(cond, code, ...)            \
  do {                                             \
    if (!(cond)) return ::salr::set_error(code, __VA_ARGS__); \
  } while (0)

#define SALR_CUDA_TRY(expr)                                                              \
  do {                                                                                   \
    cudaError_t _e = (expr);                                                             \
    if (_e != cudaSuccess)                                                               \
      return ::salr::set_error(SALR_ERR_CUDA, "%s: %s", #expr, cudaGetErrorString(_e));  \
  } while (0)

#define SALR_LAUNCH_CHECK()                                                                     \
  do {                                                                                          \
    cudaError_t _e = cudaGetLastError();                                                        \
    if (_e != cudaSuccess)                                                                      \
      return ::salr::set_error(SALR_ERR_CUDA, "kernel launch: %s", cudaGetErrorString(_e));     \
  } while (0)

}  // namespace salr
