// Device-side bounds checks for the checked build (NKB_CHECKED, built as
// lib/libnekb200_checked.so by build(checked=True)).  compute-sanitizer is
// closed on the GPU pool, so the hot kernels check their own shared- and
// global-memory indices instead: a failed check counts into a per-file
// device word (first failing line kept) and SKIPS nothing -- the access is
// still made -- so the checked build computes exactly what the product
// build computes; nkb_execute fails with NKB_ECUDA naming file:line when a
// count is non-zero.  In the product build every NKB_DCHECK is empty.
#pragma once

#include <cuda_runtime.h>

#ifdef NKB_CHECKED
namespace nkb {
namespace {
__device__ unsigned long long g_chk_count;
__device__ int g_chk_line;
}  // namespace
}  // namespace nkb
#define NKB_DCHECK(cond)                                   \
  do {                                                     \
    if (!(cond)) {                                         \
      if (atomicAdd(&::nkb::g_chk_count, 1ULL) == 0ULL)    \
        ::nkb::g_chk_line = __LINE__;                      \
    }                                                      \
  } while (0)
// host: read and clear this file's violation count (and first failing line)
#define NKB_CHECKED_ACCESSOR(fn)                                                          \
  unsigned long long fn(int* line) {                                                      \
    unsigned long long c = 0, z = 0;                                                      \
    int l = 0;                                                                            \
    cudaMemcpyFromSymbol(&c, ::nkb::g_chk_count, sizeof(c));                              \
    cudaMemcpyFromSymbol(&l, ::nkb::g_chk_line, sizeof(l));                               \
    cudaMemcpyToSymbol(::nkb::g_chk_count, &z, sizeof(z));                                \
    if (line) *line = l;                                                                  \
    return c;                                                                             \
  }
#else
#define NKB_DCHECK(cond) \
  do {                   \
  } while (0)
#define NKB_CHECKED_ACCESSOR(fn) \
  unsigned long long fn(int* line) { \
    if (line) *line = 0;             \
    return 0;                        \
  }
#endif
