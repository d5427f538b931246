// Shared device helpers for the pmedian_b200 kernels (sm_100a only).
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>
#include <stdio.h>

#ifndef __CUDACC__
#error "common.cuh is CUDA-only"
#endif

namespace pmb {

constexpr unsigned kFull = 0xffffffffu;

// Device bounds checks for the `make bounds` build (-DPMB_BOUNDS): an index
// outside its buffer prints the kernel's source line and traps, so a bad
// access surfaces as a CUDA error instead of a wrong cost.  (compute-sanitizer
// is not available on the GPU pool; tools/bounds_check.py drives this build.)
// The release build compiles every check away.
#ifdef PMB_BOUNDS
#define PMB_CHECK(cond)                                                                             \
  do {                                                                                              \
    if (!(cond)) {                                                                                  \
      printf("PMB_CHECK failed %s:%d: %s (block %d thread %d)\n", __FILE__, __LINE__, #cond,        \
             (int)blockIdx.x, (int)threadIdx.x);                                                    \
      __trap();                                                                                     \
    }                                                                                               \
  } while (0)
#else
#define PMB_CHECK(cond) \
  do {                  \
  } while (0)
#endif

__device__ __forceinline__ unsigned lane_id() { return threadIdx.x & 31; }
__device__ __forceinline__ unsigned lanemask_lt() {
  unsigned r;
  asm volatile("mov.u32 %0, %%lanemask_lt;" : "=r"(r));
  return r;
}

// 16-byte read-only global load that does not allocate in L1: every byte of
// Pi'/D' a lane streams is used once by that lane (row prefixes are reused
// across CTAs through L2, not through L1).
__device__ __forceinline__ uint4 ldg_stream(const void* p) {
  uint4 r;
  asm("ld.global.nc.L1::no_allocate.v4.u32 {%0,%1,%2,%3}, [%4];"
               : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w)
               : "l"(p));
  return r;
}

// 32-byte variant (sm_100: LDG.E.256); p must be 32-byte aligned.
__device__ __forceinline__ void ldg_stream32(const void* p, uint4& lo, uint4& hi) {
  asm("ld.global.nc.L1::no_allocate.v8.u32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
               : "=r"(lo.x), "=r"(lo.y), "=r"(lo.z), "=r"(lo.w), "=r"(hi.x), "=r"(hi.y), "=r"(hi.z),
                 "=r"(hi.w)
               : "l"(p));
}

template <class T>
__device__ __forceinline__ T warp_sum(T v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(kFull, v, o);
  return v;
}

}  // namespace pmb
