// mirror.cuh — device-side upkeep of the saturated mirror of D (kernels.h:
// struct Mirror), shared by the streaming and the sparse kernels.
#pragma once
#include "common.cuh"
#include "kernels.h"

namespace apsp {

// Mirror flag bits: kMirrorOff — some finite distance is at or above the
// width's saturation value (M is not an exact image of D); kMirrorInf — some
// active entry is INF (readers then need their INF tests).  mput returns the
// bits the write raises; callers OR them per thread and post them once per
// warp (mirror_post).
constexpr unsigned kMirrorOff = 1u, kMirrorInf = 2u;
// the transposed byte of m8[li][j] (no-op without MT)
__device__ __forceinline__ void mput_t(const Mirror& M, int64_t li, int64_t j, uint8_t b) {
  if (M.mt) M.mt[j * M.ldt + li] = b;
}
__device__ __forceinline__ unsigned mput(const Mirror& M, int64_t idx, int32_t v) {
  if (M.m8) {
    const uint8_t b = (uint8_t)min(v, kSat8i);
    M.m8[idx] = b;
    if (M.mt) {
      const int64_t li = idx / M.ld;
      mput_t(M, li, idx - li * M.ld, b);
    }
    return v >= APSP_INF_I32_DEV ? kMirrorInf : (v >= kSat8i ? kMirrorOff : 0u);
  }
  M.m[idx] = sat16(v);
  return v >= APSP_INF_I32_DEV ? kMirrorInf : (v >= kSat16i ? kMirrorOff : 0u);
}
__device__ __forceinline__ unsigned ld_acquire(const unsigned* p) {
  unsigned v;
  asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ bool has_mirror(const Mirror& M) { return M.m != nullptr || M.m8 != nullptr; }
__device__ __forceinline__ unsigned mput(const Mirror&, int64_t, float) { return 0u; }
__device__ __forceinline__ void mirror_post(const Mirror& M, unsigned bits) {
  bits = __reduce_or_sync(0xffffffffu, bits);
  if ((threadIdx.x & 31) == 0 && bits && (bits & ~*(volatile unsigned*)M.flag)) atomicOr(M.flag, bits);
}


}  // namespace apsp
