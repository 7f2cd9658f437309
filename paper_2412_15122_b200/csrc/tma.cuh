// tma.cuh — bulk-copy (TMA) row rings for the O(n^2) streaming kernels.
//
// A warp streams the rows of its (column chunk, row slab) task through a ring
// of S stages x R rows x CB bytes in shared memory.  One lane issues every
// copy with cp.async.bulk (SASS UBLKCP: the TMA engine moves the bytes, no
// register or issue slot of the warp is spent per 16 bytes) and arms the
// stage's mbarrier with the expected byte count; the warp then waits on the
// barrier's phase bit and reads the rows from shared memory.  The stage being
// refilled was consumed by the same warp one iteration earlier: a __syncwarp
// plus a generic->async proxy fence order those reads before the refill.
#pragma once
#include <cuda.h>   // CUtensorMap (the type only; maps are encoded on the host)
#include <stdint.h>

#include "common.cuh"

namespace apsp {

__device__ __forceinline__ void mbar_init(uint64_t* bar, unsigned count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}
// barrier inits (and prior generic smem writes) visible to the async proxy
__device__ __forceinline__ void fence_barrier_init() {
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}
__device__ __forceinline__ void fence_proxy_async() {
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, unsigned bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes)
               : "memory");
}
// global -> shared bulk copy of `bytes` (multiple of 16, both addresses
// 16-byte aligned), completion counted on `bar`
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, unsigned bytes, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
          smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(smem_u32(bar))
      : "memory");
}
// the same with an L2 eviction hint: the row is read once (evict_first)
__device__ __forceinline__ void bulk_g2s_stream(void* dst, const void* src, unsigned bytes, uint64_t* bar,
                                                uint64_t policy) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1], %2, [%3], "
      "%4;" ::"r"(smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(smem_u32(bar)), "l"(policy)
      : "memory");
}
// 2-D tiled tensor copy: the box at (c0, c1) of the tensor `map` describes
// -> shared memory, completion counted on `bar` (SASS UTMALDG)
__device__ __forceinline__ void tensor2d_g2s(void* dst, const CUtensorMap* map, int c0, int c1, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];" ::"r"(
          smem_u32(dst)),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(c0), "r"(c1), "r"(smem_u32(bar))
      : "memory");
}
// L2 prefetch of the box at (c0, c1) (no shared memory, no barrier): a later
// tensor2d_g2s of the same box then hits L2
__device__ __forceinline__ void tensor2d_prefetch_l2(const CUtensorMap* map, int c0, int c1) {
  asm volatile("cp.async.bulk.prefetch.tensor.2d.L2.global.tile [%0, {%1, %2}];" ::"l"(
                   reinterpret_cast<uint64_t>(map)),
               "r"(c0), "r"(c1)
               : "memory");
}
__device__ __forceinline__ uint64_t policy_evict_first() {
  uint64_t p;
  asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(p));
  return p;
}
__device__ __forceinline__ bool mbar_try_wait(uint64_t* bar, unsigned parity) {
  unsigned ok;
  asm volatile(
      "{\n"
      ".reg .pred p;\n"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n"
      "selp.u32 %0, 1, 0, p;\n"
      "}\n"
      : "=r"(ok)
      : "r"(smem_u32(bar)), "r"(parity)
      : "memory");
  return ok != 0;
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, unsigned parity) {
  while (!mbar_try_wait(bar, parity)) {
  }
}

// Per-warp ring: S stages of R rows of CB bytes, plus S mbarriers.
// Shared-memory bytes per warp: ring_bytes<S, R, CB>().
template <int S, int R, int CB>
struct WarpRing {
  static constexpr int kStageBytes = R * CB;
  // per-warp footprint, rounded to 128 bytes so that every warp's ring (and
  // each row in it) stays 16-byte aligned for the bulk copies
  static constexpr int kBytes = (S * kStageBytes + S * 8 + 127) / 128 * 128;
  uint8_t* buf;    // S * R * CB bytes, 128-byte aligned
  uint64_t* bar;   // S barriers (after the data)

  __device__ __forceinline__ void init(uint8_t* base, int lane) {
    buf = base;
    bar = reinterpret_cast<uint64_t*>(base + S * kStageBytes);
    if (lane == 0) {
#pragma unroll
      for (int s = 0; s < S; ++s) mbar_init(bar + s, 1);
      fence_barrier_init();
    }
    __syncwarp();
  }
  __device__ __forceinline__ uint8_t* row(int stage, int h) const {
    return buf + (stage % S) * kStageBytes + h * CB;
  }
  // lane 0: refill stage `stage` with rows src(h), h < R, `bytes` each.  The
  // caller's lanes finished reading the slot (the last use of it) before.
  template <typename Src, bool kFence = true>
  __device__ __forceinline__ void issue(int stage, unsigned bytes, int lane, Src src) {
    __syncwarp();
    if (lane == 0) {
      if (kFence) fence_proxy_async();
      uint64_t* b = bar + stage % S;
      mbar_expect_tx(b, R * bytes);
#pragma unroll
      for (int h = 0; h < R; ++h) bulk_g2s(row(stage, h), src(h), bytes, b);
    }
  }
  // lane 0: refill stage `stage` with one 2-D tensor box (R rows of CB bytes).
  // kFence = false: no generic->async proxy fence — for a caller whose last
  // reads of the slot fed a warp vote before this call (the values were in
  // registers, so the reads are complete before the copy can land)
  template <bool kFence = true>
  __device__ __forceinline__ void issue_box(int stage, const CUtensorMap* map, int c0, int c1, int lane) {
    __syncwarp();
    if (lane == 0) {
      if (kFence) fence_proxy_async();
      uint64_t* b = bar + stage % S;
      mbar_expect_tx(b, R * CB);
      tensor2d_g2s(row(stage, 0), map, c0, c1, b);
    }
  }
  __device__ __forceinline__ void wait(int stage) const { mbar_wait(bar + stage % S, (unsigned)(stage / S) & 1u); }
};

__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}

// CTA-wide ring: the CTA's warps cover adjacent column chunks of the SAME
// rows, so one bulk copy of CB bytes per row feeds all of them (a larger copy
// per TMA operation than a per-warp ring of one warp's chunk).  One thread
// produces; every warp consumes each stage and releases it through the
// stage's `empty` barrier (one arrival per warp), which the producer waits on
// before refilling the slot (the ordering the release/acquire pair gives; no
// proxy fence is needed for reads followed by an async-proxy refill).
template <int S, int CB>
struct CtaRing {
  static constexpr int kBytes = (S * CB + 2 * S * 8 + 127) / 128 * 128;
  uint8_t* buf;
  uint64_t* full;
  uint64_t* empty;
  // every thread of the CTA calls this (it ends with __syncthreads)
  __device__ __forceinline__ void init(uint8_t* base, int nwarps) {
    buf = base;
    full = reinterpret_cast<uint64_t*>(base + S * CB);
    empty = full + S;
    if (threadIdx.x == 0) {
#pragma unroll
      for (int s = 0; s < S; ++s) {
        mbar_init(full + s, 1);
        mbar_init(empty + s, nwarps);
      }
      fence_barrier_init();
    }
    __syncthreads();
  }
  __device__ __forceinline__ const uint8_t* row(int stage) const { return buf + (stage % S) * CB; }
  // the producer thread only: stage `stage` := `bytes` from src
  __device__ __forceinline__ void produce(int stage, const void* src, unsigned bytes) {
    const int s = stage % S;
    if (stage >= S) mbar_wait(empty + s, (unsigned)(stage / S - 1) & 1u);
    mbar_expect_tx(full + s, bytes);
    bulk_g2s(buf + s * CB, src, bytes, full + s);
  }
  __device__ __forceinline__ void wait(int stage) const { mbar_wait(full + stage % S, (unsigned)(stage / S) & 1u); }
  // every warp, after its last read of the stage
  __device__ __forceinline__ void release(int stage, int lane) {
    __syncwarp();
    if (lane == 0) mbar_arrive(empty + stage % S);
  }
};

}  // namespace apsp
