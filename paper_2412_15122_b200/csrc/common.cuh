// common.cuh — element traits, vector access and launch helpers shared by the
// sm_100a kernels of libapsp_warm.  Distances live in HBM row-major with a
// 128-byte-aligned leading dimension; every streaming kernel moves 16-byte
// vectors (int4 / float4).
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#define APSP_INF_I32_DEV 0x3FFFFFFF

// return a CUDA error from a host launcher
#define CUDA_TRY(x)                           \
  do {                                        \
    cudaError_t _e = (x);                     \
    if (_e != cudaSuccess) return _e;         \
  } while (0)

namespace apsp {

// ---------------------------------------------------------------------------
// Element traits.  int32: INF = 2^30-1, so a sum of two stored values is at
// most 2^31-2 (no overflow) and min(.) keeps every stored value <= INF.
// fp32: INF = +inf (inf + x = inf; weights >= 0, so NaN cannot arise).
// ---------------------------------------------------------------------------
// SR selects the path algebra (§6): 0 = shortest path,
// the (min, +) semiring of the paper's body; 1 = minimax / bottleneck path,
// (min, max) — "The algorithms can be revised to solve the all pairs minimax
// path problem".  Only add/relax/sat/tight differ; 0 stays the identity of
// the path composition in both (weights are >= 0).
template <typename T, int SR = 0> struct Tr;

template <> struct Tr<int32_t, 0> {
  using V4 = int4;
  static constexpr bool kFloat = false;
  __host__ __device__ static __forceinline__ int32_t inf() { return APSP_INF_I32_DEV; }
  __device__ static __forceinline__ int32_t add(int32_t a, int32_t b) { return a + b; }
  __device__ static __forceinline__ int32_t mn(int32_t a, int32_t b) { return min(a, b); }
  // relaxation d = min(d, a + b): one VIADDMNMX on sm_100a
  __device__ static __forceinline__ int32_t relax(int32_t d, int32_t a, int32_t b) {
    return min(d, a + b);
  }
  // clamp a sum of two values back into the storable range
  __device__ static __forceinline__ int32_t sat(int32_t a) { return min(a, APSP_INF_I32_DEV); }
  __device__ static __forceinline__ bool fin(int32_t a) { return a < APSP_INF_I32_DEV; }
  // "lhs == d" of Theorem 4.  lhs >= d always holds for an APSP
  // matrix, so equality is exact for integers.
  __device__ static __forceinline__ bool tight(int32_t lhs, int32_t d, float) { return lhs == d; }
  // order-preserving 32-bit key for argmin (values are >= 0)
  __device__ static __forceinline__ uint32_t key(int32_t a) { return (uint32_t)a; }
  // upper bound v has reached the lower bound lb (so it is final)
  __device__ static __forceinline__ bool at_lb(int32_t v, int32_t lb) { return v <= lb; }
};

template <> struct Tr<float, 0> {
  using V4 = float4;
  static constexpr bool kFloat = true;
  __host__ __device__ static __forceinline__ float inf() { return __builtin_huge_valf(); }
  __device__ static __forceinline__ float add(float a, float b) { return __fadd_rn(a, b); }
  __device__ static __forceinline__ float mn(float a, float b) { return fminf(a, b); }
  __device__ static __forceinline__ float relax(float d, float a, float b) {
    return fminf(d, __fadd_rn(a, b));
  }
  __device__ static __forceinline__ float sat(float a) { return a; }
  __device__ static __forceinline__ bool fin(float a) { return a < __builtin_huge_valf(); }
  // DESIGN.md Q4: flag iff lhs <= d * (1 + tau): ties and near-ties go to
  // "needs update" (a false positive only costs time).
  __device__ static __forceinline__ bool tight(float lhs, float d, float tau) {
    return lhs <= d * (1.0f + tau);
  }
  // non-negative IEEE floats order like their bit patterns
  __device__ static __forceinline__ uint32_t key(float a) { return (uint32_t)__float_as_int(a); }
  // within 2^-21 relative of the lower bound: the true value lies in [lb, v],
  // so stopping here errs by <= 5e-7 relative (fp32 bar 1e-5)
  __device__ static __forceinline__ bool at_lb(float v, float lb) { return v <= lb + lb * 0x1p-21f; }
};

// Packed pair of int16 distances (two adjacent columns per 32-bit word), the
// element of the int16x2 Floyd–Warshall (fw.cu): INF = 0x3FFF in each half, so
// a sum of two stored halves is <= 32766 (no overflow) and
// __viaddmin_s16x2 = VIADDMNMX.S16x2 relaxes both columns in one instruction.
template <> struct Tr<uint32_t, 0> {
  using V4 = uint4;
  static constexpr bool kFloat = false;
  __host__ __device__ static __forceinline__ uint32_t inf() { return 0x3FFF3FFFu; }
  __device__ static __forceinline__ uint32_t relax(uint32_t d, uint32_t a, uint32_t b) {
    return __viaddmin_s16x2(a, b, d);
  }
};

// minimax: a path's cost is its largest edge; max is exact in int32 and fp32
template <typename T> struct Tr<T, 1> : Tr<T, 0> {
  using B = Tr<T, 0>;
  __device__ static __forceinline__ T add(T a, T b) { return a > b ? a : b; }
  __device__ static __forceinline__ T relax(T d, T a, T b) { return B::mn(d, a > b ? a : b); }
  __device__ static __forceinline__ T sat(T a) { return a; }
  __device__ static __forceinline__ bool tight(T lhs, T d, float) { return lhs == d; }
};

// ---------------------------------------------------------------------------
// 16-byte vector helpers
// ---------------------------------------------------------------------------
template <typename T> struct alignas(16) Vec4 { T x, y, z, w; };

template <typename T>
__device__ __forceinline__ Vec4<T> ld4(const T* p) {
  typename Tr<T>::V4 v = *reinterpret_cast<const typename Tr<T>::V4*>(p);
  return Vec4<T>{v.x, v.y, v.z, v.w};
}
// streaming load: bypass L1 allocation (the row is read once)
template <typename T>
__device__ __forceinline__ Vec4<T> ld4_stream(const T* p) {
  int4 r;
  asm volatile("ld.global.nc.L1::no_allocate.v4.s32 {%0,%1,%2,%3}, [%4];"
               : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w)
               : "l"(p));
  Vec4<T> o;
  o.x = *reinterpret_cast<T*>(&r.x);
  o.y = *reinterpret_cast<T*>(&r.y);
  o.z = *reinterpret_cast<T*>(&r.z);
  o.w = *reinterpret_cast<T*>(&r.w);
  return o;
}
// coherent (non-.nc) 16-byte load for data this kernel may also write
template <typename T>
__device__ __forceinline__ Vec4<T> ld4_cg(const T* p) {
  int4 r;
  asm volatile("ld.global.cg.v4.s32 {%0,%1,%2,%3}, [%4];"
               : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w)
               : "l"(p));
  Vec4<T> o;
  o.x = *reinterpret_cast<T*>(&r.x);
  o.y = *reinterpret_cast<T*>(&r.y);
  o.z = *reinterpret_cast<T*>(&r.z);
  o.w = *reinterpret_cast<T*>(&r.w);
  return o;
}
template <typename T>
__device__ __forceinline__ void st4(T* p, Vec4<T> v) {
  typename Tr<T>::V4 o;
  o.x = v.x; o.y = v.y; o.z = v.z; o.w = v.w;
  *reinterpret_cast<typename Tr<T>::V4*>(p) = o;
}
template <typename T>
__device__ __forceinline__ T get(const Vec4<T>& v, int c) {
  return c == 0 ? v.x : c == 1 ? v.y : c == 2 ? v.z : v.w;
}
// replace lanes with column index >= n by INF (tail vector of a row)
template <typename T>
__device__ __forceinline__ Vec4<T> mask_tail(Vec4<T> v, int64_t col0, int64_t n) {
  const T I = Tr<T>::inf();
  if (col0 + 4 > n) {
    if (col0 + 0 >= n) v.x = I;
    if (col0 + 1 >= n) v.y = I;
    if (col0 + 2 >= n) v.z = I;
    if (col0 + 3 >= n) v.w = I;
  }
  return v;
}

// ---------------------------------------------------------------------------
// saturated mirror of int32 D, int16 / int8 (kernels.h: struct Mirror)
// ---------------------------------------------------------------------------
constexpr int32_t kSat16i = 0x3FFF;
__device__ __forceinline__ uint16_t sat16(int32_t v) { return (uint16_t)min(v, kSat16i); }
// 8 int16 mirrored values (or 16 int8 ones) in one 16-byte streaming load
// One byte of a random gather, cached in L2 only: an L1 miss would fill a
// whole 128-byte line (4 sectors from DRAM) for the one byte used.
__device__ __forceinline__ uint32_t ldg_byte_l2(const uint8_t* p) {
  uint32_t v;
  asm("ld.global.cg.u8 %0, [%1];" : "=r"(v) : "l"(p));
  return v;
}
__device__ __forceinline__ uint4 mload8(const uint16_t* p) {
  uint4 r;
  asm volatile("ld.global.nc.L1::no_allocate.v4.u32 {%0,%1,%2,%3}, [%4];"
               : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w)
               : "l"(p));
  return r;
}
// Column groups of a lane in a 512-column chunk.  int32 rows: vector v holds
// columns 4*(chunk*128 + v*32 + lane) + [0, 4).  Mirror rows are read 16 bytes
// (8 columns) at a time, so vectors 2q and 2q+1 are the halves of load q:
// columns 8*(chunk*64 + q*32 + lane) + [0, 8) — the same 512 columns per warp.
__device__ __forceinline__ int64_t group_of(bool m16, int chunk, int v, int lane) {
  return m16 ? 2 * ((int64_t)chunk * 64 + (v >> 1) * 32 + lane) + (v & 1)
             : (int64_t)chunk * 128 + v * 32 + lane;
}
// int8 mirror: 8 values widened to the int16x2 words the packed arithmetic
// uses (halves 0..0x7F)
constexpr int32_t kSat8i = 0x7F;
__device__ __forceinline__ uint4 widen8(uint2 b) {
  return make_uint4(__byte_perm(b.x, 0u, 0x4140), __byte_perm(b.x, 0u, 0x4342),
                    __byte_perm(b.y, 0u, 0x4140), __byte_perm(b.y, 0u, 0x4342));
}
// int16x2 word with halves <= 0x7F: halves equal to 0x7F (int8 INF) -> 0x3FFF
__device__ __forceinline__ uint32_t inf8to16(uint32_t x) {
  const uint32_t t = x ^ 0x007F007Fu;   // zero half <-> INF
  const uint32_t nz = (t | ((t & 0x7FFF7FFFu) + 0x7FFF7FFFu)) & 0x80008000u;
  return x | (((~nz & 0x80008000u) >> 15) * 0x3FFFu);
}

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return (uint32_t)__cvta_generic_to_shared(p);
}
// per-thread async copies (LDGSTS): 16 bytes global -> shared, no registers
__device__ __forceinline__ void cp_async16(void* dst, const void* src) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(smem_u32(dst)), "l"(src) : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_async_wait() { asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory"); }

template <typename T>
__device__ __forceinline__ T warp_min(T v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v = Tr<T>::mn(v, __shfl_xor_sync(0xffffffffu, v, o));
  return v;
}

template <typename T>
__device__ __forceinline__ T warp_max(T v) {
  if constexpr (std::is_same<T, int32_t>::value) {
    return __reduce_max_sync(0xffffffffu, v);
  } else {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v = fmaxf(v, __shfl_xor_sync(0xffffffffu, v, o));
    return v;
  }
}

constexpr int kNumSMs = 148;  // B200 (2 dies x 74); the host reads the real count

}  // namespace apsp
