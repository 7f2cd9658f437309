// microbench.cu — the roofline denominators, measured on the device (SURVEY
// §8(d-3) "K13"): the issue rate of the relaxation d = min(d, a + b) in each
// arithmetic the path uses, and the HBM read / read-modify-write stream rates.
//
//   kind 0  int32 relaxations/s      (one VIADDMNMX per relaxation on sm_100a)
//   kind 1  fp32 relaxations/s       (FADD, FADD, FMNMX3 per two relaxations)
//   kind 2  int16x2 relaxations/s    (VIADDMNMX.S16x2: two per instruction; not
//                                     used by the API, reported for reference)
//   kind 3  HBM read GB/s            (16-byte streaming loads, caller's buffer)
//   kind 4  HBM read+write GB/s      (in-place 16-byte read-modify-write)
//
// Every kernel runs on all SMs with enough independent chains per thread to
// hide pipe latency; the result is the best of 5 timed launches after 2 warm-up
// launches, CUDA events on the given stream.
#include "common.cuh"
#include "kernels.h"

namespace apsp {

constexpr int MB_THREADS = 256;
constexpr int MB_CHAINS = 16;

__global__ void __launch_bounds__(MB_THREADS) k_mb_i32(int iters, int seed, int key, int* sink) {
  int x[MB_CHAINS];
#pragma unroll
  for (int q = 0; q < MB_CHAINS; ++q) x[q] = (threadIdx.x * 7 + q * 13 + seed) & 1023;
  const int d = seed & 7;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int q = 0; q < MB_CHAINS; ++q) x[q] = min(x[q], x[(q + 5) % MB_CHAINS] + d);
  }
  int acc = 0;
#pragma unroll
  for (int q = 0; q < MB_CHAINS; ++q) acc ^= x[q];
  if (acc == key) *sink = acc;   // the host passes a key no result can equal (-1)
}

__global__ void __launch_bounds__(MB_THREADS) k_mb_f32(int iters, int seed, int key, float* sink) {
  float x[MB_CHAINS];
#pragma unroll
  for (int q = 0; q < MB_CHAINS; ++q) x[q] = (float)((threadIdx.x * 7 + q * 13 + seed) & 1023);
  const float d0 = (float)(seed & 7), d1 = d0 + 1.0f;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int q = 0; q < MB_CHAINS; ++q)   // two relaxations: FADD, FADD, FMNMX3
      x[q] = fminf(fminf(x[q], x[(q + 5) % MB_CHAINS] + d0), x[(q + 7) % MB_CHAINS] + d1);
  }
  float acc = 0.f;
#pragma unroll
  for (int q = 0; q < MB_CHAINS; ++q) acc += x[q];
  if (acc == (float)key) *sink = acc;
}

__global__ void __launch_bounds__(MB_THREADS) k_mb_s16(int iters, int seed, int key, unsigned* sink) {
  unsigned x[MB_CHAINS];
#pragma unroll
  for (int q = 0; q < MB_CHAINS; ++q) x[q] = ((threadIdx.x * 7u + q * 13u + seed) & 1023u) * 0x10001u;
  const unsigned d = (unsigned)(seed & 7) * 0x10001u;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int q = 0; q < MB_CHAINS; ++q) x[q] = __viaddmin_s16x2(x[(q + 5) % MB_CHAINS], d, x[q]);
  }
  unsigned acc = 0;
#pragma unroll
  for (int q = 0; q < MB_CHAINS; ++q) acc ^= x[q];
  if (acc == (unsigned)key) *sink = acc;
}

__global__ void k_mb_read(const int4* __restrict__ p, int64_t n16, int* sink) {
  int acc = 0;
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < n16;
       e += (int64_t)gridDim.x * blockDim.x) {
    int4 v;
    asm volatile("ld.global.nc.L1::no_allocate.v4.s32 {%0,%1,%2,%3}, [%4];"
                 : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w)
                 : "l"(p + e));
    acc ^= v.x ^ v.y ^ v.z ^ v.w;
  }
  if (acc == 0x7fffffff) *sink = acc;
}

__global__ void k_mb_rmw(int4* p, int64_t n16) {
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < n16;
       e += (int64_t)gridDim.x * blockDim.x) {
    int4 v = p[e];
    v.x += 1; v.y += 1; v.z += 1; v.w += 1;
    p[e] = v;
  }
}

// Returns the rate of `kind` (see above); -1 for bad arguments, -2 on a CUDA error.
double microbench(int kind, void* buf, size_t bytes, cudaStream_t st) {
  const int sms = num_sms();
  if (kind < 0 || kind > 4 || !buf || (kind >= 3 && bytes < 16)) return -1.0;
  cudaEvent_t a, b;
  if (cudaEventCreate(&a) != cudaSuccess) return -2.0;
  if (cudaEventCreate(&b) != cudaSuccess) { cudaEventDestroy(a); return -2.0; }
  const int iters = 4096;
  const int grid_alu = sms * 8;   // 8 CTAs x 256 threads per SM: full occupancy
  double work = 0.0;
  auto launch = [&](int rep) {
    switch (kind) {
      case 0: k_mb_i32<<<grid_alu, MB_THREADS, 0, st>>>(iters, rep, -1, reinterpret_cast<int*>(buf)); break;
      case 1: k_mb_f32<<<grid_alu, MB_THREADS, 0, st>>>(iters, rep, -1, reinterpret_cast<float*>(buf)); break;
      case 2: k_mb_s16<<<grid_alu, MB_THREADS, 0, st>>>(iters, rep, -1, reinterpret_cast<unsigned*>(buf)); break;
      case 3: k_mb_read<<<sms * 16, 512, 0, st>>>(reinterpret_cast<const int4*>(buf), (int64_t)(bytes / 16),
                                                  reinterpret_cast<int*>(buf)); break;
      case 4: k_mb_rmw<<<sms * 16, 512, 0, st>>>(reinterpret_cast<int4*>(buf), (int64_t)(bytes / 16)); break;
    }
  };
  const double threads = (double)grid_alu * MB_THREADS;
  switch (kind) {
    case 0: work = threads * iters * MB_CHAINS; break;           // relaxations
    case 1: work = threads * iters * MB_CHAINS * 2; break;       // relaxations
    case 2: work = threads * iters * MB_CHAINS * 2; break;       // relaxations (2 lanes)
    case 3: work = (double)(bytes / 16 * 16); break;             // bytes read
    case 4: work = 2.0 * (double)(bytes / 16 * 16); break;       // bytes read + written
  }
  float best = 1e30f;
  bool ok = true;
  for (int rep = 0; rep < 7 && ok; ++rep) {
    cudaEventRecord(a, st);
    launch(rep);
    cudaEventRecord(b, st);
    ok = cudaEventSynchronize(b) == cudaSuccess;
    float ms = 0.f;
    if (ok) cudaEventElapsedTime(&ms, a, b);
    if (ok && rep >= 2) best = std::min(best, ms);
  }
  cudaEventDestroy(a);
  cudaEventDestroy(b);
  if (!ok || cudaGetLastError() != cudaSuccess) return -2.0;
  return work / (best * 1e-3);
}

}  // namespace apsp
