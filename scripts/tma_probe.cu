// tma_probe.cu — measurement probe (not product code): HBM read bandwidth of
// bulk-copy (TMA) rings in the shapes the streaming kernels use.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -I../paper_2412_15122_b200/csrc \
//        scripts/tma_probe.cu -o /tmp/tma_probe && /tmp/tma_probe
// Variants: (a) per-warp rings, lane 0 copies `piece` bytes per stage;
// (b) a CTA ring filled by one producer thread, rows of `row` bytes cut into
// `piece`-byte copies, S stages, 8 consumer warps; (c) as (b) with the
// copies of a row issued by `np` producer lanes.
#include <cstdio>
#include <cuda_runtime.h>

#include "tma.cuh"

using namespace apsp;

__global__ void k_warp_ring(const uint8_t* src, size_t bytes, int piece, int S, unsigned long long* sink) {
  extern __shared__ __align__(128) uint8_t sm[];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, nw = blockDim.x >> 5;
  uint8_t* buf = sm + warp * (S * piece + 128);
  uint64_t* bar = reinterpret_cast<uint64_t*>(buf + S * piece);
  if (lane == 0) {
    for (int s = 0; s < S; ++s) mbar_init(bar + s, 1);
    fence_barrier_init();
  }
  __syncwarp();
  const size_t gw = (size_t)blockIdx.x * nw + warp, W = (size_t)gridDim.x * nw;
  const size_t np = bytes / piece;
  const size_t mine = (np > gw) ? (np - gw + W - 1) / W : 0;   // pieces gw, gw + W, ...
  unsigned acc = 0;
  auto issue = [&](size_t k) {
    if (k < mine && lane == 0) {
      fence_proxy_async();
      mbar_expect_tx(bar + k % S, piece);
      bulk_g2s(buf + (k % S) * piece, src + (gw + k * W) * piece, piece, bar + k % S);
    }
  };
  for (int k = 0; k < S - 1; ++k) issue(k);
  for (size_t k = 0; k < mine; ++k) {
    __syncwarp();
    issue(k + S - 1);
    mbar_wait(bar + k % S, (unsigned)(k / S) & 1u);
    const uint4* p = reinterpret_cast<const uint4*>(buf + (k % S) * piece);
    for (int e = lane; e < piece / 16; e += 32) acc += p[e].x ^ p[e].w;
  }
  if (acc == 0x12345678u) atomicAdd(sink, 1ull);
}

__global__ void k_cta_ring(const uint8_t* src, size_t bytes, int row, int piece, int S, int nprod,
                           unsigned long long* sink) {
  extern __shared__ __align__(128) uint8_t sm[];
  uint64_t* full = reinterpret_cast<uint64_t*>(sm + (size_t)S * row);
  uint64_t* empty = full + S;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int ncons = (blockDim.x >> 5) - 1;
  if (threadIdx.x == 0) {
    for (int s = 0; s < S; ++s) { mbar_init(full + s, 1); mbar_init(empty + s, ncons); }
    fence_barrier_init();
  }
  __syncthreads();
  const size_t nrows = bytes / row;
  const size_t per = (nrows + gridDim.x - 1) / gridDim.x;
  const size_t r0 = blockIdx.x * per, r1 = r0 + per < nrows ? r0 + per : nrows;
  const int rows = r1 > r0 ? (int)(r1 - r0) : 0;
  if (warp == ncons) {   // producer warp
    if (lane < nprod) {
      for (int rr = 0; rr < rows; ++rr) {
        const int s = rr % S;
        if (rr >= S) mbar_wait(empty + s, (unsigned)(rr / S - 1) & 1u);
        if (lane == 0) mbar_expect_tx(full + s, row);
        __syncwarp((1u << nprod) - 1);
        for (int o = lane * piece; o < row; o += nprod * piece)
          bulk_g2s(sm + (size_t)s * row + o, src + (r0 + rr) * (size_t)row + o, piece, full + s);
      }
    }
    return;
  }
  unsigned acc = 0;
  for (int rr = 0; rr < rows; ++rr) {
    const int s = rr % S;
    mbar_wait(full + s, (unsigned)(rr / S) & 1u);
    const uint4* p = reinterpret_cast<const uint4*>(sm + (size_t)s * row);
    for (int e = warp * 32 + lane; e < row / 16; e += ncons * 32) acc += p[e].x ^ p[e].w;
    __syncwarp();
    if (lane == 0) mbar_arrive(empty + s);
  }
  if (acc == 0x12345678u) atomicAdd(sink, 1ull);
}

int main() {
  const size_t bytes = (size_t)1 << 30;
  uint8_t* src;
  unsigned long long* sink;
  cudaMalloc(&src, bytes);
  cudaMemset(src, 1, bytes);
  cudaMalloc(&sink, 8);
  int sms;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  cudaFuncSetAttribute(k_warp_ring, cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024);
  cudaFuncSetAttribute(k_cta_ring, cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024);
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  auto timeit = [&](auto launch) {
    float best = 1e9f;
    for (int it = 0; it < 5; ++it) {
      cudaEventRecord(a);
      launch();
      cudaEventRecord(b);
      cudaEventSynchronize(b);
      float ms;
      cudaEventElapsedTime(&ms, a, b);
      if (it > 0 && ms < best) best = ms;
    }
    return bytes / (best * 1e-3) / 1e9;
  };
  struct W { int piece, S, warps, ctas; } wv[] = {
      {1024, 3, 8, 3}, {2048, 3, 8, 2}, {2048, 4, 8, 2}, {4096, 3, 8, 2}, {4096, 4, 4, 4}, {8192, 3, 4, 2}, {16384, 3, 4, 1}};
  for (auto v : wv) {
    const int smem = v.warps * (v.S * v.piece + 128);
    double g = timeit([&] { k_warp_ring<<<sms * v.ctas, 32 * v.warps, smem>>>(src, bytes, v.piece, v.S, sink); });
    printf("warp-ring piece=%5d S=%d warps/cta=%d ctas/sm=%d : %7.1f GB/s  (%s)\n", v.piece, v.S, v.warps, v.ctas, g,
           cudaGetErrorString(cudaGetLastError()));
  }
  struct C { int row, piece, S, nprod, cons, ctas; } cv[] = {
      {32768, 2048, 5, 1, 8, 1}, {32768, 2048, 5, 16, 8, 1}, {32768, 4096, 5, 8, 8, 1}, {32768, 32768, 5, 1, 8, 1},
      {32768, 2048, 3, 16, 8, 2}, {16384, 2048, 6, 8, 8, 2}, {8192, 2048, 8, 4, 8, 3}, {8192, 8192, 8, 1, 8, 3},
      {32768, 1024, 6, 32, 12, 1}};
  for (auto v : cv) {
    const int smem = v.S * v.row + 2 * v.S * 8;
    double g = timeit([&] {
      k_cta_ring<<<sms * v.ctas, 32 * (v.cons + 1), smem>>>(src, bytes, v.row, v.piece, v.S, v.nprod, sink);
    });
    printf("cta-ring row=%5d piece=%5d S=%d producers=%2d consumers=%2d ctas/sm=%d : %7.1f GB/s  (%s)\n", v.row,
           v.piece, v.S, v.nprod, v.cons, v.ctas, g, cudaGetErrorString(cudaGetLastError()));
  }
  return 0;
}
