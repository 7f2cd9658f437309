// sparse.cu — sparse affected-pair recompute.
//
// The paper recomputes every affected source with Dijkstra ("If the Cost is
// small, we use Dijkstra's algorithm to calculate a node's distance to other
// nodes in the new graph").  On the GPU the work is re-expressed at
// pair level: only the listed pairs (i, j) in A are recomputed, each from
// the Bellman equation of its last hop,
//     D'[i][j] = min_m D'[i][m] + W'[m][j],
// on D0 (affected entries reset to W'[i][j], unaffected entries exact by
// Theorem 4).  Round 0 scans all m (one streaming dot-min of row i of D with
// row j of WT per pair); rounds r >= 1 re-relax each pair only over the
// affected m of its own row (A_i), for rows that changed in the previous
// round, until no entry changes.  A fixpoint of these upper bounds is the
// exact distance; rows read only their own D row and the
// read-only WT, so rows never race and no grid-wide sync is needed.
#include "common.cuh"
#include "kernels.h"

namespace apsp {

static inline int64_t cdiv(int64_t a, int64_t b) { return (a + b - 1) / b; }

// warp per pair: est = min_m D[i][m] + WT[j][m] over all m < n
template <typename T>
__global__ void __launch_bounds__(256) k_sparse_round0(T* D, int64_t ld, int64_t row0,
                                                       const T* __restrict__ WT, int64_t ldw,
                                                       int64_t n, const int* __restrict__ prow,
                                                       const int* __restrict__ pcol,
                                                       int64_t npairs) {
  const int lane = threadIdx.x & 31;
  const int64_t nw = (int64_t)gridDim.x * (blockDim.x >> 5);
  const int64_t n4 = (n + 3) / 4;
  const T I = Tr<T>::inf();
  for (int64_t p = blockIdx.x * (int64_t)(blockDim.x >> 5) + (threadIdx.x >> 5); p < npairs;
       p += nw) {
    const int64_t i = prow[p], j = pcol[p];
    T* Drow = D + (i - row0) * ld;
    const T* Wrow = WT + j * ldw;
    T acc = I;
    int64_t q = lane;
    for (; q + 32 < n4; q += 64) {
      // two vectors per lane in flight; other warps may lower entries of this
      // row concurrently — any value read is a valid upper bound
      Vec4<T> d0 = ld4_cg<T>(Drow + 4 * q), d1 = ld4_cg<T>(Drow + 4 * (q + 32));
      Vec4<T> w0 = ld4<T>(Wrow + 4 * q), w1 = ld4<T>(Wrow + 4 * (q + 32));
      d1 = mask_tail<T>(d1, 4 * (q + 32), n);
      w1 = mask_tail<T>(w1, 4 * (q + 32), n);
      acc = Tr<T>::relax(acc, d0.x, w0.x); acc = Tr<T>::relax(acc, d0.y, w0.y);
      acc = Tr<T>::relax(acc, d0.z, w0.z); acc = Tr<T>::relax(acc, d0.w, w0.w);
      acc = Tr<T>::relax(acc, d1.x, w1.x); acc = Tr<T>::relax(acc, d1.y, w1.y);
      acc = Tr<T>::relax(acc, d1.z, w1.z); acc = Tr<T>::relax(acc, d1.w, w1.w);
    }
    for (; q < n4; q += 32) {
      Vec4<T> d0 = mask_tail<T>(ld4_cg<T>(Drow + 4 * q), 4 * q, n);
      Vec4<T> w0 = mask_tail<T>(ld4<T>(Wrow + 4 * q), 4 * q, n);
      acc = Tr<T>::relax(acc, d0.x, w0.x); acc = Tr<T>::relax(acc, d0.y, w0.y);
      acc = Tr<T>::relax(acc, d0.z, w0.z); acc = Tr<T>::relax(acc, d0.w, w0.w);
    }
    acc = warp_min<T>(acc);
    if (lane == 0) {
      T old = Drow[j];
      if (acc < old) Drow[j] = acc;
    }
  }
}

template <typename T>
cudaError_t sparse_round0(T* D, int64_t ld, int64_t row0, const T* WT, int64_t ldw, int64_t n,
                          const int* prow, const int* pcol, int64_t npairs, cudaStream_t st) {
  if (npairs <= 0) return cudaSuccess;
  int grid = (int)std::min<int64_t>(cdiv(npairs, 8), (int64_t)num_sms() * 8);
  k_sparse_round0<T><<<grid, 256, 0, st>>>(D, ld, row0, WT, ldw, n, prow, pcol, npairs);
  return cudaGetLastError();
}

// warp per pair of a changed row: est = min over m in A_i of D[i][m] + WT[j][m]
template <typename T>
__global__ void __launch_bounds__(256) k_sparse_round(T* D, int64_t ld, int64_t row0,
                                                      const T* __restrict__ WT, int64_t ldw,
                                                      const int* __restrict__ prow,
                                                      const int* __restrict__ pcol, int64_t npairs,
                                                      const int64_t* __restrict__ rowoff,
                                                      const int* __restrict__ rowcnt,
                                                      const int* chg_in, int* chg_out, int* any) {
  const int lane = threadIdx.x & 31;
  const int64_t nw = (int64_t)gridDim.x * (blockDim.x >> 5);
  for (int64_t p = blockIdx.x * (int64_t)(blockDim.x >> 5) + (threadIdx.x >> 5); p < npairs;
       p += nw) {
    const int64_t i = prow[p];
    const int cnt = rowcnt[i];
    if (cnt <= 1 || !chg_in[i]) continue;      // a lone affected target is exact after round 0
    const int64_t j = pcol[p];
    const int64_t off = rowoff[i];
    T* Drow = D + (i - row0) * ld;
    const T* Wrow = WT + j * ldw;
    T acc = Tr<T>::inf();
    for (int t = lane; t < cnt; t += 32) {
      const int64_t m = pcol[off + t];
      acc = Tr<T>::relax(acc, *(volatile T*)(Drow + m), Wrow[m]);
    }
    acc = warp_min<T>(acc);
    if (lane == 0) {
      T old = Drow[j];
      if (acc < old) {
        Drow[j] = acc;
        chg_out[i] = 1;
        *any = 1;
      }
    }
  }
}

template <typename T>
cudaError_t sparse_round(T* D, int64_t ld, int64_t row0, const T* WT, int64_t ldw, int64_t n,
                         const int* prow, const int* pcol, int64_t npairs, const int64_t* rowoff,
                         const int* rowcnt, const int* chg_in, int* chg_out, int* any,
                         cudaStream_t st) {
  (void)n;
  if (npairs <= 0) return cudaSuccess;
  int grid = (int)std::min<int64_t>(cdiv(npairs, 8), (int64_t)num_sms() * 8);
  k_sparse_round<T><<<grid, 256, 0, st>>>(D, ld, row0, WT, ldw, prow, pcol, npairs, rowoff, rowcnt,
                                          chg_in, chg_out, any);
  return cudaGetLastError();
}

#define INST(T)                                                                                  \
  template cudaError_t sparse_round0<T>(T*, int64_t, int64_t, const T*, int64_t, int64_t,        \
                                        const int*, const int*, int64_t, cudaStream_t);          \
  template cudaError_t sparse_round<T>(T*, int64_t, int64_t, const T*, int64_t, int64_t,         \
                                       const int*, const int*, int64_t, const int64_t*,          \
                                       const int*, const int*, int*, int*, cudaStream_t);
INST(int32_t)
INST(float)
#undef INST

}  // namespace apsp
