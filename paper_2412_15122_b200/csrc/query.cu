// query.cu — warm-start single-pair shortest path (alg:sp_apsp).
//
// "It use the conclusion of Theorem 4 to exclude unnecessary nodes from node
// i to node j, generate the candidate_node_list; then form a small graph
// which is composed of nodes in candidate_node_list; then use Dijkstra's
// algorithm to calculate the shortest path from node i to node j, on the
// small graph; then translate the path into original node index."
//
// One CTA per query:
//   1. candidate scan: C = {k : D[s][k] + D[k][t] == D[s][t]} over row s
//      (contiguous) and column t (stride ld), compacted in node order with
//      warp ballots + popc into shared memory;
//   2. Dijkstra on the induced subgraph of C (warp 0; argmin by 64-bit
//      (label, index) keys so ties go to the smaller node id), early
//      stop when t is finalised; edge weights W[m][c] = WT[c][m];
//   3. predecessor walk t -> s, written in original ids.
//
// Row-sharded mode (world > 1): D is split by rows, so
// row s lives on one rank and column t is spread over all of them.  The host
// first gathers, for a chunk of QC queries, every rank's slice of each column
// t (k_query_colslice + one all-gather of QC x R entries per rank); then the
// rank owning row s runs the query exactly as above, reading D[k][t] from the
// gathered slices, while the other ranks write zeros, and one all-reduce(sum)
// of the outputs leaves every rank with the owner's answer.  WT is replicated,
// so the Dijkstra step needs no communication.
#include "common.cuh"
#include "kernels.h"

namespace apsp {

constexpr int QT = 256;   // threads per query CTA

// Sharded-mode description (sh.colbuf == nullptr: single GPU, D holds every row).
template <typename T>
struct QShard {
  const T* colbuf;   // gathered column slices: colbuf[(r * qc + b) * R + i] = D[r*R + i][t_b]
  int64_t R;         // rows per rank
  int64_t row0, rows;   // this rank's rows (D points at global row row0)
  int qc;            // queries in this chunk
};

template <typename T, int SR>
__global__ void __launch_bounds__(QT) k_query(const T* __restrict__ D, int64_t ld,
                                              const T* __restrict__ WT, int64_t ldw, int64_t n,
                                              int q, const int* __restrict__ S,
                                              const int* __restrict__ Tq, T* dist, int* paths,
                                              int path_cap, int* path_lens, int* ncand, float tau,
                                              QShard<T> sh) {
  __shared__ int cid[kQueryCap];
  __shared__ T lab[kQueryCap];
  __shared__ short pred[kQueryCap];
  __shared__ unsigned char done[kQueryCap];
  __shared__ int s_cnt, s_is, s_it;
  __shared__ int s_wcnt[4 * (QT / 32)];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const T I = Tr<T>::inf();

  for (int b = blockIdx.x; b < q; b += gridDim.x) {
    const int s = S[b], t = Tq[b];
    const bool bad = s < 0 || s >= n || t < 0 || t >= n;
    if (sh.colbuf) {
      // sharded: the owner of row s answers (rank 0 answers invalid pairs);
      // every other rank contributes zeros to the all-reduce(sum)
      const bool mine = bad ? sh.row0 == 0 : (s >= sh.row0 && s < sh.row0 + sh.rows);
      if (!mine) {
        if (tid == 0) { path_lens[b] = 0; if (ncand) ncand[b] = 0; dist[b] = T(0); }
        for (int c = tid; c < path_cap; c += QT) paths[(int64_t)b * path_cap + c] = 0;
        continue;
      }
      for (int c = tid; c < path_cap; c += QT) paths[(int64_t)b * path_cap + c] = -1;
      __syncthreads();
    }
    if (bad) {
      if (tid == 0) { path_lens[b] = -3; if (ncand) ncand[b] = 0; dist[b] = I; }
      continue;
    }
    const T* Ds = D + ((int64_t)s - sh.row0) * ld;
    const T st = Ds[t];
    if (s == t || !Tr<T>::fin(st)) {
      if (tid == 0) {
        dist[b] = s == t ? T(0) : I;
        if (s == t) {
          if (path_cap >= 1) { paths[(int64_t)b * path_cap] = s; path_lens[b] = 1; }
          else path_lens[b] = -1;
        } else {
          path_lens[b] = 0;
        }
        if (ncand) ncand[b] = s == t ? 1 : 0;
      }
      continue;
    }
    if (tid == 0) { s_cnt = 0; s_is = -1; s_it = -1; }
    __syncthreads();

    // ---- 1. candidate scan (Theorem 4 equality), ordered compaction ----
    // Candidates are rare (|C| ~ tens out of n), so a block-wide OR skips the
    // compaction for almost every group of QT*U nodes.
    constexpr int U = 4;   // nodes per thread per step (loads in flight)
    for (int64_t base = 0; base < n; base += (int64_t)QT * U) {
      T dsk[U], dkt[U];
#pragma unroll
      for (int u = 0; u < U; ++u) {
        int64_t k = base + (int64_t)u * QT + tid;
        dsk[u] = k < n ? Ds[k] : I;
        if (sh.colbuf) {
          const int64_t r = k / sh.R;
          dkt[u] = k < n ? sh.colbuf[(r * sh.qc + b) * sh.R + (k - r * sh.R)] : I;
        } else {
          dkt[u] = k < n ? D[k * ld + t] : I;
        }
      }
      bool f[U];
      bool anyf = false;
#pragma unroll
      for (int u = 0; u < U; ++u) {
        int64_t k = base + (int64_t)u * QT + tid;
        f[u] = k < n && Tr<T>::fin(dsk[u]) && Tr<T>::fin(dkt[u]) &&
               Tr<T, SR>::tight(Tr<T, SR>::add(dsk[u], dkt[u]), st, tau);
        anyf |= f[u];
      }
      if (!__syncthreads_or(anyf)) continue;
      unsigned bal[U];
#pragma unroll
      for (int u = 0; u < U; ++u) {
        bal[u] = __ballot_sync(0xffffffffu, f[u]);
        if (lane == 0) s_wcnt[u * (QT / 32) + warp] = __popc(bal[u]);
      }
      __syncthreads();
      int tot = 0;
#pragma unroll
      for (int u = 0; u < U; ++u) {
        int off = s_cnt + tot;
        for (int w = 0; w < warp; ++w) off += s_wcnt[u * (QT / 32) + w];
        for (int w = 0; w < QT / 32; ++w) tot += s_wcnt[u * (QT / 32) + w];
        if (f[u]) {
          const int64_t k = base + (int64_t)u * QT + tid;
          const int pos = off + __popc(bal[u] & ((1u << lane) - 1));
          if (pos < kQueryCap) {
            cid[pos] = (int)k;
            if (k == s) s_is = pos;
            if (k == t) s_it = pos;
          }
        }
      }
      __syncthreads();
      if (tid == 0) s_cnt += tot;
      __syncthreads();
    }
    const int cnt = s_cnt;
    if (cnt > kQueryCap || s_is < 0 || s_it < 0) {
      if (tid == 0) { path_lens[b] = -2; if (ncand) ncand[b] = cnt; dist[b] = st; }
      __syncthreads();
      continue;
    }

    // ---- 2. Dijkstra on the candidate subgraph (warp 0) ----
    if (warp == 0) {
      for (int c = lane; c < cnt; c += 32) { lab[c] = I; pred[c] = -1; done[c] = 0; }
      __syncwarp();
      if (lane == 0) lab[s_is] = T(0);
      __syncwarp();
      for (int it = 0; it < cnt; ++it) {
        unsigned long long best = ~0ull;
        for (int c = lane; c < cnt; c += 32)
          if (!done[c]) {
            unsigned long long key = ((unsigned long long)Tr<T>::key(lab[c]) << 32) | (unsigned)c;
            best = key < best ? key : best;
          }
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) {
          unsigned long long y = __shfl_xor_sync(0xffffffffu, best, o);
          best = y < best ? y : best;
        }
        if (best == ~0ull) break;
        const int m = (int)(best & 0xffffffffu);
        const T lm = lab[m];
        if (!Tr<T>::fin(lm)) break;
        __syncwarp();
        if (lane == 0) done[m] = 1;
        __syncwarp();
        if (m == s_it) break;
        const int64_t gm = cid[m];
        for (int c = lane; c < cnt; c += 32) {
          if (done[c]) continue;
          const T w = WT[(int64_t)cid[c] * ldw + gm];   // W[m][c]
          if (!Tr<T>::fin(w)) continue;
          const T cand = Tr<T, SR>::add(lm, w);
          if (cand < lab[c]) { lab[c] = cand; pred[c] = (short)m; }
        }
        __syncwarp();
      }
      // ---- 3. path t -> s ----
      if (lane == 0) {
        int len = 0, last = -1;
        for (int c = s_it; c >= 0 && len <= cnt; c = (c == s_is) ? -1 : pred[c]) { ++len; last = c; }
        dist[b] = st;
        if (ncand) ncand[b] = cnt;
        if (len > cnt || last != s_is) {
          path_lens[b] = -2;       // no path through the candidates (cannot happen)
        } else if (len > path_cap) {
          path_lens[b] = -1;
        } else {
          int* out = paths + (int64_t)b * path_cap;
          int pos = len - 1;
          for (int c = s_it; c >= 0; c = (c == s_is) ? -1 : pred[c]) out[pos--] = cid[c];
          path_lens[b] = len;
        }
      }
    }
    __syncthreads();
  }
}

// out[b * R + i] = D[row0 + i][t_b] for local rows i < rows, INF for i in [rows, R)
// (also for an out-of-range t_b).  One warp per (query, 32-row group): the
// column entries are 4-byte strided reads, so this is sector-bound (32 B per
// entry) — 2·qc·R sectors, small next to the candidate scan's row stream.
template <typename T>
__global__ void k_query_colslice(const T* __restrict__ D, int64_t ld, int64_t rows, int64_t R,
                                 int64_t n, const int* __restrict__ Tq, int qc, T* __restrict__ out) {
  const int64_t total = (int64_t)qc * R;
  for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < total;
       e += (int64_t)gridDim.x * blockDim.x) {
    const int b = (int)(e / R);
    const int64_t i = e - (int64_t)b * R;
    const int t = Tq[b];
    out[e] = (i < rows && t >= 0 && t < n) ? D[i * ld + t] : Tr<T>::inf();
  }
}

template <typename T>
cudaError_t query_colslice(const T* D, int64_t ld, int64_t rows, int64_t R, int64_t n,
                           const int* t, int qc, T* out, cudaStream_t st) {
  const int64_t total = (int64_t)qc * R;
  if (total <= 0) return cudaSuccess;
  const int blocks = (int)std::min<int64_t>((total + 255) / 256, (int64_t)num_sms() * 8);
  k_query_colslice<T><<<blocks, 256, 0, st>>>(D, ld, rows, R, n, t, qc, out);
  return cudaGetLastError();
}

template <typename T>
cudaError_t query_batch(const T* D, int64_t ld, const T* WT, int64_t ldw, int64_t n, int q,
                        const int* s, const int* t, T* dist, int* paths, int path_cap,
                        int* path_lens, int* ncand, float tau, int sr, cudaStream_t st,
                        const T* colbuf, int64_t R, int64_t row0, int64_t rows) {
  if (q <= 0) return cudaSuccess;
  int grid = std::min(q, num_sms() * 4);
  QShard<T> sh{colbuf, R, colbuf ? row0 : 0, rows, q};
  if (sr)
    k_query<T, 1><<<grid, QT, 0, st>>>(D, ld, WT, ldw, n, q, s, t, dist, paths, path_cap, path_lens,
                                       ncand, tau, sh);
  else
    k_query<T, 0><<<grid, QT, 0, st>>>(D, ld, WT, ldw, n, q, s, t, dist, paths, path_cap, path_lens,
                                       ncand, tau, sh);
  return cudaGetLastError();
}

#define INST(T)                                                                                  \
  template cudaError_t query_batch<T>(const T*, int64_t, const T*, int64_t, int64_t, int,       \
                                      const int*, const int*, T*, int*, int, int*, int*, float,  \
                                      int, cudaStream_t, const T*, int64_t, int64_t, int64_t);   \
  template cudaError_t query_colslice<T>(const T*, int64_t, int64_t, int64_t, int64_t,          \
                                         const int*, int, T*, cudaStream_t);
INST(int32_t)
INST(float)
#undef INST

}  // namespace apsp
