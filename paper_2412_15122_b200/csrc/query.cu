// query.cu — warm-start single-pair shortest path (alg:sp_apsp).
//
// "It use the conclusion of Theorem 4 to exclude unnecessary nodes from node
// i to node j, generate the candidate_node_list; then form a small graph
// which is composed of nodes in candidate_node_list; then use Dijkstra's
// algorithm to calculate the shortest path from node i to node j, on the
// small graph; then translate the path into original node index."
//
// Two kernels per chunk of queries:
//   k_query_scan  — the candidate_node_list C = {k : D[s][k] + D[k][t] ==
//                   D[s][t]}.  Grid (node chunks x queries), so even ONE query
//                   spreads its scan of row s (contiguous) and column t
//                   (stride ld: one 32-byte sector per entry, ~128 B of DRAM
//                   traffic measured — this column is what bounds the query)
//                   over every SM.  Candidates are rare (|C| ~ tens of n),
//                   appended with one warp-aggregated atomic per warp that
//                   found any, together with D[s][k].
//   k_query_solve — one warp per query: Dijkstra on the small graph induced by
//                   C, ties to the smaller node id, early stop at t,
//                   path in original ids.  The append order of C is arbitrary,
//                   so every tie-break compares node ids, never positions.
//
// Dijkstra's labels on the small graph are known in advance: for k in C a
// whole shortest s->k path lies in C (each node y on it has D[s][y] + D[y][t]
// <= D[s][k] + D[k][t] = D[s][t]), so the label Dijkstra settles k with is
// D[s][k], which the scan read.  With positive weights Dijkstra therefore
// settles C in (D[s][k], id) order, and the predecessor it records for k is the
// first m in that order with D[s][m] + W[m][k] == D[s][k].  For int32 shortest
// paths the kernel computes exactly that tree, hop by hop backwards from t
// (one parallel pass over C per hop instead of one sequential Dijkstra
// iteration per candidate), identical to Dijkstra's output.  With zero-weight
// edges (Q2) every hop still satisfies the equality, so a walk that reaches s
// is a shortest path (though possibly another tie than Dijkstra's); a walk that
// finds no predecessor ordered before the current node falls back to the
// sequential Dijkstra.  fp32 (tolerant equality, Q4) and minimax always run
// the sequential Dijkstra.
//
// Row-sharded mode (world > 1): D is split by rows,
// so row s lives on one rank and column t is spread over all of them.  For a
// chunk of queries: row s of each query goes to every rank (the owner writes
// it, the others zeros, one all-reduce(sum)); every rank tests the candidates
// k among ITS rows — D[s][k] from the shared row, D[k][t] local — and keeps
// the hits; one all-gather of the hit lists (|C| ids per query, no column
// data) gives every rank the candidate set, and every rank solves the small
// graph itself (WT is replicated), so the answer is on every rank without a
// further exchange.
#include <cub/device/device_radix_sort.cuh>
#include "common.cuh"
#include "kernels.h"

namespace apsp {

constexpr int QS_T = 256;   // scan threads
constexpr int QS_U = 4;     // nodes per thread per step (loads in flight)

// Sharded-mode description (colbuf == nullptr: single GPU, D holds every row).
template <typename T>
struct QShard {
  const T* colbuf;   // gathered column slices: colbuf[(r * qc + b) * R + i] = D[r*R + i][t_b]
  int64_t R;         // rows per rank
  int64_t row0, rows;   // this rank's rows (D points at global row row0)
  int qc;            // queries in this chunk
  const T* rowbuf;   // gather-free mode: row s_b of every query (rowbuf[b * ldr + j]); every rank solves
  int64_t ldr;
};

template <typename T>
__device__ __forceinline__ T ld_col(const T* D, int64_t ld, int64_t k, int t, int b,
                                    const QShard<T>& sh) {
  if (sh.colbuf) {
    const int64_t r = k / sh.R;
    return sh.colbuf[(r * sh.qc + b) * sh.R + (k - r * sh.R)];
  }
  return __ldg(D + k * ld + t);
}

template <typename T, int SR>
__global__ void __launch_bounds__(QS_T) k_query_scan(const T* __restrict__ D, int64_t ld, int64_t n,
                                                     const int* __restrict__ S,
                                                     const int* __restrict__ Tq, int64_t chunk,
                                                     int* __restrict__ cand, T* __restrict__ cand_d,
                                                     int qcap, int* __restrict__ cnt, float tau,
                                                     T wmin, QShard<T> sh) {
  const int b = blockIdx.y;
  const int s = S[b], t = Tq[b];
  if (s < 0 || s >= n || t < 0 || t >= n || s == t) return;
  if (sh.colbuf && !(s >= sh.row0 && s < sh.row0 + sh.rows)) return;
  const T* Ds = D + ((int64_t)s - sh.row0) * ld;
  const T st = Ds[t];
  if (!Tr<T>::fin(st)) return;
  const int lane = threadIdx.x & 31;
  const T I = Tr<T>::inf();
  const int64_t k0 = (int64_t)blockIdx.x * chunk, k1 = min(n, k0 + chunk);
  int* out = cand + (int64_t)b * qcap;
  T* outd = cand_d + (int64_t)b * qcap;
  // Column t is the expensive read (one sector per entry), so it is read only
  // for k that can pass the test: D[k][t] >= 0, and for k != t a path of at
  // least one edge, so D[k][t] >= wmin (the smallest edge weight present since
  // creation).  Hence k needs D[s][k] <= D[s][t] - wmin (int32 shortest path;
  // fp32: D[s][k] <= D[s][t](1+tau); minimax: D[s][k] <= D[s][t]).
  T lim;
  if (SR == 1) lim = st;
  else if (Tr<T>::kFloat) lim = st * (1.0f + tau);
  else lim = st - wmin;
  for (int64_t base = k0; base < k1; base += (int64_t)QS_T * QS_U) {
    T dsk[QS_U], dkt[QS_U];
#pragma unroll
    for (int u = 0; u < QS_U; ++u) {
      const int64_t k = base + (int64_t)u * QS_T + threadIdx.x;
      dsk[u] = k < k1 ? Ds[k] : I;
    }
#pragma unroll
    for (int u = 0; u < QS_U; ++u) {
      const int64_t k = base + (int64_t)u * QS_T + threadIdx.x;
      dkt[u] = (k < k1 && (dsk[u] <= lim || k == t)) ? ld_col<T>(D, ld, k, t, b, sh) : I;
    }
#pragma unroll
    for (int u = 0; u < QS_U; ++u) {
      const int64_t k = base + (int64_t)u * QS_T + threadIdx.x;
      const bool f = k < k1 && Tr<T>::fin(dsk[u]) && Tr<T>::fin(dkt[u]) &&
                     Tr<T, SR>::tight(Tr<T, SR>::add(dsk[u], dkt[u]), st, tau);
      const unsigned bal = __ballot_sync(0xffffffffu, f);
      if (bal) {
        int pos0 = 0;
        if (lane == 0) pos0 = atomicAdd(cnt + b, __popc(bal));
        pos0 = __shfl_sync(0xffffffffu, pos0, 0);
        const int pos = pos0 + __popc(bal & ((1u << lane) - 1));
        if (f && pos < qcap) { out[pos] = (int)k; outd[pos] = dsk[u]; }
      }
    }
  }
}

// shared memory of k_query_solve (one warp per CTA); candidate sets larger
// than kSmall use the per-query global scratch instead
constexpr int kSmall = 512;
template <typename T>
struct QSolveSmem {
  int ids[kSmall];
  T dsv[kSmall];   // D[s][ids[x]]
  T lab[kSmall];
  int pred[kSmall];
  int path[kSmall];
  unsigned char done[kSmall];
};

// per-query global scratch (slot b of the chunk, qcap entries each)
template <typename T>
struct QScratch {
  int* ids;            // candidate ids (written by the scan)
  T* dsv;              // D[s][id] (written by the scan)
  T* lab;
  int* pred;
  int* path;
  unsigned char* done;
  int qcap;
};

__device__ __forceinline__ void warp_argmin(unsigned long long& key, int& pos) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    const unsigned long long k2 = __shfl_xor_sync(0xffffffffu, key, o);
    const int p2 = __shfl_xor_sync(0xffffffffu, pos, o);
    if (k2 < key) { key = k2; pos = p2; }
  }
}

template <typename T>
__device__ __forceinline__ unsigned long long qkey(T v, int id) {
  return ((unsigned long long)Tr<T>::key(v) << 32) | (unsigned)id;
}

template <typename T, int SR>
__global__ void __launch_bounds__(32) k_query_solve(
    const T* __restrict__ D, int64_t ld, const T* __restrict__ WT, int64_t ldw, int64_t n, int q,
    const int* __restrict__ S, const int* __restrict__ Tq, const int* __restrict__ cnt,
    QScratch<T> gs, T* dist, int* paths, int path_cap, int* path_lens, int* ncand, QShard<T> sh,
    const int* __restrict__ perm = nullptr /* output slot of query b (t-grouped batches), or null: b */) {
  __shared__ QSolveSmem<T> sm;
  const int lane = threadIdx.x;
  const T I = Tr<T>::inf();

  for (int b = blockIdx.x; b < q; b += gridDim.x) {
    const int ob = perm ? perm[b] : b;   // (scratch is indexed by b, the outputs by ob)
    const int s = S[b], t = Tq[b];
    const bool bad = s < 0 || s >= n || t < 0 || t >= n;
    if (sh.colbuf && !sh.rowbuf) {
      // sharded: the owner of row s answers (rank 0 answers invalid pairs);
      // every other rank contributes zeros to the all-reduce(sum)
      const bool mine = bad ? sh.row0 == 0 : (s >= sh.row0 && s < sh.row0 + sh.rows);
      if (!mine) {
        if (lane == 0) { path_lens[ob] = 0; if (ncand) ncand[ob] = 0; dist[ob] = T(0); }
        for (int c = lane; c < path_cap; c += 32) paths[(int64_t)ob * path_cap + c] = 0;
        continue;
      }
      for (int c = lane; c < path_cap; c += 32) paths[(int64_t)ob * path_cap + c] = -1;
      __syncwarp();
    }
    if (bad) {
      if (lane == 0) { path_lens[ob] = -3; if (ncand) ncand[ob] = 0; dist[ob] = I; }
      continue;
    }
    const T st = sh.rowbuf ? sh.rowbuf[(int64_t)b * sh.ldr + t] : D[((int64_t)s - sh.row0) * ld + t];
    if (s == t || !Tr<T>::fin(st)) {
      if (lane == 0) {
        dist[ob] = s == t ? T(0) : I;
        if (s == t) {
          if (path_cap >= 1) { paths[(int64_t)ob * path_cap] = s; path_lens[ob] = 1; }
          else path_lens[ob] = -1;
        } else {
          path_lens[ob] = 0;
        }
        if (ncand) ncand[ob] = s == t ? 1 : 0;
      }
      continue;
    }
    const int c = cnt[b];
    if (c > gs.qcap) {
      if (lane == 0) { path_lens[ob] = -2; if (ncand) ncand[ob] = c; dist[ob] = st; }
      continue;
    }
    const int64_t slot = (int64_t)b * gs.qcap;
    const bool small = c <= kSmall;
    int* ids = small ? sm.ids : gs.ids + slot;
    T* dsv = small ? sm.dsv : gs.dsv + slot;
    T* lab = small ? sm.lab : gs.lab + slot;
    int* pred = small ? sm.pred : gs.pred + slot;
    int* path = small ? sm.path : gs.path + slot;
    unsigned char* done = small ? sm.done : gs.done + slot;
    int is = -1, it = -1;
    for (int x = lane; x < c; x += 32) {
      const int id = gs.ids[slot + x];
      const T d = gs.dsv[slot + x];
      if (small) { ids[x] = id; dsv[x] = d; }
      if (id == s) is = x;
      if (id == t) it = x;
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      is = max(is, __shfl_xor_sync(0xffffffffu, is, o));
      it = max(it, __shfl_xor_sync(0xffffffffu, it, o));
    }
    __syncwarp();
    if (is < 0 || it < 0) {   // cannot happen: s and t satisfy the equality
      if (lane == 0) { path_lens[ob] = -2; if (ncand) ncand[ob] = c; dist[ob] = st; }
      continue;
    }

    int len = -1;   // path length found (path[] holds it backwards, t first)
    if (SR == 0 && !Tr<T>::kFloat) {
      // ---- predecessor walk with the known labels (int32 shortest path) ----
      int cur = it, hops = 0;
      if (lane == 0) path[0] = it;
      while (cur != is && hops < c) {
        const T dc = dsv[cur];
        const unsigned long long kc = qkey<T>(dc, ids[cur]);
        const T* wrow = WT + (int64_t)ids[cur] * ldw;   // W[m][cur] = WT[cur][m]
        unsigned long long best = ~0ull;
        int bpos = -1;
        for (int x = lane; x < c; x += 32) {
          const unsigned long long kx = qkey<T>(dsv[x], ids[x]);
          if (kx < kc) {
            const T w = wrow[ids[x]];
            if (Tr<T>::fin(w) && Tr<T>::add(dsv[x], w) == dc && kx < best) { best = kx; bpos = x; }
          }
        }
        warp_argmin(best, bpos);
        if (bpos < 0) break;   // no settled predecessor: a zero-weight hop (see above)
        cur = bpos;
        ++hops;
        if (lane == 0) path[hops] = cur;
      }
      if (cur == is) len = hops + 1;
      __syncwarp();
    }
    if (len < 0) {
      // ---- Dijkstra on the candidate subgraph ----
      for (int x = lane; x < c; x += 32) { lab[x] = I; pred[x] = -1; done[x] = 0; }
      __syncwarp();
      if (lane == 0) lab[is] = T(0);
      __syncwarp();
      for (int iter = 0; iter < c; ++iter) {
        unsigned long long best = ~0ull;
        int m = -1;
        for (int x = lane; x < c; x += 32)
          if (!done[x]) {
            const unsigned long long key = qkey<T>(lab[x], ids[x]);
            if (key < best) { best = key; m = x; }
          }
        warp_argmin(best, m);
        if (m < 0) break;
        const T lm = lab[m];
        if (!Tr<T>::fin(lm)) break;
        __syncwarp();
        if (lane == 0) done[m] = 1;
        __syncwarp();
        if (m == it) break;
        const int64_t gm = ids[m];
        for (int x = lane; x < c; x += 32) {
          if (done[x]) continue;
          const T w = WT[(int64_t)ids[x] * ldw + gm];   // W[m][x]
          if (!Tr<T>::fin(w)) continue;
          const T cd = Tr<T, SR>::add(lm, w);
          if (cd < lab[x]) { lab[x] = cd; pred[x] = m; }
        }
        __syncwarp();
      }
      if (lane == 0) {
        int l = 0, last = -1;
        for (int x = it; x >= 0 && l < c; x = (x == is) ? -1 : pred[x]) { path[l++] = x; last = x; }
        len = last == is ? l : -1;
      }
      len = __shfl_sync(0xffffffffu, len, 0);
    }
    // ---- output: the path s -> t in original ids ----
    __syncwarp();
    if (lane == 0) {
      dist[ob] = st;
      if (ncand) ncand[ob] = c;
      path_lens[ob] = len < 0 ? -2 : (len > path_cap ? -1 : len);
    }
    if (len > 0 && len <= path_cap) {
      int* o = paths + (int64_t)ob * path_cap;
      for (int x = lane; x < len; x += 32) o[x] = ids[path[len - 1 - x]];
    }
    __syncwarp();
  }
}

// out[b * R + i] = D[row0 + i][t_b] for local rows i < rows, INF for i in [rows, R)
// (also for an out-of-range t_b).  4-byte strided reads: sector-bound (32 B per
// entry), the sharded counterpart of the scan's column reads.
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

// ---- gather-free sharded queries (f3) -------------------------------------
// rowbuf[b * ldr + j] = D[s_b][j] if this rank owns row s_b, else 0 (summed
// over the ranks next)
template <typename T>
__global__ void k_query_rowsend(const T* __restrict__ D, int64_t ld, int64_t row0, int64_t rows, int64_t n,
                                const int* __restrict__ S, int qc, T* rowbuf, int64_t ldr) {
  const int b = blockIdx.y;
  const int s = S[b];
  const bool mine = s >= row0 && s < row0 + rows && s < n;
  for (int64_t j = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; j < ldr; j += (int64_t)gridDim.x * blockDim.x)
    rowbuf[b * ldr + j] = (mine && j < n) ? D[((int64_t)s - row0) * ld + j] : T(0);
}
// hits[b * (hcap + 1)] = |C ∩ local rows| of query b, then their ids (global)
template <typename T, int SR>
__global__ void k_query_localscan(const T* __restrict__ D, int64_t ld, int64_t row0, int64_t rows, int64_t n,
                                  const int* __restrict__ S, const int* __restrict__ Tq, const T* __restrict__ rowbuf,
                                  int64_t ldr, int* hits, int hcap, float tau, T wmin) {
  const int b = blockIdx.y;
  const int s = S[b], t = Tq[b];
  int* out = hits + (int64_t)b * (hcap + 1);
  if (s < 0 || s >= n || t < 0 || t >= n || s == t) return;
  const T* Rs = rowbuf + (int64_t)b * ldr;
  const T st = Rs[t];
  if (!Tr<T>::fin(st)) return;
  T lim;
  if (SR == 1) lim = st;
  else if (Tr<T>::kFloat) lim = st * (1.0f + tau);
  else lim = st - wmin;
  const int lane = threadIdx.x & 31;
  const int64_t hi = min(rows, n - row0);
  for (int64_t l0 = blockIdx.x * (int64_t)blockDim.x; l0 < hi; l0 += (int64_t)gridDim.x * blockDim.x) {
    const int64_t l = l0 + threadIdx.x;
    const int64_t k = row0 + l;
    bool f = false;
    if (l < hi) {
      const T dsk = Rs[k];
      if (Tr<T>::fin(dsk) && (dsk <= lim || k == t)) {
        const T dkt = D[l * ld + t];
        f = Tr<T>::fin(dkt) && Tr<T, SR>::tight(Tr<T, SR>::add(dsk, dkt), st, tau);
      }
    }
    const unsigned bal = __ballot_sync(0xffffffffu, f);
    if (bal) {
      int pos0 = 0;
      if (lane == 0) pos0 = atomicAdd(out, __popc(bal));
      pos0 = __shfl_sync(0xffffffffu, pos0, 0);
      const int pos = pos0 + __popc(bal & ((1u << lane) - 1));
      if (f && pos < hcap) out[1 + pos] = (int)k;
    }
  }
}
// the candidate set of query b from every rank's hits -> the solve's scratch
// (ids, D[s][id], |C|); |C| > qcap is left to the solve's capacity check
template <typename T>
__global__ void k_query_mergehits(const int* __restrict__ all, int world, int qc, int hcap, const T* __restrict__ rowbuf,
                                  int64_t ldr, int* ids, T* dsv, int qcap, int* cnt) {
  const int b = blockIdx.x;
  int base = 0;
  for (int rk = 0; rk < world; ++rk) {
    const int* h = all + ((int64_t)rk * qc + b) * (hcap + 1);
    const int c = min(h[0], hcap);
    for (int x = threadIdx.x; x < c; x += blockDim.x) {
      const int pos = base + x;
      if (pos < qcap) {
        const int k = h[1 + x];
        ids[(int64_t)b * qcap + pos] = k;
        dsv[(int64_t)b * qcap + pos] = rowbuf[(int64_t)b * ldr + k];
      }
    }
    base += h[0];
  }
  if (threadIdx.x == 0) cnt[b] = base;
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

template <typename T, int SR>
cudaError_t query_launch(const T* D, int64_t ld, const T* WT, int64_t ldw, int64_t n, int q,
                         const int* s, const int* t, T* dist, int* paths, int path_cap,
                         int* path_lens, int* ncand, float tau, cudaStream_t st, QShard<T> sh,
                         const QueryScratch& qs, T wmin, const int* perm = nullptr) {
  cudaError_t e = cudaMemsetAsync(qs.cnt, 0, sizeof(int) * q, st);
  if (e != cudaSuccess) return e;
  // node chunks: >= 4 CTAs per SM over the whole grid, >= 1 step per CTA
  const int64_t step = (int64_t)QS_T * QS_U;
  const int64_t steps = (n + step - 1) / step;
  int64_t nch = std::max<int64_t>(1, ((int64_t)num_sms() * 4 + q - 1) / q);
  nch = std::min(nch, steps);
  const int64_t chunk = (steps + nch - 1) / nch * step;
  nch = (n + chunk - 1) / chunk;
  T* cand_d = reinterpret_cast<T*>(qs.dsv);
  k_query_scan<T, SR><<<dim3((unsigned)nch, (unsigned)q), QS_T, 0, st>>>(
      D, ld, n, s, t, chunk, qs.ids, cand_d, qs.qcap, qs.cnt, tau, wmin, sh);
  e = cudaGetLastError();
  if (e != cudaSuccess) return e;
  QScratch<T> gs{qs.ids, cand_d, reinterpret_cast<T*>(qs.lab), qs.pred, qs.path, qs.done, qs.qcap};
  const int grid = std::min(q, num_sms() * 16);
  k_query_solve<T, SR><<<grid, 32, 0, st>>>(D, ld, WT, ldw, n, q, s, t, qs.cnt, gs, dist, paths,
                                            path_cap, path_lens, ncand, sh, perm);
  return cudaGetLastError();
}

// t-grouped batches (f3: "very large batches grouped by t"): the
// queries of a group sorted by t, so that the queries sharing a target run
// back to back and column t — the scan's expensive read, one sector per
// entry — comes from L2 after its first reader.  keys/vals: t and the
// original slot of each query of the group; the solve writes each answer to
// its original slot (perm).
__global__ void k_qgroup_init(const int* __restrict__ t, int b0, int c, int* keys, int* vals) {
  for (int b = blockIdx.x * blockDim.x + threadIdx.x; b < c; b += gridDim.x * blockDim.x) {
    keys[b] = t[b0 + b];
    vals[b] = b0 + b;
  }
}
__global__ void k_qgroup_gather(const int* __restrict__ s, const int* __restrict__ vals, int c, int* s_out) {
  for (int b = blockIdx.x * blockDim.x + threadIdx.x; b < c; b += gridDim.x * blockDim.x) s_out[b] = s[vals[b]];
}
// bytes of cub temp storage a group sort needs (host query, no launch)
size_t query_group_temp_bytes() {
  size_t bytes = 0;
  cub::DeviceRadixSort::SortPairs(nullptr, bytes, (const int*)nullptr, (int*)nullptr, (const int*)nullptr,
                                  (int*)nullptr, kQueryGroup, 0, 32);
  return bytes;
}

// Gather-free sharded chunk (qc <= qs.batch queries): phases 1 and 2 of f3
// (the caller runs the two collectives between them and solve_sharded).
template <typename T>
cudaError_t query_rowsend(const T* D, int64_t ld, int64_t row0, int64_t rows, int64_t n, const int* s, int qc,
                          T* rowbuf, int64_t ldr, cudaStream_t st) {
  const int bx = (int)std::min<int64_t>((ldr + 255) / 256, 64);
  k_query_rowsend<T><<<dim3(bx, qc), 256, 0, st>>>(D, ld, row0, rows, n, s, qc, rowbuf, ldr);
  return cudaGetLastError();
}
template <typename T>
cudaError_t query_localscan(const T* D, int64_t ld, int64_t row0, int64_t rows, int64_t n, const int* s,
                            const int* t, int qc, const T* rowbuf, int64_t ldr, int* hits, int hcap, float tau,
                            int sr, T wmin, cudaStream_t st) {
  cudaError_t e = cudaMemsetAsync(hits, 0, sizeof(int) * (size_t)qc * (hcap + 1), st);
  if (e != cudaSuccess) return e;
  const int bx = (int)std::max<int64_t>(1, std::min<int64_t>((rows + 255) / 256, (int64_t)num_sms() * 4 / std::max(qc, 1) + 1));
  if (sr)
    k_query_localscan<T, 1><<<dim3(bx, qc), 256, 0, st>>>(D, ld, row0, rows, n, s, t, rowbuf, ldr, hits, hcap, tau, wmin);
  else
    k_query_localscan<T, 0><<<dim3(bx, qc), 256, 0, st>>>(D, ld, row0, rows, n, s, t, rowbuf, ldr, hits, hcap, tau, wmin);
  return cudaGetLastError();
}
template <typename T>
cudaError_t query_solve_sharded(const T* D, int64_t ld, const T* WT, int64_t ldw, int64_t n, int qc, const int* s,
                                const int* t, T* dist, int* paths, int path_cap, int* path_lens, int* ncand,
                                float tau, int sr, const int* allhits, int world, int hcap, const T* rowbuf,
                                int64_t ldr, const QueryScratch& qs, cudaStream_t st) {
  T* cand_d = reinterpret_cast<T*>(qs.dsv);
  k_query_mergehits<T><<<qc, 256, 0, st>>>(allhits, world, qc, hcap, rowbuf, ldr, qs.ids, cand_d, qs.qcap, qs.cnt);
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return e;
  QScratch<T> gs{qs.ids, cand_d, reinterpret_cast<T*>(qs.lab), qs.pred, qs.path, qs.done, qs.qcap};
  QShard<T> sh{nullptr, 0, 0, 0, qc, rowbuf, ldr};
  const int grid = std::min(qc, num_sms() * 16);
  if (sr)
    k_query_solve<T, 1><<<grid, 32, 0, st>>>(D, ld, WT, ldw, n, qc, s, t, qs.cnt, gs, dist, paths, path_cap,
                                             path_lens, ncand, sh);
  else
    k_query_solve<T, 0><<<grid, 32, 0, st>>>(D, ld, WT, ldw, n, qc, s, t, qs.cnt, gs, dist, paths, path_cap,
                                             path_lens, ncand, sh);
  return cudaGetLastError();
}

template <typename T>
cudaError_t query_batch(const T* D, int64_t ld, const T* WT, int64_t ldw, int64_t n, int q,
                        const int* s, const int* t, T* dist, int* paths, int path_cap,
                        int* path_lens, int* ncand, float tau, int sr, cudaStream_t st,
                        const QueryScratch& qs, T wmin, const T* colbuf, int64_t R, int64_t row0,
                        int64_t rows) {
  if (q <= 0) return cudaSuccess;
  if (colbuf && q > qs.batch) return cudaErrorInvalidValue;   // the host chunks sharded batches
  if (!colbuf && q > qs.batch && qs.sort) {   // large batch: t-grouped, kQueryGroup queries per sort
    int* keys_in = qs.sort;
    int* keys_out = keys_in + kQueryGroup;
    int* vals_in = keys_out + kQueryGroup;
    int* vals_out = vals_in + kQueryGroup;
    void* temp = vals_out + kQueryGroup;
    int bits = 1;
    while (bits < 31 && (int64_t(1) << bits) < n) ++bits;
    for (int g0 = 0; g0 < q; g0 += kQueryGroup) {
      const int c = std::min(kQueryGroup, q - g0);
      const int blocks = (c + 255) / 256;
      k_qgroup_init<<<blocks, 256, 0, st>>>(t, g0, c, keys_in, vals_in);
      size_t tb = qs.sort_temp;
      cudaError_t e = cub::DeviceRadixSort::SortPairs(temp, tb, keys_in, keys_out, vals_in, vals_out, c, 0, bits, st);
      if (e != cudaSuccess) return e;
      k_qgroup_gather<<<blocks, 256, 0, st>>>(s, vals_out, c, keys_in);   // keys_in := s in t order
      for (int b0 = 0; b0 < c; b0 += qs.batch) {
        const int cc = std::min(qs.batch, c - b0);
        QShard<T> sh{nullptr, 0, 0, 0, cc, nullptr, 0};
        e = sr ? query_launch<T, 1>(D, ld, WT, ldw, n, cc, keys_in + b0, keys_out + b0, dist, paths, path_cap,
                                    path_lens, ncand, tau, st, sh, qs, wmin, vals_out + b0)
               : query_launch<T, 0>(D, ld, WT, ldw, n, cc, keys_in + b0, keys_out + b0, dist, paths, path_cap,
                                    path_lens, ncand, tau, st, sh, qs, wmin, vals_out + b0);
        if (e != cudaSuccess) return e;
      }
    }
    return cudaGetLastError();
  }
  for (int b0 = 0; b0 < q; b0 += qs.batch) {
    const int c = std::min(qs.batch, q - b0);
    QShard<T> sh{colbuf, R, colbuf ? row0 : 0, rows, c, nullptr, 0};
    int* pb = path_cap > 0 ? paths + (int64_t)b0 * path_cap : paths;
    int* nc = ncand ? ncand + b0 : nullptr;
    cudaError_t e = sr ? query_launch<T, 1>(D, ld, WT, ldw, n, c, s + b0, t + b0, dist + b0, pb, path_cap,
                                            path_lens + b0, nc, tau, st, sh, qs, wmin)
                       : query_launch<T, 0>(D, ld, WT, ldw, n, c, s + b0, t + b0, dist + b0, pb, path_cap,
                                            path_lens + b0, nc, tau, st, sh, qs, wmin);
    if (e != cudaSuccess) return e;
  }
  return cudaSuccess;
}

// ---------------------------------------------------------------------------
// Queries whose candidate set exceeds the per-query scratch (|C| > qcap, e.g.
// the directed unit cycle, where C is the whole arc and the path has n
// nodes): the same predecessor tree as the walk above, computed for every
// candidate at once instead of hop by hop.
//   k_qbig_bits: C as a bitmap (the scan's test, no capacity);
//   k_qbig_pred: for each k in C (one warp), pred[k] = the first m in
//     (D[s][m], id) order with m in C, key(m) < key(k) and D[s][m] + W[m][k]
//     == D[s][k] (fp32: the tolerant test of Q4) — row k of WT and row s of D
//     are read contiguously;
//   k_qbig_walk: t, pred[t], ... until s (one thread), the path written
//     forward.  Positive weights make the keys strictly decrease, so the walk
//     ends at s within |C| hops (R3); a zero-weight tie can leave a node
//     without a predecessor, and the walk then reports failure (-2).
// Shortest-path algebra only (minimax: -2 as before).
// ---------------------------------------------------------------------------
template <typename T>
__global__ void k_qbig_bits(const T* __restrict__ D, int64_t ld, int64_t n, int s, int t, unsigned* bits,
                            int* cnt, float tau, T wmin) {
  const T* Ds = D + (int64_t)s * ld;
  const T st = Ds[t];
  T lim;
  if (Tr<T>::kFloat) lim = st * (1.0f + tau);
  else lim = st - wmin;
  for (int64_t w = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; w < (n + 31) / 32;
       w += (int64_t)gridDim.x * blockDim.x) {
    unsigned m = 0;
    for (int e = 0; e < 32; ++e) {
      const int64_t k = 32 * w + e;
      if (k >= n) break;
      const T dsk = Ds[k];
      if (!Tr<T>::fin(dsk) || !(dsk <= lim || k == t)) continue;
      const T dkt = D[k * ld + t];
      if (Tr<T>::fin(dkt) && Tr<T>::tight(Tr<T>::add(dsk, dkt), st, tau)) m |= 1u << e;
    }
    bits[w] = m;
    if (m) atomicAdd(cnt, __popc(m));
  }
}
template <typename T>
__global__ void k_qbig_pred(const T* __restrict__ D, int64_t ld, const T* __restrict__ WT, int64_t ldw, int64_t n,
                            int s, const unsigned* __restrict__ bits, int* pred, float tau) {
  const int lane = threadIdx.x & 31;
  const T* Ds = D + (int64_t)s * ld;
  const int64_t nw = (int64_t)gridDim.x * (blockDim.x >> 5);
  for (int64_t k = blockIdx.x * (int64_t)(blockDim.x >> 5) + (threadIdx.x >> 5); k < n; k += nw) {
    if (!((bits[k >> 5] >> (k & 31)) & 1u) || k == s) continue;   // warp-uniform
    const T dk = Ds[k];
    const unsigned long long kk = ((unsigned long long)Tr<T>::key(dk) << 32) | (unsigned)k;
    const T* wrow = WT + k * ldw;   // W[m][k] = WT[k][m]
    unsigned long long best = ~0ull;
    for (int64_t m = lane; m < n; m += 32) {
      if (!((bits[m >> 5] >> (m & 31)) & 1u)) continue;
      const T dm = Ds[m];
      const unsigned long long km = ((unsigned long long)Tr<T>::key(dm) << 32) | (unsigned)m;
      if (km >= kk || km >= best) continue;
      const T w = wrow[m];
      if (!Tr<T>::fin(w)) continue;
      const T via = Tr<T>::add(dm, w);
      const bool eq = Tr<T>::kFloat ? Tr<T>::tight(via, dk, tau) : via == dk;
      if (eq) best = km;
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) best = min(best, __shfl_xor_sync(0xffffffffu, best, o));
    if (lane == 0) pred[k] = best == ~0ull ? -1 : (int)(best & 0xFFFFFFFFull);
  }
}
// out[0] = path length (or -2: no chain to s), path written forward into out + 1
__global__ void k_qbig_walk(int s, int t, const int* __restrict__ pred, int64_t n, int* out, int cap) {
  if (threadIdx.x != 0 || blockIdx.x != 0) return;
  int len = 1;
  int cur = t;
  while (cur != s && len <= n) {
    cur = pred[cur];
    if (cur < 0) { out[0] = -2; return; }
    ++len;
  }
  if (cur != s) { out[0] = -2; return; }
  out[0] = len;
  if (len > cap) return;
  cur = t;
  for (int x = len - 1; x >= 0; --x) {
    out[1 + x] = cur;
    if (x) cur = pred[cur];
  }
}
template <typename T>
cudaError_t query_big(const T* D, int64_t ld, const T* WT, int64_t ldw, int64_t n, int s, int t, unsigned* bits,
                      int* pred, int* cnt, int* out, int cap, float tau, T wmin, cudaStream_t st) {
  CUDA_TRY(cudaMemsetAsync(cnt, 0, sizeof(int), st));
  const int wwords = (int)((n + 31) / 32);
  k_qbig_bits<T><<<std::max(1, std::min((wwords + 255) / 256, num_sms() * 4)), 256, 0, st>>>(D, ld, n, s, t, bits,
                                                                                            cnt, tau, wmin);
  CUDA_TRY(cudaGetLastError());
  k_qbig_pred<T><<<num_sms() * 8, 256, 0, st>>>(D, ld, WT, ldw, n, s, bits, pred, tau);
  CUDA_TRY(cudaGetLastError());
  k_qbig_walk<<<1, 32, 0, st>>>(s, t, pred, n, out, cap);
  return cudaGetLastError();
}

#define INST(T)                                                                                  \
  template cudaError_t query_big<T>(const T*, int64_t, const T*, int64_t, int64_t, int, int, unsigned*, int*, \
                                    int*, int*, int, float, T, cudaStream_t);                    \
  template cudaError_t query_batch<T>(const T*, int64_t, const T*, int64_t, int64_t, int,       \
                                      const int*, const int*, T*, int*, int, int*, int*, float,  \
                                      int, cudaStream_t, const QueryScratch&, T, const T*, int64_t, \
                                      int64_t, int64_t);                                         \
  template cudaError_t query_colslice<T>(const T*, int64_t, int64_t, int64_t, int64_t,          \
                                         const int*, int, T*, cudaStream_t);                     \
  template cudaError_t query_rowsend<T>(const T*, int64_t, int64_t, int64_t, int64_t, const int*, int, T*, \
                                        int64_t, cudaStream_t);                                  \
  template cudaError_t query_localscan<T>(const T*, int64_t, int64_t, int64_t, int64_t, const int*, const int*, \
                                          int, const T*, int64_t, int*, int, float, int, T, cudaStream_t); \
  template cudaError_t query_solve_sharded<T>(const T*, int64_t, const T*, int64_t, int64_t, int, const int*, \
                                              const int*, T*, int*, int, int*, int*, float, int, const int*, int, \
                                              int, const T*, int64_t, const QueryScratch&, cudaStream_t);
INST(int32_t)
INST(float)
#undef INST

}  // namespace apsp
