// sparse.cu — sparse affected-pair recompute.
//
// The paper recomputes every affected source with Dijkstra ("If the Cost is
// small, we use Dijkstra's algorithm to calculate a node's distance to other
// nodes in the new graph").  On the GPU the work is re-expressed at
// pair level: only the listed pairs (i, j) of the need_update_list are
// recomputed, from the Bellman equation of their last hop
//     D'[i][j] = min_m D'[i][m] + W'[m][j]                         (*)
// on D0 (listed entries reset to W'[i][j]; unlisted entries are exact by
// Theorem 4 / Corollary 3).  Three facts make it cheap:
//  (a) lower bound: distances never decrease under a removal / increase, so
//      lb = D_old[i][j] <= D'[i][j]; an upper bound that reaches lb is final.
//      (Most listed pairs are ties — another shortest path avoids the
//      removed element — and are certified this way.)
//  (b) shortlist: per node j the library keeps SL(j), a set of in-edges
//      (m, W[m][j]) and a bound wnext(j) <= W[m][j] for every in-edge NOT in
//      SL(j).  Since D >= 0, if min over SL(j) of D[i][m] + W[m][j] is
//      <= wnext(j), it equals the min over all m of (*) for the current D.
//  (c) only pairs neither certified by (a) nor exact by (b) need the full
//      O(n) scan of row i of D against row j of WT.
// Affected m can still improve after a pair was evaluated (chains in the
// affected set), so open pairs are re-relaxed over the open entries of their
// own row until no entry changes.  A fixpoint of these upper bounds is the
// exact distance.  Rows read only their own D row and the
// read-only WT / shortlists, so rows never race and no grid sync is needed.
#include <cooperative_groups.h>

#include "common.cuh"
#include "kernels.h"
#include "mirror.cuh"

namespace apsp {

static inline int64_t cdiv(int64_t a, int64_t b) { return (a + b - 1) / b; }

// ---------------------------------------------------------------------------
// shortlists: lane-local top-kSLK in-edges of node j (kSL = 32 * kSLK entries)
// ---------------------------------------------------------------------------
// Sort SL(j) ascending by (weight, id) (dead entries — id -1, INF — sink to
// the end): a warp-level bitonic network on the 512 entries held in registers
// (entry t * 32 + lane in slot t of the lane), compare-exchanges across slots
// in-register and across lanes by shuffles.  Phase A then finds the cheapest
// in-edges — the likeliest last hops of a tie — in the first positions.  Runs
// at build (the previous in-global-memory network was latency-bound: ~100 us
// per list on the add-node side stream).
template <typename T>
__device__ __forceinline__ bool sl_less(T wa, int ia, T wb, int ib) {
  return wa < wb || (wa == wb && ia < ib);
}
template <typename T, int TJ>
__device__ __forceinline__ void sl_stage_slots(T (&w)[kSLK], int (&id)[kSLK], int k, int lane) {
#pragma unroll
  for (int t = 0; t < kSLK; ++t) {
    if ((t & TJ) == 0) {
      const int t2 = t | TJ;
      const bool up = (((t << 5) | lane) & k) == 0;
      const bool sw = up ? sl_less(w[t2], id[t2], w[t], id[t]) : sl_less(w[t], id[t], w[t2], id[t2]);
      if (sw) {
        const T tw = w[t]; w[t] = w[t2]; w[t2] = tw;
        const int ti = id[t]; id[t] = id[t2]; id[t2] = ti;
      }
    }
  }
}
template <typename T>
__device__ void sl_sort_regs(T (&w)[kSLK], int (&id)[kSLK]) {
  static_assert(kSLK == 16, "slot stages below are written for 16 slots per lane");
  const int lane = threadIdx.x & 31;
  for (int k = 2; k <= kSL; k <<= 1)
    for (int jj = k >> 1; jj > 0; jj >>= 1) {
      if (jj >= 32) {
        switch (jj >> 5) {
          case 1: sl_stage_slots<T, 1>(w, id, k, lane); break;
          case 2: sl_stage_slots<T, 2>(w, id, k, lane); break;
          case 4: sl_stage_slots<T, 4>(w, id, k, lane); break;
          default: sl_stage_slots<T, 8>(w, id, k, lane); break;
        }
      } else {
        const bool lower = (lane & jj) == 0;
#pragma unroll
        for (int t = 0; t < kSLK; ++t) {
          const T ow = __shfl_xor_sync(0xffffffffu, w[t], jj);
          const int oi = __shfl_xor_sync(0xffffffffu, id[t], jj);
          const bool up = (((t << 5) | lane) & k) == 0;
          // the lower index of the pair keeps the min when ascending, else the max
          const bool take = (lower == up) ? sl_less(ow, oi, w[t], id[t]) : sl_less(w[t], id[t], ow, oi);
          if (take) { w[t] = ow; id[t] = oi; }
        }
      }
    }
}

// Replace slot `bq` of a sorted SL(j) by (m, w) keeping the live entries in
// ascending order (dead entries — INF — may sit anywhere): p = the first live
// entry heavier than w; the entries between p and bq shift by one.  One warp,
// two passes over the 512 entries (a full re-sort per insertion was too heavy
// for the add-node side stream).
template <typename T>
__device__ void sl_place_warp(int* sid, T* sw, int bq, int m, T w) {
  const int lane = threadIdx.x & 31;
  int p = kSL;
#pragma unroll 4
  for (int t = 0; t < kSL / 32; ++t) {
    const int e = t * 32 + lane;
    if (e != bq && sid[e] >= 0 && sw[e] > w) p = min(p, e);
  }
  p = __reduce_min_sync(0xffffffffu, p);
  // target slot of (m, w): before p if p <= bq (shift [p, bq) right), else
  // just before p after shifting (bq, p) left; p == kSL means "at the end"
  const int lo = p <= bq ? p : bq + 1, hi = p <= bq ? bq : p;   // moved range [lo, hi)
  const int dst = p <= bq ? p : p - 1;
  const int dir = p <= bq ? 1 : -1;
  int ids[kSL / 32];
  T ws[kSL / 32];
#pragma unroll
  for (int t = 0; t < kSL / 32; ++t) {
    const int e = t * 32 + lane;
    if (e >= lo && e < hi) { ids[t] = sid[e]; ws[t] = sw[e]; }
  }
  __syncwarp();
#pragma unroll
  for (int t = 0; t < kSL / 32; ++t) {
    const int e = t * 32 + lane;
    if (e >= lo && e < hi) { sid[e + dir] = ids[t]; sw[e + dir] = ws[t]; }
  }
  __syncwarp();
  if (lane == 0) { sid[dst] = m; sw[dst] = w; }
  __syncwarp();
}

template <typename T>
__global__ void __launch_bounds__(256) k_shortlist_build(const T* __restrict__ WT, int64_t ldw,
                                                         int64_t n, const int* rows, int64_t r0,
                                                         int64_t r1, int* SLid, T* SLw, T* wnext) {
  const int lane = threadIdx.x & 31;
  const int64_t nw = (int64_t)gridDim.x * (blockDim.x >> 5);
  const T I = Tr<T>::inf();
  for (int64_t w = blockIdx.x * (int64_t)(blockDim.x >> 5) + (threadIdx.x >> 5); w < r1 - r0;
       w += nw) {
    const int64_t j = rows ? rows[r0 + w] : r0 + w;
    if (j < 0 || j >= n) continue;
    const T* row = WT + j * ldw;
    T bw[kSLK];
    int bi[kSLK];
#pragma unroll
    for (int q = 0; q < kSLK; ++q) { bw[q] = I; bi[q] = -1; }
    T rej = I;   // smallest weight this lane did not keep
    for (int64_t m = lane; m < n; m += 32) {
      T x = row[m];
      if (m == j || !Tr<T>::fin(x)) continue;
      if (x < bw[kSLK - 1]) {
        rej = Tr<T>::mn(rej, bw[kSLK - 1]);   // the evicted maximum becomes a rejected value
        // sorted insertion (ascending)
        T cw = x;
        int ci = (int)m;
#pragma unroll
        for (int q = 0; q < kSLK; ++q) {
          if (cw < bw[q]) {
            T tw = bw[q]; int ti = bi[q];
            bw[q] = cw; bi[q] = ci;
            cw = tw; ci = ti;
          }
        }
      } else {
        rej = Tr<T>::mn(rej, x);
      }
    }
    sl_sort_regs<T>(bw, bi);
    int* oid = SLid + j * kSL;
    T* ow = SLw + j * kSL;
#pragma unroll
    for (int q = 0; q < kSLK; ++q) {
      oid[q * 32 + lane] = bi[q];
      ow[q * 32 + lane] = bw[q];
    }
    rej = warp_min<T>(rej);
    if (lane == 0) wnext[j] = rej;
  }
}

template <typename T>
cudaError_t shortlist_build(const T* WT, int64_t ldw, int64_t n, const int* rows, int64_t r0,
                            int64_t r1, int* SLid, T* SLw, T* wnext, cudaStream_t st) {
  if (r1 <= r0) return cudaSuccess;
  int grid = (int)std::min<int64_t>(cdiv(r1 - r0, 8), (int64_t)num_sms() * 8);
  k_shortlist_build<T><<<grid, 256, 0, st>>>(WT, ldw, n, rows, r0, r1, SLid, SLw, wnext);
  return cudaGetLastError();
}

// SL(x) of one node (the add-node side stream): the kSL cheapest in-edges by
// (weight, id), exactly, and wnext = the smallest weight left out.  Two
// kernels instead of one CTA walking the row (that was latency-bound at ~117
// us for n = 32768):
//   k_sl_one_part  — CTA g sorts kSLC-entry chunks of the row in shared memory
//                    (bitonic) and keeps a running sorted top-kSL: merged as
//                    min(run[i], chunk[kSL-1-i]) (a bitonic sequence holding the
//                    kSL smallest of both) + a bitonic merge.  Writes its list
//                    and the min of everything it discarded.
//   k_sl_one_merge — one CTA merges the <= kSLG lists pairwise the same way.
// Every in-edge left out was discarded at one step, so it is >= the min over
// all discarded values = wnext(j).
constexpr int kSLC = 1024;   // chunk (one entry per thread)
template <typename T>
__device__ __forceinline__ void sl_cx(T* w, int* id, int lo, int hi) {   // ascending compare-exchange
  const T a = w[lo], b = w[hi];
  const int ia = id[lo], ib = id[hi];
  if (sl_less(b, ib, a, ia)) { w[lo] = b; w[hi] = a; id[lo] = ib; id[hi] = ia; }
}
// bitonic merge of `lists` bitonic sequences of kSL entries each, list q at
// w + q * stride (ascending); all threads of the CTA
template <typename T>
__device__ void sl_merge_lists(T* w, int* id, int lists, int stride) {
  for (int jj = kSL / 2; jj > 0; jj >>= 1) {
    for (int idx = threadIdx.x; idx < lists * (kSL / 2); idx += blockDim.x) {
      const int q = idx / (kSL / 2), t = idx % (kSL / 2);
      const int lo = (t / jj) * 2 * jj + (t % jj);
      sl_cx(w + q * stride, id + q * stride, lo, lo + jj);
    }
    __syncthreads();
  }
}
template <typename T>
__device__ __forceinline__ T sl_block_min(T v, T* red) {
  v = warp_min<T>(v);
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = v;
  __syncthreads();
  if (threadIdx.x < 32) {
    v = threadIdx.x < (blockDim.x >> 5) ? red[threadIdx.x] : Tr<T>::inf();
    v = warp_min<T>(v);
  }
  return v;   // valid in thread 0
}
template <typename T>
__global__ void __launch_bounds__(kSLC) k_sl_one_part(const T* __restrict__ row, int64_t n, int64_t j,
                                                      T* cw_out, int* ci_out, T* rej_out, const int* gate) {
  if (*(volatile const int*)gate == 0) return;   // the selection path did it
  __shared__ T cw[kSLC], rw[kSL];
  __shared__ int ci[kSLC], ri[kSL];
  __shared__ T red[32];
  const int tid = threadIdx.x;
  const T I = Tr<T>::inf();
  T rej = I;
  bool first = true;
  for (int64_t c0 = (int64_t)blockIdx.x * kSLC; c0 < n; c0 += (int64_t)gridDim.x * kSLC) {
    const int64_t e = c0 + tid;
    const T x = e < n ? row[e] : I;
    const bool ok = e < n && e != j && Tr<T>::fin(x);
    cw[tid] = ok ? x : I;
    ci[tid] = ok ? (int)e : -1;
    __syncthreads();
    for (int k = 2; k <= kSLC; k <<= 1)
      for (int jj = k >> 1; jj > 0; jj >>= 1) {
        const int l = tid ^ jj;
        if (l > tid) {
          if ((tid & k) == 0) sl_cx(cw, ci, tid, l);
          else sl_cx(cw, ci, l, tid);
        }
        __syncthreads();
      }
    if (tid >= kSL) rej = Tr<T>::mn(rej, cw[tid]);   // the upper half of the chunk is discarded
    if (first) {
      if (tid < kSL) { rw[tid] = cw[tid]; ri[tid] = ci[tid]; }
      __syncthreads();
    } else {
      if (tid < kSL) {
        const T a = rw[tid], b = cw[kSL - 1 - tid];
        const int ia = ri[tid], ib = ci[kSL - 1 - tid];
        const bool bl = sl_less(b, ib, a, ia);
        rej = Tr<T>::mn(rej, bl ? a : b);
        if (bl) { rw[tid] = b; ri[tid] = ib; }
      }
      __syncthreads();
      sl_merge_lists<T>(rw, ri, 1, 0);
    }
    first = false;
  }
  if (first && tid < kSL) { rw[tid] = I; ri[tid] = -1; }   // (no chunk: launched with fewer CTAs)
  if (tid < kSL) {
    cw_out[(int64_t)blockIdx.x * kSL + tid] = rw[tid];
    ci_out[(int64_t)blockIdx.x * kSL + tid] = ri[tid];
  }
  rej = sl_block_min<T>(rej, red);
  if (tid == 0) rej_out[blockIdx.x] = rej;
}
template <typename T>
__global__ void __launch_bounds__(kSLC) k_sl_one_merge(const T* __restrict__ cw_in, const int* __restrict__ ci_in,
                                                       const T* __restrict__ rej_in, int G, int Gp, int64_t j,
                                                       int* SLid, T* SLw, T* wnext, int* gate) {
  if (*(volatile const int*)gate == 0) return;   // the selection path did it
  extern __shared__ __align__(16) unsigned char sm_raw[];
  T* w = reinterpret_cast<T*>(sm_raw);
  int* id = reinterpret_cast<int*>(sm_raw + sizeof(T) * (size_t)Gp * kSL);
  __shared__ T red[32];
  const int tid = threadIdx.x;
  const T I = Tr<T>::inf();
  T rej = tid < G ? rej_in[tid] : I;
  for (int e = tid; e < Gp * kSL; e += blockDim.x) {
    const bool ok = e < G * kSL;
    w[e] = ok ? cw_in[e] : I;
    id[e] = ok ? ci_in[e] : -1;
  }
  __syncthreads();
  for (int s = 1; s < Gp; s <<= 1) {   // lists q (multiples of 2s) absorb lists q + s
    const int lists = Gp / (2 * s);
    for (int idx = tid; idx < lists * kSL; idx += blockDim.x) {
      const int q = (idx / kSL) * 2 * s, i = idx % kSL;
      const int pa = q * kSL + i, pb = (q + s) * kSL + (kSL - 1 - i);
      const bool bl = sl_less(w[pb], id[pb], w[pa], id[pa]);
      rej = Tr<T>::mn(rej, bl ? w[pa] : w[pb]);
      if (bl) { w[pa] = w[pb]; id[pa] = id[pb]; }
    }
    __syncthreads();
    sl_merge_lists<T>(w, id, lists, 2 * s * kSL);
  }
  if (tid < kSL) {
    SLid[j * kSL + tid] = id[tid];
    SLw[j * kSL + tid] = w[tid];
  }
  rej = sl_block_min<T>(rej, red);
  if (tid == 0) {
    wnext[j] = rej;
    *gate = 0;   // reset for the next call
  }
}

// The selection path (round 2): a histogram of the weights' order-preserving
// 32-bit keys on a log scale (keys < 128 exact, above that 128 bins per power
// of two) finds the bin b* holding the kSL-th smallest entry; one CTA then
// collects every entry in bins <= b* (if at most kSelCap of them), sorts them
// by (weight, id) and keeps the first kSL; wnext = the smallest weight left
// out (a collected entry past kSL, or the smallest entry above b*).  Exactly
// the sort path's result; that path runs instead when bin b* is too full.
constexpr int kSelCap = 4096;
__device__ __forceinline__ int sl_bin(uint32_t k) {
  if (k < 128u) return (int)k;
  const int e = 31 - __clz(k);                         // >= 7
  return (e - 6) * 128 + (int)((k >> (e - 7)) & 127u);   // < (31 - 6) * 128 + 128 = 3328
}
template <typename T>
__device__ __forceinline__ uint32_t sl_key32(T w) {
  uint32_t k;
  memcpy(&k, &w, 4);   // int32 >= 0 and IEEE floats >= 0 order like their bits
  return k;
}
template <typename T>
__global__ void __launch_bounds__(256) k_sl_hist(const T* __restrict__ row, int64_t n, int64_t j, int* hist) {
  __shared__ int h[kSLBins];
  for (int b = threadIdx.x; b < kSLBins; b += blockDim.x) h[b] = 0;
  __syncthreads();
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < n; e += (int64_t)gridDim.x * blockDim.x) {
    const T x = row[e];
    if (e != j && Tr<T>::fin(x)) atomicAdd(&h[sl_bin(sl_key32<T>(x))], 1);
  }
  __syncthreads();
  for (int b = threadIdx.x; b < kSLBins; b += blockDim.x)
    if (h[b]) atomicAdd(hist + b, h[b]);
}
template <typename T>
__global__ void __launch_bounds__(1024) k_sl_select(const T* __restrict__ row, int64_t n, int64_t j, int* hist,
                                                    int* gate, int* SLid, T* SLw, T* wnext) {
  extern __shared__ __align__(16) unsigned long long keys[];   // kSelCap
  __shared__ int cum[1024];
  __shared__ int s_b, s_c;
  __shared__ unsigned long long s_out;
  const int tid = threadIdx.x;
  // per thread 4 consecutive bins: inclusive scan of the bin counts
  int c4[4], tot = 0;
#pragma unroll
  for (int q = 0; q < 4; ++q) { c4[q] = hist[4 * tid + q]; hist[4 * tid + q] = 0; tot += c4[q]; }
  cum[tid] = tot;
  if (tid == 0) { s_b = kSLBins - 1; s_c = 0; s_out = ~0ull; }
  __syncthreads();
  for (int o = 1; o < 1024; o <<= 1) {   // Hillis-Steele scan
    const int v = tid >= o ? cum[tid - o] : 0;
    __syncthreads();
    cum[tid] += v;
    __syncthreads();
  }
  const int total = cum[1023];
  const int want = min(total, kSL);
  {   // the first bin whose inclusive count reaches `want`
    int run = cum[tid] - tot;
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      const int before = run;
      run += c4[q];
      if (want > 0 && before < want && run >= want) { s_b = 4 * tid + q; s_c = run; }
    }
  }
  __syncthreads();
  const int bstar = want > 0 ? s_b : -1, cnt = want > 0 ? s_c : 0;
  if (cnt > kSelCap) {   // bin b* too full: the sort path (gated kernels after this one)
    if (tid == 0) *gate = 1;
    return;
  }
  __syncthreads();
  if (tid == 0) s_c = 0;
  __syncthreads();
  // collect the entries of bins <= b*; the smallest entry above b* for wnext
  unsigned long long out = ~0ull;
  for (int64_t e0 = 0; e0 < n; e0 += 8 * (int64_t)blockDim.x) {   // 8 loads in flight per thread
    T x[8];
#pragma unroll
    for (int q = 0; q < 8; ++q) {
      const int64_t e = e0 + q * (int64_t)blockDim.x + tid;
      x[q] = e < n ? row[e] : Tr<T>::inf();
    }
#pragma unroll
    for (int q = 0; q < 8; ++q) {
      const int64_t e = e0 + q * (int64_t)blockDim.x + tid;
      if (e >= n || e == j || !Tr<T>::fin(x[q])) continue;
      const uint32_t k = sl_key32<T>(x[q]);
      const unsigned long long key = (unsigned long long)k << 32 | (unsigned)e;
      if (sl_bin(k) <= bstar) keys[atomicAdd(&s_c, 1)] = key;
      else out = min(out, key);
    }
  }
  atomicMin(&s_out, out);
  __syncthreads();
  int P = 1;
  while (P < cnt) P <<= 1;
  if (P <= 1024) {   // one key per thread: strides < 32 by shuffles, the rest through shared memory
    unsigned long long x = tid < cnt ? keys[tid] : ~0ull;
    for (int k = 2; k <= 1024; k <<= 1)   // bitonic sort, ascending (weight, id)
      for (int jj = k >> 1; jj > 0; jj >>= 1) {
        unsigned long long y;
        if (jj >= 32) {
          __syncthreads();
          keys[tid] = x;
          __syncthreads();
          y = keys[tid ^ jj];
        } else {
          y = __shfl_xor_sync(0xffffffffu, x, jj);
        }
        const bool up = (tid & k) == 0, lo = (tid & jj) == 0;
        x = (up == lo) ? min(x, y) : max(x, y);
      }
    __syncthreads();
    keys[tid] = x;
    __syncthreads();
  } else {
    for (int e = cnt + tid; e < P; e += blockDim.x) keys[e] = ~0ull;
    __syncthreads();
    for (int k = 2; k <= P; k <<= 1)   // bitonic sort, ascending (weight, id)
      for (int jj = k >> 1; jj > 0; jj >>= 1) {
        for (int i = tid; i < P; i += blockDim.x) {
          const int l = i ^ jj;
          if (l > i) {
            const unsigned long long a = keys[i], b = keys[l];
            if (((i & k) == 0) == (a > b)) { keys[i] = b; keys[l] = a; }
          }
        }
        __syncthreads();
      }
  }
  for (int i = tid; i < kSL; i += blockDim.x) {
    const unsigned long long key = i < cnt ? keys[i] : ~0ull;
    T w;
    const uint32_t k = (uint32_t)(key >> 32);
    memcpy(&w, &k, 4);
    SLid[j * kSL + i] = key == ~0ull ? -1 : (int)(key & 0xFFFFFFFFull);
    SLw[j * kSL + i] = key == ~0ull ? Tr<T>::inf() : w;
  }
  if (tid == 0) {
    const unsigned long long left = min(cnt > kSL ? keys[kSL] : ~0ull, s_out);
    T w = Tr<T>::inf();
    if (left != ~0ull) {
      const uint32_t k = (uint32_t)(left >> 32);
      memcpy(&w, &k, 4);
    }
    wnext[j] = w;
  }
}

template <typename T>
cudaError_t shortlist_build_one(const T* WT, int64_t ldw, int64_t n, int64_t j, int* SLid, T* SLw,
                                T* wnext, void* scratch, cudaStream_t st) {
  const int G = (int)std::max<int64_t>(1, std::min<int64_t>(kSLG, cdiv(n, kSLC)));
  int Gp = 1;
  while (Gp < G) Gp <<= 1;
  int* gate = reinterpret_cast<int*>(scratch);                      // control word 0
  int* hist = reinterpret_cast<int*>(static_cast<char*>(scratch) + 256);
  T* cw = reinterpret_cast<T*>(hist + kSLBins);
  int* ci = reinterpret_cast<int*>(cw + (size_t)kSLG * kSL);
  T* rj = reinterpret_cast<T*>(ci + (size_t)kSLG * kSL);
  const T* row = WT + j * ldw;
  k_sl_hist<T><<<(int)std::min<int64_t>(cdiv(n, 1024), 2 * num_sms()), 256, 0, st>>>(row, n, j, hist);
  CUDA_TRY(cudaGetLastError());
  static bool attr_sel = false;
  if (!attr_sel) {
    CUDA_TRY(cudaFuncSetAttribute(k_sl_select<int32_t>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                  (int)(8 * kSelCap)));
    CUDA_TRY(cudaFuncSetAttribute(k_sl_select<float>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                  (int)(8 * kSelCap)));
    attr_sel = true;
  }
  k_sl_select<T><<<1, 1024, 8 * kSelCap, st>>>(row, n, j, hist, gate, SLid, SLw, wnext);
  CUDA_TRY(cudaGetLastError());
  k_sl_one_part<T><<<G, kSLC, 0, st>>>(row, n, j, cw, ci, rj, gate);
  CUDA_TRY(cudaGetLastError());
  const size_t smem = (sizeof(T) + sizeof(int)) * (size_t)Gp * kSL;
  static bool attr = false;
  if (!attr) {
    CUDA_TRY(cudaFuncSetAttribute(k_sl_one_merge<int32_t>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                  (int)((sizeof(int32_t) + sizeof(int)) * (size_t)kSLG * kSL)));
    CUDA_TRY(cudaFuncSetAttribute(k_sl_one_merge<float>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                  (int)((sizeof(float) + sizeof(int)) * (size_t)kSLG * kSL)));
    attr = true;
  }
  k_sl_one_merge<T><<<1, kSLC, smem, st>>>(cw, ci, rj, G, Gp, j, SLid, SLw, wnext, gate);
  return cudaGetLastError();
}

// Insert in-edge (m -> j, weight w) into SL(j) when it would otherwise have to
// lower wnext(j): evict the heaviest entry instead (its weight joins the
// excluded set, so wnext(j) = min(wnext(j), evicted)).  One warp; the caller
// guarantees m is not already listed.
template <typename T>
__device__ __forceinline__ void shortlist_insert_warp(int* SLid, T* SLw, T* wnext, int64_t j, int m,
                                                      T w) {
  const int lane = threadIdx.x & 31;
  if (!(w < wnext[j])) return;   // warp-uniform: already covered by the bound
  int* sid = SLid + j * kSL;
  T* sw = SLw + j * kSL;
  // warp argmax over the entries (dead entries count as +INF: evicted first)
  T best = -Tr<T>::inf();
  int bq = -1;
#pragma unroll
  for (int q = 0; q < kSLK; ++q) {
    const int e = q * 32 + lane;
    const T x = sid[e] < 0 ? Tr<T>::inf() : sw[e];
    if (x > best || bq < 0) { best = x; bq = e; }
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    const T ob = __shfl_xor_sync(0xffffffffu, best, o);
    const int oq = __shfl_xor_sync(0xffffffffu, bq, o);
    if (ob > best || (ob == best && oq < bq)) { best = ob; bq = oq; }
  }
  if (w < best) {   // warp-uniform (best is the warp's): evict slot bq
    if (lane == 0 && sid[bq] >= 0) wnext[j] = Tr<T>::mn(wnext[j], best);
    sl_place_warp<T>(sid, sw, bq, m, w);
  } else if (lane == 0) {
    wnext[j] = Tr<T>::mn(wnext[j], w);
  }
}

// A new node x adds in-edge x -> j (weight out_w[j]) to every j.
template <typename T>
__global__ void k_shortlist_add_edges(int* SLid, T* SLw, T* wnext, const T* out_w, int64_t n, int x) {
  const int64_t nw = (int64_t)gridDim.x * (blockDim.x >> 5);
  for (int64_t j = blockIdx.x * (int64_t)(blockDim.x >> 5) + (threadIdx.x >> 5); j < n; j += nw)
    shortlist_insert_warp<T>(SLid, SLw, wnext, j, x, out_w[j]);
}
template <typename T>
cudaError_t shortlist_add_bound(int* SLid, T* SLw, T* wnext, const T* out_w, int64_t n, int64_t x,
                                cudaStream_t st) {
  int grid = (int)std::min<int64_t>(cdiv(n, 8), 8 * num_sms());
  k_shortlist_add_edges<T><<<grid, 256, 0, st>>>(SLid, SLw, wnext, out_w, n, (int)x);
  return cudaGetLastError();
}

// Edge u -> v now has weight w: refresh its entry in SL(v) if present,
// otherwise make wnext(v) cover it (one warp).
template <typename T>
__global__ void k_shortlist_set_edge(int* SLid, T* SLw, T* wnext, int64_t u, int64_t v, T w) {
  const int lane = threadIdx.x & 31;
  int at = -1;
#pragma unroll
  for (int q = 0; q < kSLK; ++q) {
    const int e = q * 32 + lane;
    if (SLid[v * kSL + e] == (int)u) at = e;
  }
  at = __reduce_max_sync(0xffffffffu, at);
  if (at >= 0) sl_place_warp<T>(SLid + v * kSL, SLw + v * kSL, at, (int)u, w);   // re-place the entry
  else shortlist_insert_warp<T>(SLid, SLw, wnext, v, (int)u, w);
}
template <typename T>
cudaError_t shortlist_set_edge(int* SLid, T* SLw, T* wnext, int64_t u, int64_t v, T w,
                               int directed, cudaStream_t st) {
  k_shortlist_set_edge<T><<<1, 32, 0, st>>>(SLid, SLw, wnext, u, v, w);
  if (!directed) k_shortlist_set_edge<T><<<1, 32, 0, st>>>(SLid, SLw, wnext, v, u, w);
  return cudaGetLastError();
}

// An edge update's first step on one GPU, one warp: read
// W[u][v] and D[u][v]; if the update exits early — same weight, a decrease
// with w_new >= D[u][v], or an increase of an edge that is not tight — apply
// it here (W, both directions when undirected, and the shortlist entries),
// so the host's one read finds it done.  host (mapped): [0] = W[u][v] and
// [1] = D[u][v] as bits of T, [2] = 1 if applied here.
template <typename T>
__global__ void k_edge_early(T* WT, int64_t ldw, const T* Du, int* SLid, T* SLw, T* wnext, int64_t u, int64_t v,
                             T w, int directed, float tau, unsigned* host) {
  const int lane = threadIdx.x & 31;
  const T w_old = WT[v * ldw + u], duv = Du[v];
  bool early;
  if (w == w_old) early = true;
  else if (w < w_old) early = !(w < duv);
  else if (Tr<T>::kFloat) early = !((double)w_old <= (double)duv * (1.0 + (double)tau));
  else early = w_old != duv;
  if (early && w != w_old) {
    if (lane == 0) {
      WT[v * ldw + u] = w;
      if (!directed) WT[u * ldw + v] = w;
    }
    __syncwarp();
    for (int dir = 0; dir < (directed ? 1 : 2); ++dir) {
      const int64_t a = dir ? v : u, b = dir ? u : v;   // entry a of SL(b)
      int at = -1;
#pragma unroll
      for (int q = 0; q < kSLK; ++q) {
        const int e = q * 32 + lane;
        if (SLid[b * kSL + e] == (int)a) at = e;
      }
      at = __reduce_max_sync(0xffffffffu, at);
      if (at >= 0) sl_place_warp<T>(SLid + b * kSL, SLw + b * kSL, at, (int)a, w);
      else shortlist_insert_warp<T>(SLid, SLw, wnext, b, (int)a, w);
      __syncwarp();
    }
  }
  if (lane == 0) {
    unsigned b0, b1;
    memcpy(&b0, &w_old, sizeof b0);
    memcpy(&b1, &duv, sizeof b1);
    volatile unsigned* hv = host;
    hv[0] = b0;
    hv[1] = b1;
    hv[2] = early ? 1u : 0u;
    __threadfence_system();
  }
}
template <typename T>
cudaError_t edge_early(T* WT, int64_t ldw, const T* Du, int* SLid, T* SLw, T* wnext, int64_t u, int64_t v, T w,
                       int directed, float tau, void* host_dev, cudaStream_t st) {
  k_edge_early<T><<<1, 32, 0, st>>>(WT, ldw, Du, SLid, SLw, wnext, u, v, w, directed, tau,
                                    reinterpret_cast<unsigned*>(host_dev));
  return cudaGetLastError();
}

// Removal of k with node `last` moving into slot k: entries naming k die
// (weight INF), entries naming `last` are renamed k, row k takes row last.
template <typename T>
__global__ void k_shortlist_remove(int* SLid, T* SLw, T* wnext, int64_t n, int k, int last) {
  const int64_t tot4 = n * kSL / 4;   // kSL is a multiple of 4: 16-byte id vectors
  int4* ids4 = reinterpret_cast<int4*>(SLid);
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < tot4;
       e += (int64_t)gridDim.x * blockDim.x) {
    int4 v = ids4[e];
    const bool hk = v.x == k || v.y == k || v.z == k || v.w == k;
    const bool hl = last != k && (v.x == last || v.y == last || v.z == last || v.w == last);
    if (!hk && !hl) continue;   // the common case: one 16-byte read
    int* id = &v.x;
#pragma unroll
    for (int c = 0; c < 4; ++c) {
      if (id[c] == k) { id[c] = -1; SLw[4 * e + c] = Tr<T>::inf(); }
      else if (hl && id[c] == last) id[c] = k;
    }
    ids4[e] = v;
  }
}
template <typename T>
__global__ void k_shortlist_move_row(int* SLid, T* SLw, T* wnext, int k, int last) {
  const int t = threadIdx.x;
  for (int q = t; q < kSL; q += blockDim.x) {
    int id = SLid[(int64_t)last * kSL + q];
    SLid[(int64_t)k * kSL + q] = (id == k) ? -1 : id;   // (renamed already)
    SLw[(int64_t)k * kSL + q] = (id == k) ? Tr<T>::inf() : SLw[(int64_t)last * kSL + q];
  }
  if (t == 0) wnext[k] = wnext[last];
}
template <typename T>
cudaError_t shortlist_remove(int* SLid, T* SLw, T* wnext, int64_t n, int64_t k, int64_t last,
                             cudaStream_t st) {
  int grid = (int)std::min<int64_t>(cdiv(n * kSL / 4, 256), 16 * num_sms());
  k_shortlist_remove<T><<<grid, 256, 0, st>>>(SLid, SLw, wnext, n, (int)k, (int)last);
  if (k != last) k_shortlist_move_row<T><<<1, 256, 0, st>>>(SLid, SLw, wnext, (int)k, (int)last);
  return cudaGetLastError();
}

// Open-pair bookkeeping of phase A (replaces a separate compaction pass):
// the pair joins its row's open list (order within a row is irrelevant) and
// the global open list consumed by phases A2/B and the rounds.
template <typename T>
struct OpenLists {
  int* ocnt; int* ocol; const int64_t* rowoff;
  int* gprow; int* gpcol; T* glb; unsigned char* gfull; int64_t ocap;
  DetectCounters* ctr;
  __device__ __forceinline__ void append(int64_t i, int64_t j, T lb) const {
    const int s1 = atomicAdd(ocnt + i, 1);
    ocol[rowoff[i] + s1] = (int)j;
    const unsigned long long s2 = atomicAdd(&ctr->open_total, 1ull);
    if ((int64_t)s2 < ocap) {
      gprow[s2] = (int)i;
      gpcol[s2] = (int)j;
      glb[s2] = lb;
      gfull[s2] = 1;
    } else {
      atomicOr(&ctr->overflow, 2u);
    }
  }
};

// A warp's staging buffer for the global open list: pairs collect in shared
// memory and go out 32 or more at a time behind ONE atomic on open_total (an
// atomic per warp step on that one word serialised the whole pass at L2).
template <typename T>
struct OpenStage {
  int i[64], j[64];
  T lb[64];
  // every lane of the warp; cnt <= 64 staged pairs
  __device__ __forceinline__ void flush(int cnt, const OpenLists<T>& ol, int lane) {
    if (cnt == 0) return;
    __syncwarp();
    unsigned long long g0 = 0;
    if (lane == 0) g0 = atomicAdd(&ol.ctr->open_total, (unsigned long long)cnt);
    g0 = __shfl_sync(0xffffffffu, g0, 0);
    for (int e = lane; e < cnt; e += 32) {
      const unsigned long long s2 = g0 + e;
      if ((int64_t)s2 < ol.ocap) {
        ol.gprow[s2] = i[e];
        ol.gpcol[s2] = j[e];
        ol.glb[s2] = lb[e];
        ol.gfull[s2] = 1;
      } else {
        atomicOr(&ol.ctr->overflow, 2u);
      }
    }
    __syncwarp();
  }
};

// Swap the ids of nodes p and q in every shortlist (rows and entries).
template <typename T>
__global__ void k_shortlist_swap(int* SLid, T* SLw, T* wnext, int64_t n, int p, int q) {
  const int64_t tot = n * kSL;
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < tot;
       e += (int64_t)gridDim.x * blockDim.x) {
    const int64_t row = e / kSL;
    if (row == p || row == q) continue;
    const int id = SLid[e];
    if (id == p) SLid[e] = q;
    else if (id == q) SLid[e] = p;
  }
}
template <typename T>
__global__ void k_shortlist_swap_rows(int* SLid, T* SLw, T* wnext, int p, int q) {
  for (int t = threadIdx.x; t < kSL; t += blockDim.x) {
    const int64_t a = (int64_t)p * kSL + t, b = (int64_t)q * kSL + t;
    int ia = SLid[a], ib = SLid[b];
    T wa = SLw[a], wb = SLw[b];
    ia = ia == p ? q : ia == q ? p : ia;
    ib = ib == p ? q : ib == q ? p : ib;
    SLid[a] = ib; SLw[a] = wb;
    SLid[b] = ia; SLw[b] = wa;
  }
  if (threadIdx.x == 0) {
    T x = wnext[p];
    wnext[p] = wnext[q];
    wnext[q] = x;
  }
}
template <typename T>
cudaError_t shortlist_swap(int* SLid, T* SLw, T* wnext, int64_t n, int64_t p, int64_t q,
                           cudaStream_t st) {
  int grid = (int)std::min<int64_t>(cdiv(n * kSL, 256), 8 * num_sms());
  k_shortlist_swap<T><<<grid, 256, 0, st>>>(SLid, SLw, wnext, n, (int)p, (int)q);
  k_shortlist_swap_rows<T><<<1, 256, 0, st>>>(SLid, SLw, wnext, (int)p, (int)q);
  return cudaGetLastError();
}

// ---------------------------------------------------------------------------
// phase A / A2: shortlist evaluation of a list of pairs
//   classify = 0 (phase A, all listed pairs):   out = 0 final (reached lb), 1 open
//   classify = 1 (phase A2, open pairs, after A): out = 0 final,
//            1 exact for the current D (est <= wnext), 2 needs the full scan.
// Phase A2 must run after phase A has finished: the certified (final) values
// of other pairs of the row are then visible, so a class-1 value is the
// exact min of (*) over every m whose value can no longer change.
// ---------------------------------------------------------------------------
constexpr int kPhaseASteps = 3;   // phase A: sorted shortlist positions 0-7, 8-39, 40-71

// Pair counts live on the device (the host reads them once per update, after
// the sparse recompute): which = 0, the need_update_list (nothing to do if it
// overflowed: some flagged entries were never reset); 1, the open pairs
// (nothing to do if either list overflowed — the dense path follows).
// which = 2: the pairs the fused detection + phase A kernel spilled to the
// global list (fused.cu).
__device__ __forceinline__ int64_t device_count(const DetectCounters* dc, int64_t cap, int which) {
  if (!dc) return cap;
  if (dc->overflow & (which == 1 ? 3u : 1u)) return 0;
  const int64_t c = (int64_t)(which == 1 ? dc->open_total : which == 2 ? dc->spill : dc->total);
  return c < cap ? c : cap;
}

// (the body: every warp of the grid; returns the mirror flag bits it raised)
template <typename T, int SR>
__device__ __forceinline__ unsigned sparse_short_body(T* D, int64_t ld, int64_t row0,
                                                      const int* __restrict__ SLid,
                                                      const T* __restrict__ SLw,
                                                      const T* __restrict__ wnext,
                                                      const int* __restrict__ prow,
                                                      const int* __restrict__ pcol,
                                                      const T* __restrict__ plb, int64_t npairs,
                                                      unsigned char* out, int classify,
                                                      const OpenLists<T>& ol, const DetectCounters* dc,
                                                      const Mirror& M, int64_t skip) {
  const int lane = threadIdx.x & 31;
  const int64_t nw = (int64_t)gridDim.x * (blockDim.x >> 5);
  npairs = device_count(dc, npairs, classify ? 1 : 0);
  // A2 gathers from the int8 mirror: every listed entry was mirrored by phase
  // A (final or not, a walk length of G'), later writes are mirrored too, and
  // 0x7F reads as INF — each value read is >= the current D entry, so e is an
  // upper bound and e <= wnext(j) still proves no m outside SL(j) does better
  const uint8_t* M8 = nullptr;
  if constexpr (std::is_same<T, int32_t>::value && SR == 0) M8 = M.m8;
  unsigned mbits = 0;
  for (int64_t p = blockIdx.x * (int64_t)(blockDim.x >> 5) + (threadIdx.x >> 5); p < npairs;
       p += nw) {
    const int64_t i = prow[p], j = pcol[p];
    T* Drow = D + (i - row0) * ld;
    const uint8_t* Mrow = M8 ? M8 + (i - row0) * ld : nullptr;
    const int* sid = SLid + j * kSL;
    const T* sw = SLw + j * kSL;
    const T lbp = plb[p];
    T acc = Tr<T>::inf();
    // Phase A only certifies: it walks SL(j) in ascending weight order (the
    // list is kept sorted) and stops as soon as the warp's bound reaches lb
    // (the value is then final); after kPhaseASteps stages a pair that has not
    // is left open — A2 evaluates the whole shortlist once the certified
    // values are in place.  (A pair that certifies almost always does so on
    // one of its cheapest few in-edges; scanning all 512 entries for the pairs
    // that never do was ~90% of phase A's time.)
    if (!classify) {
      // SL(j) is sorted ascending: positions 0-7 first (8 gathers — most ties
      // certify on the cheapest few in-edges), then 8-39, then 40-71
#pragma unroll
      for (int st = 0; st < kPhaseASteps; ++st) {
        const int e = st == 0 ? lane : 8 + 32 * (st - 1) + lane;
        if (st > 0 || lane < 8) {
          const int m = sid[e];
          if (m >= 0) acc = Tr<T, SR>::relax(acc, *(volatile T*)(Drow + m), sw[e]);
        }
        if (Tr<T>::at_lb(warp_min<T>(acc), lbp)) break;
      }
    } else {
      // the whole shortlist, in ascending weight order, stopping once no
      // later entry can improve: every later live entry weighs >= the
      // heaviest live one seen (SL(j) is sorted) and D >= 0, so D + w >= w
      // (minimax: max(D, w) >= w) — the result is min over all of SL(j)
      T wseen = T(0);
#pragma unroll
      for (int q = 0; q < kSLK; ++q) {
        const int m = sid[q * 32 + lane];
        const T w = sw[q * 32 + lane];
        if (m >= 0) {
          T d;
          // column `skip` (the removed node) is not tombstoned in the mirror,
          // nor yet in D (the swap-with-last overwrites it): read as INF
          if (Mrow) {
            const int32_t b8 = Mrow[m];
            d = (b8 == kSat8i || m == skip) ? Tr<T>::inf() : (T)b8;
          } else {
            d = m == skip ? Tr<T>::inf() : *(volatile T*)(Drow + m);
          }
          acc = Tr<T, SR>::relax(acc, d, w);
          wseen = w > wseen ? w : wseen;
        }
        if ((q & 1) && q + 1 < kSLK && __any_sync(0xffffffffu, acc <= warp_max<T>(wseen))) break;
      }
    }
    acc = warp_min<T>(acc);
    if (lane == 0) {
      const T lb = lbp;
      const T cur = *(volatile T*)(Drow + j);
      const T v = Tr<T>::mn(acc, cur);
      if (v < cur) {
        Drow[j] = v;
        if (M.m || M.m8) mbits |= mput(M, (i - row0) * ld + j, v);
      }
      unsigned char st;
      if (Tr<T>::at_lb(v, lb)) st = 0;
      else if (!classify || acc <= wnext[j]) st = 1;
      else st = 2;
      out[p] = st;
      if (!classify && st != 0) ol.append(i, j, lb);
    }
  }
  return mbits;
}
#ifndef SS_WPC
#define SS_WPC 8   // warps per CTA of k_sparse_short
#endif
template <typename T, int SR>
__global__ void __launch_bounds__(32 * SS_WPC) k_sparse_short(T* D, int64_t ld, int64_t row0,
                                                      const int* __restrict__ SLid,
                                                      const T* __restrict__ SLw,
                                                      const T* __restrict__ wnext,
                                                      const int* __restrict__ prow,
                                                      const int* __restrict__ pcol,
                                                      const T* __restrict__ plb, int64_t npairs,
                                                      unsigned char* out, int classify,
                                                      OpenLists<T> ol, const DetectCounters* dc, Mirror M,
                                                      int64_t skip) {
  const unsigned mbits = sparse_short_body<T, SR>(D, ld, row0, SLid, SLw, wnext, prow, pcol, plb, npairs, out,
                                                  classify, ol, dc, M, skip);
  if (M.m || M.m8) mirror_post(M, mbits);
}

template <typename T>
cudaError_t sparse_short(T* D, int64_t ld, int64_t row0, const int* SLid, const T* SLw,
                         const T* wnext, const int* prow, const int* pcol, const T* plb,
                         int64_t npairs, unsigned char* out, int classify, int sr,
                         const DetectCounters* dc, cudaStream_t st, Mirror M, int64_t skip) {
  if (npairs <= 0) return cudaSuccess;
  int grid = (int)std::min<int64_t>(cdiv(npairs, 8), (int64_t)num_sms() * 16);
  OpenLists<T> ol{};
  if (sr)
    k_sparse_short<T, 1><<<grid * (8 / SS_WPC), 32 * SS_WPC, 0, st>>>(D, ld, row0, SLid, SLw, wnext, prow, pcol, plb, npairs,
                                               out, classify, ol, dc, M, skip);
  else
    k_sparse_short<T, 0><<<grid * (8 / SS_WPC), 32 * SS_WPC, 0, st>>>(D, ld, row0, SLid, SLw, wnext, prow, pcol, plb, npairs,
                                               out, classify, ol, dc, M, skip);
  return cudaGetLastError();
}

// Phase A, one lane per pair, straight off the detection list (32 pairs per
// warp in flight: the stage is a chain of dependent gathers — pair, shortlist,
// D[i][m] — so the pairs a warp overlaps set its speed).  Nothing has been
// reset: every listed entry still holds D_old, which is the pair's lower
// bound lb (read here; only this lane writes (i, j)) but is stale as a
// candidate.  A stale D[i][m] is recognised by the detection predicate itself
// (same function of the same values: m's entry is listed iff it still tests
// tight against the pivot snapshots) and skipped; an entry another lane has
// already rewritten holds a walk length of G' and is used.  Skipping only
// weakens the bound, so the value written — min over the usable candidates,
// INF if none — is a walk length of G' (>= the new distance) either way.
// Each lane walks SL(j) in ascending weight order, 8 entries per batch, and
// stops at the first batch whose bound reaches lb (certified); after
// kPhaseABatches batches the pair is left open for A2 / B / the rounds.
#ifndef PA_BATCHES
#define PA_BATCHES 9
#endif
constexpr int kPhaseABatches = PA_BATCHES;   // 9: sorted positions 0-71
#ifndef PA_MINB
#define PA_MINB 4   // 4 CTAs per SM (64 registers, no spills): latency-bound, occupancy wins
#endif

template <typename T, int SR, bool TWO>
__global__ void __launch_bounds__(256, PA_MINB) k_sparse_phase_a(T* D, int64_t ld, int64_t row0,
                                                        const int* __restrict__ SLid,
                                                        const T* __restrict__ SLw,
                                                        const int* __restrict__ srow,
                                                        const int* __restrict__ scol, int64_t npairs,
                                                        const T* __restrict__ c1, const T* __restrict__ r1,
                                                        const T* __restrict__ c2, const T* __restrict__ r2,
                                                        float tau, OpenLists<T> ol,
                                                        const DetectCounters* dc, Mirror M, int nbatch,
                                                        int list) {
  const int lane = threadIdx.x & 31;
  unsigned mbits = 0;   // mirror flag bits raised by this thread's writes
  npairs = device_count(dc, npairs, list);
  // the gathers read the int8 mirror while it is valid (exact; a quarter of
  // the bytes).  An entry this kernel rewrites meanwhile reads as its old
  // value (stale: skipped by the test below), its new final value, or 0x7F
  // (INF: skipped) if that is >= 0x7F — each case only weakens the bound.
  const uint8_t* M8 = nullptr;
  if constexpr (std::is_same<T, int32_t>::value && SR == 0)
    if (M.m8 && (*(volatile unsigned*)M.flag & 1u) == 0u) M8 = M.m8;
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t base = blockIdx.x * (int64_t)blockDim.x + (threadIdx.x & ~31); base < npairs;
       base += stride) {
    const int64_t p = base + lane;
    int64_t i = 0, j = 0;
    T lb = Tr<T>::inf(), acc = Tr<T>::inf();
    bool open = false;
    if (p < npairs) {
      i = srow[p];
      j = scol[p];
      T* Drow = D + (i - row0) * ld;
      const uint8_t* Mrow = M8 ? M8 + (i - row0) * ld : nullptr;
      const int4* sid = reinterpret_cast<const int4*>(SLid + j * kSL);
      const int4* sw = reinterpret_cast<const int4*>(SLw + j * kSL);
      lb = *(volatile T*)(Drow + j);   // D_old[i][j]
      const T ci = c1[i], cj = TWO ? c2[i] : Tr<T>::inf();
      for (int b = 0; b < nbatch; ++b) {
        const int4 m0 = sid[2 * b], m1 = sid[2 * b + 1];
        const int4 w0 = sw[2 * b], w1 = sw[2 * b + 1];
        const int m[8] = {m0.x, m0.y, m0.z, m0.w, m1.x, m1.y, m1.z, m1.w};
        const int wi[8] = {w0.x, w0.y, w0.z, w0.w, w1.x, w1.y, w1.z, w1.w};
        // the first batch in two steps: the 2 cheapest in-edges certify most
        // pairs, so the other 6 gathers are issued only when they did not
        bool done = false;
#pragma unroll
        for (int h = 0; h < 2; ++h) {
          const int q0 = h == 0 ? 0 : (b == 0 ? 2 : 8), q1 = h == 0 ? (b == 0 ? 2 : 8) : 8;
          if (q0 >= q1) continue;
          T dv[8], rv[8], rv2[8];
#pragma unroll
          for (int q = 0; q < 8; ++q) {
            if (q < q0 || q >= q1) continue;
            const int mq = m[q] >= 0 ? m[q] : 0;
            if (Mrow) {
              const int32_t b8 = Mrow[mq];
              dv[q] = (m[q] >= 0 && b8 != kSat8i) ? (T)b8 : Tr<T>::inf();
            } else {
              dv[q] = m[q] >= 0 ? *(volatile const T*)(Drow + mq) : Tr<T>::inf();
            }
            rv[q] = r1[mq];
            if (TWO) rv2[q] = r2[mq];
          }
#pragma unroll
          for (int q = 0; q < 8; ++q) {
            if (q < q0 || q >= q1) continue;
            bool stale = Tr<T, SR>::tight(Tr<T, SR>::add(ci, rv[q]), dv[q], tau);
            if (TWO) stale = stale || Tr<T, SR>::tight(Tr<T, SR>::add(cj, rv2[q]), dv[q], tau);
            if (m[q] >= 0 && !stale) {
              T w;
              memcpy(&w, &wi[q], sizeof(T));
              acc = Tr<T, SR>::relax(acc, dv[q], w);
            }
          }
          if (Tr<T>::at_lb(acc, lb)) { done = true; break; }
        }
        if (done) break;
      }
      // D_old is not an upper bound of D': every listed entry gets acc — a
      // write only where it differs (a certified pair, acc == lb, already
      // holds it; mirrors included: A2 reads them; later writes — A2, B, the
      // rounds — are mirrored as they happen)
      if (acc != lb) {
        Drow[j] = acc;
        if (M.m || M.m8) mbits |= mput(M, (i - row0) * ld + j, acc);
      }
      open = !Tr<T>::at_lb(acc, lb);
    }
    // open-pair lists: per-row slot by atomic, the global slot warp-aggregated
    const unsigned bal = __ballot_sync(0xffffffffu, open);
    if (bal) {
      unsigned long long g0 = 0;
      if (lane == __ffs(bal) - 1) g0 = atomicAdd(&ol.ctr->open_total, (unsigned long long)__popc(bal));
      g0 = __shfl_sync(0xffffffffu, g0, __ffs(bal) - 1);
      if (open) {
        const int s1 = atomicAdd(ol.ocnt + i, 1);
        ol.ocol[ol.rowoff[i] + s1] = (int)j;
        const unsigned long long s2 = g0 + __popc(bal & ((1u << lane) - 1));
        if ((int64_t)s2 < ol.ocap) {
          ol.gprow[s2] = (int)i;
          ol.gpcol[s2] = (int)j;
          ol.glb[s2] = lb;
          ol.gfull[s2] = 1;
        } else {
          atomicOr(&ol.ctr->overflow, 2u);
        }
      }
    }
  }
  if (M.m || M.m8) mirror_post(M, mbits);
}

// Phase A with a per-warp work queue: the same per-pair computation as
// k_sparse_phase_a, one gather step per loop iteration (step 0: the 2
// cheapest in-edges, step 1: the other 6 of the first batch, then one 8-entry
// batch per step), and a lane whose pair is finished takes the next pair of
// the warp's chunk at once.  In the one-pair-per-lane kernel a warp runs as
// many steps as its slowest lane (ncu: ~6 batches per 32 pairs where the
// average pair needs ~1.3); here a warp runs ~sum(steps)/32.
constexpr int kPAChunk = 8;   // pairs per warp chunk = 32 * kPAChunk
#ifndef PA_WPC
#define PA_WPC 8   // warps per CTA of the work-queue kernel
#endif
template <typename T, int SR, bool TWO>
__global__ void __launch_bounds__(32 * PA_WPC, PA_MINB * 8 / PA_WPC) k_sparse_phase_aq(T* D, int64_t ld, int64_t row0,
                                                         const int* __restrict__ SLid,
                                                         const T* __restrict__ SLw,
                                                         const int* __restrict__ srow,
                                                         const int* __restrict__ scol, int64_t npairs,
                                                         const T* __restrict__ c1, const T* __restrict__ r1,
                                                         const T* __restrict__ c2, const T* __restrict__ r2,
                                                         float tau, OpenLists<T> ol,
                                                         const DetectCounters* dc, Mirror M, int nbatch,
                                                         int list, const uint8_t* __restrict__ r1b) {
  const int lane = threadIdx.x & 31;
  unsigned mbits = 0;
  npairs = device_count(dc, npairs, list);
  __shared__ OpenStage<T> stage_all[PA_WPC];
  OpenStage<T>& stg = stage_all[threadIdx.x >> 5];
  int scnt = 0;   // (warp-uniform) pairs in the warp's stage
  const uint8_t* M8 = nullptr;
  if constexpr (std::is_same<T, int32_t>::value && SR == 0)
    if (M.m8 && (*(volatile unsigned*)M.flag & 1u) == 0u) M8 = M.m8;
  // with the mirror, the stale test reads r1 as saturated bytes too: exact,
  // since a byte of 0x7F (r1 >= 0x7F) makes c + r >= 0x7F > every mirrored
  // d it is compared with (d = 0x7F entries are skipped as INF); a 32 KB row
  // of bytes stays in L1 where 4-byte values spill to L2
  const uint8_t* R8 = M8 ? r1b : nullptr;
  const int64_t nw = (int64_t)gridDim.x * (blockDim.x >> 5);
  const int64_t wid = blockIdx.x * (int64_t)(blockDim.x >> 5) + (threadIdx.x >> 5);
  // chunk: up to 32 * kPAChunk pairs, fewer when the list would leave warps
  // idle (a multiple of 32, >= 32: every lane starts with a pair)
  const int64_t CH = min((int64_t)(32 * kPAChunk), max((int64_t)32, ((npairs + nw - 1) / nw + 31) / 32 * 32));
  for (int64_t c0 = wid * CH; c0 < npairs; c0 += nw * CH) {
    const int64_t cend = c0 + CH < npairs ? c0 + CH : npairs;
    int64_t next = c0;   // warp-uniform
    bool busy = false;
    int i = 0, j = 0, b = 0, h = 0;
    T lb = Tr<T>::inf(), acc = Tr<T>::inf(), ci = Tr<T>::inf(), cj = Tr<T>::inf();
    int m[8], wi[8];
    while (true) {
      const unsigned need = __ballot_sync(0xffffffffu, !busy);
      if (need) {
        const int64_t mine = next + __popc(need & ((1u << lane) - 1));
        if (!busy && mine < cend) {
          busy = true;
          i = srow[mine];
          j = scol[mine];
          ci = c1[i];
          cj = TWO ? c2[i] : Tr<T>::inf();
          // D_old[i][j]: an integer listed pair is exactly tight, D_old = c1[i] +
          // r1[j] (or the c2 + r2 term; D_old <= both), read from the pivot
          // vectors (L2-resident) instead of a DRAM gather of D; fp32 pairs are
          // listed with a tolerance, so D itself is read
          if constexpr (!Tr<T>::kFloat) {
            lb = Tr<T, SR>::add(ci, r1[j]);
            if (TWO) lb = Tr<T>::mn(lb, Tr<T, SR>::add(cj, r2[j]));
          } else {
            lb = *(volatile T*)(D + (int64_t)(i - row0) * ld + j);
          }
          acc = Tr<T>::inf();
          b = 0;
          h = 0;
        }
        next += __popc(need);
      }
      if (!__any_sync(0xffffffffu, busy)) break;
      bool fin = false;
      if (busy) {
        if (h == 0) {   // a new batch: its 8 sorted shortlist entries
          const int4* sid = reinterpret_cast<const int4*>(SLid + (int64_t)j * kSL) + 2 * b;
          const int4* sw = reinterpret_cast<const int4*>(SLw + (int64_t)j * kSL) + 2 * b;
          const int4 m0 = sid[0], m1 = sid[1], w0 = sw[0], w1 = sw[1];
          m[0] = m0.x; m[1] = m0.y; m[2] = m0.z; m[3] = m0.w; m[4] = m1.x; m[5] = m1.y; m[6] = m1.z; m[7] = m1.w;
          wi[0] = w0.x; wi[1] = w0.y; wi[2] = w0.z; wi[3] = w0.w; wi[4] = w1.x; wi[5] = w1.y; wi[6] = w1.z;
          wi[7] = w1.w;
        }
        const int q0 = h == 0 ? 0 : 2, q1 = (b == 0 && h == 0) ? 2 : 8;
        const T* Drow = D + (int64_t)(i - row0) * ld;
        const uint8_t* Mrow = M8 ? M8 + (int64_t)(i - row0) * ld : nullptr;
        T dv[8], rv[8], rv2[8];
#pragma unroll
        for (int q = 0; q < 8; ++q) {
          if (q < q0 || q >= q1) continue;
          const int mq = m[q] >= 0 ? m[q] : 0;
          if (Mrow) {
            const int32_t b8 = Mrow[mq];
            dv[q] = (m[q] >= 0 && b8 != kSat8i) ? (T)b8 : Tr<T>::inf();
          } else {
            dv[q] = m[q] >= 0 ? *(volatile const T*)(Drow + mq) : Tr<T>::inf();
          }
          rv[q] = R8 ? (T)R8[mq] : r1[mq];
          if (TWO) rv2[q] = r2[mq];
        }
#pragma unroll
        for (int q = 0; q < 8; ++q) {
          if (q < q0 || q >= q1) continue;
          bool stale = Tr<T, SR>::tight(Tr<T, SR>::add(ci, rv[q]), dv[q], tau);
          if (TWO) stale = stale || Tr<T, SR>::tight(Tr<T, SR>::add(cj, rv2[q]), dv[q], tau);
          if (m[q] >= 0 && !stale) {
            T w;
            memcpy(&w, &wi[q], sizeof(T));
            acc = Tr<T, SR>::relax(acc, dv[q], w);
          }
        }
        if (Tr<T>::at_lb(acc, lb)) {
          fin = true;
        } else if (b == 0 && h == 0) {
          h = 1;
        } else {
          ++b;
          h = 0;
          fin = b >= nbatch;
        }
      }
      bool open = false;
      if (fin) {
        if (acc != lb) {   // D_old is not an upper bound of D' (a certified pair already holds acc)
          D[(int64_t)(i - row0) * ld + j] = acc;
          if (M.m || M.m8) mbits |= mput(M, (int64_t)(i - row0) * ld + j, acc);
        }
        open = !Tr<T>::at_lb(acc, lb);
        busy = false;
      }
      const unsigned bal = __ballot_sync(0xffffffffu, open);
      if (bal) {
        if (open) {   // the row's open list now; the global list through the warp's stage
          const int s1 = atomicAdd(ol.ocnt + i, 1);
          ol.ocol[ol.rowoff[i] + s1] = j;
          const int sp = scnt + __popc(bal & ((1u << lane) - 1));
          stg.i[sp] = i;
          stg.j[sp] = j;
          stg.lb[sp] = lb;
        }
        scnt += __popc(bal);
        if (scnt >= 32) {
          stg.flush(scnt, ol, lane);
          scnt = 0;
        }
      }
    }
  }
  stg.flush(scnt, ol, lane);
  if (M.m || M.m8) mirror_post(M, mbits);
}

// Phase A's first step as a separate, write-free pass (int32 shortest path,
// one pivot term, int8 mirror valid): each pair's two cheapest in-edges of
// SL(j), against lb = D_old[i][j] = c1[i] + r1[j].  A pair certified here keeps
// D_old (its new distance, P:173-178 / DESIGN.md §4.6); every other pair goes
// to the continuation list (crow, ccol; count ctr->spill) that the work-queue
// kernel then finishes from scratch.  Nothing is written to D, so every
// gathered D[i][m] is D_old and the detection predicate recognises the stale
// ones exactly.  A lane takes kA0P pairs at once and issues each level of
// the chain (pair -> shortlist -> D[i][m]) for all of them together: the
// chain is three dependent DRAM reads, and the pairs one lane overlaps set the
// pass's speed (the work-queue kernel holds one pair per lane).
constexpr int kA0P = 4;
#ifndef PA_SPLIT
#define PA_SPLIT 1
#endif
__global__ void __launch_bounds__(256, PA_MINB) k_phase_a0(const int* __restrict__ SLid,
                                                          const int32_t* __restrict__ SLw,
                                                          const int* __restrict__ srow,
                                                          const int* __restrict__ scol, int64_t npairs,
                                                          const int32_t* __restrict__ c1,
                                                          const int32_t* __restrict__ r1,
                                                          const uint8_t* __restrict__ r1b, int64_t ld, int64_t row0,
                                                          Mirror M, int* crow, int* ccol, DetectCounters* dc) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  npairs = device_count(dc, npairs, 0);
  const bool mv = (*(volatile unsigned*)M.flag & 1u) == 0u;   // (CTA-uniform: nothing here writes D)
  __shared__ unsigned s_cnt[8];
  __shared__ unsigned long long s_base;
  // block-stride: every warp of the CTA runs the same iterations, so the
  // continuation slots are reserved once per CTA and iteration (one atomic)
  constexpr int kBlk = 8 * 32 * kA0P;
  for (int64_t b0 = blockIdx.x * (int64_t)kBlk; b0 < npairs; b0 += (int64_t)gridDim.x * kBlk) {
    const int64_t c0 = b0 + warp * (32 * kA0P);
    int i[kA0P], j[kA0P];
    bool ok[kA0P], open[kA0P];
#pragma unroll
    for (int q = 0; q < kA0P; ++q) {
      const int64_t p = c0 + q * 32 + lane;
      ok[q] = p < npairs;
      i[q] = ok[q] ? srow[p] : 0;
      j[q] = ok[q] ? scol[p] : 0;
    }
    if (mv) {
      int2 m[kA0P], w[kA0P];
      int32_t lb[kA0P], ci[kA0P];
#pragma unroll
      for (int q = 0; q < kA0P; ++q) {
        m[q] = ok[q] ? *reinterpret_cast<const int2*>(SLid + (int64_t)j[q] * kSL) : make_int2(-1, -1);
        w[q] = ok[q] ? *reinterpret_cast<const int2*>(SLw + (int64_t)j[q] * kSL) : make_int2(0, 0);
        ci[q] = ok[q] ? c1[i[q]] : 0;
        lb[q] = ok[q] ? ci[q] + r1[j[q]] : 0;
      }
#pragma unroll
      for (int q = 0; q < kA0P; ++q) {
        const uint8_t* Mrow = M.m8 + (int64_t)(i[q] - row0) * ld;
        const int ma = m[q].x >= 0 ? m[q].x : 0, mb = m[q].y >= 0 ? m[q].y : 0;
        const int32_t da = Mrow[ma], db = Mrow[mb], ra = r1b[ma], rb = r1b[mb];
        int32_t acc = APSP_INF_I32_DEV;
        // usable: a finite mirrored entry (0x7F reads as INF) that does not
        // test tight against the pivot snapshots (a stale D_old, Theorem 4)
        if (m[q].x >= 0 && da != kSat8i && ci[q] + ra != da) acc = min(acc, da + w[q].x);
        if (m[q].y >= 0 && db != kSat8i && ci[q] + rb != db) acc = min(acc, db + w[q].y);
        open[q] = ok[q] && acc > lb[q];
      }
    } else {   // the mirror is not valid: every pair to the continuation
#pragma unroll
      for (int q = 0; q < kA0P; ++q) open[q] = ok[q];
    }
    unsigned bal[kA0P], wcnt = 0;
#pragma unroll
    for (int q = 0; q < kA0P; ++q) {
      bal[q] = __ballot_sync(0xffffffffu, open[q]);
      wcnt += __popc(bal[q]);
    }
    if (lane == 0) s_cnt[warp] = wcnt;
    __syncthreads();
    if (threadIdx.x == 0) {
      unsigned tot = 0;
      for (int w2 = 0; w2 < 8; ++w2) tot += s_cnt[w2];
      s_base = tot ? atomicAdd(&dc->spill, (unsigned long long)tot) : 0ull;
    }
    __syncthreads();
    unsigned long long pos = s_base;
    for (int w2 = 0; w2 < warp; ++w2) pos += s_cnt[w2];
#pragma unroll
    for (int q = 0; q < kA0P; ++q) {
      if (open[q]) {
        const unsigned long long s = pos + __popc(bal[q] & ((1u << lane) - 1));
        crow[s] = i[q];   // (s < npairs <= the list's capacity)
        ccol[s] = j[q];
      }
      pos += __popc(bal[q]);
    }
    __syncthreads();   // (s_cnt / s_base are rewritten by the next iteration)
  }
}

// Phase A over the detection list (pairs in append order; every pair reads
// and writes only its own row).
template <typename T>
cudaError_t sparse_phase_a(T* D, int64_t ld, Rows r, const int* SLid, const T* SLw,
                           const int64_t* rowoff, const int* srow, const int* scol, int64_t npairs,
                           const T* c1, const T* r1, const T* c2, const T* r2, float tau, int* ocnt,
                           int* ocol, int* gprow, int* gpcol, T* glb, unsigned char* gfull, int64_t ocap,
                           DetectCounters* ctr, int sr, Mirror M, cudaStream_t st, int list, const uint8_t* r1b,
                           int* crow, int* ccol) {
  if (npairs <= 0) return cudaSuccess;
  OpenLists<T> ol{ocnt, ocol, rowoff, gprow, gpcol, glb, gfull, ocap, ctr};
  // the write-free first step (k_phase_a0), then the work queue over the pairs
  // it left (list 2)
  if constexpr (std::is_same<T, int32_t>::value) {
    if (PA_SPLIT && crow && ccol && r1b && M.m8 && !sr && !c2 && list == 0) {
      const int g0 = (int)std::min<int64_t>(cdiv(npairs, 32 * kA0P * 8), (int64_t)num_sms() * PA_MINB);   // (256 threads)
      k_phase_a0<<<g0, 256, 0, st>>>(SLid, SLw, srow, scol, npairs, c1, r1, r1b, ld, r.row0, M, crow, ccol, ctr);
      srow = crow;
      scol = ccol;
      list = 2;
    }
  }
  // npairs is the capacity bound (the device count decides): full occupancy
  int grid = (int)std::min<int64_t>(cdiv(npairs, 256), (int64_t)num_sms() * 8);
#define PA(SRV, TWOV)                                                                              \
  do {                                                                                             \
    if (queue)                                                                                     \
      k_sparse_phase_aq<T, SRV, TWOV><<<grid * (8 / PA_WPC), 32 * PA_WPC, 0, st>>>(D, ld, r.row0, SLid, SLw, srow, scol,  \
                                                            npairs, c1, r1, c2, r2, tau, ol, ctr, M, nb, list, \
                                                            r1b);                                       \
    else                                                                                           \
      k_sparse_phase_a<T, SRV, TWOV><<<grid, 256, 0, st>>>(D, ld, r.row0, SLid, SLw, srow, scol,   \
                                                           npairs, c1, r1, c2, r2, tau, ol, ctr, M, nb, list); \
  } while (0)
  constexpr int nb = std::min(kSL / 8, kPhaseABatches);
#ifndef PA_QUEUE
#define PA_QUEUE 1   // 0: the one-pair-per-lane kernel (measured slower)
#endif
  constexpr bool queue = PA_QUEUE == 1;
  const bool two = c2 != nullptr;
  if (sr) { if (two) PA(1, true); else PA(1, false); }
  else { if (two) PA(0, true); else PA(0, false); }
#undef PA
  return cudaGetLastError();
}

// ---------------------------------------------------------------------------
// phase B: full scan (*) for open pairs marked 2, early exit at the lower bound
// ---------------------------------------------------------------------------
// One CTA per pair: the scan of a row is a latency chain (one warp per pair
// took ~1 us per 64 vectors: a few pairs at n = 65536 ran 0.3 ms), so all 8
// warps split it, with a block-wide early-exit test every 4 steps.
// (the body: every CTA of the grid, 256 threads; wm: 8 T of shared memory)
template <typename T, int SR>
__device__ __forceinline__ unsigned sparse_full_body(T* D, int64_t ld, int64_t row0,
                                                     const T* __restrict__ WT, int64_t ldw,
                                                     int64_t n, const int* __restrict__ gprow,
                                                     const int* __restrict__ gpcol,
                                                     const T* __restrict__ glb,
                                                     const unsigned char* __restrict__ gfull,
                                                     int64_t nopen, const DetectCounters* dc, const Mirror& M,
                                                     T* wm) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  unsigned mbits = 0;
  const int64_t n4 = (n + 3) / 4;
  nopen = device_count(dc, nopen, 1);
  const T I = Tr<T>::inf();
  for (int64_t p = blockIdx.x; p < nopen; p += gridDim.x) {
    if (gfull[p] != 2) continue;   // block-uniform
    const int64_t i = gprow[p], j = gpcol[p];
    const T lb = glb[p];
    T* Drow = D + (i - row0) * ld;
    const T* Wrow = WT + j * ldw;
    T acc = I;
    // block-uniform trip count: the early-exit test below synchronises the CTA
    for (int64_t base = 0, iter = 1; base < n4; base += 512, ++iter) {
      const int64_t q0 = base + threadIdx.x, q1 = base + 256 + threadIdx.x;
      Vec4<T> d0{I, I, I, I}, w0{I, I, I, I}, d1{I, I, I, I}, w1{I, I, I, I};
      if (q0 < n4) {
        d0 = mask_tail<T>(ld4_cg<T>(Drow + 4 * q0), 4 * q0, n);
        w0 = mask_tail<T>(ld4<T>(Wrow + 4 * q0), 4 * q0, n);
      }
      if (q1 < n4) {
        d1 = mask_tail<T>(ld4_cg<T>(Drow + 4 * q1), 4 * q1, n);
        w1 = mask_tail<T>(ld4<T>(Wrow + 4 * q1), 4 * q1, n);
      }
      acc = Tr<T, SR>::relax(acc, d0.x, w0.x); acc = Tr<T, SR>::relax(acc, d0.y, w0.y);
      acc = Tr<T, SR>::relax(acc, d0.z, w0.z); acc = Tr<T, SR>::relax(acc, d0.w, w0.w);
      acc = Tr<T, SR>::relax(acc, d1.x, w1.x); acc = Tr<T, SR>::relax(acc, d1.y, w1.y);
      acc = Tr<T, SR>::relax(acc, d1.z, w1.z); acc = Tr<T, SR>::relax(acc, d1.w, w1.w);
      if ((iter & 3) == 0 && base + 512 < n4) {   // reached the lower bound?
        const T m = warp_min<T>(acc);
        if (lane == 0) wm[warp] = m;
        __syncthreads();
        T b = wm[0];
#pragma unroll
        for (int w = 1; w < 8; ++w) b = Tr<T>::mn(b, wm[w]);
        __syncthreads();
        if (Tr<T>::at_lb(b, lb)) break;
      }
    }
    acc = warp_min<T>(acc);
    if (lane == 0) wm[warp] = acc;
    __syncthreads();
    if (threadIdx.x == 0) {
      T b = wm[0];
#pragma unroll
      for (int w = 1; w < 8; ++w) b = Tr<T>::mn(b, wm[w]);
      const T old = Drow[j];
      if (b < old) {
        Drow[j] = b;
        if (M.m || M.m8) mbits |= mput(M, (i - row0) * ld + j, b);
      }
    }
    __syncthreads();   // wm is reused by the next pair
  }
  return mbits;
}
template <typename T, int SR>
__global__ void __launch_bounds__(256) k_sparse_full(T* D, int64_t ld, int64_t row0,
                                                     const T* __restrict__ WT, int64_t ldw,
                                                     int64_t n, const int* __restrict__ gprow,
                                                     const int* __restrict__ gpcol,
                                                     const T* __restrict__ glb,
                                                     const unsigned char* __restrict__ gfull,
                                                     int64_t nopen, const DetectCounters* dc, Mirror M) {
  __shared__ T wm[8];
  const unsigned mbits = sparse_full_body<T, SR>(D, ld, row0, WT, ldw, n, gprow, gpcol, glb, gfull, nopen, dc, M, wm);
  if (M.m || M.m8) mirror_post(M, mbits);
}
template <typename T>
cudaError_t sparse_full(T* D, int64_t ld, int64_t row0, const T* WT, int64_t ldw, int64_t n,
                        const int* gprow, const int* gpcol, const T* glb, const unsigned char* gfull,
                        int64_t nopen, int sr, const DetectCounters* dc, cudaStream_t st, Mirror M) {
  if (nopen <= 0) return cudaSuccess;
  int grid = (int)std::min<int64_t>(nopen, (int64_t)num_sms() * 8);
  if (sr)
    k_sparse_full<T, 1><<<grid, 256, 0, st>>>(D, ld, row0, WT, ldw, n, gprow, gpcol, glb, gfull, nopen, dc, M);
  else
    k_sparse_full<T, 0><<<grid, 256, 0, st>>>(D, ld, row0, WT, ldw, n, gprow, gpcol, glb, gfull, nopen, dc, M);
  return cudaGetLastError();
}

// ---------------------------------------------------------------------------
// rounds: open pair of a changed row, min over the open entries m of its row
// ---------------------------------------------------------------------------
// Per-row minimum of the open entries' current values, kept as a key that
// atomicMax orders like the value's min (values are >= 0: int32 and IEEE
// floats order like their bits; ~bits reverses it; key 0 = "none").
template <typename T>
__device__ __forceinline__ unsigned open_key(T v) {
  unsigned b;
  memcpy(&b, &v, 4);
  return ~b;
}
template <typename T>
__device__ __forceinline__ T open_min(unsigned key) {
  const unsigned b = ~key;
  T v;
  memcpy(&v, &b, 4);
  return v;
}
template <typename T>
__global__ void k_open_rowmin(const T* __restrict__ D, int64_t ld, int64_t row0, const int* __restrict__ gprow,
                              const int* __restrict__ gpcol, int64_t nopen, unsigned* rowkey,
                              const DetectCounters* dc) {
  nopen = device_count(dc, nopen, 1);
  for (int64_t p = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; p < nopen; p += (int64_t)gridDim.x * blockDim.x) {
    const int64_t i = gprow[p];
    atomicMax(rowkey + i, open_key<T>(D[(i - row0) * ld + gpcol[p]]));
  }
}
template <typename T>
cudaError_t open_rowmin(const T* D, int64_t ld, int64_t row0, const int* gprow, const int* gpcol, int64_t nopen,
                        unsigned* rowkey, const DetectCounters* dc, cudaStream_t st) {
  if (nopen <= 0) return cudaSuccess;
  k_open_rowmin<T><<<2 * num_sms(), 256, 0, st>>>(D, ld, row0, gprow, gpcol, nopen, rowkey, dc);
  return cudaGetLastError();
}

// One round (see the rounds' description at recompute(), apsp_warm.cu): each
// open pair (i, j) of a row whose entries changed last round is relaxed
// through those entries; a lower value is written and becomes part of the
// next round's frontier.
// ---------------------------------------------------------------------------
// heavy rows (one GPU): a row with many open pairs is a large
// single-source problem for the rounds, whose cost per round is the row's open
// pairs x its frontier.  Its row of D' is taken instead from the other rows,
// final once the rounds converged (every pair (i, j) of a row is resolved from
// row i alone, so excluding the heavy rows does not delay the others): with H
// the heavy rows and
//   X_h[j] = min over m not in H of  W'[h][m] + D'[m][j]          (first hop)
//   C      = shortest paths inside H over the edges W' between heavy nodes
// every shortest h -> j path leaves H after a prefix inside H (at h', via a
// first hop to a node outside H) or stays inside H (j in H), so
//   D'[h][j] = min( min_h' C[h][h'] + X_h'[j],  C[h][j] if j in H ).
// ---------------------------------------------------------------------------
// X keys: atomicMin on the value's order-preserving bits (values >= 0); the
// buffer holds "INF or above" between recomputes, clamped when read
template <typename T>
__device__ __forceinline__ T heavy_xval(int k) {
  if (Tr<T>::kFloat) {
    const float f = k >= 0x7F800000 ? __builtin_huge_valf() : __int_as_float(k);
    return (T)f;
  }
  return (T)min(k, (int)Tr<T>::inf());
}
template <typename T>
__device__ __forceinline__ int heavy_xkey(T v) {
  int k;
  memcpy(&k, &v, 4);
  return k;
}

constexpr int kHxSlab = 32;   // rows m per staging step
constexpr int kHxGroup = 8;   // heavy rows per X work item
// Shared memory of the heavy-row phases (inside the cooperative rounds kernel)
template <typename T>
struct HeavySmem {
  int hrow[kHeavy];
  T w[kHxSlab][kHxGroup];
  T red[8][kHxGroup][128];
  T C[kHeavy][kHeavy];
};
// X_h[j] for the group of 8 selected rows starting at g0, over a 128-column
// stripe and the rows m in [m0, m1): the 8 warps take every 8th row, the
// weights W'[h][m] of 32 rows at a time staged in shared memory (prefetched
// one stage ahead); the warps' partial minima are reduced in shared memory,
// then one atomicMin per (h, column).  Every thread of the block calls it.
template <typename T, int SR>
__device__ void heavy_x_item(const T* __restrict__ D, int64_t ld, int64_t n, const T* __restrict__ WT, int64_t ldw,
                             int hc, int g0, int64_t stripe, int64_t m0, int64_t m1, int* x, int64_t ldx,
                             int64_t skip, HeavySmem<T>& sm, const int* __restrict__ mlist) {
  // rows m: mlist[m0 .. m1) (the pruned first hops), or m0 .. m1 - 1
  auto row_at = [&](int64_t q) -> int64_t { return mlist ? (int64_t)mlist[q] : q; };
  const int gc = min(kHxGroup, hc - g0);
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const T I = Tr<T>::inf();
  const int64_t c0 = stripe * 128 + 4 * lane;   // this lane's columns c0 .. c0+3
  T acc[kHxGroup][4];
#pragma unroll
  for (int k = 0; k < kHxGroup; ++k)
#pragma unroll
    for (int e = 0; e < 4; ++e) acc[k][e] = I;
  const int wr = threadIdx.x / kHxGroup, wk = threadIdx.x % kHxGroup;
  auto wload = [&](int64_t b) -> T {
    if (b + wr >= m1 || wk >= gc) return I;
    const int64_t m = row_at(b + wr);
    bool out = m != skip;
    for (int t = 0; t < hc; ++t) out &= sm.hrow[t] != (int)m;   // m outside H
    return out ? WT[m * ldw + sm.hrow[g0 + wk]] : I;             // W'[h][m] (WT row m: in-edges of m)
  };
  T wnext = wload(m0);
  for (int64_t b = m0; b < m1; b += kHxSlab) {
    __syncthreads();
    sm.w[wr][wk] = wnext;
    __syncthreads();
    if (b + kHxSlab < m1) wnext = wload(b + kHxSlab);
    if (c0 >= n) continue;
    Vec4<T> d[kHxSlab / 8];
#pragma unroll
    for (int rr = 0; rr < kHxSlab / 8; ++rr) {
      const int64_t q = b + rr * 8 + warp;
      d[rr] = q < m1 ? mask_tail<T>(ld4<T>(D + row_at(q) * ld + c0), c0, n) : Vec4<T>{I, I, I, I};
    }
#pragma unroll
    for (int rr = 0; rr < kHxSlab / 8; ++rr) {
      const int r = rr * 8 + warp;
#pragma unroll
      for (int k = 0; k < kHxGroup; ++k) {
        if (k >= gc) break;
        const T wv = sm.w[r][k];
        acc[k][0] = Tr<T, SR>::relax(acc[k][0], wv, d[rr].x);
        acc[k][1] = Tr<T, SR>::relax(acc[k][1], wv, d[rr].y);
        acc[k][2] = Tr<T, SR>::relax(acc[k][2], wv, d[rr].z);
        acc[k][3] = Tr<T, SR>::relax(acc[k][3], wv, d[rr].w);
      }
    }
  }
  __syncthreads();
#pragma unroll
  for (int k = 0; k < kHxGroup; ++k)
#pragma unroll
    for (int e = 0; e < 4; ++e) sm.red[warp][k][4 * lane + e] = acc[k][e];
  __syncthreads();
  for (int o = threadIdx.x; o < kHxGroup * 128; o += blockDim.x) {
    const int k = o / 128, cc = o % 128;
    const int64_t j = stripe * 128 + cc;
    if (k >= gc || j >= n) continue;
    T v = sm.red[0][k][cc];
#pragma unroll
    for (int q = 1; q < 8; ++q) v = Tr<T>::mn(v, sm.red[q][k][cc]);
    if (v < I) atomicMin(x + (g0 + k) * ldx + j, heavy_xkey<T>(Tr<T>::sat(v)));
  }
}

// The heavy rows' closure C (shortest paths inside H over W'), in shared
// memory; every thread of the block calls it.
template <typename T, int SR>
__device__ void heavy_closure(const T* __restrict__ WT, int64_t ldw, int hc, HeavySmem<T>& sm) {
  for (int e = threadIdx.x; e < hc * hc; e += blockDim.x) {
    const int a = e / hc, b = e % hc;
    sm.C[a][b] = a == b ? T(0) : WT[(int64_t)sm.hrow[b] * ldw + sm.hrow[a]];   // W'[h_a][h_b]
  }
  // Floyd–Warshall inside H, in place (row and column k do not change in step k)
  for (int k = 0; k < hc; ++k) {
    __syncthreads();
    for (int e = threadIdx.x; e < hc * hc; e += blockDim.x) {
      const int a = e / hc, b = e % hc;
      sm.C[a][b] = Tr<T>::sat(Tr<T, SR>::relax(sm.C[a][b], sm.C[a][k], sm.C[k][b]));
    }
  }
  __syncthreads();
}

// D[h][j] := min(D[h][j], min_h' C[h][h'] + X_h'[j], C[h][j] if j in H) for
// column j; resets X_h'[j] to "INF" for the next recompute
template <typename T, int SR>
__device__ __forceinline__ unsigned heavy_fix_col(T* D, int64_t ld, int64_t j, int hc, int* x, int64_t ldx,
                                                  int64_t skip, const Mirror& M, const HeavySmem<T>& sm) {
  unsigned mbits = 0;
  T xb[kHeavy];
#pragma unroll
  for (int b = 0; b < kHeavy; ++b) {
    if (b >= hc) break;
    xb[b] = heavy_xval<T>(x[b * ldx + j]);
    x[b * ldx + j] = 0x7F7F7F7F;
  }
  if (j == skip) return 0u;
  for (int a = 0; a < hc; ++a) {
    T v = Tr<T>::inf();
#pragma unroll
    for (int b = 0; b < kHeavy; ++b) {
      if (b >= hc) break;
      v = Tr<T, SR>::relax(v, sm.C[a][b], xb[b]);
      if (sm.hrow[b] == (int)j) v = Tr<T>::mn(v, sm.C[a][b]);
    }
    v = Tr<T>::sat(v);
    T* dp = D + (int64_t)sm.hrow[a] * ld + j;
    if (v < *dp) {
      *dp = v;
      if (M.m || M.m8) mbits |= mput(M, (int64_t)sm.hrow[a] * ld + j, v);
    }
  }
  return mbits;
}

constexpr int kRoundLocal = 16;   // frontier length a single lane relaxes on its own
// The whole warp relaxes pair (i, j) (current value cur) through the cnt
// frontier entries of row i; a lower value is written and joins the next
// round's frontier.
template <typename T, int SR>
__device__ __forceinline__ unsigned round_pair_warp(T* D, int64_t ld, int64_t row0, const T* __restrict__ WT,
                                                    int64_t ldw, const int64_t* __restrict__ rowoff,
                                                    const int* fcol_in, int* fcnt_out, int* ftot_out, int* fcol_out,
                                                    int* any, unsigned* rowkey, const Mirror& M, int64_t pi,
                                                    int64_t pj, int pc, T pcur, int lane) {
  unsigned mbits = 0;
  T* Drow = D + (pi - row0) * ld;
  const T* Wrow = WT + pj * ldw;
  const int* fl = fcol_in + rowoff[pi];
  T acc = Tr<T>::inf();
  int t = lane;
  for (; t + 32 < pc; t += 64) {   // two gathers in flight per lane
    const int64_t m0 = *(volatile const int*)(fl + t), m1 = *(volatile const int*)(fl + t + 32);
    const T d0 = *(volatile T*)(Drow + m0), d1 = *(volatile T*)(Drow + m1);
    const T w0 = Wrow[m0], w1 = Wrow[m1];
    acc = Tr<T, SR>::relax(Tr<T, SR>::relax(acc, d0, w0), d1, w1);
  }
  if (t < pc) {
    const int64_t m = *(volatile const int*)(fl + t);
    acc = Tr<T, SR>::relax(acc, *(volatile T*)(Drow + m), Wrow[m]);
  }
  acc = warp_min<T>(acc);
  if (lane == 0 && acc < pcur) {
    Drow[pj] = acc;
    if (M.m || M.m8) mbits |= mput(M, (pi - row0) * ld + pj, acc);
    fcol_out[rowoff[pi] + atomicAdd(fcnt_out + pi, 1)] = (int)pj;   // j changed: next round's frontier
    atomicAdd(ftot_out, 1);
    if (rowkey) atomicMax(rowkey + pi, open_key<T>(acc));
    *any = 1;
  }
  return mbits;
}

// One round over the open pairs: each lane screens one pair of its warp's 32
// (row changed last round, not heavy, not at its bound, not provably final);
// a pair whose row's frontier is short is relaxed by its lane alone, a long
// one by the whole warp — right away, or (bigq != null) appended to a queue
// that every warp of the grid drains after a barrier (round_big_drain), so a
// few long rows do not serialise on the warps that happen to hold them.
template <typename T, int SR>
__device__ __forceinline__ unsigned sparse_round_body(T* D, int64_t ld, int64_t row0, const T* __restrict__ WT,
                                                      int64_t ldw, const int* __restrict__ gprow,
                                                      const int* __restrict__ gpcol, const T* __restrict__ glb,
                                                      int64_t nopen, const int64_t* __restrict__ rowoff,
                                                      const int* fcnt_in, const int* fcol_in, int* fcnt_out,
                                                      int* ftot_out, int* fcol_out, int* any, unsigned* rowkey,
                                                      T wmin, const Mirror& M, const int* hrow = nullptr,
                                                      int hc = 0, int* bigq = nullptr, int* bigq_tail = nullptr) {
  unsigned mbits = 0;
  const int lane = threadIdx.x & 31;
  const int64_t nw = (int64_t)gridDim.x * (blockDim.x >> 5);
  for (int64_t p0 = (blockIdx.x * (int64_t)(blockDim.x >> 5) + (threadIdx.x >> 5)) * 32; p0 < nopen;
       p0 += nw * 32) {
    const int64_t p = p0 + lane;
    int i = 0, j = 0, cnt = 0;
    T cur = Tr<T>::inf();
    bool need = false;
    if (p < nopen) {
      i = gprow[p];
      cnt = *(volatile const int*)(fcnt_in + i);   // entries of row i changed last round
      bool heavy = false;   // a heavy row: resolved after the rounds (heavy_rows)
      for (int q = 0; q < hc; ++q) heavy |= hrow[q] == i;
      if (cnt != 0 && !heavy) {
        j = gpcol[p];
        cur = *(volatile T*)(D + (int64_t)(i - row0) * ld + j);   // only this pair's warp writes it
        // at its lower bound: final; or no open entry of the row can lower
        // it: every one is >= the row's smallest open value and every
        // weight >= wmin
        need = !Tr<T>::at_lb(cur, glb[p]) &&
               !(rowkey && cur <= Tr<T, SR>::add(open_min<T>(*(volatile unsigned*)(rowkey + i)), wmin));
      }
    }
    const bool local = need && cnt <= kRoundLocal;
    if (local) {
      T* Drow = D + (int64_t)(i - row0) * ld;
      const T* Wrow = WT + (int64_t)j * ldw;
      const int* fl = fcol_in + rowoff[i];
      T acc = Tr<T>::inf();
      for (int t = 0; t < cnt; ++t) {
        const int64_t m = *(volatile const int*)(fl + t);
        acc = Tr<T, SR>::relax(acc, *(volatile T*)(Drow + m), Wrow[m]);
      }
      if (acc < cur) {
        Drow[j] = acc;
        if (M.m || M.m8) mbits |= mput(M, (int64_t)(i - row0) * ld + j, acc);
        fcol_out[rowoff[i] + atomicAdd(fcnt_out + i, 1)] = j;   // j changed: next round's frontier
        atomicAdd(ftot_out, 1);
        if (rowkey) atomicMax(rowkey + i, open_key<T>(acc));
        *any = 1;
      }
    }
    unsigned todo = __ballot_sync(0xffffffffu, need && !local);
    if (bigq) {
      if (todo) {   // one atomic per warp
        int base = 0;
        if (lane == 0) base = atomicAdd(bigq_tail, __popc(todo));
        base = __shfl_sync(0xffffffffu, base, 0);
        if (need && !local) bigq[base + __popc(todo & ((1u << lane) - 1))] = (int)p;
      }
      continue;
    }
    while (todo) {
      const int src = __ffs(todo) - 1;
      todo &= todo - 1;
      const int64_t pi = __shfl_sync(0xffffffffu, i, src), pj = __shfl_sync(0xffffffffu, j, src);
      const int pc = __shfl_sync(0xffffffffu, cnt, src);
      const T pcur = __shfl_sync(0xffffffffu, cur, src);
      mbits |= round_pair_warp<T, SR>(D, ld, row0, WT, ldw, rowoff, fcol_in, fcnt_out, ftot_out, fcol_out, any,
                                      rowkey, M, pi, pj, pc, pcur, lane);
    }
  }
  return mbits;
}

// Drains the queue of long-frontier pairs sparse_round_body appended (after
// a grid barrier): each warp takes the next pair with one atomic.
template <typename T, int SR>
__device__ __forceinline__ unsigned round_big_drain(T* D, int64_t ld, int64_t row0, const T* __restrict__ WT,
                                                    int64_t ldw, const int* __restrict__ gprow,
                                                    const int* __restrict__ gpcol, const int64_t* __restrict__ rowoff,
                                                    const int* fcnt_in, const int* fcol_in, int* fcnt_out,
                                                    int* ftot_out, int* fcol_out, int* any, unsigned* rowkey,
                                                    const Mirror& M, const int* bigq, int tail, int* head) {
  unsigned mbits = 0;
  const int lane = threadIdx.x & 31;
  while (true) {
    int k = 0;
    if (lane == 0) k = atomicAdd(head, 1);
    k = __shfl_sync(0xffffffffu, k, 0);
    if (k >= tail) break;
    const int64_t p = bigq[k];
    const int64_t i = gprow[p], j = gpcol[p];
    const int cnt = *(volatile const int*)(fcnt_in + i);
    const T cur = *(volatile T*)(D + (i - row0) * ld + j);
    mbits |= round_pair_warp<T, SR>(D, ld, row0, WT, ldw, rowoff, fcol_in, fcnt_out, ftot_out, fcol_out, any,
                                    rowkey, M, i, j, cnt, cur, lane);
  }
  return mbits;
}

template <typename T, int SR>
__global__ void __launch_bounds__(256) k_sparse_round(T* D, int64_t ld, int64_t row0,
                                                      const T* __restrict__ WT, int64_t ldw,
                                                      const int* __restrict__ gprow,
                                                      const int* __restrict__ gpcol,
                                                      const T* __restrict__ glb, int64_t nopen,
                                                      const int64_t* __restrict__ rowoff,
                                                      const int* __restrict__ fcnt_in,
                                                      const int* __restrict__ ftot_in,
                                                      const int* __restrict__ fcol_in,
                                                      int* fcnt_out, int* ftot_out, int* fcol_out, int* any,
                                                      const DetectCounters* dc, unsigned* rowkey, T wmin,
                                                      Mirror M) {
  // an empty frontier (nothing changed last round): the round is a no-op
  if (ftot_in && *(volatile const int*)ftot_in == 0) return;
  nopen = device_count(dc, nopen, 1);
  const unsigned mbits = sparse_round_body<T, SR>(D, ld, row0, WT, ldw, gprow, gpcol, glb, nopen, rowoff, fcnt_in,
                                                  fcol_in, fcnt_out, ftot_out, fcol_out, any, rowkey, wmin, M);
  if (M.m || M.m8) mirror_post(M, mbits);
}

// Rounds r0 .. r1 - 1 in ONE cooperative launch, a grid-wide barrier between
// rounds, stopping after the first round that changes nothing: no host round
// trip per batch of rounds.  Buffers as the one-round kernel's: frontier
// counts per round in chg[round % 4] (their totals at [cap]; rounds 0-3
// zeroed by the caller, round r + 1's during round r — that buffer was last
// read in round r - 2 — so no extra barrier), frontier lists alternating between
// fcol[0] / fcol[1]; round 0 reads the open lists (ocnt / ocol).  *rounds_run
// receives the number of rounds executed; *last_total the last round's total.
template <typename T, int SR>
__global__ void __launch_bounds__(256) k_sparse_rounds_coop(T* D, int64_t ld, int64_t row0, const T* __restrict__ WT,
                                                            int64_t ldw, const int* __restrict__ gprow,
                                                            const int* __restrict__ gpcol, const T* __restrict__ glb,
                                                            int64_t nopen, const int64_t* __restrict__ rowoff,
                                                            const int* ocnt, const int* ocol, RoundBufs rb, int r0,
                                                            int r1, int* any, const DetectCounters* dc,
                                                            unsigned* rowkey, T wmin, Mirror M) {
  namespace cg = cooperative_groups;
  cg::grid_group grid = cg::this_grid();
  nopen = device_count(dc, nopen, 1);
  __shared__ HeavySmem<T> sm;
  int* hrow = sm.hrow;
  unsigned mbits = 0;
  if (rb.tail) {   // A2, then B, then the open rows' minima (each reads the one before)
    const OpenLists<T> ol{};
    mbits |= sparse_short_body<T, SR>(D, ld, row0, rb.slid, static_cast<const T*>(rb.slw),
                                      static_cast<const T*>(rb.wnext), gprow, gpcol, glb, nopen, rb.gfull, 1, ol,
                                      dc, M, rb.skip);
    grid.sync();
    mbits |= sparse_full_body<T, SR>(D, ld, row0, WT, ldw, rb.n, gprow, gpcol, glb, rb.gfull, nopen, dc, M,
                                     &sm.w[0][0]);
    grid.sync();
    for (int64_t p = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; p < nopen; p += (int64_t)gridDim.x * blockDim.x) {
      const int64_t i = gprow[p];
      atomicMax(rowkey + i, open_key<T>(D[(i - row0) * ld + gpcol[p]]));
    }
    if (rb.heavy_thr <= 0) grid.sync();   // (else the selection's barrier below)
  }
  if (rb.heavy_thr > 0) {   // heavy rows: >= heavy_thr open pairs (the first kHeavy found)
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < rb.rows;
         i += (int64_t)gridDim.x * blockDim.x)
      if (ocnt[i] >= rb.heavy_thr) {
        const int s = atomicAdd(rb.heavy, 1);
        if (s < kHeavy) rb.heavy[1 + s] = (int)i;
      }
    grid.sync();
  }
  const int hc = rb.heavy_thr > 0 ? min(*(volatile const int*)rb.heavy, kHeavy) : 0;
  if (threadIdx.x < hc) hrow[threadIdx.x] = *(volatile const int*)(rb.heavy + 1 + threadIdx.x);
  __syncthreads();
  int round = r0;
  for (; round < r1; ++round) {
    const int o = round & 3, oi = (round + 3) & 3;
    int* chg_o = rb.chg + (int64_t)o * rb.stride;
    const int* fin_c = round == 0 ? ocnt : rb.chg + (int64_t)oi * rb.stride;
    const int* fin_l = round == 0 ? ocol : rb.fcol[(round & 1) ^ 1];
    // the previous round changed nothing: converged (grid-uniform after the barrier)
    if (round > 0 && *(volatile const int*)(fin_c + rb.cap) == 0) break;
    // this round's queue counters (tail, head) at bq[2 (round & 1)]; the other
    // pair is reset for the next round (nobody uses it now)
    int* bq = rb.bigq_ctr + 2 * (round & 1);
    if (blockIdx.x == 0 && threadIdx.x < 2) rb.bigq_ctr[2 * ((round + 1) & 1) + threadIdx.x] = 0;
    if (round + 1 >= 4) {   // the next round's counts (last read two rounds ago) start at zero
      int* chg_n = rb.chg + (int64_t)((round + 1) & 3) * rb.stride;
      for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e <= rb.cap; e += (int64_t)gridDim.x * blockDim.x)
        chg_n[e] = 0;
    }
    mbits |= sparse_round_body<T, SR>(D, ld, row0, WT, ldw, gprow, gpcol, glb, nopen, rowoff, fin_c, fin_l, chg_o,
                                      chg_o + rb.cap, rb.fcol[round & 1], any, rowkey, wmin, M, hrow, hc, rb.bigq,
                                      bq);
    grid.sync();
    const int tail = *(volatile int*)bq;
    if (tail > 0) {   // grid-uniform
      mbits |= round_big_drain<T, SR>(D, ld, row0, WT, ldw, gprow, gpcol, rowoff, fin_c, fin_l, chg_o, chg_o + rb.cap,
                                      rb.fcol[round & 1], any, rowkey, M, rb.bigq, tail, bq + 1);
      grid.sync();
    }
  }
  if (hc > 0) {   // the heavy rows, from the other rows (final once the rounds converged)
    const int64_t n = rb.n;
    // Pruning the first hops: D'[h][j] <= B_h = max_j D[h][j] (every entry is
    // already a walk length of G'), so a first hop m with W'[h][m] > B_h lies
    // on no shortest h -> j path — only the m with W'[h][m] <= B_h for some
    // heavy h are read.  B_h as order keys in heavy[1 + kHeavy + k].
    int* bkey = rb.heavy + 1 + kHeavy;
    int* nlive = rb.heavy + 1 + 2 * kHeavy;
    int* mlist = rb.bigq;   // free again: the rounds are over
    for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < (int64_t)hc * n;
         e += (int64_t)gridDim.x * blockDim.x) {
      const int k = (int)(e / n);
      const int64_t j = e - (int64_t)k * n;
      if (j == rb.skip) continue;
      int kv = heavy_xkey<T>(D[(int64_t)hrow[k] * ld + j]);
      kv = __reduce_max_sync(__activemask(), kv);
      atomicMax(bkey + k, kv);
    }
    grid.sync();
    for (int64_t m = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; m < n; m += (int64_t)gridDim.x * blockDim.x) {
      bool live = false, inh = m == rb.skip;
      for (int k = 0; k < hc; ++k) inh |= hrow[k] == (int)m;
      if (!inh)
        for (int k = 0; k < hc && !live; ++k) live = WT[m * ldw + hrow[k]] <= heavy_xval<T>(bkey[k]);
      if (live) mlist[atomicAdd(nlive, 1)] = (int)m;
    }
    grid.sync();
    const int64_t nl = *(volatile int*)nlive;
    const int64_t gx = (n + 127) / 128;
    const int ng = (hc + kHxGroup - 1) / kHxGroup;
    const int64_t ny = max((int64_t)1, min((nl + kHxSlab - 1) / kHxSlab, 2 * (int64_t)gridDim.x / (gx * ng)));
    const int64_t slab = ((nl + ny - 1) / ny + kHxSlab - 1) / kHxSlab * kHxSlab;
    const int64_t items = nl > 0 ? gx * ng * ((nl + slab - 1) / slab) : 0;
    for (int64_t it = blockIdx.x; it < items; it += gridDim.x) {
      const int64_t stripe = it % gx, rest = it / gx;
      const int g = (int)(rest % ng);
      const int64_t m0 = (rest / ng) * slab;
      heavy_x_item<T, SR>(D, ld, n, WT, ldw, hc, g * kHxGroup, stripe, m0, min(nl, m0 + slab), rb.heavy_x, rb.ldx,
                          rb.skip, sm, mlist);
    }
    grid.sync();
    heavy_closure<T, SR>(WT, ldw, hc, sm);
    for (int64_t j = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; j < n; j += (int64_t)gridDim.x * blockDim.x)
      mbits |= heavy_fix_col<T, SR>(D, ld, j, hc, rb.heavy_x, rb.ldx, rb.skip, M, sm);
  }
  if (M.m || M.m8) mirror_post(M, mbits);
  if (blockIdx.x == 0 && threadIdx.x == 0) {
    *rb.rounds_run = round - r0;
    // the last round that ran (or the one that found nothing): its total
    const int last = round > r0 ? round - 1 : r0;
    *rb.last_total = rb.chg[(int64_t)(last & 3) * rb.stride + rb.cap];
  }
  if (rb.host) {   // every block's writes and flag bits in place: the host's read
    grid.sync();
    if (blockIdx.x == 0 && threadIdx.x == 0) {
      volatile long long* host = static_cast<volatile long long*>(rb.host);
      reinterpret_cast<volatile unsigned*>(host)[14] = (unsigned)*rb.rounds_run;
      host[0] = (long long)dc->total;
      host[1] = (long long)dc->rows;
      host[2] = (dc->overflow & 1u) ? 1 : 0;
      host[3] = (dc->overflow & 2u) ? 1 : 0;
      host[4] = *(volatile int*)rb.last_total ? 1 : 0;
      host[5] = (long long)dc->maxrow;
      reinterpret_cast<volatile unsigned*>(host)[12] = *(volatile const unsigned*)rb.mflag;
      __threadfence_system();
    }
  }
}
template <typename T>
cudaError_t sparse_rounds_coop(T* D, int64_t ld, int64_t row0, const T* WT, int64_t ldw, const int* gprow,
                               const int* gpcol, const T* glb, int64_t nopen, const int64_t* rowoff, const int* ocnt,
                               const int* ocol, const RoundBufs& rb, int r0, int r1, int* any, int sr,
                               const DetectCounters* dc, cudaStream_t st, unsigned* rowkey, T wmin, Mirror M) {
  auto kern = sr ? k_sparse_rounds_coop<T, 1> : k_sparse_rounds_coop<T, 0>;
  static int per_sm[2] = {0, 0};
  int& bps = per_sm[sr ? 1 : 0];
  if (!bps) {
    CUDA_TRY(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&bps, kern, 256, 0));
    if (bps <= 0) return cudaErrorInvalidConfiguration;
  }
#ifndef COOP_BPS
#define COOP_BPS 2
#endif
  const int grid = std::min(bps, COOP_BPS) * num_sms();
  void* args[] = {&D, &ld, &row0, &WT, &ldw, &gprow, &gpcol, &glb, &nopen, &rowoff, &ocnt, &ocol,
                  const_cast<RoundBufs*>(&rb), &r0, &r1, &any, &dc, &rowkey, &wmin, &M};
  return cudaLaunchCooperativeKernel(reinterpret_cast<void*>(kern), grid, 256, args, 0, st);
}
template <typename T>
cudaError_t sparse_round(T* D, int64_t ld, int64_t row0, const T* WT, int64_t ldw,
                         const int* gprow, const int* gpcol, const T* glb, int64_t nopen,
                         const int64_t* rowoff, const int* fcnt_in, const int* ftot_in, const int* fcol_in,
                         int* fcnt_out, int* ftot_out, int* fcol_out, int* any, int sr,
                         const DetectCounters* dc, cudaStream_t st, unsigned* rowkey, T wmin, Mirror M) {
  if (nopen <= 0) return cudaSuccess;
  // round 0 relaxes every open pair through its row's open entries; later
  // rounds only the pairs whose row changed (often none: a small grid keeps
  // the no-op round cheap)
  int grid = (int)std::min<int64_t>(cdiv(nopen, 256), (int64_t)num_sms() * (ftot_in ? 2 : 8));
  if (sr)
    k_sparse_round<T, 1><<<grid, 256, 0, st>>>(D, ld, row0, WT, ldw, gprow, gpcol, glb, nopen, rowoff,
                                               fcnt_in, ftot_in, fcol_in, fcnt_out, ftot_out, fcol_out, any,
                                               dc, rowkey, wmin, M);
  else
    k_sparse_round<T, 0><<<grid, 256, 0, st>>>(D, ld, row0, WT, ldw, gprow, gpcol, glb, nopen, rowoff,
                                               fcnt_in, ftot_in, fcol_in, fcnt_out, ftot_out, fcol_out, any,
                                               dc, rowkey, wmin, M);
  return cudaGetLastError();
}

#define INST(T)                                                                                   \
  template cudaError_t shortlist_build<T>(const T*, int64_t, int64_t, const int*, int64_t, int64_t, \
                                          int*, T*, T*, cudaStream_t);                            \
  template cudaError_t shortlist_add_bound<T>(int*, T*, T*, const T*, int64_t, int64_t,            \
                                              cudaStream_t);                                      \
  template cudaError_t shortlist_build_one<T>(const T*, int64_t, int64_t, int64_t, int*, T*, T*, void*, \
                                              cudaStream_t);                                      \
  template cudaError_t shortlist_set_edge<T>(int*, T*, T*, int64_t, int64_t, T, int, cudaStream_t); \
  template cudaError_t shortlist_swap<T>(int*, T*, T*, int64_t, int64_t, int64_t, cudaStream_t);    \
  template cudaError_t shortlist_remove<T>(int*, T*, T*, int64_t, int64_t, int64_t, cudaStream_t); \
  template cudaError_t edge_early<T>(T*, int64_t, const T*, int*, T*, T*, int64_t, int64_t, T, int, float, void*, \
                                     cudaStream_t);                                                  \
  template cudaError_t sparse_short<T>(T*, int64_t, int64_t, const int*, const T*, const T*,       \
                                       const int*, const int*, const T*, int64_t, unsigned char*,  \
                                       int, int, const DetectCounters*, cudaStream_t, Mirror, int64_t);            \
  template cudaError_t sparse_phase_a<T>(T*, int64_t, Rows, const int*, const T*, const int64_t*,  \
                                         const int*, const int*, int64_t, const T*, const T*,      \
                                         const T*, const T*, float, int*, int*, int*, int*, T*,    \
                                         unsigned char*, int64_t, DetectCounters*, int, Mirror,    \
                                         cudaStream_t, int, const uint8_t*, int*, int*);           \
  template cudaError_t sparse_full<T>(T*, int64_t, int64_t, const T*, int64_t, int64_t,            \
                                      const int*, const int*, const T*, const unsigned char*,      \
                                      int64_t, int, const DetectCounters*, cudaStream_t, Mirror);         \
  template cudaError_t open_rowmin<T>(const T*, int64_t, int64_t, const int*, const int*, int64_t,      \
                                      unsigned*, const DetectCounters*, cudaStream_t);             \
  template cudaError_t sparse_rounds_coop<T>(T*, int64_t, int64_t, const T*, int64_t, const int*, const int*, \
                                             const T*, int64_t, const int64_t*, const int*, const int*,      \
                                             const RoundBufs&, int, int, int*, int, const DetectCounters*,    \
                                             cudaStream_t, unsigned*, T, Mirror);                               \
  template cudaError_t sparse_round<T>(T*, int64_t, int64_t, const T*, int64_t, const int*,        \
                                       const int*, const T*, int64_t, const int64_t*, const int*,  \
                                       const int*, const int*, int*, int*, int*, int*, int,        \
                                       const DetectCounters*, cudaStream_t, unsigned*, T, Mirror);
INST(int32_t)
INST(float)
#undef INST

}  // namespace apsp
