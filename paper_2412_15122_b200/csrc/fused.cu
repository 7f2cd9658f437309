// fused.cu — detection and the sparse recompute's phase A in ONE pass over
// the int8 mirror (removal of a node / increase of a directed edge, int32
// shortest path, int8 mirror valid).
//
// The need_update_list (Corollary 3 / Theorem 4) of
// row i and phase A of every pair on it (sparse.cu: the last-hop bound
// D'[i][j] <= min_m D[i][m] + W'[m][j] over the cheapest in-edges m of j,
// certified when it reaches lb = D_old[i][j]) need only row i of D — which
// the detection pass streams anyway.  Done separately, phase A re-reads
// D[i][m] and D_old[i][j] by random one-byte gathers (each a DRAM sector:
// ~0.2 GB and ~0.1 ms per BJ.c4 removal, measured); here row i sits whole
// in shared memory while its pairs are certified.
//
// CTA = 8 worker warps + 1 producer warp; a CTA owns a slab of whole rows.
// The producer bulk-copies each row (TMA, one copy of the row's n bytes: a
// single large copy streams at ~6.8 TB/s over the chip, measured by
// scripts/tma_probe.cu) into a ring of S stages.  Worker warp w, at step rr:
//   scan   row rr: its 512-byte segments w, w + 8, ... with the SWAR byte test
//          of k_detect_p8 (stream.cu) against the pivot row (staged in shared
//          memory once); for each flagged pair (i, j) it records j and starts
//          an asynchronous copy (cp.async) of the head of SL(j) — the 8
//          cheapest in-edges (ids and weights, 64 bytes) — into shared memory;
//   certify row rr - 1 (its copies have landed meanwhile): phase A on the
//          first 8 in-edges of each pair, reading D[i][m] from the row in
//          shared memory; a stale D_old[i][m] (m itself listed) is recognised
//          by the detection predicate and skipped, exactly as in
//          k_sparse_phase_a.  A certified pair keeps its value (it equals
//          D_old): nothing is written.  Pairs not certified — and pairs beyond
//          a warp's per-row slots — are appended to the global list, whose
//          phase A is the stand-alone kernel (sparse.cu), run right after
//          with its full shortlist walk and the open-list appends;
//   release row rr - 1 to the producer (one arrival per warp).
// The row counts |A_i| are written per row (rowcnt); the per-row slices of
// the open lists, Phi and max |A_i| come from detect_lists afterwards.
#include "common.cuh"
#include "kernels.h"
#include "mirror.cuh"
#include "tma.cuh"

namespace apsp {

__host__ __device__ static inline int64_t cdiv_f(int64_t a, int64_t b) { return (a + b - 1) / b; }

constexpr int kFW = 16;                        // worker warps (latency hiding: the per-row work is a chain)
constexpr int kFThreads = 32 * (kFW + 1);      // + the producer warp
constexpr int kFSlots = 8;                     // certified-in-kernel pairs per warp and row
constexpr int kFSeg = 6;                       // 512-byte row segments per worker (pivot row in registers)

constexpr int kFQ = 64;                        // per-warp queue of pairs for the global list
struct FusedSmem {   // byte offsets into the dynamic shared memory
  int64_t ring, r1b, slj, slh, dq, pcnt, dcnt, bars, total;
};
// slh: [2][kFW][kFSlots] heads of SL(j), 8 ids + 8 weights (64 B) each;
// slj: [2][kFW][kFSlots] the pairs' columns j (double-buffered by row parity)
__host__ __device__ inline FusedSmem fused_layout(int S, int64_t RB) {
  FusedSmem L;
  int64_t o = 0;
  L.ring = o; o += S * RB;
  L.r1b = o; o += RB;
  L.slh = o; o += 2 * kFW * kFSlots * 64;
  L.slj = o; o += 2 * kFW * kFSlots * 4;
  L.dq = o; o += kFW * kFQ * 8;
  L.pcnt = o; o += S * 4;
  L.dcnt = o; o += S * 4;
  o = (o + 7) / 8 * 8;
  L.bars = o; o += 2 * S * 8;
  L.total = o;
  return L;
}

struct FusedArgs {
  int32_t* D; int64_t ld; Rows r; int64_t n; int64_t skip;
  const int32_t* c1; const int32_t* r1;
  const int* SLid; const int32_t* SLw;
  uint8_t* M8; unsigned* mflag;
  int* rowcnt;
  int* srow; int* scol; int64_t lcap;   // the pairs left to the stand-alone phase A (all, if export_only)
  DetectCounters* ctr;
  int64_t slab, RB;
  int export_only;                      // 1: every pair on the global list, no certification
};

__device__ __forceinline__ uint32_t sat8u(int32_t v) { return (uint32_t)min(v, kSat8i); }

template <int S>
__global__ void __launch_bounds__(kFThreads, 1) k_detect_fix_p8(FusedArgs a) {
  extern __shared__ __align__(128) uint8_t sm[];
  const FusedSmem L = fused_layout(S, a.RB);
  uint8_t* ring = sm + L.ring;
  uint8_t* r1b = sm + L.r1b;
  uint4* slh = reinterpret_cast<uint4*>(sm + L.slh);   // 4 uint4 per slot
  int* slj = reinterpret_cast<int*>(sm + L.slj);
  int2* dq = reinterpret_cast<int2*>(sm + L.dq) + (threadIdx.x >> 5) * kFQ;   // this warp's queue
  int* pcnt = reinterpret_cast<int*>(sm + L.pcnt);
  int* dcnt = reinterpret_cast<int*>(sm + L.dcnt);
  uint64_t* full = reinterpret_cast<uint64_t*>(sm + L.bars);
  uint64_t* empty = full + S;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int64_t n = a.n, ld = a.ld, skip = a.skip, row0 = a.r.row0;
  const int64_t i_lo = a.r.lo + (int64_t)blockIdx.x * a.slab;
  const int64_t i_hi = min(a.r.hi, i_lo + a.slab);
  const int rows = (int)max((int64_t)0, i_hi - i_lo);
  if (rows == 0) return;   // CTA-uniform
  // the pivot row as saturated bytes (0x7F = INF; columns >= n read as INF)
  for (int64_t j = tid; j < a.RB / 4; j += blockDim.x) {
    uint32_t w = 0;
#pragma unroll
    for (int e = 0; e < 4; ++e) {
      const int64_t c = 4 * j + e;
      w |= (c < n ? sat8u(a.r1[c]) : (uint32_t)kSat8i) << (8 * e);
    }
    reinterpret_cast<uint32_t*>(r1b)[j] = w;
  }
  if (tid < S) { pcnt[tid] = 0; dcnt[tid] = 0; }
  if (tid == 0) {
    for (int s = 0; s < S; ++s) {
      mbar_init(full + s, 1);
      mbar_init(empty + s, kFW);
    }
    fence_barrier_init();
  }
  __syncthreads();
  const unsigned cb = (unsigned)((n + 15) & ~15);

  if (warp == kFW) {   // ---------------- producer: one bulk copy per row
    if (lane == 0) {
      const uint8_t* src = a.M8 + (i_lo - row0) * ld;
      for (int rr = 0; rr < rows; ++rr) {
        const int s = rr % S;
        if (rr >= S) mbar_wait(empty + s, (unsigned)(rr / S - 1) & 1u);
        mbar_expect_tx(full + s, cb);
        bulk_g2s(ring + s * a.RB, src + (int64_t)rr * ld, cb, full + s);
      }
    }
    return;
  }

  // ---------------- worker warps
  const int nseg = (int)cdiv_f(n, 512);
  uint32_t rreg[kFSeg][4];   // this lane's 16 bytes of the pivot row in each of the warp's segments
#pragma unroll
  for (int t = 0; t < kFSeg; ++t) {
    const int seg = warp + t * kFW;
    const uint4 v = seg < nseg ? *reinterpret_cast<const uint4*>(r1b + (int64_t)seg * 512 + 16 * lane)
                               : make_uint4(0x7F7F7F7Fu, 0x7F7F7F7Fu, 0x7F7F7F7Fu, 0x7F7F7F7Fu);
    rreg[t][0] = v.x; rreg[t][1] = v.y; rreg[t][2] = v.z; rreg[t][3] = v.w;
  }
  const int32_t I = APSP_INF_I32_DEV;
  uint32_t cl = 0, cw_prev = 0;      // the pivot column's byte of row rr - 1 (stale test)
  int ncur = 0, nprev = 0;            // slots this warp filled for row rr / rr - 1 (warp-uniform)
  unsigned long long my_pairs = 0;
  // pairs for the global list go through a per-warp shared-memory queue,
  // flushed 32+ at a time (one atomic on the list cursor per flush: its
  // round trip would otherwise hold the row's slot)
  int qn = 0;   // queued pairs (warp-uniform)
  auto flush = [&]() {
    if (qn == 0) return;
    __syncwarp();
    unsigned long long q0 = 0;
    if (lane == 0) q0 = atomicAdd(&a.ctr->spill, (unsigned long long)qn);
    q0 = __shfl_sync(0xffffffffu, q0, 0);
    for (int e = lane; e < qn; e += 32) {
      const unsigned long long q = q0 + e;
      if ((int64_t)q < a.lcap) {
        a.srow[q] = dq[e].x;
        a.scol[q] = dq[e].y;
      } else {
        atomicOr(&a.ctr->overflow, 1u);
      }
    }
    __syncwarp();
    qn = 0;
  };
  auto spill = [&](bool want, int64_t i, int j) {   // warp-collective: queue (i, j) for want lanes
    const unsigned bal = __ballot_sync(0xffffffffu, want);
    if (!bal) return;
    if (qn + 32 > kFQ) flush();
    if (want) dq[qn + __popc(bal & ((1u << lane) - 1))] = make_int2((int)i, j);
    qn += __popc(bal);
    if (qn >= 32) flush();
  };
  uint32_t cw_prev_next = 0;
  auto cgroup = [&](int r0) -> uint32_t {
    const int64_t il = i_lo + r0 + lane;
    return (r0 + lane < rows && il != skip) ? sat8u(a.c1[il]) * 0x01010101u : 0x7F7F7F7Fu;
  };
  uint32_t cl_next = cgroup(0);
  for (int rr = 0; rr <= rows; ++rr) {
    // ---- scan row rr
    if (rr < rows) {
      const int s = rr % S;
      const int64_t i = i_lo + rr;
      if ((rr & 31) == 0) {   // the pivot column for 32 rows, one per lane (INF on row k),
        cl = cl_next;         // loaded a group ahead
        cl_next = cgroup(rr + 32);
      }
      const uint32_t cw = __shfl_sync(0xffffffffu, cl, rr & 31);
      mbar_wait(full + s, (unsigned)(rr / S) & 1u);
      const uint8_t* row = ring + s * a.RB;
      const int par = rr & 1;
      ncur = 0;
      int found = 0;
      // the SWAR test of the warp's segments w, w + kFW, ... (at most kFSeg)
      uint32_t accs[kFSeg];
      uint32_t anyacc = 0;
#pragma unroll
      for (int t = 0; t < kFSeg; ++t) {
        accs[t] = 0;
        const int seg = warp + t * kFW;
        if (seg < nseg) {
          const uint4 dv = *reinterpret_cast<const uint4*>(row + (int64_t)seg * 512 + 16 * lane);
          const uint32_t d[4] = {dv.x, dv.y, dv.z, dv.w};
#pragma unroll
          for (int q = 0; q < 4; ++q) {
            // every byte <= 0x7F and D <= c + r: no carries or borrows between
            // bytes; the entry is tight iff its byte of u is 0 (k_detect_p8)
            const uint32_t u = cw + rreg[t][q] - d[q];
            accs[t] |= (u - 0x01010101u) & ~u;
          }
          anyacc |= accs[t];
        }
      }
      if (__any_sync(0xffffffffu, (anyacc & 0x80808080u) != 0u)) {
#pragma unroll
        for (int t = 0; t < kFSeg; ++t) {
          const int seg = warp + t * kFW;
          if (seg >= nseg || !__any_sync(0xffffffffu, (accs[t] & 0x80808080u) != 0u)) continue;
          const int64_t off = (int64_t)seg * 512 + 16 * lane;
          unsigned bits = 0;   // bit b <-> column off + b
          if (accs[t] & 0x80808080u) {
            const uint4 dv = *reinterpret_cast<const uint4*>(row + off);
            const uint32_t d[4] = {dv.x, dv.y, dv.z, dv.w};
#pragma unroll
            for (int q = 0; q < 4; ++q) {
              // exact zero bytes of u, minus the INF entries (d == 0x7F: a row
              // whose c is INF and a column whose r is 0 would test tight; INF
              // pairs are never listed, Q5)
              const uint32_t u = cw + rreg[t][q] - d[q];
              const uint32_t di = d[q] ^ 0x7F7F7F7Fu;
              const uint32_t z = ~(u | ((u & 0x7F7F7F7Fu) + 0x7F7F7F7Fu)) &
                                 (di | ((di & 0x7F7F7F7Fu) + 0x7F7F7F7Fu)) & 0x80808080u;
              bits |= (((((z >> 7) & 0x01010101u) * 0x01020408u) >> 24) & 0xFu) << (4 * q);
            }
#pragma unroll
            for (int b = 0; b < 16; ++b) {
              const int64_t j = off + b;
              if (j >= n || j == skip || j == i) bits &= ~(1u << b);
            }
          }
          // the flagged pairs: slots (with the head of SL(j) on its way) or the list
          while (__any_sync(0xffffffffu, bits != 0u)) {
            const bool have = bits != 0u;
            const int b = have ? __ffs(bits) - 1 : 0;
            if (have) bits &= bits - 1;
            const int j = (int)(off + b);
            const unsigned bal = __ballot_sync(0xffffffffu, have);
            const int k = ncur + __popc(bal & ((1u << lane) - 1));
            const bool slot = have && !a.export_only && k < kFSlots;
            if (slot) {
              const int e = (par * kFW + warp) * kFSlots + k;
              slj[e] = j;
              cp_async16(slh + 4 * e + 0, a.SLid + (int64_t)j * kSL);
              cp_async16(slh + 4 * e + 1, a.SLid + (int64_t)j * kSL + 4);
              cp_async16(slh + 4 * e + 2, a.SLw + (int64_t)j * kSL);
              cp_async16(slh + 4 * e + 3, a.SLw + (int64_t)j * kSL + 4);
            }
            spill(have && !slot, i, j);
            if (!a.export_only) ncur = min(ncur + __popc(bal), kFSlots);   // (slots filled)
            found += __popc(bal);
          }
        }
      }
      cp_async_commit();   // (one group per row, possibly empty)
      if (lane == 0 && found) atomicAdd(pcnt + s, found);
      my_pairs += (unsigned)found;
      cw_prev_next = cw;
    }
    // ---- certify row rr - 1 (its heads of SL(j) have landed), then release it
    if (rr >= 1) {
      const int rp = rr - 1, s = rp % S, par = rp & 1;
      const int64_t i = i_lo + rp;
      if (rr < rows) cp_async_wait<1>(); else cp_async_wait<0>();
      __syncwarp();
      const uint8_t* row = ring + s * a.RB;
      bool defer = false;
      int j = 0;
      if (lane < nprev) {
        const int e = (par * kFW + warp) * kFSlots + lane;
        j = slj[e];
        // c[i] saturated at 0x7F: exact for the stale test (ci + r == d with
        // d <= 0x7E needs ci < 0x7F; a saturated ci never tests stale, nor
        // does the true one)
        const int32_t ci = (int32_t)(cw_prev & 0xFFu);
        const int32_t lb = (int32_t)row[j];   // D_old[i][j]: finite (a listed pair)
        const uint4 m0 = slh[4 * e + 0], m1 = slh[4 * e + 1], w0 = slh[4 * e + 2], w1 = slh[4 * e + 3];
        const int m[8] = {(int)m0.x, (int)m0.y, (int)m0.z, (int)m0.w, (int)m1.x, (int)m1.y, (int)m1.z, (int)m1.w};
        const int w[8] = {(int)w0.x, (int)w0.y, (int)w0.z, (int)w0.w, (int)w1.x, (int)w1.y, (int)w1.z, (int)w1.w};
        int32_t acc = I;
#pragma unroll
        for (int q = 0; q < 8; ++q) {
          if (m[q] < 0) continue;
          const int32_t d8 = (int32_t)row[m[q]];
          const int32_t r8 = (int32_t)r1b[m[q]];
          if (d8 == kSat8i) continue;                        // INF: no candidate
          if (r8 != kSat8i && ci + r8 == d8) continue;       // stale: m is listed itself
          acc = min(acc, min(d8 + w[q], I));
        }
        // certified iff the bound reaches lb (then it equals D_old: nothing
        // to write); otherwise the stand-alone phase A takes the pair
        defer = acc > lb;
      }
      spill(defer, i, j);
      __syncwarp();
      if (lane == 0) {
        if (atomicAdd(dcnt + s, 1) == kFW - 1) {   // the row's last warp: its |A_i|
          __threadfence_block();
          const int cnt = *(volatile int*)(pcnt + s);
          if (cnt > 0) a.rowcnt[i] = cnt;
          pcnt[s] = 0;
          dcnt[s] = 0;
        }
        mbar_arrive(empty + s);
      }
    }
    nprev = ncur;
    cw_prev = cw_prev_next;
  }
  flush();
  if (lane == 0 && my_pairs) atomicAdd(&a.ctr->total, my_pairs);
}

// Ring depth for a row of `n` bytes (0: the row does not fit; use the
// separate kernels).
int fused_stages(int64_t n) {
  const int64_t RB = (n + 511) / 512 * 512;
  if (RB / 512 > (int64_t)kFW * kFSeg) return 0;   // more segments than the workers hold
  for (int S = 5; S >= 3; --S)
    if (fused_layout(S, RB).total <= 227 * 1024) return S;
  return 0;
}

cudaError_t detect_fix_p8(int32_t* D, int64_t ld, Rows r, int64_t n, int64_t skip, const int32_t* c1,
                          const int32_t* r1, const int* SLid, const int32_t* SLw, Mirror M, int* rowcnt,
                          int* srow, int* scol, int64_t lcap, DetectCounters* ctr, int export_only,
                          cudaStream_t st) {
  const int S = fused_stages(n);
  if (!S || !M.m8) return cudaErrorInvalidValue;
  const int64_t m = r.hi - r.lo;
  if (m <= 0) return cudaSuccess;
  FusedArgs a;
  a.D = D; a.ld = ld; a.r = r; a.n = n; a.skip = skip; a.c1 = c1; a.r1 = r1; a.SLid = SLid; a.SLw = SLw;
  a.M8 = M.m8; a.mflag = M.flag; a.rowcnt = rowcnt; a.srow = srow; a.scol = scol;
  a.lcap = lcap; a.ctr = ctr; a.export_only = export_only;
  a.RB = (n + 511) / 512 * 512;
  const int grid = (int)std::min<int64_t>(m, num_sms());
  a.slab = cdiv_f(m, grid);
  const int ctas = (int)cdiv_f(m, a.slab);
  const size_t smem = (size_t)fused_layout(S, a.RB).total;
  static const cudaError_t attr = [] {
    const int mx = 227 * 1024;
    cudaError_t e = cudaFuncSetAttribute(k_detect_fix_p8<5>, cudaFuncAttributeMaxDynamicSharedMemorySize, mx);
    if (e == cudaSuccess) e = cudaFuncSetAttribute(k_detect_fix_p8<4>, cudaFuncAttributeMaxDynamicSharedMemorySize, mx);
    if (e == cudaSuccess) e = cudaFuncSetAttribute(k_detect_fix_p8<3>, cudaFuncAttributeMaxDynamicSharedMemorySize, mx);
    return e;
  }();
  CUDA_TRY(attr);
  if (S == 5) k_detect_fix_p8<5><<<ctas, kFThreads, smem, st>>>(a);
  else if (S == 4) k_detect_fix_p8<4><<<ctas, kFThreads, smem, st>>>(a);
  else k_detect_fix_p8<3><<<ctas, kFThreads, smem, st>>>(a);
  return cudaGetLastError();
}

}  // namespace apsp
