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
// scripts/tma_probe.cu) into a ring of S stages.  Worker warp w scans its
// 512-byte segments w, w + 8, ... of each row with the SWAR byte test of
// k_detect_p8 (stream.cu) against the pivot row (held in registers), keeps
// each flagged pair (i, j) with lb = D_old[i][j], starts an asynchronous copy
// (cp.async) of the head of SL(j) — the 8 cheapest in-edges m of j, ids and
// weights — and releases the row's stage at once (the ring keeps S - 1 rows
// in flight).  Pairs are processed in batches of kB per warp, pipelined:
//   batch k fills (shortlist heads on their way);
//   batch k - 1: heads landed -> asynchronous gathers of D[i][m] (from the
//     mirror in global memory — its rows were streamed moments ago, so these
//     hit L2) and of the pivot row at m;
//   batch k - 2: gathers landed -> phase A on the first 8 in-edges: a stale
//     D_old[i][m] (m itself listed) is recognised by the detection predicate
//     and skipped, exactly as in k_sparse_phase_a.  A certified pair keeps
//     its value (it equals D_old): nothing is written.  A pair not certified
//     goes to the deferred list with its bound acc (a walk length of G', or
//     INF); k_defer_apply then writes it and appends it to the open lists,
//     for A2 / B / the rounds — so every listed entry ends up final or open
//     with a walk length, as after k_sparse_phase_a.
// The row counts |A_i| are written per row (rowcnt); the per-row slices of
// the open lists, Phi and max |A_i| come from detect_lists afterwards.
#include "common.cuh"
#include "kernels.h"
#include "mirror.cuh"
#include "tma.cuh"

namespace apsp {

__host__ __device__ static inline int64_t cdiv_f(int64_t a, int64_t b) { return (a + b - 1) / b; }

constexpr int kFW = 8;                         // worker warps
constexpr int kFThreads = 32 * (kFW + 1);      // + the producer warp
constexpr int kFSeg = 9;                       // 512-byte row segments per worker (pivot row in registers)
constexpr int kB = 16;                         // pairs per batch (per warp)
constexpr int kFQ = 64;                        // per-warp queue of deferred pairs for the global list

// One pair in a worker's batch pipeline: the head of SL(j), then the gathered bytes.
struct alignas(16) FSlot {
  uint4 slh[4];        // ids m[0..7], weights w[0..7]
  uint32_t dw[8];      // the 4-byte words of the mirror row holding D[i][m_q]
  int32_t rw[8];       // the pivot row at m_q
  int i, j, lb, cw;    // the pair, D_old[i][j], the row's pivot-column byte
};
struct FusedSmem {   // byte offsets into the dynamic shared memory
  int64_t ring, slots, dq, pcnt, dcnt, bars, total;
};
__host__ __device__ inline FusedSmem fused_layout(int S, int64_t RB) {
  FusedSmem L;
  int64_t o = 0;
  L.ring = o; o += S * RB;
  L.slots = o; o += (int64_t)3 * kFW * kB * sizeof(FSlot);   // batches k, k - 1, k - 2
  L.dq = o; o += kFW * kFQ * 16;
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
  int* srow; int* scol; int* sacc; int* slb; int64_t lcap;   // the deferred pairs (all pairs if export_only)
  DetectCounters* ctr;
  int64_t slab, RB;
  int export_only;                      // 1: every pair on the global list, no certification
};

__device__ __forceinline__ uint32_t sat8u(int32_t v) { return (uint32_t)min(v, kSat8i); }
// 4-byte asynchronous copy global -> shared (cp.async.ca, LDGSTS.32)
__device__ __forceinline__ void cp_async4(void* dst, const void* src) {
  asm volatile("cp.async.ca.shared.global [%0], [%1], 4;" ::"r"(smem_u32(dst)), "l"(src) : "memory");
}

template <int S>
__global__ void __launch_bounds__(kFThreads, 1) k_detect_fix_p8(FusedArgs a) {
  extern __shared__ __align__(128) uint8_t sm[];
  const FusedSmem L = fused_layout(S, a.RB);
  uint8_t* ring = sm + L.ring;
  FSlot* slots = reinterpret_cast<FSlot*>(sm + L.slots);
  int4* dq = reinterpret_cast<int4*>(sm + L.dq) + (threadIdx.x >> 5) * kFQ;   // this warp's queue
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
  const int32_t I = APSP_INF_I32_DEV;
  // this lane's 16 bytes of the pivot row (saturated) in each of the warp's segments
  uint32_t rreg[kFSeg][4];
#pragma unroll
  for (int t = 0; t < kFSeg; ++t) {
    const int64_t c0 = (int64_t)(warp + t * kFW) * 512 + 16 * lane;
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      uint32_t w = 0;
#pragma unroll
      for (int e = 0; e < 4; ++e) {
        const int64_t c = c0 + 4 * q + e;
        w |= (c < n ? sat8u(a.r1[c]) : (uint32_t)kSat8i) << (8 * e);
      }
      rreg[t][q] = w;
    }
  }
  // deferred pairs go through a per-warp shared-memory queue, flushed 32+ at
  // a time (one atomic on the list cursor per flush)
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
        const int4 v = dq[e];
        a.srow[q] = v.x;
        a.scol[q] = v.y;
        a.sacc[q] = v.z;
        a.slb[q] = v.w;
      } else {
        atomicOr(&a.ctr->overflow, 1u);
      }
    }
    __syncwarp();
    qn = 0;
  };
  auto defer = [&](bool want, int4 v) {   // warp-collective: queue v for want lanes
    const unsigned bal = __ballot_sync(0xffffffffu, want);
    if (!bal) return;
    if (qn + 32 > kFQ) flush();
    if (want) dq[qn + __popc(bal & ((1u << lane) - 1))] = v;
    qn += __popc(bal);
    if (qn >= 32) flush();
  };
  // ---- batch pipeline (kB pairs per batch, three batches in the ring)
  auto bslot = [&](int bk, int e) -> FSlot& { return slots[((bk % 3) * kFW + warp) * kB + e]; };
  int bk = 0;                 // the batch being filled
  int bfill = 0;              // pairs in it (warp-uniform)
  int bn1 = 0, bn2 = 0;       // pairs in batches bk - 1, bk - 2
  auto advance = [&]() {      // close batch bk; gather for bk - 1; certify bk - 2
    cp_async_commit();        // G1(bk): the heads of batch bk
    cp_async_wait<1>();       // every group but G1(bk) is complete
    __syncwarp();
    if (lane < bn1) {         // batch bk - 1: heads landed -> gathers
      FSlot& sl = bslot(bk + 2, lane);   // (bk - 1) mod 3
      const uint8_t* mrow = a.M8 + ((int64_t)sl.i - row0) * ld;
      const uint4 m0 = sl.slh[0], m1 = sl.slh[1];
      const int m[8] = {(int)m0.x, (int)m0.y, (int)m0.z, (int)m0.w, (int)m1.x, (int)m1.y, (int)m1.z, (int)m1.w};
#pragma unroll
      for (int q = 0; q < 8; ++q) {
        const int mq = m[q] >= 0 ? m[q] : 0;
        cp_async4(&sl.dw[q], mrow + (mq & ~3));
        cp_async4(&sl.rw[q], a.r1 + mq);
      }
    }
    cp_async_commit();        // G2(bk - 1)
    bool want = false;        // batch bk - 2 (its gathers completed at the wait above): certify
    int4 v = make_int4(0, 0, 0, 0);
    if (lane < bn2) {
      const FSlot& sl = bslot(bk + 1, lane);   // (bk - 2) mod 3
      // c[i] saturated at 0x7F: exact for the stale test (ci + r == d with
      // d <= 0x7E needs ci < 0x7F; a saturated ci never tests stale, nor does
      // the true one)
      const int32_t ci = sl.cw;
      const uint4 m0 = sl.slh[0], m1 = sl.slh[1], w0 = sl.slh[2], w1 = sl.slh[3];
      const int m[8] = {(int)m0.x, (int)m0.y, (int)m0.z, (int)m0.w, (int)m1.x, (int)m1.y, (int)m1.z, (int)m1.w};
      const int w[8] = {(int)w0.x, (int)w0.y, (int)w0.z, (int)w0.w, (int)w1.x, (int)w1.y, (int)w1.z, (int)w1.w};
      int32_t acc = I;
#pragma unroll
      for (int q = 0; q < 8; ++q) {
        if (m[q] < 0) continue;
        const int32_t d8 = (int32_t)((sl.dw[q] >> (8 * (m[q] & 3))) & 0xFFu);
        if (d8 == kSat8i) continue;                          // INF: no candidate
        if (sl.rw[q] < I && ci + sl.rw[q] == d8) continue;   // stale: m is listed itself
        acc = min(acc, min(d8 + w[q], I));
      }
      // certified iff the bound reaches lb (then it equals D_old: nothing to
      // write); otherwise deferred with its bound
      want = acc > sl.lb;
      v = make_int4(sl.i, sl.j, acc, sl.lb);
    }
    defer(want, v);
    bn2 = bn1;
    bn1 = bfill;
    bfill = 0;
    ++bk;
  };
  auto cgroup = [&](int r0) -> uint32_t {
    const int64_t il = i_lo + r0 + lane;
    return (r0 + lane < rows && il != skip) ? sat8u(a.c1[il]) * 0x01010101u : 0x7F7F7F7Fu;
  };
  uint32_t cl = 0, cl_next = cgroup(0);
  unsigned long long my_pairs = 0;
  for (int rr = 0; rr < rows; ++rr) {
    const int s = rr % S;
    const int64_t i = i_lo + rr;
    if ((rr & 31) == 0) {   // the pivot column for 32 rows, one per lane (INF on row k),
      cl = cl_next;         // loaded a group ahead
      cl_next = cgroup(rr + 32);
    }
    const uint32_t cw = __shfl_sync(0xffffffffu, cl, rr & 31);
    mbar_wait(full + s, (unsigned)(rr / S) & 1u);
    const uint8_t* row = ring + s * a.RB;
    int found = 0;
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
        uint4 dv = make_uint4(0, 0, 0, 0);
        if (accs[t] & 0x80808080u) {
          dv = *reinterpret_cast<const uint4*>(row + off);
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
        found += __reduce_add_sync(0xffffffffu, (unsigned)__popc(bits));
        if (a.export_only) {   // the list only: every pair to the global list
          while (__any_sync(0xffffffffu, bits != 0u)) {
            const bool have = bits != 0u;
            const int b = have ? __ffs(bits) - 1 : 0;
            if (have) bits &= bits - 1;
            defer(have, make_int4((int)i, (int)(off + b), I, 0));
          }
          continue;
        }
        // the flagged pairs into the batch (the head of SL(j) on its way)
        while (__any_sync(0xffffffffu, bits != 0u)) {
          const bool have = bits != 0u;
          const unsigned bal = __ballot_sync(0xffffffffu, have);
          const int k = bfill + __popc(bal & ((1u << lane) - 1));
          if (have && k < kB) {
            const int b = __ffs(bits) - 1;
            bits &= bits - 1;
            const int j = (int)(off + b);
            FSlot& sl = bslot(bk, k);
            const uint32_t dword = b < 4 ? dv.x : b < 8 ? dv.y : b < 12 ? dv.z : dv.w;
            sl.i = (int)i;
            sl.j = j;
            sl.lb = (int)((dword >> (8 * (b & 3))) & 0xFFu);   // D_old[i][j]
            sl.cw = (int)(cw & 0xFFu);
            cp_async16(&sl.slh[0], a.SLid + (int64_t)j * kSL);
            cp_async16(&sl.slh[1], a.SLid + (int64_t)j * kSL + 4);
            cp_async16(&sl.slh[2], a.SLw + (int64_t)j * kSL);
            cp_async16(&sl.slh[3], a.SLw + (int64_t)j * kSL + 4);
          }
          bfill = min(bfill + __popc(bal), kB);
          if (bfill == kB) advance();
        }
      }
    }
    // the row's bytes are no longer needed: release the stage
    __syncwarp();
    if (lane == 0) {
      if (found) atomicAdd(pcnt + s, found);
      __threadfence_block();
      if (atomicAdd(dcnt + s, 1) == kFW - 1) {   // the row's last warp: its |A_i|
        __threadfence_block();
        const int cnt = *(volatile int*)(pcnt + s);
        if (cnt > 0) a.rowcnt[i] = cnt;
        pcnt[s] = 0;
        dcnt[s] = 0;
      }
      mbar_arrive(empty + s);
    }
    my_pairs += (unsigned)found;
  }
  // drain the pipeline: the partial batch, then two empty ones
  if (!a.export_only) {
    advance();
    advance();
    advance();
  }
  cp_async_wait<0>();
  flush();
  if (lane == 0 && my_pairs) atomicAdd(&a.ctr->total, my_pairs);
}

// Deferred pairs (count ctr->spill): D[i][j] := acc (a walk length of G' or
// INF) mirrored, and the pair appended to its row's open list and the global
// one (lb = D_old[i][j]) — what k_sparse_phase_a does for a pair it leaves
// open.
__global__ void k_defer_apply(int32_t* D, int64_t ld, int64_t row0, const int* __restrict__ srow,
                              const int* __restrict__ scol, const int* __restrict__ sacc,
                              const int* __restrict__ slb, int64_t lcap, int* ocnt, int* ocol,
                              const int64_t* __restrict__ rowoff, int* gprow, int* gpcol, int32_t* glb,
                              unsigned char* gfull, int64_t ocap, DetectCounters* ctr, Mirror M) {
  const int64_t np = (ctr->overflow & 1u) ? 0 : min((int64_t)ctr->spill, lcap);
  unsigned mbits = 0;
  const int lane = threadIdx.x & 31;
  for (int64_t p0 = blockIdx.x * (int64_t)blockDim.x; p0 < np; p0 += (int64_t)gridDim.x * blockDim.x) {
    const int64_t p = p0 + threadIdx.x;
    const bool on = p < np;
    int i = 0, j = 0, acc = 0, lb = 0;
    if (on) {
      i = srow[p]; j = scol[p]; acc = sacc[p]; lb = slb[p];
      const int64_t idx = ((int64_t)i - row0) * ld + j;
      D[idx] = acc;
      mbits |= mput(M, idx, acc);
      const int s1 = atomicAdd(ocnt + i, 1);
      ocol[rowoff[i] + s1] = j;
    }
    const unsigned bal = __ballot_sync(0xffffffffu, on);
    unsigned long long g0 = 0;
    if (bal) {
      if (lane == __ffs(bal) - 1) g0 = atomicAdd(&ctr->open_total, (unsigned long long)__popc(bal));
      g0 = __shfl_sync(0xffffffffu, g0, __ffs(bal) - 1);
    }
    if (on) {
      const unsigned long long s2 = g0 + __popc(bal & ((1u << lane) - 1));
      if ((int64_t)s2 < ocap) {
        gprow[s2] = i;
        gpcol[s2] = j;
        glb[s2] = lb;
        gfull[s2] = 1;
      } else {
        atomicOr(&ctr->overflow, 2u);
      }
    }
  }
  mirror_post(M, mbits);
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
                          int* srow, int* scol, int* sacc, int* slb, int64_t lcap, DetectCounters* ctr,
                          int export_only, cudaStream_t st) {
  const int S = fused_stages(n);
  if (!S || !M.m8) return cudaErrorInvalidValue;
  const int64_t m = r.hi - r.lo;
  if (m <= 0) return cudaSuccess;
  FusedArgs a;
  a.D = D; a.ld = ld; a.r = r; a.n = n; a.skip = skip; a.c1 = c1; a.r1 = r1; a.SLid = SLid; a.SLw = SLw;
  a.M8 = M.m8; a.mflag = M.flag; a.rowcnt = rowcnt; a.srow = srow; a.scol = scol; a.sacc = sacc; a.slb = slb;
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

cudaError_t defer_apply(int32_t* D, int64_t ld, int64_t row0, const int* srow, const int* scol, const int* sacc,
                        const int* slb, int64_t lcap, int* ocnt, int* ocol, const int64_t* rowoff, int* gprow,
                        int* gpcol, int32_t* glb, unsigned char* gfull, int64_t ocap, DetectCounters* ctr, Mirror M,
                        cudaStream_t st) {
  k_defer_apply<<<num_sms() * 2, 256, 0, st>>>(D, ld, row0, srow, scol, sacc, slb, lcap, ocnt, ocol, rowoff, gprow,
                                               gpcol, glb, gfull, ocap, ctr, M);
  return cudaGetLastError();
}

}  // namespace apsp
