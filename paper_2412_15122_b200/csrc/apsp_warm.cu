// apsp_warm.cu — host orchestration behind the C ABI of include/apsp_warm.h.
//
// Every step of the hot path runs in the sm_100a kernels of fw.cu, stream.cu,
// sparse.cu and query.cu; this file validates arguments, takes the O(1) host
// decisions the paper's algorithms contain (early exits, the cost gate of
// P:196), carves the caller's workspace, and issues NCCL collectives when D
// is row-sharded over several GPUs.
#include <nccl.h>
#include <nvtx3/nvToolsExt.h>   // header-only NVTX: named ranges per API call (free without a tool attached)

#include <algorithm>
#include <cstdarg>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <map>
#include <string>
#include <type_traits>
#include <vector>

#include "../../include/apsp_warm.h"
#include "common.cuh"
#include "comm.h"
#include "kernels.h"

using namespace apsp;

namespace {

// one NVTX range per C-ABI call (profilers show the update types on the timeline)
struct NvtxRange {
  explicit NvtxRange(const char* name) { nvtxRangePushA(name); }
  ~NvtxRange() { nvtxRangePop(); }
};

constexpr int64_t kTile = 128;       // FW pivot block / row-partition granule
constexpr int kMaxSlabs = 256;       // add-node column partial slabs
constexpr int kAddColLimit = 2048;   // columns the add-node gathers may read per row (else the stream)
constexpr int64_t kAddShortcutMinN = 4096;   // the add-node shortcuts from this n on
constexpr int64_t kVecs = 9;         // scratch vectors of ld elements
constexpr int kQueryChunk = 32;      // sharded queries per column all-gather

int64_t round_up(int64_t a, int64_t b) { return (a + b - 1) / b * b; }
int64_t cdiv(int64_t a, int64_t b) { return (a + b - 1) / b; }


// ------------------------------------------------------------------ workspace plan
struct Plan {
  int64_t ld, lcap, ocap, maxchunk;
  size_t off_wt, off_vec, off_rowpart, off_colpart, off_rowoff, off_rowcnt, off_chg, off_prow,
      off_pcol, off_ocol, off_ocnt, off_gprow, off_gpcol, off_glb, off_gfull,
      off_srow, off_scol, off_slid, off_slw, off_wnext, off_slscr, off_panel, off_pt, off_anyrow, off_qsend, off_qcol,
      off_qids, off_qdsv, off_qlab, off_qpred, off_qpath, off_qdone, off_qcnt, off_p16, off_p8, off_mt, off_ptd,
      off_small, off_qbits, off_qbpred, off_qbout, off_qhit, off_heavy, off_bigq, off_qsort, total;
  size_t qsort_temp = 0;
  int64_t ldt;   // row stride of the transposed int8 mirror (bytes >= local rows)
  int qcap, qbatch;
  int64_t ldpt;
};

// ld: leading dimension of D, also used for WT and every scratch vector.
Plan make_plan(int64_t cap, int world, int64_t ld) {
  Plan p;
  p.ld = ld;
  p.maxchunk = cdiv(cdiv(p.ld, 4), 128);   // add-node pass-1 column chunks (512 columns)
  int64_t lc = cap * cap / 32;
  p.lcap = std::min<int64_t>(std::max<int64_t>(lc, 1 << 20), (int64_t)1 << 28);
  size_t o = 0;
  auto take = [&](size_t bytes) {
    size_t at = o;
    o = (size_t)round_up((int64_t)(o + bytes), 256);
    return at;
  };
  p.off_wt = take(sizeof(int32_t) * (size_t)cap * p.ld);
  p.off_vec = take(sizeof(int32_t) * (size_t)kVecs * p.ld);
  p.off_rowpart = take(sizeof(int32_t) * (size_t)p.maxchunk * p.ld * 2);   // min and max partials
  p.off_colpart = take(sizeof(int32_t) * (size_t)kMaxSlabs * p.ld);
  p.off_rowoff = take(sizeof(int64_t) * (size_t)cap);
  p.off_rowcnt = take(sizeof(int32_t) * (size_t)cap);
  p.off_chg = take(sizeof(int32_t) * (size_t)(cap + 32) * 4);   // 4 rounds' counts + frontier totals
  p.ocap = std::max<int64_t>(p.lcap / 4, 1 << 18);
  p.off_prow = take(sizeof(int32_t) * (size_t)p.lcap);
  p.off_pcol = take(sizeof(int32_t) * (size_t)p.lcap);
  p.off_ocol = take(sizeof(int32_t) * (size_t)p.lcap);
  p.off_ocnt = take(sizeof(int32_t) * (size_t)cap);
  p.off_gprow = take(sizeof(int32_t) * (size_t)p.ocap);
  p.off_gpcol = take(sizeof(int32_t) * (size_t)p.ocap);
  p.off_glb = take(sizeof(int32_t) * (size_t)p.ocap);
  p.off_gfull = take((size_t)p.ocap);
  p.off_srow = take(sizeof(int32_t) * (size_t)p.lcap);   // staging list of the detection pass
  p.off_scol = take(sizeof(int32_t) * (size_t)p.lcap);
  p.off_slid = take(sizeof(int32_t) * (size_t)cap * kSL);
  p.off_slw = take(sizeof(int32_t) * (size_t)cap * kSL);
  p.off_wnext = take(sizeof(int32_t) * (size_t)cap);
  p.off_slscr = take(kSLScratch);
  p.off_panel = take(world > 1 ? 2 * sizeof(int32_t) * (size_t)kTile * p.ld : 256);   // two receive buffers
  // transposed pivot column panel for the FW phase-3 kernel (kTile x ldpt)
  p.ldpt = round_up(world > 1 ? round_up(cdiv(cap, world), kTile) : cap, kTile);
  p.off_pt = take(sizeof(int32_t) * (size_t)kTile * p.ldpt);
  const int64_t rows_max = world > 1 ? round_up(cdiv(cap, world), kTile) : cap;
  p.off_anyrow = take(sizeof(int32_t) * (size_t)cap);
  // query scratch: qbatch slots of qcap candidates (|C| <= n <= cap)
  p.qcap = (int)std::min<int64_t>(kQueryCap, cap);
  // sharded queries (f3, gather-free): rows s of a chunk of queries (qsend),
  // this rank's hit lists and every rank's (qcol, all-gathered)
  p.off_qsend = take(world > 1 ? sizeof(int32_t) * (size_t)kQueryChunk * p.ld : 256);
  p.off_qhit = take(world > 1 ? sizeof(int32_t) * (size_t)kQueryChunk * (p.qcap + 1) : 256);
  p.off_qcol = take(world > 1 ? sizeof(int32_t) * (size_t)kQueryChunk * (p.qcap + 1) * world : 256);
  p.qbatch = world > 1 ? kQueryChunk : kQueryBatch;
  const size_t qe = (size_t)p.qcap * p.qbatch;
  p.off_qids = take(4 * qe);
  p.off_qdsv = take(4 * qe);
  p.off_qlab = take(4 * qe);
  p.off_qpred = take(4 * qe);
  p.off_qpath = take(4 * qe);
  p.off_qdone = take(qe);
  p.off_qcnt = take(sizeof(int32_t) * (size_t)p.qbatch);
  // t-grouped large batches (one GPU): keys, values (in, out) + cub temp
  p.qsort_temp = world > 1 ? 0 : query_group_temp_bytes();
  p.off_qsort = take(world > 1 ? 256 : 4 * sizeof(int32_t) * (size_t)kQueryGroup + p.qsort_temp);
  // a single query whose candidate set exceeds qcap (query_big): bitmap,
  // predecessors, [length, path] (one GPU)
  p.off_qbits = take(sizeof(uint32_t) * (size_t)(cap / 32 + 1));
  p.off_qbpred = take(sizeof(int32_t) * (size_t)cap);
  p.off_qbout = take(sizeof(int32_t) * (size_t)(cap + 4));
  // int16x2 FW (one GPU): packed copy of D (two columns per word) + the
  // transposed diagonal tile
  p.off_p16 = take(sizeof(uint16_t) * (size_t)rows_max * p.ld);
  p.off_p8 = take((size_t)rows_max * p.ld);   // the int8 mirror (int32 handles)
  p.ldt = round_up(rows_max, 128);
  p.off_mt = take((size_t)cap * p.ldt);       // its transpose (column j of D = row j)
  p.off_ptd = take(sizeof(uint32_t) * (size_t)kTile * kTile);
  // heavy rows of the sparse recompute (one GPU): the set, then kHeavy rows of X keys
  p.off_heavy = take(512 + sizeof(int32_t) * (size_t)kHeavy * p.ld);
  p.off_bigq = take(sizeof(int32_t) * (size_t)p.ocap);   // the rounds' long-frontier pair queue (one GPU)
  p.off_small = take(64 * 1024);
  p.total = o;
  return p;
}

void layout_rows(int64_t cap, int world, int rank, int64_t* row0, int64_t* rows) {
  int64_t R = world > 1 ? round_up(cdiv(cap, world), kTile) : cap;
  int64_t r0 = std::min<int64_t>((int64_t)rank * R, cap);
  *row0 = r0;
  *rows = std::max<int64_t>(0, std::min<int64_t>(R, cap - r0));
}

}  // namespace

// ------------------------------------------------------------------ handle
struct apsp_handle {
  apsp_dtype dt;
  int directed;
  int64_t n, cap, ld;
  void* D;
  int64_t row0, rows;            // local row block [row0, row0 + rows)
  int64_t R;                     // rows per rank (partition granule)
  unsigned char* ws;
  Plan plan;
  cudaStream_t st;
  cudaStream_t st2 = nullptr;    // side stream: shortlist upkeep overlapped with the D passes
  cudaEvent_t ev_fork = nullptr, ev_join = nullptr, ev_row = nullptr;
  cudaStream_t stc = nullptr;    // sharded FW: panel broadcasts (look-ahead), world > 1
  cudaEvent_t ev_pan = nullptr, ev_bc = nullptr;
  int rank, world;
  Comm* comm = nullptr;          // world > 1: NCCL or in-process group (comm.h)
  // options
  int force_path = 0;
  double theta = 0.02;
  float tau = 1e-5f;
  int max_rounds = 64;
  int rounds_hint = 2;           // rounds the last sparse recompute needed (its first batch)
  int fw16 = 1;                  // int16x2 FW when exact (int32 shortest path, one GPU)
  int last_fw16 = 0;             // 1: the last FW ran packed, 2: it fell back to int32
  bool mirror_built = false;     // the mirror was built (or invalidated) from D
  bool mirror_hint = false;      // last host read of the mirror flag said "valid" (gates the shortcuts / twins; see mirror_fresh)
  bool mirror_fresh = false;     // no kernel that can write a new value ran since that observation
  bool sl_join = false;          // shortlist upkeep pending on st2: join (ev_join) before reading them
  int mirror_level = 16;         // width of the mirror: 8 or 16 bits
  int mirror8 = 1;               // APSP_OPT_MIRROR8: try the int8 width at each build
  int use_mirror = 1;            // APSP_OPT_MIRROR: 0 = no mirror, the streams read D (4 B/entry)
  int heavy_min = 0;             // APSP_OPT_HEAVY: 0 = max(512, n/8), -1 = off
  int fused = 0;                 // APSP_OPT_FUSED: detection + phase A in one pass (fused.cu; off:
                                 // measured slower than the separate kernels)
  bool mirror8_failed = false;   // an int8 build found a distance >= 0x7F: int16 from then on
  // bytes per entry the O(n^2) streams read: 1 / 2 on a valid int8 / int16 mirror, else 4
  template <typename T> double stream_bytes() const {
    if (!(std::is_same<T, int32_t>::value && sr == 0 && mirror_hint)) return 4.0;
    return mirror_level == 8 ? 1.0 : 2.0;
  }
  double row_delta = 0.0;        // > 0: the paper's Definition-1 gate (ablation)
  int sr = 0;                    // path algebra: 0 shortest path, 1 minimax
  // state
  bool poisoned = false;
  std::string err;
  int64_t launches = 0;
  void* host_small = nullptr;    // pinned, mapped host scratch for small D2H reads
  void* host_small_dev = nullptr;   // its device address
  // profiling (apsp_profile_*)
  struct ProfRec { int cls; cudaEvent_t a, b; double work; };
  bool prof_on = false;
  // one GPU: captured FW pivot loops, keyed by (variant, n); a key is captured
  // the second time it runs (fw_graph)
  struct FwGraph { cudaGraphExec_t exec; int64_t launches; };
  std::map<uint64_t, FwGraph> fw_graphs;
  cudaStream_t stcap = nullptr;  // capture stream (the caller's may be the legacy default stream)
  std::vector<uint64_t> fw_seen;
  std::vector<ProfRec> prof_pending;
  std::vector<cudaEvent_t> ev_pool;
  double prof_ms[APSP_K_COUNT] = {};
  int64_t prof_cnt[APSP_K_COUNT] = {};
  double prof_work[APSP_K_COUNT] = {};
  cudaEvent_t ev() {
    if (ev_pool.empty()) {
      cudaEvent_t e;
      cudaEventCreate(&e);
      return e;
    }
    cudaEvent_t e = ev_pool.back();
    ev_pool.pop_back();
    return e;
  }
  cudaError_t prof_resolve() {
    if (prof_pending.empty()) return cudaSuccess;
    cudaError_t e = cudaStreamSynchronize(st);
    if (e != cudaSuccess) return e;
    for (auto& r : prof_pending) {
      float ms = 0.f;
      cudaEventElapsedTime(&ms, r.a, r.b);
      prof_ms[r.cls] += ms;
      prof_cnt[r.cls] += 1;
      prof_work[r.cls] += r.work;
      ev_pool.push_back(r.a);
      ev_pool.push_back(r.b);
    }
    prof_pending.clear();
    unsigned long long rb = 0;
    e = cudaMemcpy(&rb, rank1_bytes(), sizeof rb, cudaMemcpyDeviceToHost);
    if (e != cudaSuccess) return e;
    prof_work[APSP_K_RANK1] += (double)rb;
    e = cudaMemset(rank1_bytes(), 0, sizeof rb);
    if (e != cudaSuccess) return e;
    unsigned long long cb = 0;   // the add's column pass (k_addcol_mt)
    e = cudaMemcpy(&cb, add_scratch().work, sizeof cb, cudaMemcpyDeviceToHost);
    if (e != cudaSuccess) return e;
    prof_work[APSP_K_ADD_PASS1] += (double)cb;
    return cudaMemset(add_scratch().work, 0, sizeof cb);
  }

  template <typename T> T* WT() { return reinterpret_cast<T*>(ws + plan.off_wt); }
  template <typename T> T* vec(int idx) {
    return reinterpret_cast<T*>(ws + plan.off_vec) + (size_t)idx * plan.ld;
  }
  template <typename T> T* rowpart() { return reinterpret_cast<T*>(ws + plan.off_rowpart); }
  template <typename T> T* colpart() { return reinterpret_cast<T*>(ws + plan.off_colpart); }
  int64_t* rowoff() { return reinterpret_cast<int64_t*>(ws + plan.off_rowoff); }
  int* rowcnt() { return reinterpret_cast<int*>(ws + plan.off_rowcnt); }
  // round frontier counts per row; chg(k)[cap] = their total
  int* chg(int k) { return reinterpret_cast<int*>(ws + plan.off_chg) + (size_t)k * (cap + 32); }
  int* prow() { return reinterpret_cast<int*>(ws + plan.off_prow); }
  int* pcol() { return reinterpret_cast<int*>(ws + plan.off_pcol); }
  int* ocol() { return reinterpret_cast<int*>(ws + plan.off_ocol); }
  int* ocnt() { return reinterpret_cast<int*>(ws + plan.off_ocnt); }
  int* gprow() { return reinterpret_cast<int*>(ws + plan.off_gprow); }
  int* gpcol() { return reinterpret_cast<int*>(ws + plan.off_gpcol); }
  template <typename T> T* glb() { return reinterpret_cast<T*>(ws + plan.off_glb); }
  unsigned char* gfull() { return ws + plan.off_gfull; }
  int* srow() { return reinterpret_cast<int*>(ws + plan.off_srow); }
  int* scol() { return reinterpret_cast<int*>(ws + plan.off_scol); }
  int* slid() { return reinterpret_cast<int*>(ws + plan.off_slid); }
  template <typename T> T* slw() { return reinterpret_cast<T*>(ws + plan.off_slw); }
  template <typename T> T* wnext() { return reinterpret_cast<T*>(ws + plan.off_wnext); }
  void* slscr() { return ws + plan.off_slscr; }
  template <typename T> T* panel(int b = 0) {
    return reinterpret_cast<T*>(ws + plan.off_panel + (size_t)b * sizeof(int32_t) * kTile * plan.ld);
  }
  template <typename T> T* pt() { return reinterpret_cast<T*>(ws + plan.off_pt); }
  template <typename T> T* qsend() { return reinterpret_cast<T*>(ws + plan.off_qsend); }
  template <typename T> T* qcol() { return reinterpret_cast<T*>(ws + plan.off_qcol); }
  QueryScratch qscratch() {
    QueryScratch q;
    q.ids = reinterpret_cast<int*>(ws + plan.off_qids);
    q.dsv = ws + plan.off_qdsv;
    q.lab = ws + plan.off_qlab;
    q.pred = reinterpret_cast<int*>(ws + plan.off_qpred);
    q.path = reinterpret_cast<int*>(ws + plan.off_qpath);
    q.done = ws + plan.off_qdone;
    q.cnt = reinterpret_cast<int*>(ws + plan.off_qcnt);
    q.qcap = plan.qcap;
    q.batch = plan.qbatch;
    if (world == 1 && plan.qsort_temp > 0) {
      q.sort = reinterpret_cast<int*>(ws + plan.off_qsort);
      q.sort_temp = plan.qsort_temp;
    }
    return q;
  }
  int* anyrow() { return reinterpret_cast<int*>(ws + plan.off_anyrow); }
  DetectCounters* ctr() { return reinterpret_cast<DetectCounters*>(ws + plan.off_small); }
  int* anyflag() { return reinterpret_cast<int*>(ws + plan.off_small + 256); }
  unsigned long long* rank1_bytes() {   // device counter of bytes the rank-1 kernel read
    return reinterpret_cast<unsigned long long*>(ws + plan.off_small + 320);
  }
  unsigned* fw16_flag() { return reinterpret_cast<unsigned*>(ws + plan.off_small + 392); }
  unsigned* mirror_flag() { return reinterpret_cast<unsigned*>(ws + plan.off_small + 396); }
  unsigned* pass1_uncertain() { return reinterpret_cast<unsigned*>(ws + plan.off_small + 400); }
  unsigned* mirror_epoch_word() { return reinterpret_cast<unsigned*>(ws + plan.off_small + 472); }
  unsigned* validate_done() { return reinterpret_cast<unsigned*>(ws + plan.off_small + 476); }   // block counter
  int* coop_rounds_word() { return reinterpret_cast<int*>(ws + plan.off_small + 480); }
  int* coop_total_word() { return reinterpret_cast<int*>(ws + plan.off_small + 484); }
  int* heavy_set() { return reinterpret_cast<int*>(ws + plan.off_heavy); }
  // the pivot row snapshot r1 as saturated bytes (update_prep; phase A's stale test)
  uint8_t* r1_bytes() { return reinterpret_cast<uint8_t*>(vec<int32_t>(8)); }
  int* bigq() { return reinterpret_cast<int*>(ws + plan.off_bigq); }
  int* bigq_ctr() { return reinterpret_cast<int*>(ws + plan.off_small + 488); }   // 4 ints
  int* heavy_x() { return reinterpret_cast<int*>(ws + plan.off_heavy + 512); }
  alignas(64) unsigned char tmap8[128];   // CUtensorMap of the int8 mirror (detection's TMA)
  bool tmap8_ok = false;
  const void* tmap8_ptr() const { return tmap8_ok ? tmap8 : nullptr; }
  unsigned mirror_epoch = 0;     // per-launch epochs of the rank-1 gate (Mirror::epoch)
  // the add-node shortcuts' scratch words (small + 404 ... 463)
  AddScratch add_scratch() {
    unsigned char* b = ws + plan.off_small;
    return AddScratch{reinterpret_cast<unsigned long long*>(b + 448), reinterpret_cast<unsigned*>(b + 404),
                      reinterpret_cast<int*>(b + 408), reinterpret_cast<int*>(b + 412),
                      reinterpret_cast<int*>(b + 416), reinterpret_cast<int*>(b + 420),
                      reinterpret_cast<int*>(b + 424), reinterpret_cast<int*>(b + 428),
                      reinterpret_cast<unsigned*>(b + 432), reinterpret_cast<unsigned*>(b + 436),
                      reinterpret_cast<unsigned long long*>(b + 456)};
  }
  // saturated mirror of D (kernels.h), int32 handles only: int8 (own buffer)
  // or int16 (in the packed-FW buffer), the width picked at the last build
  template <typename T> Mirror mirror() {
    if constexpr (std::is_same<T, int32_t>::value) {
      if (!use_mirror) return Mirror{nullptr, nullptr, mirror_flag()};
      if (mirror_level == 8)
        return Mirror{nullptr, ws + plan.off_p8, mirror_flag(), mirror_epoch_word(), ++mirror_epoch,
                      ws + plan.off_mt, ld, plan.ldt};
      return Mirror{reinterpret_cast<uint16_t*>(p16()), nullptr, mirror_flag(), mirror_epoch_word(), ++mirror_epoch};
    } else {
      return Mirror{nullptr, nullptr, mirror_flag()};
    }
  }
  uint32_t* p16() { return reinterpret_cast<uint32_t*>(ws + plan.off_p16); }
  uint32_t* ptd() { return reinterpret_cast<uint32_t*>(ws + plan.off_ptd); }
  unsigned* wmin_dev() {   // accumulator of the smallest edge weight (bits of a T >= 0)
    return reinterpret_cast<unsigned*>(ws + plan.off_small + 384);
  }
  unsigned char* small() { return ws + plan.off_small + 512; }   // query scratch etc.
  // host copy: the smallest weight of any edge present since creation, as the
  // bits of a T >= 0 (~0u: none).  A lower bound of every distance between
  // distinct nodes (removals and increases only remove weights).
  unsigned wmin_bits = ~0u;
  template <typename T> T wmin() const {
    if (wmin_bits == ~0u) return T(0);
    if constexpr (std::is_same<T, float>::value) { float f; std::memcpy(&f, &wmin_bits, 4); return f; }
    else return (T)wmin_bits;
  }
  template <typename T> void fold_wmin(T w) {   // host code: no device traits here
    unsigned b;
    if constexpr (std::is_same<T, float>::value) {
      if (!(w >= 0.0f) || std::isinf(w)) return;
      std::memcpy(&b, &w, 4);
    } else {
      if (w < 0 || w >= APSP_INF_I32) return;
      b = (unsigned)w;
    }
    wmin_bits = std::min(wmin_bits, b);
  }
  template <typename T> T* Dl() { return reinterpret_cast<T*>(D); }
  template <typename T> T* Drow(int64_t gi) { return Dl<T>() + (gi - row0) * ld; }
  bool local(int64_t gi) const { return gi >= row0 && gi < row0 + rows; }
  int owner(int64_t gi) const { return world > 1 ? (int)(gi / R) : 0; }
  Rows active() const {
    Rows r;
    r.row0 = row0;
    r.lo = std::min(row0, n);
    r.hi = std::min(row0 + rows, n);
    if (r.hi < r.lo) r.hi = r.lo;
    return r;
  }
};

namespace {

apsp_status fail(apsp_handle* h, apsp_status s, const char* fmt, ...) {
  if (h) {
    char buf[512];
    va_list ap;
    va_start(ap, fmt);
    vsnprintf(buf, sizeof buf, fmt, ap);
    va_end(ap);
    h->err = buf;
    if (s == APSP_E_CUDA || s == APSP_E_NCCL) h->poisoned = true;
  }
  return s;
}

// Launch a kernel class `cls` with algorithmic work `wk`; with profiling on,
// bracket it with CUDA events on the handle's stream.
#define PK(cls, wk, expr)                                                                 \
  do {                                                                                    \
    cudaEvent_t _a = nullptr;                                                             \
    if (h->prof_on) {                                                                     \
      _a = h->ev();                                                                       \
      cudaEventRecord(_a, h->st);                                                         \
    }                                                                                     \
    cudaError_t _e = (expr);                                                              \
    ++h->launches;                                                                        \
    if (_e != cudaSuccess)                                                                \
      return fail(h, APSP_E_CUDA, "%s failed: %s", #expr, cudaGetErrorString(_e));       \
    if (h->prof_on) {                                                                     \
      cudaEvent_t _b = h->ev();                                                           \
      cudaEventRecord(_b, h->st);                                                         \
      h->prof_pending.push_back({(int)(cls), _a, _b, (double)(wk)});                      \
    }                                                                                     \
  } while (0)
#define CK(expr) PK(APSP_K_OTHER, 0, expr)
// a launch on the side stream (not bracketed by the profiling events)
#define CK2(expr)                                                                         \
  do {                                                                                    \
    cudaError_t _e = (expr);                                                              \
    ++h->launches;                                                                        \
    if (_e != cudaSuccess)                                                                \
      return fail(h, APSP_E_CUDA, "%s failed: %s", #expr, cudaGetErrorString(_e));       \
  } while (0)
#define CKR(expr)                                                                         \
  do {                                                                                    \
    cudaError_t _e = (expr);                                                              \
    if (_e != cudaSuccess)                                                                \
      return fail(h, APSP_E_CUDA, "%s failed: %s", #expr, cudaGetErrorString(_e));       \
  } while (0)
#define NK(expr)                                                                          \
  do {                                                                                    \
    int _r = (expr);                                                                      \
    if (_r != 0)                                                                          \
      return fail(h, APSP_E_NCCL, "%s failed: %s", #expr, h->comm->errstr(_r));          \
  } while (0)
#define CHECK_HANDLE(h)                                                                   \
  do {                                                                                    \
    if (!(h)) return APSP_E_INVAL;                                                        \
    if ((h)->poisoned) return APSP_E_POISONED;                                            \
  } while (0)

template <typename T> ncclDataType_t nccl_type();
template <> ncclDataType_t nccl_type<int32_t>() { return ncclInt32; }
template <> ncclDataType_t nccl_type<float>() { return ncclFloat32; }

// broadcast a length-`count` vector from the rank owning global row `gi`
template <typename T>
apsp_status bcast_from_owner(apsp_handle* h, T* buf, int64_t count, int64_t gi) {
  if (h->world <= 1) return APSP_OK;
  NK(h->comm->bcast(buf, (size_t)count, nccl_type<T>(), h->owner(gi), h->st));
  return APSP_OK;
}

// snapshot row gi of D (+ add) into out (padded to ld with INF), all ranks
// Pivot snapshots: c[i] = D[i][col] + add over the local rows and r = row `ri`
// of D (every rank) — one launch on one GPU, gather + broadcast otherwise.
template <typename T>
apsp_status snap_row(apsp_handle* h, int64_t gi, T add, T* out);
template <typename T>
apsp_status snap_pivots(apsp_handle* h, int64_t col, T add, T* c, int64_t ri, T* rout) {
  if (h->world == 1) {
    CK(gather_col_row<T>(h->Dl<T>(), h->ld, h->active(), col, add, c, h->Drow<T>(ri), h->n, h->ld, rout,
                         h->sr, h->st));
    return APSP_OK;
  }
  CK(gather_col<T>(h->Dl<T>(), h->ld, h->active(), col, add, c, h->sr, h->st));
  return snap_row<T>(h, ri, T(0), rout);
}

template <typename T>
apsp_status snap_row(apsp_handle* h, int64_t gi, T add, T* out) {
  if (h->local(gi)) CK(copy_vec<T>(h->Drow<T>(gi), h->n, h->ld, add, out, h->st));
  return bcast_from_owner<T>(h, out, h->ld, gi);
}

// ------------------------------------------------------------------ cold FW
// Blocked FW over the current D (the dense fallback a7 runs it on D0).
template <typename T>
apsp_status fw_impl_elem(apsp_handle* h);

// (Re)build the mirror of D: at the first update of a handle whose D
// the caller filled (warm start), and after an int32 FW.  Mirror flag bit 0
// set iff some finite local distance is >= the saturation value, bit 1 iff some local entry
// is INF (stream.cu: kMirrorOff, kMirrorInf).
// The int8 width is tried first (unless an earlier int8 build failed): if some
// finite distance is >= 0x7F the build is redone at int16 (one host read of
// the flag; builds are rare — warm start, after an int32 FW).
bool try_mirror8(const apsp_handle* h) { return h->mirror8 && !h->mirror8_failed && h->sr == 0; }

// read the mirror flag; if the int8 build came out invalid, fall back to int16
// for the rest of the handle's life (returns true if the caller must build it)
apsp_status mirror8_settle(apsp_handle* h, bool* need16) {
  unsigned* hf = reinterpret_cast<unsigned*>(h->host_small);
  CKR(cudaMemcpyAsync(hf, h->mirror_flag(), sizeof(unsigned), cudaMemcpyDeviceToHost, h->st));
  CKR(cudaStreamSynchronize(h->st));
  *need16 = (*hf & 1u) != 0u;
  h->mirror_fresh = true;
  if (*need16) {
    h->mirror8_failed = true;
    h->mirror_level = 16;
  }
  return APSP_OK;
}

template <typename T>
apsp_status mirror_rebuild(apsp_handle* h) {
  if constexpr (std::is_same<T, int32_t>::value) {
    if (!h->use_mirror) {   // APSP_OPT_MIRROR = 0: the streams read D itself
      CKR(cudaMemsetAsync(h->mirror_flag(), 0xff, sizeof(unsigned), h->st));
      h->mirror_hint = false;
      h->mirror_built = true;
      return APSP_OK;
    }
    bool need16 = true;
    if (try_mirror8(h)) {
      h->mirror_level = 8;
      CKR(cudaMemsetAsync(h->mirror_flag(), 0, sizeof(unsigned), h->st));
      CK(mirror_build(h->Dl<int32_t>(), h->ld, h->active(), h->n, h->mirror<int32_t>(), h->st));
      apsp_status s = mirror8_settle(h, &need16);
      if (s != APSP_OK) return s;
    }
    if (need16) {
      h->mirror_level = 16;
      CKR(cudaMemsetAsync(h->mirror_flag(), 0, sizeof(unsigned), h->st));
      // per rank: each rank's readers stream only its own rows
      CK(mirror_build(h->Dl<int32_t>(), h->ld, h->active(), h->n, h->mirror<int32_t>(), h->st));
    }
    h->mirror_hint = true;   // corrected at the next host read of the flag
  }
  h->mirror_built = true;
  return APSP_OK;
}
// Build the mirror if it was never built — or if it is the int8 one and the
// host has seen it invalidated (a distance reached 0x7F): rebuilt once, it is
// the int16 one from then on (an invalid int16 mirror stays invalid until a
// FW or apsp_sync_distances rebuilds it: its distances are >= 0x3FFF).
template <typename T>
apsp_status ensure_mirror(apsp_handle* h) {
  const bool stale8 = h->mirror_built && h->mirror_level == 8 && !h->mirror_hint;
  return (h->mirror_built && !stale8) ? APSP_OK : mirror_rebuild<T>(h);
}

// One GPU: the pivot loop of a blocked FW is a fixed launch sequence for a
// given (variant, n) over the handle's fixed buffers — captured into a CUDA
// graph the second time it runs and replayed after that (one launch instead
// of ~4 per pivot block).  Not under the per-kernel profile (its events would
// be captured too) and never when sharded (the loop holds collectives).
constexpr size_t kFwGraphs = 8;
template <typename Body>
apsp_status fw_graph(apsp_handle* h, uint64_t key, Body body) {
  if (h->prof_on || h->world > 1) return body();
  auto it = h->fw_graphs.find(key);
  if (it == h->fw_graphs.end()) {
    if (std::find(h->fw_seen.begin(), h->fw_seen.end(), key) == h->fw_seen.end()) {
      if (h->fw_seen.size() >= 64) h->fw_seen.erase(h->fw_seen.begin());
      h->fw_seen.push_back(key);
      return body();   // first run of this key: plain launches
    }
    if (h->fw_graphs.size() >= kFwGraphs) {   // bounded cache: drop one
      cudaGraphExecDestroy(h->fw_graphs.begin()->second.exec);
      h->fw_graphs.erase(h->fw_graphs.begin());
    }
    const int64_t l0 = h->launches;
    // captured on a stream of its own (capturing the legacy default stream is
    // not allowed): the body enqueues on h->st, swapped for the capture; the
    // graph is then launched on the caller's stream
    if (!h->stcap) CKR(cudaStreamCreateWithFlags(&h->stcap, cudaStreamNonBlocking));
    cudaStream_t user = h->st;
    h->st = h->stcap;
    cudaError_t eb = cudaStreamBeginCapture(h->st, cudaStreamCaptureModeRelaxed);
    const apsp_status s = eb == cudaSuccess ? body() : APSP_OK;
    cudaGraph_t g = nullptr;
    const cudaError_t e = eb == cudaSuccess ? cudaStreamEndCapture(h->st, &g) : eb;
    h->st = user;
    if (s != APSP_OK) {
      if (g) cudaGraphDestroy(g);
      return s;
    }
    CKR(e);
    cudaGraphExec_t ex = nullptr;
    const cudaError_t e2 = cudaGraphInstantiate(&ex, g, 0);
    cudaGraphDestroy(g);
    CKR(e2);
    it = h->fw_graphs.emplace(key, apsp_handle::FwGraph{ex, h->launches - l0}).first;
    h->launches = l0;   // counted when replayed
  }
  CKR(cudaGraphLaunch(it->second.exec, h->st));
  h->launches += it->second.launches;
  return APSP_OK;
}

// Sharded blocked FW (world > 1) with look-ahead: the owner of pivot block
// K+1 first relaxes that block's rows through pivot K, closes it (diagonal +
// row panel) and broadcasts it on the comm stream, while the rest of pivot
// K's phase 3 runs on the compute stream; receivers alternate between two
// panel buffers.  close(K0, kb) -> the owner's panel (on h->st);
// phase3(K0, kb, P, lo, hi, skip_ti) relaxes local rows [lo, hi) through
// pivot block K0 with panel P (skipping row tile skip_ti of that range);
// recv(b) = receive buffer b; words = panel elements per row.
template <typename E, typename Close, typename Phase3, typename Recv>
apsp_status fw_sharded(apsp_handle* h, int64_t n, int64_t m, size_t words, ncclDataType_t dt, Close close,
                       Phase3 phase3, Recv recv) {
  const int64_t T = kTile;
  auto bcast = [&](E* P, int64_t K0, int kb) -> apsp_status {
    CKR(cudaEventRecord(h->ev_pan, h->st));   // panel closed / receive buffer free
    CKR(cudaStreamWaitEvent(h->stc, h->ev_pan, 0));
    NK(h->comm->bcast(P, (size_t)kb * words, dt, h->owner(K0), h->stc));
    CKR(cudaEventRecord(h->ev_bc, h->stc));
    return APSP_OK;
  };
  E* P = nullptr;
  {
    const int kb0 = (int)std::min<int64_t>(T, n);
    if (h->local(0)) {
      apsp_status s = close(int64_t(0), kb0, &P);
      if (s != APSP_OK) return s;
    } else {
      P = recv(0);
    }
    apsp_status s = bcast(P, 0, kb0);
    if (s != APSP_OK) return s;
  }
  for (int64_t K0 = 0, kbi = 0; K0 < n; K0 += T, ++kbi) {
    const int kb = (int)std::min<int64_t>(T, n - K0);
    const bool own = h->local(K0);
    const int skip_ti = own ? (int)((K0 - h->row0) / T) : -1;
    CKR(cudaStreamWaitEvent(h->st, h->ev_bc, 0));   // panel K in place everywhere
    E* P1 = nullptr;
    const int64_t K1 = K0 + T;
    apsp_status s = APSP_OK;
    if (K1 < n) {
      const int kb1 = (int)std::min<int64_t>(T, n - K1);
      const bool own1 = h->local(K1);
      const int64_t l1 = K1 - h->row0;
      if (own1) {   // look-ahead: block K+1's rows through pivot K, then close it
        s = phase3(K0, kb, P, l1, std::min<int64_t>(l1 + T, m), -1);
        if (s == APSP_OK) s = close(K1, kb1, &P1);
      } else {
        P1 = recv((int)((kbi + 1) & 1));
      }
      if (s == APSP_OK) s = bcast(P1, K1, kb1);
      if (s != APSP_OK) return s;
      if (own1) {   // the rest of pivot K's phase 3, around block K+1
        s = phase3(K0, kb, P, 0, l1, skip_ti);
        if (s == APSP_OK) s = phase3(K0, kb, P, std::min<int64_t>(l1 + T, m), m, -1);
      } else {
        s = phase3(K0, kb, P, 0, m, skip_ti);
      }
    } else {
      s = phase3(K0, kb, P, 0, m, skip_ti);
    }
    if (s != APSP_OK) return s;
    P = P1;
  }
  return APSP_OK;
}

// int16x2 blocked FW (fw.cu) over the packed copy of this rank's rows, with the
// same pivot schedule and panel broadcast as fw_impl_elem.  Sets *saturated
// (summed over ranks) when some entry reached 0x3FFF: D then holds the exact
// entries below it and walk lengths elsewhere.
apsp_status fw16_impl(apsp_handle* h, int64_t skip, bool* saturated) {
  const int64_t n = h->n, ld = h->ld;
  Rows r = h->active();
  const int64_t m = r.hi - r.lo;
  uint32_t* P = h->p16();
  uint32_t* PT = h->pt<uint32_t>();
  CK(p16_from_d32(h->Dl<int32_t>(), ld, m, n, P, h->st));
  if (h->world > 1) {
    const int64_t lw = ld / 2;   // words per packed row
    auto close = [&](int64_t K0, int kb, uint32_t** out) -> apsp_status {
      uint32_t* rowK = P + (K0 - h->row0) * lw;
      PK(APSP_K_FW_DIAG, (double)kb * kb * kb, p16_diag(rowK + K0 / 2, ld, kb, h->st));
      CK(p16_transpose_rep(rowK, ld, kb, K0, kb, h->ptd(), kTile, h->st));
      PK(APSP_K_FW_PANEL, (double)kb * kb * (n - kb), p16_tile3(rowK, ld, h->ptd(), kTile, rowK, kb, n, kb, -1, h->st));
      *out = rowK;
      return APSP_OK;
    };
    auto phase3 = [&](int64_t K0, int kb, uint32_t* panel, int64_t lo, int64_t hi, int skip_ti) -> apsp_status {
      if (hi <= lo) return APSP_OK;
      uint32_t* Pr = P + lo * lw;
      const int64_t rows = hi - lo;
      const double mo = (double)(rows - (skip_ti >= 0 ? kb : 0));
      CK(p16_transpose_rep(Pr, ld, rows, K0, kb, PT, h->plan.ldpt, h->st));   // old column panel
      PK(APSP_K_FW_PANEL, mo * kb * kb,
         p16_tile3(Pr + K0 / 2, ld, PT, h->plan.ldpt, panel + K0 / 2, rows, kb, kb, skip_ti, h->st));
      CK(p16_transpose_rep(Pr, ld, rows, K0, kb, PT, h->plan.ldpt, h->st));   // updated column panel
      PK(APSP_K_FW_TILE, mo * (double)(n - kb) * kb,
         p16_tile3(Pr, ld, PT, h->plan.ldpt, panel, rows, n, kb, skip_ti, h->st));
      return APSP_OK;
    };
    auto recv = [&](int b) { return h->panel<uint32_t>(b); };
    apsp_status s = fw_sharded<uint32_t>(h, n, m, (size_t)lw, ncclUint32, close, phase3, recv);
    if (s != APSP_OK) return s;
  }
  if (h->world == 1) {   // every row local: no panel exchange
    auto loop = [&]() -> apsp_status {
      for (int64_t K0 = 0; K0 < n; K0 += kTile) {
        const int kb = (int)std::min<int64_t>(kTile, n - K0);
        uint32_t* rowK = P + K0 * (ld / 2);
        PK(APSP_K_FW_DIAG, (double)kb * kb * kb, p16_diag(rowK + K0 / 2, ld, kb, h->st));
        CK(p16_transpose_rep(rowK, ld, kb, K0, kb, h->ptd(), kTile, h->st));
        PK(APSP_K_FW_PANEL, (double)kb * kb * (n - kb),
           p16_tile3(rowK, ld, h->ptd(), kTile, rowK, kb, n, kb, -1, h->st));
        const int skip_ti = (int)(K0 / kTile);
        const double mo = (double)(m - kb);
        CK(p16_transpose_rep(P, ld, m, K0, kb, PT, h->plan.ldpt, h->st));   // old column panel
        PK(APSP_K_FW_PANEL, mo * kb * kb,
           p16_tile3(P + K0 / 2, ld, PT, h->plan.ldpt, rowK + K0 / 2, m, kb, kb, skip_ti, h->st));
        CK(p16_transpose_rep(P, ld, m, K0, kb, PT, h->plan.ldpt, h->st));   // updated column panel
        PK(APSP_K_FW_TILE, mo * (double)(n - kb) * kb,
           p16_tile3(P, ld, PT, h->plan.ldpt, rowK, m, n, kb, skip_ti, h->st));
      }
      return APSP_OK;
    };
    apsp_status s = fw_graph(h, (uint64_t)n << 8 | 1u, loop);
    if (s != APSP_OK) return s;
  }
  CKR(cudaMemsetAsync(h->fw16_flag(), 0, sizeof(unsigned), h->st));
  CK(p16_to_d32(P, ld, m, n, h->row0, skip, h->Dl<int32_t>(), h->fw16_flag(), h->st));
  if (h->world > 1) NK(h->comm->allreduce(h->fw16_flag(), 1, ncclUint32, ncclMax, h->st));
  unsigned* hf = reinterpret_cast<unsigned*>(h->host_small);
  CKR(cudaMemcpyAsync(hf, h->fw16_flag(), sizeof(unsigned), cudaMemcpyDeviceToHost, h->st));
  CKR(cudaStreamSynchronize(h->st));
  *saturated = *hf != 0;
  return APSP_OK;
}

// Blocked FW: the int16x2 path first where it is exact, the element-type
// path otherwise (and whenever an entry saturated).
// `skip`: a tombstoned node (its row and column are INF and stay so), or -1.
template <typename T>
apsp_status fw_impl(apsp_handle* h, int64_t skip = -1) {
  if constexpr (std::is_same<T, int32_t>::value) {
    if (h->fw16 && h->sr == 0) {
      bool saturated = false;
      apsp_status s = fw16_impl(h, skip, &saturated);
      if (s != APSP_OK) return s;
      h->last_fw16 = saturated ? 2 : 1;
      if (!saturated && !h->use_mirror) return mirror_rebuild<T>(h);
      if (!saturated) {   // the packed buffer now holds sat16(D): the int16 mirror is valid
        bool need16 = true;
        if (try_mirror8(h)) {   // narrow it to int8 if every distance is < 0x7F
          h->mirror_level = 8;
          CKR(cudaMemsetAsync(h->mirror_flag(), 0, sizeof(unsigned), h->st));
          CK(mirror8_from_p16(h->p16(), h->ld, h->active().hi - h->active().lo, h->n, h->mirror<int32_t>(),
                              h->st));
          apsp_status s2 = mirror8_settle(h, &need16);
          if (s2 != APSP_OK) return s2;
        }
        if (need16) h->mirror_level = 16;
        CKR(cudaMemsetAsync(h->mirror_flag(), 0, sizeof(unsigned), h->st));
        h->mirror_built = true;
        h->mirror_hint = true;
        return APSP_OK;
      }
      // some distance is >= 0x3FFF or infinite: finish in int32 (exact from any
      // matrix of walk lengths, which D still is)
    }
  }
  apsp_status s = fw_impl_elem<T>(h);
  if (s != APSP_OK) return s;
  return mirror_rebuild<T>(h);   // the packed buffer was work space (or never mirrored D)
}

template <typename T>
apsp_status fw_impl_elem(apsp_handle* h) {
  const int64_t n = h->n, ld = h->ld;
  Rows r = h->active();
  const int64_t m = r.hi - r.lo;   // local active rows (local row 0 = global row0)
  T* D = h->Dl<T>();
  if (h->world > 1) {
    auto close = [&](int64_t K0, int kb, T** out) -> apsp_status {
      T* rowK = D + (K0 - h->row0) * ld;
      PK(APSP_K_FW_DIAG, (double)kb * kb * kb, fw_diag<T>(rowK + K0, ld, kb, h->sr, h->st));
      PK(APSP_K_FW_PANEL, (double)kb * kb * (n - kb), fw_row_panel<T>(rowK, ld, K0, kb, n, h->sr, h->st));
      *out = rowK;
      return APSP_OK;
    };
    auto phase3 = [&](int64_t K0, int kb, T* P, int64_t lo, int64_t hi, int skip_ti) -> apsp_status {
      if (hi <= lo) return APSP_OK;
      T* Dr = D + lo * ld;
      const int64_t rows = hi - lo;
      const double mo = (double)(rows - (skip_ti >= 0 ? kb : 0));
      PK(APSP_K_FW_PANEL, mo * kb * kb, fw_col_panel<T>(Dr, ld, rows, K0, kb, P + K0, ld, skip_ti, h->sr, h->st));
      PK(APSP_K_FW_TILE, mo * (double)(n - kb) * kb,
         fw_rest_pt<T>(Dr, ld, rows, n, K0, kb, P, ld, skip_ti, h->pt<T>(), h->plan.ldpt, h->sr, h->st));
      return APSP_OK;
    };
    auto recv = [&](int b) { return h->panel<T>(b); };
    return fw_sharded<T>(h, n, m, (size_t)ld, nccl_type<T>(), close, phase3, recv);
  }
  auto loop = [&]() -> apsp_status {   // one GPU: every row local
    for (int64_t K0 = 0; K0 < n; K0 += kTile) {
      const int kb = (int)std::min<int64_t>(kTile, n - K0);
      T* rowK = D + K0 * ld;
      PK(APSP_K_FW_DIAG, (double)kb * kb * kb, fw_diag<T>(rowK + K0, ld, kb, h->sr, h->st));
      PK(APSP_K_FW_PANEL, (double)kb * kb * (n - kb), fw_row_panel<T>(rowK, ld, K0, kb, n, h->sr, h->st));
      const int skip_ti = (int)(K0 / kTile);
      const double mo = (double)(m - kb);   // rows outside the pivot block
      PK(APSP_K_FW_PANEL, mo * kb * kb, fw_col_panel<T>(D, ld, m, K0, kb, rowK + K0, ld, skip_ti, h->sr, h->st));
      PK(APSP_K_FW_TILE, mo * (double)(n - kb) * kb,
         fw_rest_pt<T>(D, ld, m, n, K0, kb, rowK, ld, skip_ti, h->pt<T>(), h->plan.ldpt, h->sr, h->st));
    }
    return APSP_OK;
  };
  return fw_graph(h, (uint64_t)n << 8 | (std::is_same<T, float>::value ? 2u : 4u) | (uint64_t)h->sr << 3, loop);
}

// Cold start (a1): D := W, then blocked FW.
template <typename T>
apsp_status cold_fw_impl(apsp_handle* h) {
  CK(init_d<T>(h->Dl<T>(), h->ld, h->active(), h->n, h->WT<T>(), h->ld, h->st));
  return fw_impl<T>(h);
}

// ------------------------------------------------------------------ detect + recompute
// Shared by remove_node (skip = k, tombstone) and edge increases (skip = -1).
// c1/r1 (and c2/r2 when undirected increase) must be set up by the caller.
// The int8 mirror is valid as of this update's host read of its flag (valid
// only where no kernel that writes D/the mirror ran since that read).
// (the last observation only, possibly stale: for speculative work that is
// re-checked after the next host read)
inline bool mirror8_hint(const apsp_handle* h) {
  return h->mirror_built && h->mirror_level == 8 && h->mirror_hint && h->sr == 0;
}
inline bool mirror8_known_valid(const apsp_handle* h) {
  return h->mirror_built && h->mirror_level == 8 && h->mirror_hint && h->mirror_fresh && h->sr == 0;
}

// Removal of node k: SL upkeep (drop k's entries, node n-1 takes slot k) on
// the side stream; the next shortlist reader or writer on the compute stream
// joins it (join_side / recompute's sl_join).
template <typename T>
apsp_status fork_shortlist_remove(apsp_handle* h, int64_t k) {
  CKR(cudaEventRecord(h->ev_fork, h->st));
  CKR(cudaStreamWaitEvent(h->st2, h->ev_fork, 0));
  CK2(shortlist_remove<T>(h->slid(), h->slw<T>(), h->wnext<T>(), h->n, k, h->n - 1, h->st2));
  CKR(cudaEventRecord(h->ev_join, h->st2));
  return APSP_OK;
}

// The compute stream waits for pending shortlist upkeep on the side stream
// (a removal's, an increase's) before it touches the shortlists itself.
apsp_status join_side(apsp_handle* h) {
  if (h->sl_join) {
    CKR(cudaStreamWaitEvent(h->st, h->ev_join, 0));
    h->sl_join = false;
  }
  return APSP_OK;
}

// The fused detection + phase A kernel (fused.cu) applies: int32 shortest
// path, the int8 mirror known valid, one pivot term (removal or a directed
// increase), and a row of the mirror fits in shared memory.
template <typename T>
bool use_fused(const apsp_handle* h, bool two) {
  return std::is_same<T, int32_t>::value && !two && mirror8_known_valid(h) && h->fused && fused_stages(h->n) > 0;
}

// Every per-update counter of the recompute: per-row counts, the counters,
// the open-list cursors, the first four rounds' frontier counts, the flag.
ZeroSet recompute_zero_set(apsp_handle* h) {
  ZeroSet z{};
  z.add(h->rowcnt(), h->cap);
  z.add(reinterpret_cast<int*>(h->ctr()), (int64_t)(sizeof(DetectCounters) / sizeof(int)));
  z.add(h->ocnt(), h->cap);
  for (int q = 0; q < 4; ++q) z.add(h->chg(q), h->cap + 1);
  z.add(h->anyflag(), 1);
  z.add(h->anyrow(), h->cap);   // the rounds' per-row open minima (keys)
  z.add(h->heavy_set(), 2 + 2 * kHeavy);   // heavy rows: count, ids, bounds, pruned-list length
  z.add(h->bigq_ctr(), 4);      // the rounds' queue counters
  return z;
}

// One GPU: A2, B and the open rows' minima inside the cooperative rounds
// launch (1) or as their own launches before it (0: measured faster — the
// cooperative grid, 2 CTAs per SM, has an eighth of the warps A2's
// one-warp-per-pair gathers get from a full launch: 90 vs 58 us per BJ.c4 removal)
#ifndef COOP_TAIL
#define COOP_TAIL 0
#endif
constexpr bool kCoopTail = COOP_TAIL != 0;

// Phase A's algorithmic bytes per listed pair: the list entry (8), the first
// two shortlist entries of column j (ids + weights, 16), their D entries on
// the int8 mirror (2) and pivot values (8)
constexpr double kPhaseABytes = 34.0;

// prepped: the counters were zeroed — and for a removal WT tombstoned — by the
// update's first launch (update_prep, one GPU)
template <typename T>
apsp_status recompute(apsp_handle* h, int64_t skip, const T* c1, const T* r1, const T* c2,
                      const T* r2, bool removal, apsp_update_info* info, bool prepped = false,
                      const uint8_t* r1b = nullptr /* r1 as saturated bytes, written by update_prep */) {
  const int64_t n = h->n;
  Rows r = h->active();
  const int64_t lcap = h->plan.lcap, ocap = h->plan.ocap;
  if (!prepped) CK(zero_set(recompute_zero_set(h), h->st));
  // ---- sparse recompute (a6), enqueued without a host round trip: the pair
  // counts stay on the device, and the kernels do nothing if a list
  // overflowed.  Every value they write is a walk length of G' (>= the new
  // distance), so if the gate below picks the dense path after all, FW on
  // the result is still exact.
  const bool try_sparse = h->force_path != 2;
  const bool fused = use_fused<T>(h, c2 != nullptr) && try_sparse;
  auto sl_join = [&]() -> apsp_status {   // the side stream's shortlist upkeep (update_edge)
    if (h->sl_join) {
      CKR(cudaStreamWaitEvent(h->st, h->ev_join, 0));
      h->sl_join = false;
    }
    return APSP_OK;
  };
  if (fused) {
    { apsp_status sj = sl_join(); if (sj != APSP_OK) return sj; }
    // detection + phase A in one pass over the int8 mirror (fused.cu); the
    // pairs it could not buffer get the stand-alone phase A below
    PK(APSP_K_DETECT, (double)(r.hi - r.lo) * (double)n,
       detect_fix_p8(reinterpret_cast<int32_t*>(h->Dl<T>()), h->ld, r, n, skip,
                     reinterpret_cast<const int32_t*>(c1), reinterpret_cast<const int32_t*>(r1), h->slid(),
                     reinterpret_cast<const int32_t*>(h->slw<T>()), h->mirror<T>(), h->rowcnt(), h->srow(),
                     h->scol(), h->prow(), h->pcol(), lcap, h->ctr(), 0, h->st));
    PK(APSP_K_EMIT, 0.0, detect_lists(r, h->rowcnt(), h->rowoff(), h->ctr(), h->st));
    if (removal && !prepped) CK(tombstone<T>(h->Dl<T>(), h->ld, r, n, skip, h->WT<T>(), h->ld, h->st));
    // the pairs it did not certify: their bounds into D, onto the open lists
    PK(APSP_K_SPARSE0, 0.0,
       defer_apply(reinterpret_cast<int32_t*>(h->Dl<T>()), h->ld, h->row0, h->srow(), h->scol(), h->prow(),
                   h->pcol(), lcap, h->ocnt(), h->ocol(), h->rowoff(), h->gprow(), h->gpcol(),
                   reinterpret_cast<int32_t*>(h->glb<T>()), h->gfull(), ocap, h->ctr(), h->mirror<T>(), h->st));
  } else {
    // one streaming pass appends the need_update_list; then the per-row slices
    // of the open lists and Phi / max|A_i|
    PK(APSP_K_DETECT, h->stream_bytes<T>() * (double)(r.hi - r.lo) * (double)n,
       detect<T>(h->Dl<T>(), h->ld, r, n, skip, c1, r1, c2, r2, h->tau, 1, nullptr, h->rowcnt(),
                 h->srow(), h->scol(), nullptr, lcap, h->ctr(), h->WT<T>(), h->ld, h->sr,
                 h->mirror<T>(), h->st, h->tmap8_ptr(), !mirror8_known_valid(h)));
    PK(APSP_K_EMIT, 0.0, detect_lists(r, h->rowcnt(), h->rowoff(), h->ctr(), h->st));
    // (prepped: WT was tombstoned by update_prep; D's row and column of the
    // removed node are only read again by the dense path, which tombstones
    // them itself, or overwritten by the swap-with-last)
    if (removal && !prepped) CK(tombstone<T>(h->Dl<T>(), h->ld, r, n, skip, h->WT<T>(), h->ld, h->st));
  }
  // Rounds are frontier-based Bellman-Ford over each row's open entries: round
  // r relaxes every open pair of a row through the entries of that row that
  // changed in round r-1 (round 0: all open entries).  Frontier lists live in
  // the row slices of two spare pair-list buffers; counts (and, at [cap], the
  // round's total of changes) in chg(r % 4) — zeroed with the counters for
  // rounds 0-3, by a memset for later ones.  "Converged" = the last round of
  // a batch changed nothing: its total, read with the counters.
  int rounds = 0;
  int* fcol[2] = {h->prow(), h->pcol()};
  // one GPU: the rounds run in one cooperative kernel (sparse_rounds_coop);
  // sharded: batches of single-round launches with a flag all-reduce between
  const bool coop = h->world == 1;
  int* last_total = h->anyflag();   // no round enqueued: 0
  auto enqueue_rounds = [&](int batch) -> apsp_status {
    for (int b = 0; b < batch; ++b, ++rounds) {
      const int o = rounds & 3, oi = (rounds + 3) & 3;
      const int* fin_c = rounds == 0 ? h->ocnt() : h->chg(oi);
      const int* fin_l = rounds == 0 ? h->ocol() : fcol[(rounds & 1) ^ 1];
      if (rounds >= 4) CKR(cudaMemsetAsync(h->chg(o), 0, sizeof(int) * (h->cap + 1), h->st));
      PK(APSP_K_SPARSE_R, 0.0,
         sparse_round<T>(h->Dl<T>(), h->ld, h->row0, h->WT<T>(), h->ld, h->gprow(), h->gpcol(),
                         h->glb<T>(), ocap, h->rowoff(), fin_c, rounds == 0 ? nullptr : fin_c + h->cap,
                         fin_l, h->chg(o), h->chg(o) + h->cap, fcol[rounds & 1], h->anyflag(), h->sr, h->ctr(),
                         h->st, reinterpret_cast<unsigned*>(h->anyrow()), h->wmin<T>(), h->mirror<T>()));
      last_total = h->chg(o) + h->cap;
    }
    return APSP_OK;
  };
  if (try_sparse) {
    // A: every listed entry rewritten with a walk length of G' (stale entries
    // skipped by the detection predicate), certified where it reaches lb
    { apsp_status sj = sl_join(); if (sj != APSP_OK) return sj; }
    if (!fused)
    PK(APSP_K_SPARSE0, 0.0,
       sparse_phase_a<T>(h->Dl<T>(), h->ld, r, h->slid(), h->slw<T>(), h->rowoff(), h->srow(), h->scol(),
                         lcap, c1, r1, c2, r2, h->tau, h->ocnt(), h->ocol(), h->gprow(), h->gpcol(),
                         h->glb<T>(), h->gfull(), ocap, h->ctr(), h->sr, h->mirror<T>(), h->st, 0, r1b,
                         h->prow(), h->pcol()));   // (the rounds' frontier buffers: free until the rounds)
    if (!coop || !kCoopTail) {   // (kCoopTail: inside the cooperative launch instead)
      // A2: whole-shortlist pass over the open pairs, now that certified values are final
      PK(APSP_K_SPARSE_R, 0.0,
         sparse_short<T>(h->Dl<T>(), h->ld, h->row0, h->slid(), h->slw<T>(), h->wnext<T>(), h->gprow(),
                         h->gpcol(), h->glb<T>(), ocap, h->gfull(), 1, h->sr, h->ctr(), h->st, h->mirror<T>(),
                         removal ? skip : -1));
      // the removal's shortlist upkeep needs nothing after A2 (the last reader of
      // SL): it runs on the side stream, joined before the update returns
      if (removal) {
        apsp_status s2 = fork_shortlist_remove<T>(h, skip);
        if (s2 != APSP_OK) return s2;
      }
      // B: full O(n) scan for the pairs the shortlist could not settle
      PK(APSP_K_SPARSE_R, 0.0,
         sparse_full<T>(h->Dl<T>(), h->ld, h->row0, h->WT<T>(), h->ld, n, h->gprow(), h->gpcol(),
                        h->glb<T>(), h->gfull(), ocap, h->sr, h->ctr(), h->st, h->mirror<T>()));
      CK(open_rowmin<T>(h->Dl<T>(), h->ld, h->row0, h->gprow(), h->gpcol(), ocap,
                        reinterpret_cast<unsigned*>(h->anyrow()), h->ctr(), h->st));
    }
    // rounds over the open entries of each row, a first batch of 4
    // the first batch is enqueued blind: as many rounds as the previous
    // recompute needed (at least 2: round 1 finding nothing proves convergence)
    if (coop) {   // every round in one cooperative launch, to convergence (no host round trips)
      // rows with >= max(512, n/8) open pairs skip the rounds and are resolved
      // from the other rows afterwards, inside the same launch
      RoundBufs rb{h->chg(0),      h->cap + 32,     h->cap,    {fcol[0], fcol[1]}, h->coop_rounds_word(),
                   h->coop_total_word(), h->bigq(), h->bigq_ctr(), h->heavy_set(), h->heavy_x(), h->ld,
                   h->heavy_min < 0 ? 0 : (h->heavy_min > 0 ? h->heavy_min : (int)std::max<int64_t>(512, n / 8)),
                   r.hi - r.lo, n, removal ? skip : -1,
                   kCoopTail ? 1 : 0, h->slid(), h->slw<T>(), h->wnext<T>(), h->gfull(), h->host_small_dev,
                   h->mirror_flag()};
      PK(APSP_K_SPARSE_R, 0.0,
         sparse_rounds_coop<T>(h->Dl<T>(), h->ld, h->row0, h->WT<T>(), h->ld, h->gprow(), h->gpcol(), h->glb<T>(),
                               ocap, h->rowoff(), h->ocnt(), h->ocol(), rb, 0, h->max_rounds, h->anyflag(), h->sr,
                               h->ctr(), h->st, reinterpret_cast<unsigned*>(h->anyrow()), h->wmin<T>(),
                               h->mirror<T>()));
      last_total = h->coop_total_word();
      if (removal && kCoopTail) {   // the shortlist upkeep after A2, its last reader (inside the launch above)
        apsp_status s2 = fork_shortlist_remove<T>(h, skip);
        if (s2 != APSP_OK) return s2;
      }
    } else {
      apsp_status s = enqueue_rounds(std::min(std::max(2, h->rounds_hint), h->max_rounds));
      if (s != APSP_OK) return s;
    }
  }

  if (removal && !try_sparse) {
    apsp_status s2 = fork_shortlist_remove<T>(h, skip);
    if (s2 != APSP_OK) return s2;
  }
  { apsp_status sj = sl_join(); if (sj != APSP_OK) return sj; }   // (forced dense: joined here)
  // ---- the one host read of this update: counters (summed over ranks) ----
  long long* hv = reinterpret_cast<long long*>(h->host_small);
  unsigned* hmf = reinterpret_cast<unsigned*>(h->host_small) + 12;
  if (h->world == 1 && coop && try_sparse) {
    // (the cooperative launch packed the counters into mapped host memory)
  } else if (h->world == 1) {   // packed straight into mapped host memory
    CK(pack_to_host(h->ctr(), last_total, h->mirror_flag(), h->host_small_dev, h->st, nullptr));
  } else {
    long long* v = reinterpret_cast<long long*>(h->small());
    CK(pack_counters(h->ctr(), last_total, v, h->st));   // total rows ovf1 ovf2 changed | maxrow
    NK(h->comm->allreduce(v, 5, ncclInt64, ncclSum, h->st));
    NK(h->comm->allreduce(v + 5, 1, ncclInt64, ncclMax, h->st));
    ReadSet rs{};
    rs.add(v, 6 * sizeof(long long));
    rs.add(h->mirror_flag(), sizeof(unsigned));
    CK(readback(rs, h->host_small_dev, h->st));
  }
  CKR(cudaStreamSynchronize(h->st));
  h->mirror_hint = (*hmf & 1u) == 0u;
  h->mirror_fresh = true;
  if (coop && try_sparse) rounds = (int)reinterpret_cast<unsigned*>(h->host_small)[14];
  const int64_t total = hv[0], rows = hv[1], maxrow = hv[5];
  if (h->prof_on && try_sparse)   // phase A's algorithmic bytes, now that |A| is known
    for (auto it = h->prof_pending.rbegin(); it != h->prof_pending.rend(); ++it)
      if (it->cls == APSP_K_SPARSE0) {
        it->work = kPhaseABytes * (double)total;
        break;
      }
  const bool overflow = hv[2] != 0 || hv[3] != 0;   // a list overflowed on some rank
  bool changed = hv[4] != 0;
  if (info) {
    info->affected_pairs = total;
    info->affected_rows = rows;
    info->max_row_affected = maxrow;
    info->cost = removal ? (n > 1 ? (double)rows / (double)(n - 1) : 0.0) : (double)rows / (double)n;
  }
  const double cost = removal ? (n > 1 ? (double)rows / (double)(n - 1) : 0.0) : (double)rows / n;
  const bool gate = h->row_delta > 0 ? cost > h->row_delta   // paper: "Cost larger than delta"
                                     : (double)total > h->theta * (double)n * (double)n;
  bool dense = h->force_path == 2 || (h->force_path == 0 && gate) || overflow;
  // rounds until no entry changes (rarely more than the first batch); later
  // batches double (a round whose frontier is empty costs one small launch)
  int batch = std::max(2, rounds);
  while (!coop && !dense && changed && rounds < h->max_rounds) {
    batch *= 2;
    apsp_status s = enqueue_rounds(std::min(batch, h->max_rounds - rounds));
    if (s != APSP_OK) return s;
    if (h->world > 1) NK(h->comm->allreduce(last_total, 1, ncclInt32, ncclMax, h->st));
    int* hflag = reinterpret_cast<int*>(h->host_small);
    CKR(cudaMemcpyAsync(hflag, last_total, sizeof(int), cudaMemcpyDeviceToHost, h->st));
    CKR(cudaStreamSynchronize(h->st));
    changed = *hflag != 0;
  }
  if (info) info->rounds = rounds;
  if (try_sparse && !dense && !changed) h->rounds_hint = rounds;   // converged within `rounds`
  if (!dense && changed) dense = true;   // not converged: every entry is still a valid upper bound
  if (dense) {
    if (info) info->path = 3;
    if (removal && prepped)   // FW needs the removed node's row and column of D at INF
      CK(tombstone<T>(h->Dl<T>(), h->ld, r, n, skip, h->WT<T>(), h->ld, h->st));
    if (hv[2] != 0)   // the need_update_list missed pairs: reset every flagged entry in place
      PK(APSP_K_DETECT, 4.0 * (double)(r.hi - r.lo) * (double)n,
         detect<T>(h->Dl<T>(), h->ld, r, n, skip, c1, r1, c2, r2, h->tau, 2, nullptr, nullptr, nullptr,
                   nullptr, nullptr, 0, nullptr, h->WT<T>(), h->ld, h->sr, h->mirror<T>(), h->st));
    else if (!try_sparse)   // no phase A ran: the listed entries still hold D_old
      CK(reset_pairs<T>(h->Dl<T>(), h->ld, h->row0, h->WT<T>(), h->ld, h->srow(), h->scol(), h->ctr(), lcap,
                        h->st));
    // the sparse kernels' values are walk lengths of G' but may exceed a
    // listed pair's own edge: FW needs D0 <= W' too (one O(n^2) pass, against
    // the O(n^3) FW that follows)
    if (try_sparse) CK(min_with_w<T>(h->Dl<T>(), h->ld, r, n, h->WT<T>(), h->ld, h->st));
    return fw_impl<T>(h, removal ? skip : -1);
  }
  if (info) info->path = 2;
  // (the sparse kernels mirrored every value they wrote)
  return APSP_OK;
}

// ------------------------------------------------------------------ add node
template <typename T>
apsp_status add_node_impl(apsp_handle* h, const void* out_w, const void* in_w, int64_t* new_index,
                          apsp_update_info* info) {
  {
    apsp_status ms = ensure_mirror<T>(h);
    if (ms != APSP_OK) return ms;
  }
  const int64_t n = h->n, ld = h->ld, x = n;
  T* ow = h->vec<T>(0);
  T* iw = h->vec<T>(1);
  T* col = h->vec<T>(2);
  T* row = h->vec<T>(3);
  // (the scratch words start reset: at creation, then by each add's last
  // kernel, addnode_write, or on a rejected call below)
  const AddScratch as = h->add_scratch();
  // both vectors in one launch; its last block writes the host's read (the
  // validation flag, the smallest weight, the mirror flag) to mapped memory
  CK(validate_vec<T>(reinterpret_cast<const T*>(out_w), nullptr, n, ld, ow, &h->ctr()->err, h->wmin_dev(),
                     h->st, reinterpret_cast<const T*>(in_w),
                     h->directed ? nullptr : reinterpret_cast<const T*>(out_w), iw,
                     std::is_same<T, int32_t>::value ? as.argmin_out : nullptr,
                     std::is_same<T, int32_t>::value ? as.in_min : nullptr,
                     ValidateReadback{reinterpret_cast<unsigned*>(h->host_small_dev), h->validate_done(),
                                      h->mirror_flag()}));
  // the new row from the few rows that can attain it (one GPU, int8 mirror
  // valid): on the side stream, launched before the validation read so it
  // overlaps the host round trip (it writes scratch only; a rejected call
  // waits for it before returning, and if that read shows the mirror
  // invalidated the shortcuts are dropped)
  bool srow = false;
  // (small graphs: the one streaming pass costs less than the shortcuts' extra launches)
  const bool shortcut_shape = std::is_same<T, int32_t>::value && n >= kAddShortcutMinN && n < (int64_t(1) << 24) &&
                              h->plan.maxchunk >= 2 && 2 * kAddColLimit <= ld;   // (k_addrow packs t in 24 bits)
  if constexpr (std::is_same<T, int32_t>::value) {
    srow = h->world == 1 && shortcut_shape && mirror8_hint(h);
    if (srow) {
      CKR(cudaEventRecord(h->ev_fork, h->st));
      CKR(cudaStreamWaitEvent(h->st2, h->ev_fork, 0));
      // scratch: the (value, minimiser) row, the minimiser flags and U's in /
      // out lists live in the pass-1 partial buffer (4 ld words: unused unless
      // the gathers fall back to pass 1, which runs after they are consumed)
      CK2(addrow_s(as, ow, n, h->mirror<T>().m8, ld, h->row0, h->rows, row, ld, reinterpret_cast<int*>(h->vec<T>(5)),
                   reinterpret_cast<unsigned long long*>(h->rowpart<T>()),
                   reinterpret_cast<int*>(h->rowpart<T>()) + 2 * ld, h->st2));
      CKR(cudaEventRecord(h->ev_row, h->st2));
    }
  }
  unsigned* herr = reinterpret_cast<unsigned*>(h->host_small);
  CKR(cudaStreamSynchronize(h->st));
  h->mirror_hint = (herr[2] & 1u) == 0u;
  h->mirror_fresh = true;
  if (*herr) {
    if (srow) CKR(cudaStreamSynchronize(h->st2));   // the scratch is free again
    CK(add_init(as, &h->ctr()->err, h->wmin_dev(), h->st));   // reset for the next add
    return fail(h, APSP_E_INVAL, "add_node: %s",
                (*herr & 2) ? "undirected graph needs out_w == in_w" : "negative or NaN weight");
  }
  h->wmin_bits = std::min(h->wmin_bits, herr[1]);
  if (srow && !mirror8_known_valid(h)) {
    // the flag read just now says the int8 mirror was invalidated since the
    // last host read: no shortcuts; the row chain's scratch must be free first
    srow = false;
    CKR(cudaStreamWaitEvent(h->st, h->ev_row, 0));
  }
  if constexpr (std::is_same<T, int32_t>::value) {
    if (h->world > 1 && shortcut_shape) {
      // sharded: every rank must take the same path (collectives inside), so
      // the ranks agree on their mirrors first; then the new row from the
      // rows that can attain it, each rank over its own rows of S
      int* agree = reinterpret_cast<int*>(h->small() + 2048);
      CKR(cudaMemsetAsync(agree, mirror8_known_valid(h) ? 1 : 0, sizeof(int), h->st));
      NK(h->comm->allreduce(agree, 1, ncclInt32, ncclMin, h->st));
      CKR(cudaMemcpyAsync(h->host_small, agree, sizeof(int), cudaMemcpyDeviceToHost, h->st));
      CKR(cudaStreamSynchronize(h->st));
      srow = *reinterpret_cast<int*>(h->host_small) != 0;
      if (srow) {
        const uint8_t* m8 = h->mirror<T>().m8;
        int* slist = reinterpret_cast<int*>(h->vec<T>(5));
        auto* packed = reinterpret_cast<unsigned long long*>(h->rowpart<T>());
        int* tflag = reinterpret_cast<int*>(h->rowpart<T>()) + 2 * ld;
        CK(addrow_s(as, ow, n, m8, ld, h->row0, h->rows, row, ld, slist, packed, tflag, h->st, 1));
        NK(h->comm->allreduce(as.rmax, 1, ncclInt32, ncclMax, h->st));
        CK(addrow_s(as, ow, n, m8, ld, h->row0, h->rows, row, ld, slist, packed, tflag, h->st, 2));
        NK(h->comm->allreduce(packed, (size_t)ld, ncclUint64, ncclMin, h->st));
        CK(addrow_s(as, ow, n, m8, ld, h->row0, h->rows, row, ld, slist, packed, tflag, h->st, 3));
      }
    }
  }
  // shortlist upkeep needs only the validated edge vectors: it runs on the
  // side stream while pass 1 / rank-1 stream D (joined before returning)
  CKR(cudaEventRecord(h->ev_fork, h->st));
  CKR(cudaStreamWaitEvent(h->st2, h->ev_fork, 0));
  CK2(shortlist_add_bound<T>(h->slid(), h->slw<T>(), h->wnext<T>(), ow, n, x, h->st2));  // x -> j
  CK2(shortlist_build_one<T>(iw, 0, n + 1, x, h->slid(), h->slw<T>(), h->wnext<T>(), h->slscr(),
                             h->st2));   // in-edges of x: row x of WT is in_w
  CKR(cudaEventRecord(h->ev_join, h->st2));
  Rows r = h->active();
  int nchunk = 0, nslab = 0;
  T* rowpartM = h->rowpart<T>() + (size_t)h->plan.maxchunk * ld;
  T* ceff = h->vec<T>(4);
  // Pass 1: on the int8 / int16 mirror in packed arithmetic when it is valid
  // (shortest path, int32), else — or if a new-row/column value came out
  // >= 0x3FFF — in int32.  The choice is made on the device: each launch
  // below exits when it does not apply (gate flags, stream order).
  const bool try_packed = std::is_same<T, int32_t>::value && h->sr == 0 && h->use_mirror;
  unsigned* unc = h->pass1_uncertain();
  if (try_packed) {
    if (!srow) CKR(cudaMemsetAsync(unc, 0, sizeof(unsigned), h->st));   // (the gather path never reads it)
    const unsigned* cfull = nullptr;
    if constexpr (std::is_same<T, int32_t>::value) {
      if (srow) {   // the new row first (side stream; sharded: done above), then col / the skip bound by gathers
        if (h->world == 1) CKR(cudaStreamWaitEvent(h->st, h->ev_row, 0));
        PK(APSP_K_ADD_PASS1, 0.0,
           addcol_g(as, r, h->mirror<T>().m8, ld, n, iw, ow, reinterpret_cast<int*>(h->rowpart<T>()) + 2 * ld,
                    reinterpret_cast<int*>(h->vec<T>(5)), reinterpret_cast<int*>(h->rowpart<T>()) + 3 * ld,
                    kAddColLimit, col, ceff, h->vec<T>(6),
                    reinterpret_cast<int*>(h->vec<T>(7)), h->wmin<int32_t>(), h->st, h->mirror<T>().mt,
                    h->plan.ldt));
        cfull = as.ufull;
      }
    }
    if (srow) {
      // fallback of the gathers (|U| over its limit, *cfull set): the int32
      // pass — exact, so no int16 uncertainty to resolve — and the finish of
      // the column; both exit at once otherwise (grid-stride, small grids)
      CK(addnode_pass1<T>(h->Dl<T>(), ld, r, n, ow, iw, h->rowpart<T>(), rowpartM, h->colpart<T>(), ld,
                          &nchunk, &nslab, kMaxSlabs, h->sr, h->mirror<T>(), cfull, 0, h->st));
      CK(addnode_finish<T>(h->rowpart<T>(), rowpartM, nchunk, h->colpart<T>(), nslab, ld, r, n, ld, col,
                           ceff, row, 0, h->mirror<T>(), unc, h->st, as.rfull, cfull));
    } else {
      // the streaming pass on the mirror ...
      PK(APSP_K_ADD_PASS1, h->mirror_hint ? h->stream_bytes<T>() * (double)(r.hi - r.lo) * (double)n : 0.0,
         addnode_pass1<T>(h->Dl<T>(), ld, r, n, ow, iw, h->rowpart<T>(), rowpartM, h->colpart<T>(), ld,
                          &nchunk, &nslab, kMaxSlabs, h->sr, h->mirror<T>(), unc, 1, h->st));
      CK(addnode_finish<T>(h->rowpart<T>(), rowpartM, nchunk, h->colpart<T>(), nslab, ld, r, n, ld, col,
                           ceff, row, 1, h->mirror<T>(), unc, h->st));
    }
  }
  if (!srow) {   // ... or in int32 (gated on the packed pass' outcome when it ran)
    PK(APSP_K_ADD_PASS1, try_packed && h->mirror_hint ? 0.0 : 4.0 * (double)(r.hi - r.lo) * (double)n,
       addnode_pass1<T>(h->Dl<T>(), ld, r, n, ow, iw, h->rowpart<T>(), rowpartM, h->colpart<T>(), ld,
                        &nchunk, &nslab, kMaxSlabs, h->sr, h->mirror<T>(), try_packed ? unc : nullptr, 0,
                        h->st));
    CK(addnode_finish<T>(h->rowpart<T>(), rowpartM, nchunk, h->colpart<T>(), nslab, ld, r, n, ld, col,
                         ceff, row, try_packed ? 2 : 0, h->mirror<T>(), unc, h->st));
  }
  if (h->world > 1 && !srow)   // (the shortcut's row is already complete)
    NK(h->comm->allreduce(row, (size_t)ld, nccl_type<T>(), ncclMin, h->st));
  // rows with ceff[i] = INF provably do not change and are not read at all
  PK(APSP_K_RANK1, 0.0,   // work: bytes actually read, counted on the device
     rank1<T>(h->Dl<T>(), ld, r, n, ceff, row, nullptr, nullptr, h->rank1_bytes(), h->sr, h->mirror<T>(),
              h->st, mirror8_known_valid(h) ? 0 : 1));
  h->mirror_fresh = false;   // rank-1 and the new row / column may write values >= 0x7F
  CK(addnode_write<T>(h->Dl<T>(), ld, r, n, x, h->local(x) ? 1 : 0, col, row, h->WT<T>(), ld, ow,
                      iw, h->mirror<T>(), h->st, as, &h->ctr()->err, h->wmin_dev()));
  // (addnode_write mirrored the new row / column)
  CKR(cudaStreamWaitEvent(h->st, h->ev_join, 0));   // shortlist upkeep (side stream) done
  h->sl_join = false;   // (st2 is in order: this joined any earlier upkeep too)
  h->n = n + 1;
  if (new_index) *new_index = x;
  if (info) {
    info->kind = 3;
    info->path = 1;
    info->n_after = h->n;
  }
  return APSP_OK;
}

// ------------------------------------------------------------------ remove node
template <typename T>
apsp_status remove_node_impl(apsp_handle* h, int64_t k, int64_t* moved_from, apsp_update_info* info) {
  {
    apsp_status ms = ensure_mirror<T>(h);
    if (ms != APSP_OK) return ms;
  }
  const int64_t n = h->n, ld = h->ld;
  Rows r = h->active();
  T* c1 = h->vec<T>(4);
  T* r1 = h->vec<T>(5);
  apsp_status s;
  const bool prep = h->world == 1;
  if (prep) {   // counters, snapshots t1 = SPD(i, k), t2 = SPD(k, j), WT tombstone: one launch
    CK(update_prep<T>(h->Dl<T>(), ld, r, k, T(0), c1, h->Drow<T>(k), n, ld, r1, recompute_zero_set(h), h->WT<T>(),
                      ld, k, h->sr, h->st, h->r1_bytes()));
  } else {
    s = snap_pivots<T>(h, k, T(0), c1, k, r1);   // t1 = SPD(i, k), t2 = SPD(k, j)
    if (s != APSP_OK) return s;
  }
  if (info) info->kind = 4;
  s = recompute<T>(h, k, c1, r1, nullptr, nullptr, true, info, prep, prep ? h->r1_bytes() : nullptr);
  if (s != APSP_OK) return s;

  // swap-with-last: node n-1 moves into slot k (Q7)
  const int64_t last = n - 1;
  int row_copy = 0;
  if (k != last) {
    const bool ok_k = h->local(k), ok_l = h->local(last);
    if (ok_k && ok_l) {
      row_copy = 1;
    } else if (ok_k || ok_l) {   // the row crosses ranks: it arrives in row k first
      P2POp op = ok_l ? P2POp{1, h->Drow<T>(last), (size_t)n, nccl_type<T>(), h->owner(k)}
                      : P2POp{0, h->Drow<T>(k), (size_t)n, nccl_type<T>(), h->owner(last)};
      NK(h->comm->sendrecv(&op, 1, h->st));
    }
  }
  CK(move_last<T>(h->Dl<T>(), ld, r, n, k, row_copy, h->WT<T>(), ld, h->mirror<T>(), h->st));
  // the shortlist upkeep (side stream, forked in recompute) is joined by the
  // next reader or writer of the shortlists on the compute stream (join_side,
  // recompute's sl_join), not here: it overlaps the next update's first kernels
  h->sl_join = true;
  h->n = n - 1;
  if (moved_from) *moved_from = (k != last) ? last : -1;
  if (info) info->n_after = h->n;
  return APSP_OK;
}

// ------------------------------------------------------------------ update edge
template <typename T>
apsp_status update_edge_impl(apsp_handle* h, int64_t u, int64_t v, T w_new, apsp_update_info* info) {
  const int64_t n = h->n, ld = h->ld;
  T* WT = h->WT<T>();
  // 8-byte read: W[u][v] (replicated WT) and D[u][v] (owner of row u) —
  // one GPU: both words straight into the mapped host buffer by one kernel
  T* hv = reinterpret_cast<T*>(h->host_small);
  if (h->world == 1) {
    // one warp reads both words and, when the update exits early, applies it
    // (W and the shortlists) before the host's read — the common case costs
    // one launch and the read
    { apsp_status sj = join_side(h); if (sj != APSP_OK) return sj; }
    CK(edge_early<T>(WT, ld, h->Drow<T>(u), h->slid(), h->slw<T>(), h->wnext<T>(), u, v, w_new, h->directed,
                     h->tau, h->host_small_dev, h->st));
    CKR(cudaStreamSynchronize(h->st));
    if (reinterpret_cast<volatile unsigned*>(h->host_small)[2] != 0u) {
      const T w_old = hv[0];
      if (info) {
        info->n_after = n;
        info->kind = w_new == w_old ? 0 : (w_new < w_old ? 1 : 2);
        info->early_exit = 1;
      }
      if (w_new != w_old) h->fold_wmin<T>(w_new);
      return APSP_OK;
    }
  } else {
    T* dev2 = reinterpret_cast<T*>(h->small());
    CKR(cudaMemcpyAsync(dev2, WT + v * ld + u, sizeof(T), cudaMemcpyDeviceToDevice, h->st));
    if (h->local(u))
      CKR(cudaMemcpyAsync(dev2 + 1, h->Drow<T>(u) + v, sizeof(T), cudaMemcpyDeviceToDevice, h->st));
    NK(h->comm->bcast(dev2 + 1, 1, nccl_type<T>(), h->owner(u), h->st));
    ReadSet rs{};
    rs.add(dev2, 2 * sizeof(T));
    CK(readback(rs, h->host_small_dev, h->st));
    CKR(cudaStreamSynchronize(h->st));
  }
  const T w_old = hv[0], duv = hv[1];
  if (info) info->n_after = n;
  if (w_new == w_old) {
    if (info) { info->kind = 0; info->early_exit = 1; }
    return APSP_OK;
  }
  h->fold_wmin<T>(w_new);
  Rows r = h->active();
  T* c1 = h->vec<T>(4);
  T* r1 = h->vec<T>(5);
  T* c2 = h->vec<T>(6);
  T* r2 = h->vec<T>(7);
  const bool und = !h->directed;
  if (w_new < w_old) {
    // ---- decrease: exact early exit iff w_new >= D[u][v] ----
    if (info) info->kind = 1;
    if (!(w_new < duv)) {
      if (info) info->early_exit = 1;
      CK(set_edge<T>(WT, ld, u, v, w_new, h->directed, h->st));
      { apsp_status sj = join_side(h); if (sj != APSP_OK) return sj; }
      CK(shortlist_set_edge<T>(h->slid(), h->slw<T>(), h->wnext<T>(), u, v, w_new, h->directed, h->st));
      return APSP_OK;
    }
    // D'[i][j] = min(D[i][j], D[i][u] + w + D[v][j] (, D[i][v] + w + D[u][j]))
    apsp_status s = snap_pivots<T>(h, u, w_new, c1, v, r1);
    if (s != APSP_OK) return s;
    if (und) {
      s = snap_pivots<T>(h, v, w_new, c2, u, r2);
      if (s != APSP_OK) return s;
    }
    PK(APSP_K_RANK1, 0.0,   // work: bytes actually read, counted on the device
       rank1<T>(h->Dl<T>(), ld, r, n, c1, r1, und ? c2 : nullptr, und ? r2 : nullptr, h->rank1_bytes(),
                h->sr, h->mirror<T>(), h->st));
    h->mirror_fresh = false;   // rank-1 may write values >= 0x7F
    CK(set_edge<T>(WT, ld, u, v, w_new, h->directed, h->st));
    { apsp_status sj = join_side(h); if (sj != APSP_OK) return sj; }
    CK(shortlist_set_edge<T>(h->slid(), h->slw<T>(), h->wnext<T>(), u, v, w_new, h->directed, h->st));
    if (info) info->path = 1;
    return APSP_OK;
  }
  // ---- increase: exact early exit iff the edge is not tight (w_old > D[u][v]) ----
  if (info) info->kind = 2;
  bool tight;
  if (Tr<T>::kFloat) tight = (double)w_old <= (double)duv * (1.0 + (double)h->tau);
  else tight = (w_old == duv);
  if (!tight) {
    if (info) info->early_exit = 1;
    CK(set_edge<T>(WT, ld, u, v, w_new, h->directed, h->st));
    { apsp_status sj = join_side(h); if (sj != APSP_OK) return sj; }
    CK(shortlist_set_edge<T>(h->slid(), h->slw<T>(), h->wnext<T>(), u, v, w_new, h->directed, h->st));
    return APSP_OK;
  }
  apsp_status s;
  const bool prep = h->world == 1;
  if (prep) {   // counters and the snapshots D[i][u] + w_old, D[v][j]: one launch
    CK(update_prep<T>(h->Dl<T>(), ld, r, u, w_old, c1, h->Drow<T>(v), n, ld, r1, recompute_zero_set(h), WT, ld,
                      -1, h->sr, h->st, h->r1_bytes()));
  } else {
    s = snap_pivots<T>(h, u, w_old, c1, v, r1);   // D[i][u] + w_old, D[v][j]
    if (s != APSP_OK) return s;
  }
  if (und) {
    s = snap_pivots<T>(h, v, w_old, c2, u, r2);
    if (s != APSP_OK) return s;
  }
  // W' before the recompute reads it: WT here, the shortlists on the side
  // stream (recompute joins it before its first shortlist reader)
  CK(set_edge<T>(WT, ld, u, v, w_new, h->directed, h->st));
  CKR(cudaEventRecord(h->ev_fork, h->st));
  CKR(cudaStreamWaitEvent(h->st2, h->ev_fork, 0));
  CK2(shortlist_set_edge<T>(h->slid(), h->slw<T>(), h->wnext<T>(), u, v, w_new, h->directed, h->st2));
  CKR(cudaEventRecord(h->ev_join, h->st2));
  h->sl_join = true;
  {   // the detection pass reads the mirror (early exits and decreases do not)
    apsp_status ms = ensure_mirror<T>(h);
    if (ms != APSP_OK) return ms;
  }
  return recompute<T>(h, -1, c1, r1, und ? c2 : nullptr, und ? r2 : nullptr, false, info, prep,
                      prep ? h->r1_bytes() : nullptr);
}

// ------------------------------------------------------------------ f1: paper-faithful modify
// Definition 1's Phi for removing node k: rows with a non-empty need_update_list
// (P:184-194), counted from the detection bitmap's row marks.
template <typename T>
apsp_status removal_phi(apsp_handle* h, int64_t k, int64_t* phi) {
  const int64_t n = h->n, ld = h->ld;
  Rows r = h->active();
  T* c1 = h->vec<T>(4);
  T* r1 = h->vec<T>(5);
  CK(gather_col<T>(h->Dl<T>(), ld, r, k, T(0), c1, h->sr, h->st));
  apsp_status s = snap_row<T>(h, k, T(0), r1);
  if (s != APSP_OK) return s;
  PK(APSP_K_DETECT, h->stream_bytes<T>() * (double)(r.hi - r.lo) * (double)n,
     detect<T>(h->Dl<T>(), ld, r, n, k, c1, r1, nullptr, nullptr, h->tau, 0, h->anyrow(), nullptr,
               nullptr, nullptr, nullptr, 0, nullptr, nullptr, 0, h->sr, h->mirror<T>(), h->st, h->tmap8_ptr()));
  unsigned long long* cnt = reinterpret_cast<unsigned long long*>(h->small() + 128);
  CKR(cudaMemsetAsync(cnt, 0, sizeof *cnt, h->st));
  CK(count_nonzero(h->anyrow() + r.lo, r.hi - r.lo, cnt, h->st));
  if (h->world > 1)
    NK(h->comm->allreduce(cnt, 1, ncclUint64, ncclSum, h->st));
  unsigned long long* hv = reinterpret_cast<unsigned long long*>(h->host_small);
  CKR(cudaMemcpyAsync(hv, cnt, sizeof *cnt, cudaMemcpyDeviceToHost, h->st));
  CKR(cudaStreamSynchronize(h->st));
  *phi = (int64_t)*hv;
  return APSP_OK;
}

// Exchange the ids of nodes p and q (rows and columns of D and WT, shortlists).
template <typename T>
apsp_status swap_nodes(apsp_handle* h, int64_t p, int64_t q) {
  const int64_t n = h->n, ld = h->ld;
  const bool lp = h->local(p), lq = h->local(q);
  if (lp && lq) {
    CK(swap_vecs<T>(h->Drow<T>(p), h->Drow<T>(q), n, h->st));
  } else if (lp || lq) {
    T* mine = lp ? h->Drow<T>(p) : h->Drow<T>(q);
    const int peer = h->owner(lp ? q : p);
    T* tmp = h->panel<T>();
    P2POp ops[2] = {{1, mine, (size_t)n, nccl_type<T>(), peer}, {0, tmp, (size_t)n, nccl_type<T>(), peer}};
    NK(h->comm->sendrecv(ops, 2, h->st));
    CK(copy_row<T>(mine, tmp, n, h->st));
  }
  CK(swap_cols<T>(h->Dl<T>(), ld, h->active(), p, q, h->st));
  T* WT = h->WT<T>();
  CK(swap_vecs<T>(WT + p * ld, WT + q * ld, n, h->st));
  Rows rw{0, n, 0};
  CK(swap_cols<T>(WT, ld, rw, p, q, h->st));
  { apsp_status sj = join_side(h); if (sj != APSP_OK) return sj; }
  CK(shortlist_swap<T>(h->slid(), h->slw<T>(), h->wnext<T>(), n, p, q, h->st));
  CK(mirror_cross(h->Dl<T>(), ld, h->active(), n, p, p, h->mirror<T>(), h->st));
  CK(mirror_cross(h->Dl<T>(), ld, h->active(), n, q, q, h->mirror<T>(), h->st));
  return APSP_OK;
}

template <typename T>
apsp_status modify_readd_impl(apsp_handle* h, int64_t u, int64_t v, T w_new, int64_t* removed,
                              apsp_update_info* info) {
  {
    apsp_status ms = ensure_mirror<T>(h);
    if (ms != APSP_OK) return ms;
  }
  const int64_t n = h->n, ld = h->ld;
  T* WT = h->WT<T>();
  T* hv = reinterpret_cast<T*>(h->host_small);
  CKR(cudaMemcpyAsync(hv, WT + v * ld + u, sizeof(T), cudaMemcpyDeviceToHost, h->st));
  CKR(cudaStreamSynchronize(h->st));
  if (info) info->n_after = n;
  if (hv[0] == w_new) {
    if (info) { info->kind = 0; info->early_exit = 1; }
    return APSP_OK;
  }
  // "it calculates which node is cheaper to remove, then remove the cheaper one"
  int64_t phi_u = 0, phi_v = 0;
  apsp_status s = removal_phi<T>(h, u, &phi_u);
  if (s != APSP_OK) return s;
  s = removal_phi<T>(h, v, &phi_v);
  if (s != APSP_OK) return s;
  const int64_t p = (phi_u < phi_v || (phi_u == phi_v && u < v)) ? u : v;
  const int64_t other = p == u ? v : u;
  // p's edge vectors with the edited edge: out[t] = W[p][t], in[t] = W[t][p]
  T* so = h->vec<T>(2);
  T* si = h->vec<T>(3);
  Rows rw{0, n, 0};
  CK(gather_col<T>(WT, ld, rw, p, T(0), so, h->sr, h->st));
  CK(copy_vec<T>(WT + p * ld, n, ld, T(0), si, h->st));
  if (!h->directed || p == u) CK(vec_set_move<T>(so, other, w_new, -1, 0, h->st));
  if (!h->directed || p == v) CK(vec_set_move<T>(si, other, w_new, -1, 0, h->st));
  const int64_t last = n - 1;
  if (p != last) {   // after the removal node `last` lives in slot p
    CK(vec_set_move<T>(so, -1, T(0), p, last, h->st));
    CK(vec_set_move<T>(si, -1, T(0), p, last, h->st));
  }
  int64_t mf = -1;
  apsp_update_info rinfo;
  std::memset(&rinfo, 0, sizeof rinfo);
  s = remove_node_impl<T>(h, p, &mf, &rinfo);
  if (s != APSP_OK) return s;
  int64_t x = -1;
  s = add_node_impl<T>(h, so, si, &x, nullptr);
  if (s != APSP_OK) return s;
  if (p != last) {
    s = swap_nodes<T>(h, p, x);   // restore the original ids
    if (s != APSP_OK) return s;
  }
  if (removed) *removed = p;
  if (info) {
    *info = rinfo;
    info->kind = 5;
    info->n_after = h->n;
  }
  return APSP_OK;
}

// ------------------------------------------------------------------ query
// Batched queries on device arrays.  world == 1: one kernel.  world > 1 (row-
// sharded D, f3 of SURVEY §8(f)): per chunk of kQueryChunk queries, gather the
// column-t slices of every rank (one all-gather), let the owner of row s answer,
// and all-reduce(sum) the outputs (non-owners contribute zeros).  No rank
// gathers whole rows; WT is replicated, so the Dijkstra step is local.
template <typename T>
apsp_status query_dispatch(apsp_handle* h, int q, const int* s, const int* t, T* dist, int* paths,
                           int path_cap, int* lens, int* ncand) {
  const int64_t n = h->n, ld = h->ld;
  if (h->world <= 1) {
    PK(APSP_K_QUERY, 8.0 * (double)n * q,
       query_batch<T>(h->Dl<T>(), ld, h->WT<T>(), ld, n, q, s, t, dist, paths, path_cap, lens, ncand,
                      h->tau, h->sr, h->st, h->qscratch(), h->wmin<T>()));
    return APSP_OK;
  }
  Rows r = h->active();
  const int hcap = h->plan.qcap;
  int* hits = reinterpret_cast<int*>(h->ws + h->plan.off_qhit);
  int* allhits = reinterpret_cast<int*>(h->ws + h->plan.off_qcol);
  T* rowbuf = h->qsend<T>();
  for (int b0 = 0; b0 < q; b0 += kQueryChunk) {
    const int c = std::min(kQueryChunk, q - b0);
    // rows s to every rank, the local candidate tests, the hit lists to every
    // rank; then every rank solves (identical answers, no output exchange)
    CK(query_rowsend<T>(h->Dl<T>(), ld, h->row0, r.hi - r.lo, n, s + b0, c, rowbuf, ld, h->st));
    NK(h->comm->allreduce(rowbuf, (size_t)c * ld, nccl_type<T>(), ncclSum, h->st));
    PK(APSP_K_QUERY, 8.0 * (double)(r.hi - r.lo) * c,
       query_localscan<T>(h->Dl<T>(), ld, h->row0, r.hi - r.lo, n, s + b0, t + b0, c, rowbuf, ld, hits, hcap,
                          h->tau, h->sr, h->wmin<T>(), h->st));
    NK(h->comm->allgather(hits, allhits, (size_t)c * (hcap + 1), ncclInt32, h->st));
    int* pb = path_cap > 0 ? paths + (int64_t)b0 * path_cap : paths;
    CK(query_solve_sharded<T>(h->Dl<T>(), ld, h->WT<T>(), ld, n, c, s + b0, t + b0, dist + b0, pb, path_cap,
                              lens + b0, ncand ? ncand + b0 : nullptr, h->tau, h->sr, allhits, h->world, hcap,
                              rowbuf, ld, h->qscratch(), h->st));
  }
  return APSP_OK;
}

template <typename T>
apsp_status query_one(apsp_handle* h, int64_t s, int64_t t, void* dist, int32_t* path,
                      int32_t path_cap, int32_t* path_len, int32_t* n_candidates) {
  // device scratch: [s, t, len, ncand, dist] then the path
  int* dv = reinterpret_cast<int*>(h->small() + 1024);
  T* ddist = reinterpret_cast<T*>(dv + 4);
  int* dpath = dv + 8;
  const int cap_dev = (int)((64 * 1024 - 1024 - 512 - 64) / sizeof(int)) - 8;
  int* hv = reinterpret_cast<int*>(h->host_small);
  hv[0] = (int)s; hv[1] = (int)t;
  CKR(cudaMemcpyAsync(dv, hv, 2 * sizeof(int), cudaMemcpyHostToDevice, h->st));
  apsp_status qs = query_dispatch<T>(h, 1, dv, dv + 1, ddist, dpath, cap_dev, dv + 2, dv + 3);
  if (qs != APSP_OK) return qs;
  CKR(cudaMemcpyAsync(hv, dv, 8 * sizeof(int), cudaMemcpyDeviceToHost, h->st));
  CKR(cudaStreamSynchronize(h->st));
  const int len = hv[2], nc = hv[3];
  std::memcpy(dist, &hv[4], sizeof(T));
  if (n_candidates) *n_candidates = nc;
  if (len < 0 && nc > std::min(h->plan.qcap, cap_dev) && h->world == 1 && h->sr == 0) {
    // more candidates than the batch scratch holds: every candidate's
    // predecessor at once, then the walk (query.cu: query_big)
    int* out = reinterpret_cast<int*>(h->ws + h->plan.off_qbout);
    CK(query_big<T>(h->Dl<T>(), h->ld, h->WT<T>(), h->ld, h->n, (int)s, (int)t,
                    reinterpret_cast<unsigned*>(h->ws + h->plan.off_qbits),
                    reinterpret_cast<int*>(h->ws + h->plan.off_qbpred), out + 2, out + 3, (int)h->cap, h->tau,
                    h->wmin<T>(), h->st));
    CKR(cudaMemcpyAsync(hv, out + 3, sizeof(int), cudaMemcpyDeviceToHost, h->st));
    CKR(cudaStreamSynchronize(h->st));
    const int blen = hv[0];
    if (blen > 0) {
      if (path_len) *path_len = blen;
      if (blen > path_cap)
        return fail(h, APSP_E_RANGE, "sp_pair_query: path_cap %d < path length %d", path_cap, blen);
      CKR(cudaMemcpyAsync(path, out + 4, sizeof(int) * blen, cudaMemcpyDeviceToHost, h->st));
      CKR(cudaStreamSynchronize(h->st));
      return APSP_OK;
    }
  }
  if (len < 0) {
    if (path_len) *path_len = 0;
    return fail(h, APSP_E_RANGE, "sp_pair_query: no path from the %d candidates (capacity %d)", nc,
                std::min(h->plan.qcap, cap_dev));
  }
  if (path_len) *path_len = len;
  if (len > path_cap) return fail(h, APSP_E_RANGE, "sp_pair_query: path_cap %d < path length %d", path_cap, len);
  if (len > 0) {
    CKR(cudaMemcpyAsync(path, dpath, sizeof(int) * len, cudaMemcpyDeviceToHost, h->st));
    CKR(cudaStreamSynchronize(h->st));
  }
  return APSP_OK;
}

// ------------------------------------------------------------------ test export
// The need_update_list of a prospective update, by the same snapshot and
// detection launches the update itself runs (MODE 1), without applying it.
template <typename T>
apsp_status need_list_impl(apsp_handle* h, int kind, int64_t a, int64_t b, int32_t* rows, int32_t* cols,
                           int64_t cap, int64_t* count) {
  { apsp_status sj = join_side(h); if (sj != APSP_OK) return sj; }
  {
    apsp_status ms = ensure_mirror<T>(h);
    if (ms != APSP_OK) return ms;
  }
  const int64_t n = h->n;
  Rows r = h->active();
  T* c1 = h->vec<T>(4);
  T* r1 = h->vec<T>(5);
  T* c2 = h->vec<T>(6);
  T* r2 = h->vec<T>(7);
  const bool und = kind == 2 && !h->directed;
  int64_t skip = -1;
  apsp_status s;
  if (kind == 4) {
    skip = a;
    s = snap_pivots<T>(h, a, T(0), c1, a, r1);
  } else {
    T* hv = reinterpret_cast<T*>(h->host_small);
    CKR(cudaMemcpyAsync(hv, h->WT<T>() + b * h->ld + a, sizeof(T), cudaMemcpyDeviceToHost, h->st));
    CKR(cudaStreamSynchronize(h->st));
    const T w_old = hv[0];
    s = snap_pivots<T>(h, a, w_old, c1, b, r1);
    if (s == APSP_OK && und) s = snap_pivots<T>(h, b, w_old, c2, a, r2);
  }
  if (s != APSP_OK) return s;
  ZeroSet z{};
  z.add(h->rowcnt(), h->cap);
  z.add(reinterpret_cast<int*>(h->ctr()), (int64_t)(sizeof(DetectCounters) / sizeof(int)));
  CK(zero_set(z, h->st));
  if (use_fused<T>(h, und)) {   // the kernel the update would run, every pair on the list
    PK(APSP_K_DETECT, (double)(r.hi - r.lo) * (double)n,
       detect_fix_p8(reinterpret_cast<int32_t*>(h->Dl<T>()), h->ld, r, n, skip,
                     reinterpret_cast<const int32_t*>(c1), reinterpret_cast<const int32_t*>(r1), h->slid(),
                     reinterpret_cast<const int32_t*>(h->slw<T>()), h->mirror<T>(), h->rowcnt(), h->srow(),
                     h->scol(), h->prow(), h->pcol(), h->plan.lcap, h->ctr(), 1, h->st));
  } else {
    PK(APSP_K_DETECT, h->stream_bytes<T>() * (double)(r.hi - r.lo) * (double)n,
       detect<T>(h->Dl<T>(), h->ld, r, n, skip, c1, r1, und ? c2 : nullptr, und ? r2 : nullptr, h->tau, 1,
                 nullptr, h->rowcnt(), h->srow(), h->scol(), nullptr, h->plan.lcap, h->ctr(), h->WT<T>(), h->ld,
                 h->sr, h->mirror<T>(), h->st, h->tmap8_ptr()));
  }
  unsigned long long tot = 0;
  CKR(cudaMemcpyAsync(h->host_small, &h->ctr()->total, sizeof tot, cudaMemcpyDeviceToHost, h->st));
  CKR(cudaStreamSynchronize(h->st));
  std::memcpy(&tot, h->host_small, sizeof tot);
  *count = (int64_t)tot;
  const int64_t m = std::min<int64_t>(std::min<int64_t>((int64_t)tot, h->plan.lcap), cap);
  if (m > 0) {
    CKR(cudaMemcpyAsync(rows, h->srow(), sizeof(int32_t) * (size_t)m, cudaMemcpyDeviceToHost, h->st));
    CKR(cudaMemcpyAsync(cols, h->scol(), sizeof(int32_t) * (size_t)m, cudaMemcpyDeviceToHost, h->st));
    CKR(cudaStreamSynchronize(h->st));
  }
  return APSP_OK;
}

template <typename F>
apsp_status dispatch(apsp_dtype dt, F&& f) {
  if (dt == APSP_I32) return f(int32_t{});
  return f(float{});
}

}  // namespace

// ============================================================================
// C ABI
// ============================================================================
extern "C" {

apsp_status apsp_layout(int64_t cap, int world, int rank, int64_t* ld, int64_t* row0, int64_t* rows) {
  if (cap < 1 || world < 1 || rank < 0 || rank >= world) return APSP_E_INVAL;
  if (ld) *ld = round_up(cap, 32);
  int64_t r0, rr;
  layout_rows(cap, world, rank, &r0, &rr);
  if (row0) *row0 = r0;
  if (rows) *rows = rr;
  return APSP_OK;
}

size_t apsp_workspace_bytes(apsp_dtype dtype, int64_t cap, int world) {
  if ((dtype != APSP_I32 && dtype != APSP_F32) || cap < 1 || world < 1) return 0;
  return make_plan(cap, world, round_up(cap, 32)).total;
}

const char* apsp_status_string(apsp_status s) {
  switch (s) {
    case APSP_OK: return "ok";
    case APSP_E_INVAL: return "invalid argument";
    case APSP_E_RANGE: return "out of range";
    case APSP_E_CAPACITY: return "capacity exceeded";
    case APSP_E_PRECOND: return "precondition violated";
    case APSP_E_CUDA: return "CUDA error";
    case APSP_E_NCCL: return "NCCL error";
    case APSP_E_NOMEM: return "workspace too small";
    case APSP_E_POISONED: return "handle poisoned by an earlier failure";
    case APSP_E_UNSUPPORTED: return "unsupported";
  }
  return "unknown status";
}

apsp_status apsp_nccl_unique_id(void* out128) {
  if (!out128) return APSP_E_INVAL;
  return nccl_unique_id(out128) ? APSP_OK : APSP_E_NCCL;
}

}  // extern "C"

namespace {

// Frees everything a handle owns (never the caller's memory).
void release_handle(apsp_handle* h) {
  for (auto& g : h->fw_graphs) cudaGraphExecDestroy(g.second.exec);
  if (h->stcap) cudaStreamDestroy(h->stcap);
  for (auto e : h->ev_pool) cudaEventDestroy(e);
  for (auto& r : h->prof_pending) { cudaEventDestroy(r.a); cudaEventDestroy(r.b); }
  if (h->st2) { cudaStreamSynchronize(h->st2); cudaStreamDestroy(h->st2); }
  if (h->ev_fork) cudaEventDestroy(h->ev_fork);
  if (h->ev_join) cudaEventDestroy(h->ev_join);
  if (h->ev_row) cudaEventDestroy(h->ev_row);
  if (h->stc) { cudaStreamSynchronize(h->stc); cudaStreamDestroy(h->stc); }
  if (h->ev_pan) cudaEventDestroy(h->ev_pan);
  if (h->ev_bc) cudaEventDestroy(h->ev_bc);
  delete h->comm;
  if (h->host_small) cudaFreeHost(h->host_small);
  delete h;
}

// Shared by apsp_create (NCCL) and apsp_create_local (in-process group):
// exactly one of nccl_id / group is used when world > 1.
apsp_status create_impl(apsp_handle** out, apsp_dtype dtype, int directed, int64_t n, int64_t cap,
                        const void* W, int64_t ldw, void* D_local, int64_t ld, void* workspace,
                        size_t workspace_bytes, void* stream, int rank, int world,
                        const void* nccl_id, LocalGroup* group) {
  if (!out) return APSP_E_INVAL;
  *out = nullptr;
  if (dtype != APSP_I32 && dtype != APSP_F32) return APSP_E_INVAL;
  if (n < 1 || cap < n || cap > (int64_t)1 << 30 || !W || ldw < n || !D_local || !workspace)
    return APSP_E_INVAL;
  if (world < 1 || rank < 0 || rank >= world || (world > 1 && !nccl_id && !group)) return APSP_E_INVAL;
  if (((uintptr_t)workspace & 255) || ((uintptr_t)D_local & 15)) return APSP_E_INVAL;
  if (ld < round_up(cap, 32) || (ld & 3)) return APSP_E_INVAL;
  Plan plan = make_plan(cap, world, ld);
  if (workspace_bytes < plan.total) return APSP_E_NOMEM;

  apsp_handle* h = new apsp_handle();
  h->dt = dtype;
  h->directed = directed ? 1 : 0;
  h->n = n;
  h->cap = cap;
  h->ld = ld;
  h->plan = plan;
  h->D = D_local;
  layout_rows(cap, world, rank, &h->row0, &h->rows);
  h->R = world > 1 ? round_up(cdiv(cap, world), kTile) : cap;
  h->ws = reinterpret_cast<unsigned char*>(workspace);
  h->st = reinterpret_cast<cudaStream_t>(stream);
  h->rank = rank;
  h->world = world;
  // mapped: small host reads are written by a kernel (k_readback) instead of
  // separate device-to-host copies
  if (cudaHostAlloc(&h->host_small, 4096, cudaHostAllocMapped) != cudaSuccess ||
      cudaHostGetDevicePointer(&h->host_small_dev, h->host_small, 0) != cudaSuccess) {
    if (h->host_small) cudaFreeHost(h->host_small);
    delete h;
    return APSP_E_CUDA;
  }
  if (cudaStreamCreateWithFlags(&h->st2, cudaStreamNonBlocking) != cudaSuccess ||
      cudaEventCreateWithFlags(&h->ev_fork, cudaEventDisableTiming) != cudaSuccess ||
      cudaEventCreateWithFlags(&h->ev_join, cudaEventDisableTiming) != cudaSuccess ||
      cudaEventCreateWithFlags(&h->ev_row, cudaEventDisableTiming) != cudaSuccess) {
    cudaFreeHost(h->host_small);
    delete h;
    return APSP_E_CUDA;
  }
  if (world > 1 && (cudaStreamCreateWithFlags(&h->stc, cudaStreamNonBlocking) != cudaSuccess ||
                    cudaEventCreateWithFlags(&h->ev_pan, cudaEventDisableTiming) != cudaSuccess ||
                    cudaEventCreateWithFlags(&h->ev_bc, cudaEventDisableTiming) != cudaSuccess)) {
    release_handle(h);
    return APSP_E_CUDA;
  }
  if (world > 1) {
    int err = 0;
    h->comm = group ? make_local_comm(group, rank) : make_nccl_comm(nccl_id, world, rank, &err);
    if (!h->comm) {
      release_handle(h);
      return APSP_E_NCCL;
    }
  }
  // WT := W^T (replicated), pads INF; validate W (diag 0, w >= 0)
  apsp_status s = dispatch(dtype, [&](auto z) -> apsp_status {
    using T = decltype(z);
    CKR(cudaMemsetAsync(h->ws + h->plan.off_small, 0, 512, h->st));   // counters, flags
    CKR(cudaMemsetAsync(h->mirror_flag(), 0xff, sizeof(unsigned), h->st));   // no mirror yet
    CKR(cudaMemsetAsync(h->heavy_x(), 0x7f, sizeof(int32_t) * (size_t)kHeavy * h->ld, h->st));   // X: "INF"
    CKR(cudaMemsetAsync(h->slscr(), 0, 256 + sizeof(int) * (size_t)kSLBins, h->st));   // SL(x) selection state
    CK(fill<T>(h->WT<T>(), (int64_t)cap * h->ld, Tr<T>::inf(), h->st));
    CKR(cudaMemsetAsync(&h->ctr()->err, 0, sizeof(unsigned), h->st));
    CKR(cudaMemsetAsync(h->wmin_dev(), 0xff, sizeof(unsigned), h->st));
    CK(transpose_in<T>(reinterpret_cast<const T*>(W), ldw, n, h->WT<T>(), h->ld, &h->ctr()->err,
                       h->wmin_dev(), h->st));
    CK(shortlist_build<T>(h->WT<T>(), h->ld, n, nullptr, 0, n, h->slid(), h->slw<T>(), h->wnext<T>(), h->st));
    if (std::is_same<T, int32_t>::value && h->rows > 0) {   // the int8 detection's tensor map (fixed buffer)
      const int64_t rows_max = world > 1 ? round_up(cdiv(cap, world), kTile) : cap;
      CKR(detect8_tensor_map(h->tmap8, h->ws + h->plan.off_p8, h->ld, rows_max));
      h->tmap8_ok = true;
    }
    unsigned* herr = reinterpret_cast<unsigned*>(h->host_small);
    CKR(cudaMemcpyAsync(herr, &h->ctr()->err, sizeof(unsigned), cudaMemcpyDeviceToHost, h->st));
    CKR(cudaMemcpyAsync(herr + 1, h->wmin_dev(), sizeof(unsigned), cudaMemcpyDeviceToHost, h->st));
    CKR(cudaStreamSynchronize(h->st));
    if (*herr) return fail(h, APSP_E_INVAL, "create: W has %s", (*herr & 4) ? "a nonzero diagonal" : "a negative/NaN weight");
    h->wmin_bits = herr[1];
    CK(add_init(h->add_scratch(), &h->ctr()->err, h->wmin_dev(), h->st));   // the first add's scratch
    return APSP_OK;
  });
  if (s != APSP_OK) {
    release_handle(h);
    return s;
  }
  *out = h;
  return APSP_OK;
}

}  // namespace

extern "C" {

apsp_status apsp_create(apsp_handle** out, apsp_dtype dtype, int directed, int64_t n, int64_t cap,
                        const void* W, int64_t ldw, void* D_local, int64_t ld, void* workspace,
                        size_t workspace_bytes, void* stream, int rank, int world,
                        const void* nccl_id) {
  return create_impl(out, dtype, directed, n, cap, W, ldw, D_local, ld, workspace, workspace_bytes,
                     stream, rank, world, nccl_id, nullptr);
}

apsp_status apsp_local_group_create(int world, void** group) {
  if (!group) return APSP_E_INVAL;
  *group = nullptr;
  if (world < 1 || world > 16) return APSP_E_INVAL;
  LocalGroup* g = local_group_create(world);
  if (!g) return APSP_E_CUDA;
  *group = g;
  return APSP_OK;
}

apsp_status apsp_local_group_destroy(void* group) {
  if (!group) return APSP_E_INVAL;
  local_group_destroy(reinterpret_cast<LocalGroup*>(group));
  return APSP_OK;
}

apsp_status apsp_create_local(apsp_handle** out, apsp_dtype dtype, int directed, int64_t n,
                              int64_t cap, const void* W, int64_t ldw, void* D_local, int64_t ld,
                              void* workspace, size_t workspace_bytes, void* stream, int rank,
                              void* group) {
  if (!group) return APSP_E_INVAL;
  LocalGroup* g = reinterpret_cast<LocalGroup*>(group);
  return create_impl(out, dtype, directed, n, cap, W, ldw, D_local, ld, workspace, workspace_bytes,
                     stream, rank, local_group_world(g), nullptr, g);
}

apsp_status apsp_destroy(apsp_handle* h) {
  if (!h) return APSP_E_INVAL;
  if (h->st) cudaStreamSynchronize(h->st);
  h->prof_resolve();
  release_handle(h);
  return APSP_OK;
}

apsp_status apsp_set_option(apsp_handle* h, apsp_option opt, double value) {
  CHECK_HANDLE(h);
  switch (opt) {
    case APSP_OPT_FORCE_PATH:
      if (value != 0 && value != 1 && value != 2) return APSP_E_INVAL;
      h->force_path = (int)value;
      return APSP_OK;
    case APSP_OPT_THETA:
      if (!(value >= 0)) return APSP_E_INVAL;
      h->theta = value;
      return APSP_OK;
    case APSP_OPT_TAU:
      if (!(value >= 0) || value > 0.1) return APSP_E_INVAL;
      h->tau = (float)value;
      return APSP_OK;
    case APSP_OPT_MAX_ROUNDS:
      if (!(value >= 1)) return APSP_E_INVAL;
      h->max_rounds = (int)value;
      return APSP_OK;
    case APSP_OPT_SEMIRING:
      if (value != 0 && value != 1) return APSP_E_INVAL;
      h->sr = (int)value;
      return APSP_OK;
    case APSP_OPT_FW16:
      if (value != 0 && value != 1) return APSP_E_INVAL;
      h->fw16 = (int)value;
      return APSP_OK;
    case APSP_OPT_MIRROR8:   // takes effect at the next mirror build
      if (value != 0 && value != 1) return APSP_E_INVAL;
      h->mirror8 = (int)value;
      h->mirror8_failed = false;
      if (!value && h->mirror_level == 8) h->mirror_built = false;   // rebuild at int16
      return APSP_OK;
    case APSP_OPT_MIRROR:   // takes effect at the next update (rebuilt, or dropped)
      if (value != 0 && value != 1) return APSP_E_INVAL;
      h->use_mirror = (int)value;
      h->mirror_built = false;
      return APSP_OK;
    case APSP_OPT_FUSED:
      if (value != 0 && value != 1) return APSP_E_INVAL;
      h->fused = (int)value;
      return APSP_OK;
    case APSP_OPT_HEAVY:
      if (!(value >= -1) || value != (double)(int64_t)value || value > 1e9) return APSP_E_INVAL;
      h->heavy_min = (int)value;
      return APSP_OK;
    case APSP_OPT_ROW_DELTA:
      if (!(value >= 0) || value > 1) return APSP_E_INVAL;
      h->row_delta = value;
      return APSP_OK;
  }
  return APSP_E_INVAL;
}

int32_t apsp_mirror_width(const apsp_handle* h) {
  if (!h) return -1;
  if (h->dt != APSP_I32 || h->sr != 0 || !h->mirror_built || !h->mirror_hint) return 0;
  return h->mirror_level;
}

apsp_status apsp_sync_distances(apsp_handle* h) {
  CHECK_HANDLE(h);
  return dispatch(h->dt, [&](auto z) { return mirror_rebuild<decltype(z)>(h); });
}

apsp_status apsp_cold_fw(apsp_handle* h) {
  CHECK_HANDLE(h);
  NvtxRange nvtx_("apsp_cold_fw");
  return dispatch(h->dt, [&](auto z) { return cold_fw_impl<decltype(z)>(h); });
}

apsp_status apsp_add_node(apsp_handle* h, const void* out_w, const void* in_w, int64_t* new_index,
                          apsp_update_info* info) {
  CHECK_HANDLE(h);
  NvtxRange nvtx_("apsp_add_node");
  if (info) std::memset(info, 0, sizeof *info);
  if (!out_w || !in_w) return fail(h, APSP_E_INVAL, "add_node: null edge vector");
  if (h->n >= h->cap) return fail(h, APSP_E_CAPACITY, "add_node: n == cap == %lld", (long long)h->cap);
  return dispatch(h->dt, [&](auto z) { return add_node_impl<decltype(z)>(h, out_w, in_w, new_index, info); });
}

apsp_status apsp_remove_node(apsp_handle* h, int64_t k, int64_t* moved_from, apsp_update_info* info) {
  CHECK_HANDLE(h);
  NvtxRange nvtx_("apsp_remove_node");
  if (info) std::memset(info, 0, sizeof *info);
  if (k < 0 || k >= h->n) return fail(h, APSP_E_RANGE, "remove_node: k=%lld outside [0,%lld)", (long long)k, (long long)h->n);
  if (h->n == 1) return fail(h, APSP_E_PRECOND, "remove_node: cannot remove the last node");
  return dispatch(h->dt, [&](auto z) { return remove_node_impl<decltype(z)>(h, k, moved_from, info); });
}

apsp_status apsp_update_edge(apsp_handle* h, int64_t u, int64_t v, double w_new, apsp_update_info* info) {
  CHECK_HANDLE(h);
  NvtxRange nvtx_("apsp_update_edge");
  if (info) std::memset(info, 0, sizeof *info);
  if (u < 0 || u >= h->n || v < 0 || v >= h->n)
    return fail(h, APSP_E_RANGE, "update_edge: (%lld,%lld) outside [0,%lld)", (long long)u, (long long)v, (long long)h->n);
  if (u == v) return fail(h, APSP_E_INVAL, "update_edge: u == v (the diagonal is fixed at 0)");
  if (std::isnan(w_new) || w_new < 0) return fail(h, APSP_E_INVAL, "update_edge: negative or NaN weight");
  if (h->dt == APSP_I32) {
    if (std::isfinite(w_new) && w_new != std::floor(w_new))
      return fail(h, APSP_E_INVAL, "update_edge: non-integral weight on an int32 handle");
    int32_t w = (w_new >= (double)APSP_INF_I32) ? APSP_INF_I32 : (int32_t)w_new;
    return update_edge_impl<int32_t>(h, u, v, w, info);
  }
  float w = std::isinf(w_new) ? Tr<float>::inf() : (float)w_new;
  return update_edge_impl<float>(h, u, v, w, info);
}

apsp_status apsp_modify_edge_readd(apsp_handle* h, int64_t u, int64_t v, double w_new,
                                   int64_t* removed, apsp_update_info* info) {
  CHECK_HANDLE(h);
  NvtxRange nvtx_("apsp_modify_edge_readd");
  if (info) std::memset(info, 0, sizeof *info);
  if (u < 0 || u >= h->n || v < 0 || v >= h->n)
    return fail(h, APSP_E_RANGE, "modify_edge_readd: (%lld,%lld) outside [0,%lld)", (long long)u, (long long)v, (long long)h->n);
  if (u == v) return fail(h, APSP_E_INVAL, "modify_edge_readd: u == v");
  if (std::isnan(w_new) || w_new < 0) return fail(h, APSP_E_INVAL, "modify_edge_readd: negative or NaN weight");
  if (h->n < 3) return fail(h, APSP_E_PRECOND, "modify_edge_readd: needs n >= 3");
  if (h->dt == APSP_I32) {
    if (std::isfinite(w_new) && w_new != std::floor(w_new))
      return fail(h, APSP_E_INVAL, "modify_edge_readd: non-integral weight on an int32 handle");
    int32_t w = (w_new >= (double)APSP_INF_I32) ? APSP_INF_I32 : (int32_t)w_new;
    return modify_readd_impl<int32_t>(h, u, v, w, removed, info);
  }
  float w = std::isinf(w_new) ? Tr<float>::inf() : (float)w_new;
  return modify_readd_impl<float>(h, u, v, w, removed, info);
}

apsp_status sp_pair_query(apsp_handle* h, int64_t s, int64_t t, void* dist, int32_t* path,
                          int32_t path_cap, int32_t* path_len, int32_t* n_candidates) {
  CHECK_HANDLE(h);
  NvtxRange nvtx_("sp_pair_query");
  if (!dist || !path_len || (path_cap > 0 && !path)) return fail(h, APSP_E_INVAL, "sp_pair_query: null output");
  if (s < 0 || s >= h->n || t < 0 || t >= h->n) return fail(h, APSP_E_RANGE, "sp_pair_query: id out of range");
  return dispatch(h->dt, [&](auto z) {
    return query_one<decltype(z)>(h, s, t, dist, path, path_cap, path_len, n_candidates);
  });
}

apsp_status sp_pair_query_batch(apsp_handle* h, int32_t q, const int32_t* s, const int32_t* t,
                                void* dist, int32_t* paths, int32_t path_cap, int32_t* path_lens,
                                int32_t* n_cand) {
  CHECK_HANDLE(h);
  NvtxRange nvtx_("sp_pair_query_batch");
  if (q < 0 || (q > 0 && (!s || !t || !dist || !path_lens))) return fail(h, APSP_E_INVAL, "query_batch: null argument");
  if (path_cap > 0 && !paths) return fail(h, APSP_E_INVAL, "query_batch: null paths");
  return dispatch(h->dt, [&](auto z) -> apsp_status {
    using T = decltype(z);
    return query_dispatch<T>(h, q, s, t, reinterpret_cast<T*>(dist), paths, path_cap, path_lens, n_cand);
  });
}

apsp_status apsp_get_weight(apsp_handle* h, int64_t u, int64_t v, void* w) {
  CHECK_HANDLE(h);
  if (!w) return fail(h, APSP_E_INVAL, "get_weight: null output");
  if (u < 0 || u >= h->n || v < 0 || v >= h->n) return fail(h, APSP_E_RANGE, "get_weight: id out of range");
  const size_t es = 4;
  CKR(cudaMemcpyAsync(h->host_small, h->ws + h->plan.off_wt + (size_t)(v * h->ld + u) * es, es,
                      cudaMemcpyDeviceToHost, h->st));
  CKR(cudaStreamSynchronize(h->st));
  std::memcpy(w, h->host_small, es);
  return APSP_OK;
}

apsp_status apsp_need_update_list(apsp_handle* h, int32_t kind, int64_t a, int64_t b, int32_t* rows,
                                  int32_t* cols, int64_t cap, int64_t* count) {
  CHECK_HANDLE(h);
  if (!count || cap < 0 || (cap > 0 && (!rows || !cols)) || (kind != 2 && kind != 4))
    return fail(h, APSP_E_INVAL, "need_update_list: bad argument");
  if (a < 0 || a >= h->n || (kind == 2 && (b < 0 || b >= h->n)))
    return fail(h, APSP_E_RANGE, "need_update_list: id out of range");
  if (kind == 2 && a == b) return fail(h, APSP_E_INVAL, "need_update_list: u == v");
  return dispatch(h->dt, [&](auto z) { return need_list_impl<decltype(z)>(h, kind, a, b, rows, cols, cap, count); });
}

int64_t apsp_size(const apsp_handle* h) { return h ? h->n : -1; }

const char* apsp_last_error(const apsp_handle* h) { return h ? h->err.c_str() : "null handle"; }

int64_t apsp_kernel_launches(const apsp_handle* h) { return h ? h->launches : -1; }

apsp_status apsp_microbench(int kind, void* buf, size_t bytes, void* stream, double* rate) {
  if (!rate || kind < 0 || kind > 4) return APSP_E_INVAL;
  const double r = microbench(kind, buf, bytes, reinterpret_cast<cudaStream_t>(stream));
  if (r < 0) return r == -1.0 ? APSP_E_INVAL : APSP_E_CUDA;
  *rate = r;
  return APSP_OK;
}

apsp_status apsp_profile_enable(apsp_handle* h, int on) {
  CHECK_HANDLE(h);
  h->prof_on = on != 0;
  return APSP_OK;
}

apsp_status apsp_profile_reset(apsp_handle* h) {
  CHECK_HANDLE(h);
  CKR(h->prof_resolve());
  for (int c = 0; c < APSP_K_COUNT; ++c) { h->prof_ms[c] = 0; h->prof_cnt[c] = 0; h->prof_work[c] = 0; }
  return APSP_OK;
}

apsp_status apsp_profile_read(apsp_handle* h, int kernel_class, double* ms, int64_t* launches,
                              double* work) {
  CHECK_HANDLE(h);
  if (kernel_class < 0 || kernel_class >= APSP_K_COUNT) return APSP_E_RANGE;
  CKR(h->prof_resolve());
  if (ms) *ms = h->prof_ms[kernel_class];
  if (launches) *launches = h->prof_cnt[kernel_class];
  if (work) *work = h->prof_work[kernel_class];
  return APSP_OK;
}

}  // extern "C"
