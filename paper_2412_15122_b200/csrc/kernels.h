// kernels.h — host-callable launchers of the sm_100a kernels (internal).
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

namespace apsp {

// Saturated mirror of an int32 D (same element indexing, ld elements per row)
// at one of two widths: int16 (m: v stored as min(v, 0x3FFF), INF as 0x3FFF)
// or int8 (m8: min(v, 0x7F), INF as 0x7F).  It is exact — and the two O(n^2)
// streaming passes (add-node pass 1, detection) read it at a half / a quarter
// of the bytes — while bit 0 of *flag is clear, i.e. while every finite
// distance is below the width's saturation value.  Writers of D keep it in
// step and raise the bit on a finite value at or above it.  At most one of m,
// m8 is set (the host picks the width when it builds the mirror).
struct Mirror {
  uint16_t* m;      // int16 level (nullptr: not this width / no mirror)
  uint8_t* m8;      // int8 level
  unsigned* flag;   // bit 0 clear: the mirror images D exactly
  // k_rank1_p8's launch gate: a launch that raises bit 0 itself first stores
  // its `epoch` (unique per launch, from the host) in *ep, so its own later
  // CTAs still see the pre-launch state (rows left un-relaxed otherwise)
  unsigned* ep = nullptr;
  unsigned epoch = 0;
  // int8 level only: the transposed copy MT[j][li] = m8[li][j] (li = local row),
  // kept in step by every writer of m8, so that a COLUMN of D is a contiguous
  // row of MT (the add-node column reads it).  nullptr: none.
  uint8_t* mt = nullptr;
  int64_t ld = 0;    // row stride of m / m8 (elements)
  int64_t ldt = 0;   // row stride of mt (bytes >= local rows)
};

// Device counters written by the detection kernel.
struct DetectCounters {
  unsigned long long total;   // |A|
  unsigned int rows;          // Phi
  unsigned int maxrow;        // max |A_i|
  unsigned int overflow;      // list capacity exceeded
  unsigned int err;           // validation flag (add_node inputs)
  unsigned long long open_total;   // open pairs after the shortlist certification
  unsigned long long rowbase;      // cursor of the per-row open-list slices
  unsigned long long spill;        // fused detection + phase A: pairs left on the global list
};

// ---------------- fw.cu ----------------  (sr: 0 shortest path, 1 minimax)
template <typename T> cudaError_t fw_diag(T* Dkk, int64_t ld, int kb, int sr, cudaStream_t st);
template <typename T>
cudaError_t fw_row_panel(T* rowK, int64_t ld, int64_t K0, int kb, int64_t ncols, int sr,
                         cudaStream_t st);
template <typename T>
cudaError_t fw_col_panel(T* D, int64_t ld, int64_t m, int64_t K0, int kb, const T* Dkk,
                         int64_t lddk, int skip_ti, int sr, cudaStream_t st);
template <typename T>
cudaError_t fw_rest_pt(T* D, int64_t ld, int64_t m, int64_t ncols, int64_t K0, int kb, const T* P,
                       int64_t ldp, int skip_ti, T* PT, int64_t ldpt, int sr, cudaStream_t st);

// int16x2 blocked FW of an int32 shortest-path D (fw.cu): packed copy P of the
// local rows (two columns per 32-bit word, row stride ld/2 words), values
// saturated at 0x3FFF.  ld = D's leading dimension in int32 elements.
cudaError_t p16_from_d32(const int32_t* D, int64_t ld, int64_t m, int64_t n, uint32_t* P, cudaStream_t st);
// D := P where < 0x3FFF; *flag |= 1 if any of the m x n entries saturated
// (row / column `skip`, a tombstoned node, excluded; -1: none)
cudaError_t p16_to_d32(const uint32_t* P, int64_t ld, int64_t m, int64_t n, int64_t row0, int64_t skip,
                       int32_t* D, unsigned* flag, cudaStream_t st);
cudaError_t p16_diag(uint32_t* Pkk, int64_t ld, int kb, cudaStream_t st);
// PT[k][i] = D[i][K0 + k] in both halves (k < kb, i < m), INF padding to TB x round_up(m, 128)
cudaError_t p16_transpose_rep(const uint32_t* P, int64_t ld, int64_t m, int64_t K0, int kb, uint32_t* PT,
                              int64_t ldpt, cudaStream_t st);
// C[i][j] = min(C[i][j], min_k PT[k][i] + B[k][j]) for i < m, j < n (packed rows)
cudaError_t p16_tile3(uint32_t* C, int64_t ld, const uint32_t* PT, int64_t ldpt, const uint32_t* B, int64_t m,
                      int64_t n, int kdepth, int skip_ti, cudaStream_t st);

// ---------------- stream.cu ----------------
// Row range [lo, hi) is global; D points at global row `row0` (local block).
struct Rows {
  int64_t lo, hi, row0;
};

// validate_vec's optional read for the host: the last block writes host[0] =
// *err, host[1] = *wmin_bits, host[2] = *mflag (mapped host memory); done is
// a device counter left at 0
struct ValidateReadback {
  unsigned* host;
  unsigned* done;
  const unsigned* mflag;
};
template <typename T>
// (inb, in2b, outb): an optional second vector validated in the same launch
cudaError_t validate_vec(const T* in, const T* in2, int64_t n, int64_t npad, T* out,
                         unsigned int* err, unsigned* wmin_bits, cudaStream_t st, const T* inb = nullptr,
                         const T* in2b = nullptr, T* outb = nullptr, unsigned long long* argmin0 = nullptr,
                         unsigned* min1 = nullptr, ValidateReadback rb = ValidateReadback{nullptr, nullptr, nullptr});
template <typename T>
cudaError_t transpose_in(const T* W, int64_t ldw, int64_t n, T* WT, int64_t ldt, unsigned int* err,
                         unsigned* wmin_bits, cudaStream_t st);
template <typename T>
cudaError_t fill(T* p, int64_t count, T v, cudaStream_t st);
template <typename T>
cudaError_t init_d(T* D, int64_t ld, Rows r, int64_t n, const T* WT, int64_t ldw, cudaStream_t st);
template <typename T>
cudaError_t gather_col(const T* D, int64_t ld, Rows r, int64_t col, T add, T* out, int sr,
                       cudaStream_t st);
template <typename T>
cudaError_t gather_col_row(const T* D, int64_t ld, Rows r, int64_t col, T add, T* cout, const T* rsrc,
                           int64_t n, int64_t npad, T* rout, int sr, cudaStream_t st);
template <typename T>
cudaError_t copy_vec(const T* src, int64_t n, int64_t npad, T add, T* out, cudaStream_t st);
template <typename T>
cudaError_t addnode_pass1(const T* D, int64_t ld, Rows r, int64_t n, const T* ow, const T* iw,
                          T* rowpart, T* rowpartM, T* colpart, int64_t part_ld, int* nchunk_out,
                          int* nslab_out, int max_slabs, int sr, Mirror M, const unsigned* uncertain, int packed,
                          cudaStream_t st, int colp = 1, const unsigned* full = nullptr);
// Add-node shortcuts (int8 mirror, one GPU): scratch words, the new row from
// the rows that can attain it, then the new column / skip bound by gathers
struct AddScratch {
  unsigned long long* argmin_out; unsigned* in_min; int* s_count; int* u_count; int* th2; int* fb_count;
  int* rmax; int* rb; unsigned* ufull; unsigned* rfull;
  unsigned long long* work;   // cumulative algorithmic bytes of the column pass (profile)
};
cudaError_t add_init(const AddScratch& a, unsigned* err, unsigned* wmin, cudaStream_t st);
// The new row of an add from the rows that can attain it.  stage 0: all of
// it (one GPU); sharded: stage 1 (this rank's part of the bound, into
// *a.rmax: all-reduce(max) it), stage 2 (S and the partial row over this
// rank's rows of S, into `packed`: all-reduce(min) it as uint64), stage 3
// (the row and the minimiser flags from `packed`)
cudaError_t addrow_s(const AddScratch& a, const int32_t* ow, int64_t n, const uint8_t* m8, int64_t ld, int64_t row0,
                     int64_t rows, int32_t* row, int64_t npad, int* slist, unsigned long long* packed, int* tflag,
                     cudaStream_t st, int stage = 0);
// *a.ufull = 1 when |U| exceeded `limit`: pass 1 + the finish kernel compute col instead
cudaError_t addcol_g(const AddScratch& a, Rows r, const uint8_t* m8, int64_t ld, int64_t n, const int32_t* iw,
                     const int32_t* ow, const int* tflag, int* ulist, int* uaux /* 2 * limit */, int limit,
                     int32_t* col, int32_t* ceff, int32_t* mprime, int* fb_list,
                     int32_t wmin /* <= every edge weight */, cudaStream_t st,
                     const uint8_t* mt = nullptr, int64_t ldt = 0 /* the transposed mirror, if any */);
template <typename T>
cudaError_t addnode_finish(const T* rowpart, const T* rowpartM, int nchunk, const T* colpart,
                           int nslab, int64_t part_ld, Rows r, int64_t n, int64_t npad, T* col,
                           T* ceff, T* row, int gate, Mirror M, unsigned* uncertain,
                           cudaStream_t st, const unsigned* row_full = nullptr,   // see addrow_s
                           const unsigned* col_full = nullptr);                   // see addcol_g
template <typename T>
// twin = 0: the caller knows the int8 mirror is valid (its flag was read since
// the last write that could change it), so only the int8 pass is launched
cudaError_t rank1(T* D, int64_t ld, Rows r, int64_t n, const T* c, const T* rv, const T* c2,
                  const T* rv2, unsigned long long* bytes_read, int sr, Mirror M, cudaStream_t st,
                  int twin = 1);
// (it also resets the add's scratch words — as, *err, *wmin — for the next add)
template <typename T>
cudaError_t addnode_write(T* D, int64_t ld, Rows r, int64_t n, int64_t x, int xlocal,
                          const T* col, const T* row, T* WT, int64_t ldw, const T* ow,
                          const T* iw, Mirror M, cudaStream_t st, const AddScratch& as, unsigned* err,
                          unsigned* wmin);
// mode 0: mark rows with flags (anyrow); 1: append the need_update_list
// (pairs to prow/pcol, rowcnt, ctr->total/overflow; plb unused); 2: reset
// flagged entries to W' in place
template <typename T>
cudaError_t detect(T* D, int64_t ld, Rows r, int64_t n, int64_t skip, const T* c1, const T* r1,
                   const T* c2, const T* r2, float tau, int mode, int* anyrow, int* rowcnt,
                   int* prow, int* pcol, T* plb, int64_t lcap, DetectCounters* ctr, const T* WT,
                   int64_t ldw, int sr, Mirror M, cudaStream_t st,
                   const void* tmap8 = nullptr /* host CUtensorMap of the int8 mirror (detect8_tensor_map) */,
                   bool twin = true /* false: the host knows the int8 mirror is valid, no int32 twin launch */);
// The 2-D tensor map the int8 detection's TMA copies use: the int8 mirror m8
// as a uint32 tensor of `rows` x ld / 4 words (row stride ld bytes), boxes of
// 256 words x the kernel's rows per stage.  out: 128-byte CUtensorMap.
cudaError_t detect8_tensor_map(void* out, const uint8_t* m8, int64_t ld, int64_t rows);
cudaError_t detect_lists(Rows r, const int* rowcnt, int64_t* rowoff, DetectCounters* ctr,
                         cudaStream_t st);
// D[i][j] := W'[i][j] on every listed pair (the dense path without the sparse kernels)
template <typename T>
cudaError_t min_with_w(T* D, int64_t ld, Rows r, int64_t n, const T* WT, int64_t ldw, cudaStream_t st);
template <typename T>
cudaError_t reset_pairs(T* D, int64_t ld, int64_t row0, const T* WT, int64_t ldw, const int* srow,
                        const int* scol, const DetectCounters* ctr, int64_t lcap, cudaStream_t st);
template <typename T>
cudaError_t tombstone(T* D, int64_t ld, Rows r, int64_t n, int64_t k, T* WT, int64_t ldw,
                      cudaStream_t st);
template <typename T>
cudaError_t copy_row(T* dst, const T* src, int64_t n, cudaStream_t st);
// swap-with-last after a removal: node n-1 into slot k of D (local rows r) and
// WT, slot n-1 cleared, the mirror of row / column k re-derived.  row_copy = 0
// when row n-1 lives on another rank (it was exchanged into row k already).
template <typename T>
cudaError_t move_last(T* D, int64_t ld, Rows r, int64_t n, int64_t k, int row_copy, T* WT, int64_t ldw,
                      Mirror M, cudaStream_t st);
template <typename T>
cudaError_t copy_col(T* D, int64_t ld, Rows r, int64_t dst_col, int64_t src_col, cudaStream_t st);
template <typename T>
cudaError_t fill_col(T* D, int64_t ld, Rows r, int64_t col, T v, cudaStream_t st);
template <typename T>
cudaError_t set_edge(T* WT, int64_t ldw, int64_t u, int64_t v, T w, int directed, cudaStream_t st);
cudaError_t count_nonzero(const int* a, int64_t m, unsigned long long* out, cudaStream_t st);
template <typename T>
cudaError_t vec_set_move(T* v, int64_t set_i, T set_v, int64_t dst, int64_t src, cudaStream_t st);
template <typename T>
cudaError_t swap_vecs(T* a, T* b, int64_t n, cudaStream_t st);
template <typename T>
cudaError_t swap_cols(T* D, int64_t ld, Rows r, int64_t p, int64_t q, cudaStream_t st);
template <typename T>
cudaError_t shortlist_swap(int* SLid, T* SLw, T* wnext, int64_t n, int64_t p, int64_t q,
                           cudaStream_t st);

// ---------------- sparse.cu ----------------
constexpr int kSLK = 16;              // shortlist entries per lane
constexpr int kSL = 32 * kSLK;        // shortlist entries per node
constexpr int kSLG = 32;              // shortlist_build_one: partial lists (CTAs) at most
// its scratch: [control 256 B | histogram kSLBins ints | the sort path's lists]
// (control and histogram zero between calls: zeroed at creation, reset by the
// kernels that used them)
constexpr int kSLBins = 4096;
constexpr size_t kSLScratch = 256 + (size_t)kSLBins * 4 + (size_t)kSLG * kSL * 8 + (size_t)kSLG * 4;
template <typename T>
cudaError_t shortlist_build(const T* WT, int64_t ldw, int64_t n, const int* rows, int64_t r0,
                            int64_t r1, int* SLid, T* SLw, T* wnext, cudaStream_t st);
template <typename T>
cudaError_t shortlist_build_one(const T* WT, int64_t ldw, int64_t n, int64_t j, int* SLid, T* SLw,
                                T* wnext, void* scratch /* kSLScratch bytes */, cudaStream_t st);
template <typename T>
cudaError_t shortlist_add_bound(int* SLid, T* SLw, T* wnext, const T* out_w, int64_t n, int64_t x,
                                cudaStream_t st);
// one GPU: an edge update's early exits applied on the device (sparse.cu)
template <typename T>
cudaError_t edge_early(T* WT, int64_t ldw, const T* Du, int* SLid, T* SLw, T* wnext, int64_t u, int64_t v, T w,
                       int directed, float tau, void* host_dev, cudaStream_t st);
template <typename T>
cudaError_t shortlist_set_edge(int* SLid, T* SLw, T* wnext, int64_t u, int64_t v, T w,
                               int directed, cudaStream_t st);
template <typename T>
cudaError_t shortlist_remove(int* SLid, T* SLw, T* wnext, int64_t n, int64_t k, int64_t last,
                             cudaStream_t st);
template <typename T>
cudaError_t sparse_short(T* D, int64_t ld, int64_t row0, const int* SLid, const T* SLw,
                         const T* wnext, const int* prow, const int* pcol, const T* plb,
                         int64_t npairs, unsigned char* out, int classify, int sr, const DetectCounters* dc, cudaStream_t st,
                         Mirror M = Mirror{nullptr, nullptr, nullptr}, int64_t skip = -1);
template <typename T>
cudaError_t sparse_phase_a(T* D, int64_t ld, Rows r, const int* SLid, const T* SLw,
                           const int64_t* rowoff, const int* srow, const int* scol, int64_t npairs,
                           const T* c1, const T* r1, const T* c2, const T* r2, float tau, int* ocnt,
                           int* ocol, int* gprow, int* gpcol, T* glb, unsigned char* gfull, int64_t ocap,
                           DetectCounters* ctr, int sr, Mirror M, cudaStream_t st,
                           int list = 0 /* 0: the need_update_list, 2: the fused kernel's spills */,
                           const uint8_t* r1b = nullptr /* r1 as saturated bytes (update_prep), or null */,
                           int* crow = nullptr, int* ccol = nullptr /* continuation list of the first step (lcap) */);
template <typename T>
cudaError_t sparse_full(T* D, int64_t ld, int64_t row0, const T* WT, int64_t ldw, int64_t n,
                        const int* gprow, const int* gpcol, const T* glb, const unsigned char* gfull,
                        int64_t nopen, int sr, const DetectCounters* dc, cudaStream_t st,
                        Mirror M = Mirror{nullptr, nullptr, nullptr});
// The sparse rounds' buffers: per-round frontier counts chg + k * stride
// (k = round % 4; the total at [cap]), frontier lists fcol[round & 1]; the
// cooperative kernel reports rounds run and the last round's total.
struct RoundBufs {
  int* chg; int64_t stride; int64_t cap;
  int* fcol[2];
  int* rounds_run; int* last_total;
  int* bigq;          // queue of long-frontier pairs (capacity: the open-list size)
  int* bigq_ctr;      // 4 ints: (tail, head) per round parity; zero on entry
  // heavy rows: selected at the start (>= heavy_thr open
  // pairs, at most kHeavy; heavy_thr 0: none), skipped by the rounds, then
  // resolved from the other rows.  heavy[0] = rows selected, heavy[1..kHeavy]
  // their ids, heavy[1 + kHeavy + k] row k's bound B_h (key), heavy[1 + 2
  // kHeavy] the pruned first-hop list's length (all zero on entry); heavy_x =
  // kHeavy rows of ldx keys, 0x7F-filled at creation and reset after each use
  int* heavy; int* heavy_x; int64_t ldx; int heavy_thr;
  int64_t rows, n, skip;   // local rows (one GPU: all), nodes, removed node or -1
  // tail = 1 (one GPU): the recompute's tail in this launch — A2 (the whole
  // shortlists, classifying), B (full scans) and the open rows' minima
  // before the rounds; the counters packed into mapped host memory after
  int tail;
  const int* slid; const void* slw; const void* wnext; unsigned char* gfull;
  void* host; const unsigned* mflag;   // host: mapped memory for the counters (packed at the end), or null
};
constexpr int kHeavy = 32;
// rounds r0 .. r1 - 1 in one cooperative launch (grid barriers between rounds),
// stopping at convergence
template <typename T>
cudaError_t sparse_rounds_coop(T* D, int64_t ld, int64_t row0, const T* WT, int64_t ldw, const int* gprow,
                               const int* gpcol, const T* glb, int64_t nopen, const int64_t* rowoff, const int* ocnt,
                               const int* ocol, const RoundBufs& rb, int r0, int r1, int* any, int sr,
                               const DetectCounters* dc, cudaStream_t st, unsigned* rowkey, T wmin, Mirror M);
template <typename T>
cudaError_t sparse_round(T* D, int64_t ld, int64_t row0, const T* WT, int64_t ldw,
                         const int* gprow, const int* gpcol, const T* glb, int64_t nopen,
                         const int64_t* rowoff, const int* fcnt_in, const int* ftot_in, const int* fcol_in,
                         int* fcnt_out, int* ftot_out, int* fcol_out, int* any, int sr,
                         const DetectCounters* dc, cudaStream_t st, unsigned* rowkey = nullptr, T wmin = T(0),
                         Mirror M = Mirror{nullptr, nullptr, nullptr});
// per-row minimum of the open pairs' current values (after A2 / B), as keys
template <typename T>
cudaError_t open_rowmin(const T* D, int64_t ld, int64_t row0, const int* gprow, const int* gpcol, int64_t nopen,
                        unsigned* rowkey, const DetectCounters* dc, cudaStream_t st);

// ---------------- query.cu ----------------
constexpr int kQueryCap = 4096;    // max |C| per query (min(kQueryCap, cap) per handle)
constexpr int kQueryBatch = 1024;  // queries per scan/solve launch pair
// per-query device scratch, `batch` slots of `qcap` entries each (workspace)
struct QueryScratch {
  int* ids;             // candidate ids
  void* dsv;            // D[s][id], the handle's element type
  void* lab;            // Dijkstra labels (element type)
  int* pred;
  int* path;
  unsigned char* done;
  int* cnt;             // |C| per slot
  int qcap, batch;
  int* sort = nullptr;  // t-grouped batches (one GPU): 4 kQueryGroup ints + sort_temp bytes, or null
  size_t sort_temp = 0;
};
constexpr int kQueryGroup = 1 << 16;   // queries per t-sorted group
size_t query_group_temp_bytes();       // cub temp storage of one group sort
// One query with a candidate set beyond the batch scratch (one GPU, shortest
// path): bits (n bits), pred (n ints), cnt (1 int) scratch; out[0] = path
// length (-2: not found), path (<= cap ids) in out + 1.
template <typename T>
cudaError_t query_big(const T* D, int64_t ld, const T* WT, int64_t ldw, int64_t n, int s, int t, unsigned* bits,
                      int* pred, int* cnt, int* out, int cap, float tau, T wmin, cudaStream_t st);
template <typename T>
cudaError_t query_batch(const T* D, int64_t ld, const T* WT, int64_t ldw, int64_t n, int q,
                        const int* s, const int* t, T* dist, int* paths, int path_cap,
                        int* path_lens, int* ncand, float tau, int sr, cudaStream_t st,
                        const QueryScratch& qs, T wmin, const T* colbuf = nullptr, int64_t R = 0,
                        int64_t row0 = 0, int64_t rows = 0);
// sharded queries: out[b * R + i] = D[row0 + i][t_b] (INF beyond the local rows)
// Gather-free sharded queries (f3): row s of each query to every rank
// (rowsend + all-reduce sum), the local candidate tests (localscan: per query
// hcap + 1 ints, count then ids), the hit lists all-gathered, then every rank
// merges them and solves (solve_sharded) — identical answers on every rank.
template <typename T>
cudaError_t query_rowsend(const T* D, int64_t ld, int64_t row0, int64_t rows, int64_t n, const int* s, int qc,
                          T* rowbuf, int64_t ldr, cudaStream_t st);
template <typename T>
cudaError_t query_localscan(const T* D, int64_t ld, int64_t row0, int64_t rows, int64_t n, const int* s,
                            const int* t, int qc, const T* rowbuf, int64_t ldr, int* hits, int hcap, float tau,
                            int sr, T wmin, cudaStream_t st);
template <typename T>
cudaError_t query_solve_sharded(const T* D, int64_t ld, const T* WT, int64_t ldw, int64_t n, int qc, const int* s,
                                const int* t, T* dist, int* paths, int path_cap, int* path_lens, int* ncand,
                                float tau, int sr, const int* allhits, int world, int hcap, const T* rowbuf,
                                int64_t ldr, const QueryScratch& qs, cudaStream_t st);
template <typename T>
cudaError_t query_colslice(const T* D, int64_t ld, int64_t rows, int64_t R, int64_t n,
                           const int* t, int qc, T* out, cudaStream_t st);

// mirror upkeep (stream.cu): build from D (flag must be 0 before), re-sync
// the listed pairs / one row and one column (-1: none) after D changed there
cudaError_t mirror_build(const int32_t* D, int64_t ld, Rows r, int64_t n, Mirror M, cudaStream_t st);
// int8 mirror from the packed int16 buffer (after a packed FW left sat16(D) there)
cudaError_t mirror8_from_p16(const uint32_t* P, int64_t ld, int64_t m, int64_t n, Mirror M, cudaStream_t st);
// M := sat(D) on the listed pairs: the need_update_list (open == 0, ctr->total
// entries) or the open-pair list (open == 1, ctr->open_total entries)
cudaError_t mirror_pairs(const int32_t* D, int64_t ld, int64_t row0, const int* prow, const int* pcol,
                         const DetectCounters* ctr, int64_t lcap, int open, Mirror M, cudaStream_t st);
cudaError_t mirror_cross(const int32_t* D, int64_t ld, Rows r, int64_t n, int64_t row, int64_t col, Mirror M,
                         cudaStream_t st);
// fp32 handles have no mirror
inline cudaError_t mirror_pairs(const float*, int64_t, int64_t, const int*, const int*, const DetectCounters*,
                                int64_t, int, Mirror, cudaStream_t) { return cudaSuccess; }
inline cudaError_t mirror_cross(const float*, int64_t, Rows, int64_t, int64_t, int64_t, Mirror, cudaStream_t) {
  return cudaSuccess;
}
cudaError_t pack_counters(const DetectCounters* c, const int* any, long long* v, cudaStream_t st);
// small device values to (mapped) host memory in one launch: the pieces are
// packed back to back, 4-byte words, in the order added
struct ReadSet {
  static constexpr int kMax = 8;
  const void* p[kMax];
  int bytes[kMax];
  int k;
  void add(const void* ptr, int nbytes) {
    if (k < kMax) { p[k] = ptr; bytes[k] = nbytes; ++k; }
    else overflow = true;
  }
  bool overflow;
};
cudaError_t readback(const ReadSet& rs, void* dst_dev, cudaStream_t st);
// zero up to 12 int buffers in one launch
struct ZeroSet {
  static constexpr int kMax = 12;
  int* p[kMax];
  int64_t n[kMax];
  int k;
  void add(int* ptr, int64_t count) {
    if (k < kMax) { p[k] = ptr; n[k] = count; ++k; }
    else overflow = true;
  }
  bool overflow;
};
cudaError_t zero_set(const ZeroSet& z, cudaStream_t st);
// zero z, the pivot snapshots cout[i] = sat(D[i][col] + add) (local rows) and
// rout = rsrc (if non-null), and tombstone node `tomb` (>= 0) in WT: one launch
template <typename T>
cudaError_t update_prep(const T* D, int64_t ld, Rows r, int64_t col, T add, T* cout, const T* rsrc, int64_t n,
                        int64_t npad, T* rout, const ZeroSet& z, T* WT, int64_t ldw, int64_t tomb, int sr,
                        cudaStream_t st, uint8_t* rout8 = nullptr /* + min(rsrc, 0x7F) bytes (int32) */);
// the counters pack_counters packs, plus the mirror flag, into mapped host memory
cudaError_t pack_to_host(const DetectCounters* c, const int* any, const unsigned* mflag, void* host_dev,
                         cudaStream_t st, const int* rounds = nullptr /* -> host word 14 */);
double microbench(int kind, void* buf, size_t bytes, cudaStream_t st);   // microbench.cu
int num_sms();
// ---------------- fused.cu ----------------
// Detection + phase A in one pass over the int8 mirror (removal, or a directed
// edge increase: c1 = D[:, u] (+ w), r1 = D[v, :]); rows are staged whole in
// shared memory: fused_stages(n) > 0 iff a row of n bytes fits.
int fused_stages(int64_t n);
// Outputs: rowcnt[i] = |A_i|, ctr->total = |A|, and on (srow, scol, sacc, slb)
// with count ctr->spill the pairs it did not certify with their bound and
// D_old (all pairs, no bounds, if export_only).  defer_apply then writes
// those bounds and appends the pairs to the open lists (rowoff from
// detect_lists).
cudaError_t detect_fix_p8(int32_t* D, int64_t ld, Rows r, int64_t n, int64_t skip, const int32_t* c1,
                          const int32_t* r1, const int* SLid, const int32_t* SLw, Mirror M, int* rowcnt,
                          int* srow, int* scol, int* sacc, int* slb, int64_t lcap, DetectCounters* ctr,
                          int export_only, cudaStream_t st);
cudaError_t defer_apply(int32_t* D, int64_t ld, int64_t row0, const int* srow, const int* scol, const int* sacc,
                        const int* slb, int64_t lcap, int* ocnt, int* ocol, const int64_t* rowoff, int* gprow,
                        int* gpcol, int32_t* glb, unsigned char* gfull, int64_t ocap, DetectCounters* ctr, Mirror M,
                        cudaStream_t st);

}  // namespace apsp
