/*
 * apsp_warm.h — C ABI of the B200 warm-start APSP library.
 *
 * Maintains the all-pairs shortest-path matrix D of a dense weighted graph on
 * the GPU and re-computes it after a minor update, after
 *   G. Liu, "Solving the all pairs shortest path problem after minor update of
 *   a large dense graph", arXiv 2412.15122  (PAPER.md; "P:a-b" = its lines).
 *
 * Problem statement: the APSP matrix of the original graph
 * is already known; after adding a node, removing a node or updating an edge,
 * compute the APSP matrix of the new graph.  Weights are non-negative
 * (P:29-35); an absent edge / unreachable pair is "infinity".
 *
 * ----------------------------------------------------------------------------
 * Data model
 *   dtype APSP_I32: int32 weights/distances, infinity = APSP_INF_I32 (2^30-1).
 *         Every finite weight and every finite distance must be < APSP_INF_I32
 *         (so a sum of two stored values never overflows int32).
 *   dtype APSP_F32: float weights/distances, infinity = +INFINITY.
 *   W[i][j] = w(i -> j); W[i][i] = 0.  D[i][i] = 0.
 *   Undirected graphs keep W and D symmetric; edge edits touch both directions.
 *
 * Memory (all caller-owned; the library never allocates or frees device memory)
 *   D_local : this rank's rows of D, row-major, leading dimension `ld`
 *             (elements), rows [row0, row0+rows) of the global matrix, as given
 *             by apsp_layout().  Entries with row or column >= n are unused.
 *   workspace: apsp_workspace_bytes() bytes of device memory, 256-B aligned.
 *             Holds the replicated transposed weight matrix WT (WT[j][i] =
 *             W[i][j]), the affected-pair lists and scratch vectors.
 *   Capacity `cap` bounds n for the handle's lifetime (add_node at n == cap
 *   fails with APSP_E_CAPACITY).
 *
 * Streams and synchronisation
 *   All device work is enqueued on the handle's stream (a cudaStream_t passed
 *   as void*).  Calls that need a host decision synchronise that stream:
 *   add_node (argument validation flag, 4 B), update_edge (the 8-byte read of
 *   W[u][v], D[u][v]), remove_node and edge increases (one read of |A|, Phi,
 *   max|A_i| and the round flag after the sparse recompute was enqueued, plus
 *   one 4-byte flag per further batch of rounds), sp_pair_query (result).
 *   cold_fw and update_edge decreases after the early-exit test are
 *   asynchronous.  One handle per stream; handles are not thread-safe.
 *
 * Errors
 *   Every call returns apsp_status; nothing throws or aborts across the ABI.
 *   Argument errors (E_INVAL, E_RANGE, E_CAPACITY, E_PRECOND) are detected
 *   before any device state is modified: D, WT and n are unchanged.
 *   A CUDA or NCCL failure poisons the handle: that call returns E_CUDA/E_NCCL
 *   and every later call returns E_POISONED.  apsp_last_error() returns a
 *   per-handle message for the most recent failure.
 *
 * Multi-GPU (world > 1): one process per GPU, SPMD — every rank calls every
 * function with identical arguments.  D is row-partitioned (apsp_layout), WT
 * is replicated.  The library exchanges pivot rows / panels with NCCL over
 * NVLink using a communicator built from the 128-byte ncclUniqueId the caller
 * distributes (apsp_nccl_unique_id on rank 0, broadcast by the caller).
 * ----------------------------------------------------------------------------
 */
#ifndef APSP_WARM_H
#define APSP_WARM_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define APSP_INF_I32 0x3FFFFFFF

typedef enum { APSP_I32 = 0, APSP_F32 = 1 } apsp_dtype;

typedef enum {
  APSP_OK = 0,
  APSP_E_INVAL = 1,       /* bad argument value (u == v, negative/NaN weight, ...) */
  APSP_E_RANGE = 2,       /* node id outside [0, n), or an output buffer too small */
  APSP_E_CAPACITY = 3,    /* add_node at n == cap */
  APSP_E_PRECOND = 4,     /* operation undefined in this state (remove at n == 1) */
  APSP_E_CUDA = 5,        /* CUDA runtime error; handle poisoned */
  APSP_E_NCCL = 6,        /* NCCL error; handle poisoned */
  APSP_E_NOMEM = 7,       /* workspace smaller than apsp_workspace_bytes() */
  APSP_E_POISONED = 8,    /* an earlier CUDA/NCCL failure poisoned the handle */
  APSP_E_UNSUPPORTED = 9  /* configuration not supported by this build */
} apsp_status;

/* Tunables (apsp_set_option). */
typedef enum {
  APSP_OPT_FORCE_PATH = 0,  /* 0 auto, 1 sparse (a6), 2 dense (a7) — mirrors S:192 */
  APSP_OPT_THETA = 1,       /* gate: dense iff |A| > theta * n^2 (default 0.02)      */
  APSP_OPT_TAU = 2,         /* fp32 tie tolerance tau (default 1e-5), Q4   */
  APSP_OPT_MAX_ROUNDS = 3,  /* sparse rounds before switching to dense (default 64)  */
  APSP_OPT_ROW_DELTA = 4,   /* > 0: use the paper's own gate instead — dense FW iff
                               Definition 1's cost Phi/(N-1) > delta;
                               0 (default): the pair-level gate of APSP_OPT_THETA    */
  APSP_OPT_SEMIRING = 5,    /* path algebra: 0 (default) shortest path, D = min over
                               paths of the summed weights; 1 minimax / bottleneck
                               path, D = min over paths of the largest weight (PAPER.md
                               §6: "The algorithms can be revised to solve
                               the all pairs minimax path problem").  Every call then
                               uses that algebra; D is NOT converted: set it before
                               apsp_cold_fw (or fill D with the matching matrix).    */
  APSP_OPT_FW16 = 6,        /* 1 (default): blocked FW on int32 shortest-path handles
                               on one GPU runs on a packed int16x2 copy of D (two
                               relaxations per VIADDMNMX.S16x2), exact for every
                               distance < 0x3FFF; if any entry saturates it finishes
                               in int32 — results are identical either way.
                               0: always int32.                                       */
  APSP_OPT_MIRROR8 = 7,     /* 1 (default): on int32 shortest-path handles the two
                               O(n^2) streaming passes (add-node pass 1, detection)
                               read an int8 copy of D while every finite distance is
                               < 0x7F, else an int16 copy while every one is < 0x3FFF,
                               else D itself; results are identical on every path.
                               0: never int8 (int16 / int32 only).                    */
  APSP_OPT_MIRROR = 8,      /* 1 (default): keep the saturated mirror of APSP_OPT_MIRROR8.
                               0: no mirror at all — every O(n^2) pass streams the
                               int32 D itself (4 bytes per entry, SURVEY §8(d-4)'s
                               byte basis); for measuring the 4-byte streams.  Results
                               are identical.  Takes effect at the next update.       */
  APSP_OPT_FUSED = 9,       /* 1: removals and directed edge increases on the int8
                               mirror run detection and the first phase of the sparse
                               recompute in ONE pass, each row of the mirror staged
                               whole in shared memory (n up to ~36K).  0 (default): the
                               separate kernels, measured faster at BJ.c4 (DESIGN.md
                               §11).  Results are identical.                          */
  APSP_OPT_HEAVY = 10       /* Sparse recompute, one GPU: a row with at least this many
                               open pairs skips the frontier rounds and is resolved
                               from the other rows once they are final (at most 32
                               rows per update).  0 (default):
                               max(512, n/8); -1: never.  Results are identical.      */
} apsp_option;

/* Statistics of one update. */
typedef struct {
  int32_t kind;        /* 0 no-op, 1 edge decrease, 2 edge increase, 3 add node, 4 remove node,
                          5 edge modified by remove + re-add (apsp_modify_edge_readd) */
  int32_t early_exit;  /* 1: an O(1) tightness test proved no distance changes */
  int32_t path;        /* 0 none, 1 rank-1 relaxation, 2 sparse recompute, 3 dense FW */
  int32_t rounds;      /* sparse-recompute rounds run (path 2) */
  int64_t affected_pairs;    /* |A|: pairs on the need_update_list */
  int64_t affected_rows;     /* Phi: sources with a non-empty list (Definition 1) */
  int64_t max_row_affected;  /* max_i |A_i| */
  double cost;               /* Definition 1: Phi/(N-1) for removals, Phi/n for increases */
  int64_t n_after;           /* node count after the update */
} apsp_update_info;

typedef struct apsp_handle apsp_handle;

/* Row partition and leading dimension for a handle of capacity `cap` on
 * `world` ranks: ld = round_up(cap, 32); rank r owns global rows
 * [row0, row0 + rows).  Pure host function (no CUDA).  E_INVAL on cap < 1,
 * world < 1 or rank outside [0, world). */
apsp_status apsp_layout(int64_t cap, int world, int rank, int64_t* ld, int64_t* row0,
                        int64_t* rows);

/* Bytes of device workspace a handle needs.  Pure host function. */
size_t apsp_workspace_bytes(apsp_dtype dtype, int64_t cap, int world);

/* Create a handle.
 *   W, ldw   : the full n x n row-major weight matrix (device, read only during
 *              this call; every rank passes the whole W).  Diagonal must be 0,
 *              entries >= 0 (int32: <= APSP_INF_I32, which means absent).
 *              W is transposed into the WT replica held in the workspace.
 *   D_local  : this rank's rows of D (device), leading dimension ld (>= the ld
 *              of apsp_layout).  Not read or written here: call apsp_cold_fw,
 *              or fill it with a known APSP matrix of W (warm start).
 *   stream   : cudaStream_t (may be NULL = legacy default stream).
 *   nccl_id  : 128-byte ncclUniqueId when world > 1, else NULL.
 * Errors: E_INVAL (n < 1, n > cap, bad dtype, world/rank inconsistent,
 * diagonal != 0 or negative weight — checked on device, synchronises),
 * E_NOMEM (workspace too small), E_CUDA, E_NCCL. */
apsp_status apsp_create(apsp_handle** out, apsp_dtype dtype, int directed, int64_t n,
                        int64_t cap, const void* W, int64_t ldw, void* D_local, int64_t ld,
                        void* workspace, size_t workspace_bytes, void* stream, int rank,
                        int world, const void* nccl_id);

/* In-process rank group: the row-sharded path with every rank
 * a host THREAD of one process, all ranks on the calling threads' current
 * device.  Used to exercise the multi-rank code (partition, owner broadcasts,
 * reductions, swap-with-last across ranks) bit-for-bit on fewer GPUs than
 * ranks; production multi-GPU runs use apsp_create with NCCL.  A collective
 * is a host rendezvous of all ranks followed by device-to-device copies (and,
 * for reductions, one kernel) ordered against each rank's stream with CUDA
 * events — no kernel ever waits on another kernel.  The group owns 8 MiB of
 * device scratch (the one device allocation the library makes).
 *   apsp_local_group_create: world in [1, 16]; *group receives the group.
 *   apsp_create_local: as apsp_create with world = the group's size and the
 *     group in place of the NCCL id; every rank's thread calls every API
 *     function with identical arguments (SPMD), concurrently.
 *   apsp_local_group_destroy: after every handle of the group is destroyed.
 * Errors: E_INVAL (bad world / null), E_CUDA (scratch allocation). */
apsp_status apsp_local_group_create(int world, void** group);
apsp_status apsp_local_group_destroy(void* group);
apsp_status apsp_create_local(apsp_handle** out, apsp_dtype dtype, int directed, int64_t n,
                              int64_t cap, const void* W, int64_t ldw, void* D_local, int64_t ld,
                              void* workspace, size_t workspace_bytes, void* stream, int rank,
                              void* group);

apsp_status apsp_destroy(apsp_handle* h);

apsp_status apsp_set_option(apsp_handle* h, apsp_option opt, double value);

/* D was written by the caller (a warm start from a known APSP matrix):
 * re-derive the library's internal image of it (the int8 / int16 mirror the
 * O(n^2) passes read on int32 handles).  Optional — the first
 * update that needs it does it otherwise, inside that update's time.
 * Synchronises the stream once when it tries the int8 width (one 4-byte read
 * of the validity flag), else asynchronous.
 * D must not be modified by the caller after an update call without calling
 * this (or apsp_cold_fw) again. */
apsp_status apsp_sync_distances(apsp_handle* h);

/* Width in bits (8 or 16) of the saturated copy of D the O(n^2) streaming
 * passes read (APSP_OPT_MIRROR8), as last observed by the
 * host (the validity flag is read at each update's host synchronisation);
 * 0 when they read D itself (fp32 / minimax handles, no copy built yet, or the
 * copy was invalidated by a distance at or above its saturation value).
 * Returns -1 for a null handle.  Never blocks. */
int32_t apsp_mirror_width(const apsp_handle* h);

/* Cold start: D := APSP(W) by tiled blocked Floyd–Warshall (the comparator of
 * P:74/P:93/P:224).  Asynchronous. */
apsp_status apsp_cold_fw(apsp_handle* h);

/* Add a node (Theorems theorem2, theo_2_back P:286-304,
 * Corollaries 1-2 P:307-343, Theorem 3).
 *   out_w[t] = w(x -> t), in_w[t] = w(t -> x) for t < n (device arrays of the
 *   handle's dtype; int32 values >= APSP_INF_I32 mean absent).  Undirected:
 *   out_w must equal in_w.
 *   new_index (out, may be NULL) = x = the old n (Q8).
 * O(n^2): one read pass over D for the new row/column, one rank-1 min-plus pass.
 * Errors: E_CAPACITY (n == cap), E_INVAL (negative/NaN weight, undirected
 * asymmetry; detected on device before D is touched). */
apsp_status apsp_add_node(apsp_handle* h, const void* out_w, const void* in_w,
                          int64_t* new_index, apsp_update_info* info);

/* Remove node k: need_update_list by Corollary 3,
 * cost by Definition 1, then a sparse recompute of the listed pairs or the
 * blocked Floyd–Warshall fallback (the paper's delta gate).  Node n-1
 * is then moved into slot k (swap-with-last, Q7): moved_from = n-1,
 * or -1 when k == n-1.  Errors: E_RANGE (k outside [0,n)), E_PRECOND (n == 1). */
apsp_status apsp_remove_node(apsp_handle* h, int64_t k, int64_t* moved_from,
                             apsp_update_info* info);

/* Set w(u -> v) := w_new (undirected: both directions).  w_new >= APSP_INF_I32
 * (int32) or +inf (fp32) deletes the edge; setting an absent edge inserts it.
 * Decrease: exact early exit if w_new >= D[u][v], else a rank-1 min-plus
 * relaxation through the edge.  Increase: exact early exit if the edge is not
 * tight (w_old > D[u][v]), else affected-pair detection (Theorem 4's edge
 * analogue) and recompute as in remove_node.  Errors: E_RANGE, E_INVAL (u == v,
 * negative/NaN w_new, non-integral w_new on an int32 handle). */
apsp_status apsp_update_edge(apsp_handle* h, int64_t u, int64_t v, double w_new,
                             apsp_update_info* info);

/* Edge modification by the paper's own algorithm (alg:APSPmodify):
 * "It firstly remove a node associated with the edge from the graph, then add
 * the node back, with the edge being updated ... it calculates which node is
 * cheaper to remove, then remove the cheaper one."  The removal cost of both
 * endpoints is Definition 1 (Phi/(N-1), need_update_lists counted
 * on the GPU); ties go to the smaller index.  The chosen endpoint
 * is removed (remove_node), re-added with its edge vectors including the
 * edited edge (add_node), and swapped back into its original slot so node
 * ids are stable.  Same result as apsp_update_edge (D is unique); this is the
 * paper-faithful composition, kept for comparison.  info->kind = 5,
 * info->cost = the removed endpoint's cost, *removed = that endpoint (may be
 * NULL).  Errors as apsp_update_edge; E_PRECOND when n < 3. */
apsp_status apsp_modify_edge_readd(apsp_handle* h, int64_t u, int64_t v, double w_new,
                                   int64_t* removed, apsp_update_info* info);

/* Warm single-pair shortest path (alg:sp_apsp): candidate_node_list
 * by Theorem 4 (nodes k with D[s][k] + D[k][t] = D[s][t]), then Dijkstra on
 * the induced small graph, path in original ids.
 *   dist (host, 4 bytes of the handle's dtype) = D[s][t];
 *   path (host, path_cap int32) = s ... t; *path_len = its length
 *   (1 for s == t, 0 if unreachable); *n_candidates (may be NULL) = |C|.
 * E_RANGE: s/t out of range, or path_cap too small (*path_len then holds the
 * needed length).  A candidate set larger than the batch scratch (4096) is
 * answered by a second pass that computes every candidate's predecessor at
 * once (one GPU, shortest path; e.g. the directed unit cycle, whose path
 * has n nodes); only multi-GPU or minimax queries beyond 4096 candidates, or
 * zero-weight ties that leave the large set without a chain, still return
 * E_RANGE.  Synchronises the stream. */
apsp_status sp_pair_query(apsp_handle* h, int64_t s, int64_t t, void* dist, int32_t* path,
                          int32_t path_cap, int32_t* path_len, int32_t* n_candidates);

/* Batched form, all arrays on the device: s[q], t[q] -> dist[q],
 * paths[q*path_cap ...], path_lens[q] (-1: path_cap too small, -2: candidate
 * overflow), n_cand[q] (may be NULL).  Asynchronous.  Ids are validated on the
 * device (an out-of-range pair gets path_len -3).  One GPU, q > 1024: the
 * queries run in groups sorted by t (queries sharing a target share column
 * t's reads); every answer still lands in its own slot. */
apsp_status sp_pair_query_batch(apsp_handle* h, int32_t q, const int32_t* s, const int32_t* t,
                                void* dist, int32_t* paths, int32_t path_cap,
                                int32_t* path_lens, int32_t* n_cand);

/* TEST / DIAGNOSTIC export of the need_update_list of a
 * prospective update, computed by the same snapshot + detection kernels the
 * update runs, WITHOUT applying the update (D, WT and n are unchanged):
 *   kind 4: removal of node a — pairs (i, j), i, j != a, D[i][j] < INF, with
 *           D[i][a] + D[a][j] == D[i][j] (Corollary 3);
 *   kind 2: increase of edge (a, b) — pairs with D[i][a] + w(a,b) + D[b][j] ==
 *           D[i][j] (undirected: or D[i][b] + w + D[a][j] == D[i][j]), w the
 *           current weight (Theorem 4's edge analogue); fp32 uses
 *           the tolerant test of APSP_OPT_TAU (Q4).
 * rows/cols (host, cap entries each) receive the pairs in global ids, in the
 * kernel's flush order (unsorted); *count = |A| (only min(|A|, cap) written).
 * Multi-GPU: each rank returns the pairs of its own rows.  Synchronises.
 * Errors: E_INVAL (bad kind, null output, u == v), E_RANGE (ids). */
apsp_status apsp_need_update_list(apsp_handle* h, int32_t kind, int64_t a, int64_t b, int32_t* rows,
                                  int32_t* cols, int64_t cap, int64_t* count);

/* Current weight w(u -> v) (host, 4 bytes of the handle's dtype; INF if
 * absent).  Synchronises the stream.  E_RANGE for ids outside [0, n). */
apsp_status apsp_get_weight(apsp_handle* h, int64_t u, int64_t v, void* w);

/* Current node count n. */
int64_t apsp_size(const apsp_handle* h);

const char* apsp_last_error(const apsp_handle* h);
const char* apsp_status_string(apsp_status s);

/* Fill out[128] with a fresh ncclUniqueId (call on rank 0 only; E_NCCL if
 * NCCL cannot be loaded). */
apsp_status apsp_nccl_unique_id(void* out128);

/* Counters of the most recent operation's kernels: number of kernel launches
 * the library issued since the handle was created (monotone). */
int64_t apsp_kernel_launches(const apsp_handle* h);

/* ---------------------------------------------------------------------------
 * Measurement hooks (used by bench.py for the live roofline).
 * With profiling enabled the library brackets every kernel launch with CUDA
 * events on the handle's stream and accumulates, per kernel class, the event
 * time, the launch count and the launch's ALGORITHMIC work: bytes the method
 * must move for HBM-bound classes, relaxations for the FW tile
 * class.  apsp_profile_read synchronises the stream. */
typedef enum {
  APSP_K_FW_DIAG = 0,    /* FW closure of the diagonal tile           work: relaxations */
  APSP_K_FW_PANEL = 1,   /* FW row + column panels                    work: relaxations */
  APSP_K_FW_TILE = 2,    /* FW phase-3 min-plus tiles                 work: relaxations */
  APSP_K_ADD_PASS1 = 3,  /* add-node read pass (new row and column)   work: bytes       */
  APSP_K_RANK1 = 4,      /* rank-1 min-plus relaxation pass           work: bytes read  */
  APSP_K_DETECT = 5,     /* affected-pair detection (streaming pass)  work: bytes       */
  APSP_K_SPARSE0 = 6,    /* sparse recompute, phase A                 work: bytes       */
  APSP_K_SPARSE_R = 7,   /* sparse recompute after phase A: A2, B, rounds, heavy rows  work: bytes */
  APSP_K_QUERY = 8,      /* single-pair queries                       work: bytes       */
  APSP_K_OTHER = 9,      /* snapshots, tombstone, swap, small kernels work: bytes       */
  APSP_K_EMIT = 10,      /* detection list: per-row slices, Phi        work: bytes       */
  APSP_K_COUNT = 11
} apsp_kernel_class;

apsp_status apsp_profile_enable(apsp_handle* h, int on);
apsp_status apsp_profile_reset(apsp_handle* h);
apsp_status apsp_profile_read(apsp_handle* h, int kernel_class, double* ms, int64_t* launches,
                              double* work);

/* Roofline denominators measured on the current device:
 *   kind 0: int32 relaxations/s (d = min(d, a + b), one VIADDMNMX each)
 *   kind 1: fp32 relaxations/s (FADD, FADD, FMNMX3 per two)
 *   kind 2: int16x2 relaxations/s (VIADDMNMX.S16x2; reference only)
 *   kind 3: HBM read bytes/s over buf[0, bytes) (device; >= 1 GiB to exceed L2)
 *   kind 4: HBM read+write bytes/s, buf updated in place (contents destroyed)
 * buf: device memory (kinds 0-2 only need 4 bytes, never written).  Best of 5
 * launches after 2 warm-ups, CUDA events on `stream`; synchronises it.
 * Errors: E_INVAL (bad kind, null buf/rate), E_CUDA. */
apsp_status apsp_microbench(int kind, void* buf, size_t bytes, void* stream, double* rate);

#ifdef __cplusplus
}
#endif
#endif /* APSP_WARM_H */
