/*
 * oracle/oracle.c — TEST INFRASTRUCTURE ONLY.
 *
 * Plain, slow, obviously-correct CPU computations of what the hot path must
 * produce: the APSP matrix of a weighted graph, i.e. for every ordered pair
 * the minimum over paths of the summed edge weights (§1,
 * "minimize W(P) = sum w(v_i, v_{i+1})"; the APSP problem P:52).
 *
 * Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline /
 * --impl reference legs may load this library.  It shares no code, header or
 * constant with the CUDA path (paper_2412_15122_b200/).
 *
 * Arithmetic: integers in int64, floating point in fp64 (Q1/Q16).
 * "Infinity" (absent edge / unreachable) is the caller-supplied value `inf`,
 * which must be so large that inf + anything finite stays >= inf without
 * overflow (the Python wrapper uses 2^62 for int64 and IEEE +inf for fp64).
 *
 * Contents (each a textbook routine named by the paper):
 *   oracle_fw_*        Floyd–Warshall, k-i-j triple loop ("[FW] ... O(|V|^3)").
 *   oracle_dijkstra_*  dense array Dijkstra, O(n^2), smaller index wins ties
 *                      ("greedy algorithm ... non-negative edge weights";
 *                      tie rule from SPEC S:161).
 *   oracle_brute_*     exhaustive simple-path enumeration, n <= 9 (the plain
 *                      definition of, used to pin the two above).
 */
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

/* ---------------- Floyd–Warshall ---------------- */
/* D (n x n, row-major) holds W on entry (diag 0, absent = inf); on exit the
 * shortest-path distances.  for k: for i: for j: D[i][j] = min(D[i][j], D[i][k] + D[k][j]).
 * Parallel over i for a fixed k: row k and column k do not change during
 * pivot k (D[k][k] = 0, weights >= 0), so the i-rows are independent. */
void oracle_fw_i64(int64_t n, int64_t* D, int64_t inf) {
  for (int64_t k = 0; k < n; ++k) {
    const int64_t* Dk = D + k * n;
#pragma omp parallel for schedule(static)
    for (int64_t i = 0; i < n; ++i) {
      int64_t dik = D[i * n + k];
      if (dik >= inf) continue;
      int64_t* Di = D + i * n;
      for (int64_t j = 0; j < n; ++j) {
        int64_t cand = dik + Dk[j];
        if (cand < Di[j]) Di[j] = cand;
      }
    }
  }
}

void oracle_fw_f64(int64_t n, double* D) {
  for (int64_t k = 0; k < n; ++k) {
    const double* Dk = D + k * n;
#pragma omp parallel for schedule(static)
    for (int64_t i = 0; i < n; ++i) {
      double dik = D[i * n + k];
      double* Di = D + i * n;
      for (int64_t j = 0; j < n; ++j) {
        double cand = dik + Dk[j];
        if (cand < Di[j]) Di[j] = cand;
      }
    }
  }
}

/* Run only pivots [k0, k1) of the FW loop above (used to time a bounded
 * sample of the cold comparator; same loop body). */
void oracle_fw_i64_pivots(int64_t n, int64_t* D, int64_t inf, int64_t k0, int64_t k1) {
  for (int64_t k = k0; k < k1; ++k) {
    const int64_t* Dk = D + k * n;
#pragma omp parallel for schedule(static)
    for (int64_t i = 0; i < n; ++i) {
      int64_t dik = D[i * n + k];
      if (dik >= inf) continue;
      int64_t* Di = D + i * n;
      for (int64_t j = 0; j < n; ++j) {
        int64_t cand = dik + Dk[j];
        if (cand < Di[j]) Di[j] = cand;
      }
    }
  }
}

/* ---------------- Dijkstra, dense array form ---------------- */
/* Single source s on W (n x n, W[i][j] = w(i->j)).  dist[v] = SPD(s, v);
 * pred[v] = predecessor on the chosen shortest path (-1 for s / unreachable).
 * Each step finalises the unfinalised vertex with the smallest label,
 * smaller index first on ties.  If `stop` >= 0 the search ends once `stop`
 * is finalised (single-pair form, the Experiment III comparator P:238). */
void oracle_dijkstra_i64(int64_t n, const int64_t* W, int64_t inf, int64_t s, int64_t stop,
                         int64_t* dist, int64_t* pred) {
  char* done = (char*)calloc((size_t)n, 1);
  for (int64_t v = 0; v < n; ++v) { dist[v] = inf; pred[v] = -1; }
  dist[s] = 0;
  for (int64_t it = 0; it < n; ++it) {
    int64_t m = -1;
    for (int64_t v = 0; v < n; ++v)
      if (!done[v] && dist[v] < inf && (m < 0 || dist[v] < dist[m])) m = v;
    if (m < 0) break;
    done[m] = 1;
    if (m == stop) break;
    const int64_t* Wm = W + m * n;
    for (int64_t v = 0; v < n; ++v) {
      if (done[v] || Wm[v] >= inf) continue;
      int64_t cand = dist[m] + Wm[v];
      if (cand < dist[v]) { dist[v] = cand; pred[v] = m; }
    }
  }
  free(done);
}

void oracle_dijkstra_f64(int64_t n, const double* W, int64_t s, int64_t stop,
                         double* dist, int64_t* pred) {
  const double inf = __builtin_inf();
  char* done = (char*)calloc((size_t)n, 1);
  for (int64_t v = 0; v < n; ++v) { dist[v] = inf; pred[v] = -1; }
  dist[s] = 0;
  for (int64_t it = 0; it < n; ++it) {
    int64_t m = -1;
    for (int64_t v = 0; v < n; ++v)
      if (!done[v] && dist[v] < inf && (m < 0 || dist[v] < dist[m])) m = v;
    if (m < 0) break;
    done[m] = 1;
    if (m == stop) break;
    const double* Wm = W + m * n;
    for (int64_t v = 0; v < n; ++v) {
      if (done[v] || !(Wm[v] < inf)) continue;
      double cand = dist[m] + Wm[v];
      if (cand < dist[v]) { dist[v] = cand; pred[v] = m; }
    }
  }
  free(done);
}

/* All sources (rows [r0, r1)), parallel over sources. */
void oracle_dijkstra_rows_i64(int64_t n, const int64_t* W, int64_t inf, const int64_t* srcs,
                              int64_t count, int64_t* out /* count x n */) {
#pragma omp parallel for schedule(dynamic, 1)
  for (int64_t q = 0; q < count; ++q) {
    int64_t* pred = (int64_t*)malloc((size_t)n * sizeof(int64_t));
    oracle_dijkstra_i64(n, W, inf, srcs[q], -1, out + q * n, pred);
    free(pred);
  }
}

void oracle_dijkstra_rows_f64(int64_t n, const double* W, const int64_t* srcs, int64_t count,
                              double* out) {
#pragma omp parallel for schedule(dynamic, 1)
  for (int64_t q = 0; q < count; ++q) {
    int64_t* pred = (int64_t*)malloc((size_t)n * sizeof(int64_t));
    oracle_dijkstra_f64(n, W, srcs[q], -1, out + q * n, pred);
    free(pred);
  }
}

/* ---------------- Brute force (definition) ---------------- */
/* Minimum over all simple paths s -> t of the summed weights, by exhaustive
 * depth-first enumeration.  With w >= 0 a shortest walk can always be taken
 * simple, so this is the definition of SPD(s, t).  n <= 12. */
static void brute_rec(int64_t n, const int64_t* W, int64_t inf, int64_t cur, int64_t t,
                      int64_t len, unsigned vis, int64_t* best) {
  if (cur == t) { if (len < *best) *best = len; return; }
  for (int64_t v = 0; v < n; ++v) {
    if (vis & (1u << v)) continue;
    int64_t w = W[cur * n + v];
    if (w >= inf) continue;
    brute_rec(n, W, inf, v, t, len + w, vis | (1u << v), best);
  }
}
int64_t oracle_brute_i64(int64_t n, const int64_t* W, int64_t inf, int64_t s, int64_t t) {
  int64_t best = inf;
  if (n > 12) return -1;
  brute_rec(n, W, inf, s, t, 0, 1u << s, &best);
  return best;
}

static void brute_rec_f(int64_t n, const double* W, int64_t cur, int64_t t, double len,
                        unsigned vis, double* best) {
  if (cur == t) { if (len < *best) *best = len; return; }
  for (int64_t v = 0; v < n; ++v) {
    if (vis & (1u << v)) continue;
    double w = W[cur * n + v];
    if (!(w < __builtin_inf())) continue;
    brute_rec_f(n, W, v, t, len + w, vis | (1u << v), best);
  }
}
double oracle_brute_f64(int64_t n, const double* W, int64_t s, int64_t t) {
  double best = __builtin_inf();
  if (n > 12) return -1;
  brute_rec_f(n, W, s, t, 0.0, 1u << s, &best);
  return best;
}

/* Number of simple paths s -> t (used by tests to certify that a pair has a
 * unique shortest path when checking candidate-set minimality). */
static void count_rec(int64_t n, const int64_t* W, int64_t inf, int64_t cur, int64_t t,
                      int64_t len, int64_t target, unsigned vis, int64_t* cnt) {
  if (cur == t) { if (len == target) ++*cnt; return; }
  for (int64_t v = 0; v < n; ++v) {
    if (vis & (1u << v)) continue;
    int64_t w = W[cur * n + v];
    if (w >= inf) continue;
    count_rec(n, W, inf, v, t, len + w, target, vis | (1u << v), cnt);
  }
}
int64_t oracle_count_shortest_i64(int64_t n, const int64_t* W, int64_t inf, int64_t s, int64_t t,
                                  int64_t target) {
  int64_t cnt = 0;
  if (n > 12) return -1;
  count_rec(n, W, inf, s, t, 0, target, 1u << s, &cnt);
  return cnt;
}

/* Dijkstra from each source in srcs on an int32 matrix W (row stride ld,
 * absent edge = inf32), int64 arithmetic; rows of the APSP matrix out
 * (count x n, int64, unreachable = inf64).  Same algorithm as
 * oracle_dijkstra_i64, reading the int32 input in place (used for sampled
 * checks of full-size configurations). */
void oracle_dijkstra_rows_i32w(int64_t n, const int32_t* W, int64_t ld, int32_t inf32,
                               int64_t inf64, const int64_t* srcs, int64_t count, int64_t* out,
                               int reverse) {
#pragma omp parallel for schedule(dynamic, 1)
  for (int64_t q = 0; q < count; ++q) {
    int64_t* dist = out + q * n;
    char* done = (char*)calloc((size_t)n, 1);
    for (int64_t v = 0; v < n; ++v) dist[v] = inf64;
    dist[srcs[q]] = 0;
    for (int64_t it = 0; it < n; ++it) {
      int64_t m = -1;
      for (int64_t v = 0; v < n; ++v)
        if (!done[v] && dist[v] < inf64 && (m < 0 || dist[v] < dist[m])) m = v;
      if (m < 0) break;
      done[m] = 1;
      for (int64_t v = 0; v < n; ++v) {
        int32_t w = reverse ? W[v * ld + m] : W[m * ld + v];   /* reverse: edges into m */
        if (done[v] || w >= inf32) continue;
        int64_t cand = dist[m] + (int64_t)w;
        if (cand < dist[v]) dist[v] = cand;
      }
    }
    free(done);
  }
}

/* ---------------- minimax (bottleneck) paths, §6 ----------------
 * "The algorithms can be revised to solve the all pairs minimax path problem":
 * the cost of a path is its largest edge weight; MD(s,t) = min over paths of
 * that maximum.  Same textbook loops with (+) replaced by max. */
void oracle_fw_minimax_i64(int64_t n, int64_t* D, int64_t inf) {
  for (int64_t k = 0; k < n; ++k) {
    const int64_t* Dk = D + k * n;
#pragma omp parallel for schedule(static)
    for (int64_t i = 0; i < n; ++i) {
      int64_t dik = D[i * n + k];
      if (dik >= inf) continue;
      int64_t* Di = D + i * n;
      for (int64_t j = 0; j < n; ++j) {
        int64_t cand = dik > Dk[j] ? dik : Dk[j];
        if (cand < Di[j]) Di[j] = cand;
      }
    }
  }
}

void oracle_fw_minimax_f64(int64_t n, double* D) {
  for (int64_t k = 0; k < n; ++k) {
    const double* Dk = D + k * n;
#pragma omp parallel for schedule(static)
    for (int64_t i = 0; i < n; ++i) {
      double dik = D[i * n + k];
      double* Di = D + i * n;
      for (int64_t j = 0; j < n; ++j) {
        double cand = dik > Dk[j] ? dik : Dk[j];
        if (cand < Di[j]) Di[j] = cand;
      }
    }
  }
}

static void brute_mm_rec(int64_t n, const int64_t* W, int64_t inf, int64_t cur, int64_t t,
                         int64_t mx, unsigned vis, int64_t* best) {
  if (cur == t) { if (mx < *best) *best = mx; return; }
  for (int64_t v = 0; v < n; ++v) {
    if (vis & (1u << v)) continue;
    int64_t w = W[cur * n + v];
    if (w >= inf) continue;
    brute_mm_rec(n, W, inf, v, t, mx > w ? mx : w, vis | (1u << v), best);
  }
}
/* min over simple s->t paths of the max edge weight (n <= 12); 0 for s == t */
int64_t oracle_brute_minimax_i64(int64_t n, const int64_t* W, int64_t inf, int64_t s, int64_t t) {
  int64_t best = inf;
  if (n > 12) return -1;
  brute_mm_rec(n, W, inf, s, t, 0, 1u << s, &best);
  return best;
}
