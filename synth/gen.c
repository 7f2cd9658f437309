/*
 * synth/gen.c — seeded, counter-based synthetic INPUT generators.
 *
 * This module is shared by the oracle side (tests/, oracle checks) and the
 * product side (bench.py, smoke()).  It holds NONE of the method's arithmetic:
 * no relaxation, no min, no path sums.  It only turns (seed, stream, i, j)
 * into weights / update parameters, following SURVEY.md §8(d-2) and the
 * readings Q18–Q22 recorded in DESIGN.md §3.
 *
 * Every value is a pure function of (seed, stream, a, b):
 *     h = mix64(mix64(mix64(seed ^ stream<<56) ^ a) ^ b)
 * where mix64 is the splitmix64 output finaliser.  Hence generation order and
 * thread count never change a value.
 *
 * Streams: 1 weight, 2 presence, 3 new-node out-edges, 4 new-node in-edges,
 *          5 update type/target, 6 reweight factor, 7 query pairs.
 */
#include <math.h>
#include <stdint.h>

static inline uint64_t mix64(uint64_t z) {
  z += 0x9E3779B97F4A7C15ull;
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}

uint64_t synth_hash(uint64_t seed, uint64_t stream, uint64_t a, uint64_t b) {
  return mix64(mix64(mix64(seed ^ (stream << 56)) ^ a) ^ b);
}

/* U[lo,hi] (inclusive) from the top 32 bits: lo + ((h>>32)*(hi-lo+1))>>32 */
static inline int64_t uni_int(uint64_t h, int64_t lo, int64_t hi) {
  uint64_t span = (uint64_t)(hi - lo + 1);
  return lo + (int64_t)(((h >> 32) * span) >> 32);
}
/* u in [0,1) from 53 bits */
static inline double uni01(uint64_t h) { return (double)(h >> 11) * 0x1.0p-53; }

int64_t synth_uniform_int(uint64_t seed, uint64_t stream, uint64_t a, uint64_t b,
                          int64_t lo, int64_t hi) {
  return uni_int(synth_hash(seed, stream, a, b), lo, hi);
}
double synth_uniform01(uint64_t seed, uint64_t stream, uint64_t a, uint64_t b) {
  return uni01(synth_hash(seed, stream, a, b));
}

/* Weight distributions (Q19/Q20):
 *   kind 0: int U[lo,hi]
 *   kind 1: int round(exp(u * ln(hi/lo)) * lo)  (log-uniform; BJ.c5 uses lo=1, hi=1e6)
 *   kind 2: fp32-exact grid (m+1)*2^-24, m = top 24 bits  (BJ.c2 "uniform (0,1]")
 */
static inline double draw_weight(uint64_t h, int kind, int64_t lo, int64_t hi) {
  if (kind == 0) return (double)uni_int(h, lo, hi);
  if (kind == 1) return round(exp(uni01(h) * log((double)hi / (double)lo)) * (double)lo);
  return (double)((h >> 40) + 1) * 0x1.0p-24;
}

/* Fill a dense n x n weight matrix W (row-major, leading dimension ld) with
 * W[i][j] = w(i->j).  Diagonal 0.  Absent edges get `absent` (the caller's
 * INF sentinel).  Undirected graphs draw each unordered pair once using
 * (min(i,j), max(i,j)) as the counter, so W is exactly symmetric.
 * Presence: edge present iff density >= 1 or u01(stream 2) < density (Q21). */
static void fill(uint64_t seed, int64_t n, int directed, double density, int kind,
                 int64_t lo, int64_t hi, int is_f32, void* W, int64_t ld, double absent) {
#pragma omp parallel for schedule(dynamic, 16)
  for (int64_t i = 0; i < n; ++i) {
    for (int64_t j = 0; j < n; ++j) {
      double w;
      if (i == j) {
        w = 0.0;
      } else {
        uint64_t a = (uint64_t)i, b = (uint64_t)j;
        if (!directed && a > b) { uint64_t t = a; a = b; b = t; }
        int present = density >= 1.0 || uni01(synth_hash(seed, 2, a, b)) < density;
        w = present ? draw_weight(synth_hash(seed, 1, a, b), kind, lo, hi) : absent;
      }
      if (is_f32) ((float*)W)[i * ld + j] = (float)w;
      else ((int32_t*)W)[i * ld + j] = (int32_t)w;
    }
  }
}

void synth_graph_i32(uint64_t seed, int64_t n, int directed, double density, int kind,
                     int64_t lo, int64_t hi, int32_t* W, int64_t ld, int32_t absent) {
  fill(seed, n, directed, density, kind, lo, hi, 0, W, ld, (double)absent);
}
void synth_graph_f32(uint64_t seed, int64_t n, int directed, double density,
                     float* W, int64_t ld, float absent) {
  fill(seed, n, directed, density, 2, 0, 0, 1, W, ld, (double)absent);
}

/* Edge vectors of a node added at update index t (streams 3 = out, 4 = in).
 * out[j] = w(x->j), in[j] = w(j->x) for j < n.  Undirected: in == out (stream 3). */
void synth_node_edges_i32(uint64_t seed, uint64_t t, int64_t n, int directed, int kind,
                          int64_t lo, int64_t hi, int32_t* out_w, int32_t* in_w) {
#pragma omp parallel for schedule(static)
  for (int64_t j = 0; j < n; ++j) {
    out_w[j] = (int32_t)draw_weight(synth_hash(seed, 3, t, (uint64_t)j), kind, lo, hi);
    in_w[j] = directed ? (int32_t)draw_weight(synth_hash(seed, 4, t, (uint64_t)j), kind, lo, hi)
                       : out_w[j];
  }
}
void synth_node_edges_f32(uint64_t seed, uint64_t t, int64_t n, int directed,
                          float* out_w, float* in_w) {
#pragma omp parallel for schedule(static)
  for (int64_t j = 0; j < n; ++j) {
    out_w[j] = (float)draw_weight(synth_hash(seed, 3, t, (uint64_t)j), 2, 0, 0);
    in_w[j] = directed ? (float)draw_weight(synth_hash(seed, 4, t, (uint64_t)j), 2, 0, 0)
                       : out_w[j];
  }
}
