/*
 * graphgen.c — seeded, counter-based synthetic edge-list generators.
 *
 * This module is INPUT INFRASTRUCTURE shared by the oracle tests, the GPU
 * parity tests and bench.py. It holds none of the method's arithmetic (no
 * degrees, no CSR/CSC, no PageRank, no BFS): it only emits (src, dst) pairs,
 * which both sides consume and cross-check by checksum.
 *
 * Every random decision is a pure function of (seed, counter), so edge i is
 * reproducible in isolation and generation parallelises trivially:
 *   U(seed, ctr) = mix64(mix64(seed) + ctr) >> 11, scaled to [0, 1).
 *
 * RMAT (reading R13): edge i of ef*2^scale, for each of
 * `scale` bit levels (most significant first) draw u = U(seed, i*64 + level):
 *   u < a          -> (src bit, dst bit) = (0, 0)
 *   u < a+b        -> (0, 1)
 *   u < a+b+c      -> (1, 0)
 *   otherwise      -> (1, 1)
 * No noise, no vertex permutation. Self-loops and duplicates are emitted as
 * drawn; removing them is the graph builder's job (flags).
 *
 * Grid (reading R15): R x C lattice, id = r*C + c, 4-neighbour undirected
 * edges; horizontal edge k = r*(C-1)+c, vertical edge k = R*(C-1) + r*C + c;
 * edge k is dropped iff U(seed, k) < p_drop; survivors are emitted in both
 * directions, (a,b) then (b,a), in increasing k.
 *
 * Source selection (reading R14): candidate j is v = floor(U(seed, j) * n);
 * accepted when `eligible[v]` and not already taken, until k accepted.
 */
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

static inline uint64_t mix64(uint64_t z) {
  z += 0x9E3779B97F4A7C15ull;
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}

static inline double unif(uint64_t key, uint64_t ctr) {
  return (double)(mix64(key + ctr) >> 11) * (1.0 / 9007199254740992.0);
}

double gg_uniform(uint64_t seed, uint64_t ctr) { return unif(mix64(seed), ctr); }

/* RMAT edges [first, first+count) of the stream; writes src/dst (int32). */
void gg_rmat(int scale, double a, double b, double c, uint64_t seed, int64_t first,
             int64_t count, int32_t* src, int32_t* dst) {
  const uint64_t key = mix64(seed);
  const double ab = a + b, abc = a + b + c;
#pragma omp parallel for schedule(static)
  for (int64_t j = 0; j < count; ++j) {
    const uint64_t i = (uint64_t)(first + j);
    uint32_t s = 0, d = 0;
    for (int l = 0; l < scale; ++l) {
      const double u = unif(key, i * 64u + (uint64_t)l);
      uint32_t sb, db;
      if (u < a) { sb = 0; db = 0; }
      else if (u < ab) { sb = 0; db = 1; }
      else if (u < abc) { sb = 1; db = 0; }
      else { sb = 1; db = 1; }
      s = (s << 1) | sb;
      d = (d << 1) | db;
    }
    src[j] = (int32_t)s;
    dst[j] = (int32_t)d;
  }
}

/* Number of undirected lattice edges kept; call with src=dst=NULL to count. */
int64_t gg_grid(int32_t rows, int32_t cols, double p_drop, uint64_t seed, int32_t* src,
                int32_t* dst) {
  const uint64_t key = mix64(seed);
  const int64_t nh = (int64_t)rows * (cols > 0 ? cols - 1 : 0);
  const int64_t nv = (int64_t)(rows > 0 ? rows - 1 : 0) * cols;
  int64_t w = 0;
  for (int64_t k = 0; k < nh + nv; ++k) {
    if (unif(key, (uint64_t)k) < p_drop) continue;
    if (src) {
      int32_t x, y;
      if (k < nh) {
        const int64_t r = k / (cols - 1), cc = k % (cols - 1);
        x = (int32_t)(r * cols + cc);
        y = x + 1;
      } else {
        const int64_t q = k - nh;
        const int64_t r = q / cols, cc = q % cols;
        x = (int32_t)(r * cols + cc);
        y = x + cols;
      }
      src[2 * w] = x; dst[2 * w] = y;
      src[2 * w + 1] = y; dst[2 * w + 1] = x;
    }
    ++w;
  }
  return w;
}

/* eligible[v] = 1 iff v is the source of some non-self-loop input pair. */
void gg_has_out_edge(int64_t n, int64_t m, const int32_t* src, const int32_t* dst,
                     uint8_t* eligible) {
  memset(eligible, 0, (size_t)n);
  for (int64_t i = 0; i < m; ++i)
    if (src[i] != dst[i]) eligible[src[i]] = 1;
}

/* Draw k distinct eligible vertices; returns how many were found (k unless
 * fewer than k are eligible or `max_draws` candidates were exhausted). */
int64_t gg_pick_sources(int64_t n, const uint8_t* eligible, int64_t k, uint64_t seed,
                        int64_t max_draws, int32_t* out) {
  const uint64_t key = mix64(seed);
  uint8_t* taken = (uint8_t*)calloc((size_t)(n > 0 ? n : 1), 1);
  int64_t got = 0;
  for (int64_t j = 0; j < max_draws && got < k && n > 0; ++j) {
    int64_t v = (int64_t)(unif(key, (uint64_t)j) * (double)n);
    if (v >= n) v = n - 1;
    if (eligible[v] && !taken[v]) { taken[v] = 1; out[got++] = (int32_t)v; }
  }
  free(taken);
  return got;
}

/* Order-independent checksum of an edge list (sum of mix64 of each pair). */
uint64_t gg_edge_checksum(int64_t m, const int32_t* src, const int32_t* dst) {
  uint64_t h = 0;
#pragma omp parallel for reduction(+ : h) schedule(static)
  for (int64_t i = 0; i < m; ++i)
    h += mix64(((uint64_t)(uint32_t)src[i] << 32) | (uint32_t)dst[i]);
  return h;
}

/* Synthetic edge weights (SSSP inputs, reading R24): the weight of directed edge
 * (u, v), u and v input ids, is 1 + mix64(mix64(seed) + (u << 32 | v)) % 255,
 * an integer in [1, 255]: a pure function of (seed, u, v), so the CUDA library
 * draws the same weights from its own copy of this counter-based generator. */
uint32_t gg_edge_weight(uint64_t seed, int32_t u, int32_t v) {
  return 1u + (uint32_t)(mix64(mix64(seed) + (((uint64_t)(uint32_t)u << 32) | (uint32_t)v)) % 255u);
}

void gg_edge_weights(uint64_t seed, int64_t m, const int32_t* u, const int32_t* v, int32_t* w) {
  for (int64_t i = 0; i < m; ++i) w[i] = (int32_t)gg_edge_weight(seed, u[i], v[i]);
}
