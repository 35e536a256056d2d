/*
 * gi_oracle.c — the CPU ORACLE for the edgeset.apply hot path (PageRank, BFS, CC, SSSP).
 *
 * TEST INFRASTRUCTURE ONLY. Only tests/, __graft_entry__.smoke() and
 * bench.py's cpu_baseline / --impl reference legs may load this library.
 * It shares no code, header, table or constant generator with the CUDA
 * library (paper_1805_00923_b200/csrc, include/gi.h); neither includes the
 * other. It is plain, slow and written to be checked against the paper by eye.
 *
 * What it computes (PAPER.md = P, SPEC.md = S, readings = R):
 *
 *  Graph (or_build)   P:853-858 "edges = load(...)", "vertices =
 *      edges.getVertices()", "OutDegree = edges.getOutDegrees()"; edgeset as
 *      CSR/CSC P:3183 [draft]. V = {0..n-1} with n given explicitly (R4);
 *      self-loops removed and duplicates removed on request (R5); optional
 *      symmetrisation "duplicating the directed edges" P:3183 [draft].
 *      Rows by counting sort, each row sorted with qsort (a library
 *      primitive), repeats dropped inside the sorted row.
 *
 *  PageRank (or_pagerank), fp64, Jacobi, fixed iteration count:
 *      edge update  new_rank[dst] += old_rank[src] / out_degree[src]
 *                                                    P:3242-3244 [draft]
 *      vertex update new_rank = beta_score + damp * new_rank  P:3249 [draft]
 *      beta_score = (1 - damp) / |V|                         P:856 (R1)
 *      r_0 = 1/|V|                                           (R2)
 *      dangling mass D_k = sum_{outdeg(u)=0} r_k[u], redistributed as D_k/n
 *      inside the damped term ("uniform", default) or dropped ("drop",
 *      the paper-literal rule)                                (R3)
 *      r_{k+1}[v] = (1-d)/n + d * ( sum_{(u,v) in E} r_k[u]/outdeg(u) + D_k/n )
 *      fixed MaxIter, no convergence test
 *    Rows are summed in ascending source order (CSC rows sorted), one
 *    destination at a time; the OpenMP loop over destinations does not change
 *    any rounding, so results are bit-identical for every thread count.
 *
 *  BFS (or_bfs_depth): depth(s) = 0, depth(v) = length of the shortest
 *      directed path s ->* v along out-edges, -1 if unreachable; FIFO queue.
 *      Parent vector semantics: parent = -1 initially P:2093-2099; each vertex
 *      inserted once P:1021-1025; parent[source] = source S:509 (R8, R9).
 *
 *      or_bfs_depth_levels: the same depths level by level (OpenMP), for the
 *      billion-edge configs; pinned to or_bfs_depth.
 *
 *  CC (or_cc_labels): label propagation IDs[dst] min= IDs[src] from
 *      IDs[v] = v (P:3440-3472 [punt]) written out as its fixed point
 *      IDs[v] = min{u : u = v or u ->* v} (see the function).
 *
 *  SSSP (or_sssp): the shortest-path distances the paper's frontier
 *      Bellman-Ford reaches, written out with Dijkstra.
 *
 *  Validator (or_validate_bfs): Graph500-style. A parent vector is valid iff
 *      parent[s] = s; parent[v] = -1 <=> depth(v) = -1; otherwise
 *      (parent[v], v) in E (binary search in the CSR row of parent[v]) and
 *      depth(parent[v]) = depth(v) - 1. Several parent vectors are valid; they
 *      are validated, never compared (R8).
 */
#include <stdint.h>
#include <stdlib.h>
#include <math.h>
#include <string.h>
#include <omp.h>

typedef struct {
  int64_t n, m;
  int64_t* csr_off; /* n+1 */
  int32_t* csr_idx; /* m, ascending within each row */
  int64_t* csc_off; /* n+1 */
  int32_t* csc_idx; /* m, ascending within each row */
} or_graph;

void or_graph_free(or_graph* g);

/* OpenMP threads the oracle's parallel loops use (the CPU baseline times it on
 * all host cores and on one); returns the previous setting. */
int or_set_threads(int t) {
  const int prev = omp_get_max_threads();
  if (t > 0) omp_set_num_threads(t);
  return prev;
}

static int cmp_i32(const void* a, const void* b) {
  const int32_t x = *(const int32_t*)a, y = *(const int32_t*)b;
  return x < y ? -1 : (x > y ? 1 : 0);
}

/* Bucket the pairs (key[i], val[i]), i < k, by key into rows of a CSR over n
 * keys (counting sort), then sort every row (qsort, a library primitive) and,
 * with dedup, keep one copy of each repeated value. Returns the number of
 * entries kept, or -3 (out of memory); *off (n+1) and *idx are malloc'd; key
 * and val are freed. The counting sort runs in two passes so that no two
 * threads ever write the same counter: (1) each thread moves its slice of the
 * pairs into NB key ranges ("coarse buckets") at offsets from a prefix over
 * (bucket, thread) counts; (2) each coarse bucket is counting-sorted by key on
 * its own. Rows are independent, so the OpenMP loops change nothing but speed. */
#define OR_NB 256
static int64_t bucket_rows(int64_t n, int64_t k, int32_t* key, int32_t* val, int dedup,
                           int64_t** off_out, int32_t** idx_out) {
  const int64_t width = n / OR_NB + 1; /* keys per coarse bucket */
  const int nt = omp_get_max_threads();
  int64_t* hist = (int64_t*)calloc((size_t)nt * OR_NB + 1, sizeof(int64_t));
  int32_t* ck = (int32_t*)malloc((size_t)(k > 0 ? k : 1) * sizeof(int32_t));
  int32_t* cv = (int32_t*)malloc((size_t)(k > 0 ? k : 1) * sizeof(int32_t));
  int64_t* cnt = (int64_t*)calloc((size_t)n + 1, sizeof(int64_t));
  if (!hist || !ck || !cv || !cnt) { free(hist); free(ck); free(cv); free(cnt); free(key); free(val); return -3; }
  /* pass 1: hist[b * nt + t] = pairs of thread t's slice in bucket b */
#pragma omp parallel num_threads(nt)
  {
    const int t = omp_get_thread_num();
    const int64_t lo = k * t / nt, hi = k * (t + 1) / nt;
    int64_t* h = (int64_t*)calloc(OR_NB, sizeof(int64_t));
    for (int64_t i = lo; i < hi; ++i) h[key[i] / width]++;
    for (int b = 0; b < OR_NB; ++b) hist[(int64_t)b * nt + t] = h[b];
#pragma omp barrier
#pragma omp single
    {
      int64_t run = 0;
      for (int64_t j = 0; j < (int64_t)nt * OR_NB; ++j) {
        const int64_t c = hist[j];
        hist[j] = run;
        run += c;
      }
      hist[(int64_t)nt * OR_NB] = run;
    }
    for (int b = 0; b < OR_NB; ++b) h[b] = hist[(int64_t)b * nt + t];
    for (int64_t i = lo; i < hi; ++i) {
      const int64_t at = h[key[i] / width]++;
      ck[at] = key[i];
      cv[at] = val[i];
    }
    free(h);
  }
  free(key);
  free(val);
  /* row lengths: cnt[x + 1] = pairs with key x (each bucket's keys counted by one thread) */
#pragma omp parallel for schedule(dynamic, 1)
  for (int b = 0; b < OR_NB; ++b)
    for (int64_t i = hist[(int64_t)b * nt]; i < hist[(int64_t)(b + 1) * nt]; ++i) cnt[ck[i] + 1]++;
  for (int64_t x = 0; x < n; ++x) cnt[x + 1] += cnt[x]; /* cnt = row starts */
  int32_t* buf = (int32_t*)malloc((size_t)(k > 0 ? k : 1) * sizeof(int32_t));
  int64_t* pos = (int64_t*)malloc(((size_t)n + 1) * sizeof(int64_t));
  if (!buf || !pos) { free(hist); free(ck); free(cv); free(cnt); free(buf); free(pos); return -3; }
  memcpy(pos, cnt, ((size_t)n + 1) * sizeof(int64_t));
  /* pass 2: scatter each bucket into its rows */
#pragma omp parallel for schedule(dynamic, 1)
  for (int b = 0; b < OR_NB; ++b)
    for (int64_t i = hist[(int64_t)b * nt]; i < hist[(int64_t)(b + 1) * nt]; ++i) buf[pos[ck[i]]++] = cv[i];
  free(hist);
  free(ck);
  free(cv);
  /* sort each row; pos[x] = entries kept in row x */
#pragma omp parallel for schedule(dynamic, 1024)
  for (int64_t x = 0; x < n; ++x) {
    int32_t* row = buf + cnt[x];
    const int64_t len = cnt[x + 1] - cnt[x];
    qsort(row, (size_t)len, sizeof(int32_t), cmp_i32);
    int64_t kept = len;
    if (dedup && len > 1) {
      kept = 1;
      for (int64_t j = 1; j < len; ++j)
        if (row[j] != row[kept - 1]) row[kept++] = row[j];
    }
    pos[x] = kept;
  }
  int64_t* off = (int64_t*)malloc(((size_t)n + 1) * sizeof(int64_t));
  if (!off) { free(cnt); free(pos); free(buf); return -3; }
  off[0] = 0;
  for (int64_t x = 0; x < n; ++x) off[x + 1] = off[x] + pos[x];
  const int64_t m = off[n];
  int32_t* idx = (int32_t*)malloc((size_t)(m > 0 ? m : 1) * sizeof(int32_t));
  if (!idx) { free(cnt); free(pos); free(buf); free(off); return -3; }
#pragma omp parallel for schedule(dynamic, 1024)
  for (int64_t x = 0; x < n; ++x) memcpy(idx + off[x], buf + cnt[x], (size_t)pos[x] * sizeof(int32_t));
  free(cnt);
  free(pos);
  free(buf);
  *off_out = off;
  *idx_out = idx;
  return m;
}

/* Returns m >= 0 and *out, or -1 (bad argument) / -2 (vertex out of range) /
 * -3 (out of memory).
 * E = the input pairs without self-loops (remove_self_loops), plus (v,u) for
 * every (u,v) (symmetrize), without repeats (dedup). CSR: E bucketed by source,
 * each row sorted; CSC: the CSR's pairs bucketed by destination, each row
 * sorted (the transpose). */
int64_t or_build(int64_t n, int64_t m0, const int32_t* src, const int32_t* dst,
                 int remove_self_loops, int dedup, int symmetrize, or_graph** out) {
  *out = NULL;
  if (n < 0 || m0 < 0 || n > 2147483647LL) return -1;
  int bad = 0;
#pragma omp parallel for reduction(| : bad)
  for (int64_t i = 0; i < m0; ++i)
    if (src[i] < 0 || src[i] >= n || dst[i] < 0 || dst[i] >= n) bad = 1;
  if (bad) return -2;
  /* the cleaned pair list (u[i], v[i]) */
  const int64_t cap = symmetrize ? 2 * m0 : m0;
  int32_t* u = (int32_t*)malloc((size_t)(cap > 0 ? cap : 1) * sizeof(int32_t));
  int32_t* v = (int32_t*)malloc((size_t)(cap > 0 ? cap : 1) * sizeof(int32_t));
  if (!u || !v) { free(u); free(v); return -3; }
  int64_t k = 0;
  for (int64_t i = 0; i < m0; ++i) {
    if (remove_self_loops && src[i] == dst[i]) continue;
    u[k] = src[i];
    v[k++] = dst[i];
    if (symmetrize) {
      u[k] = dst[i];
      v[k++] = src[i];
    }
  }
  or_graph* g = (or_graph*)calloc(1, sizeof(or_graph));
  if (!g) { free(u); free(v); return -3; }
  g->n = n;
  const int64_t m = bucket_rows(n, k, u, v, dedup, &g->csr_off, &g->csr_idx); /* frees u, v */
  if (m < 0) { free(g); return m; }
  g->m = m;
  /* CSC: the same m pairs keyed by destination */
  int32_t* row = (int32_t*)malloc((size_t)(m > 0 ? m : 1) * sizeof(int32_t));
  if (!row) { or_graph_free(g); return -3; }
#pragma omp parallel for schedule(dynamic, 1024)
  for (int64_t x = 0; x < n; ++x)
    for (int64_t j = g->csr_off[x]; j < g->csr_off[x + 1]; ++j) row[j] = (int32_t)x;
  int32_t* col = (int32_t*)malloc((size_t)(m > 0 ? m : 1) * sizeof(int32_t));
  if (!col) { free(row); or_graph_free(g); return -3; }
  memcpy(col, g->csr_idx, (size_t)m * sizeof(int32_t));
  const int64_t mt = bucket_rows(n, m, col, row, 0, &g->csc_off, &g->csc_idx); /* frees col, row */
  if (mt != m) { or_graph_free(g); return mt < 0 ? mt : -3; }
  *out = g;
  return m;
}

void or_graph_arrays(const or_graph* g, int64_t* csr_off, int32_t* csr_idx, int64_t* csc_off,
                     int32_t* csc_idx) {
  memcpy(csr_off, g->csr_off, (size_t)(g->n + 1) * sizeof(int64_t));
  memcpy(csc_off, g->csc_off, (size_t)(g->n + 1) * sizeof(int64_t));
  memcpy(csr_idx, g->csr_idx, (size_t)g->m * sizeof(int32_t));
  memcpy(csc_idx, g->csc_idx, (size_t)g->m * sizeof(int32_t));
}

void or_graph_free(or_graph* g) {
  if (!g) return;
  free(g->csr_off);
  free(g->csr_idx);
  free(g->csc_off);
  free(g->csc_idx);
  free(g);
}

/* dangling_rule: 0 = uniform redistribution (R3 default), 1 = drop. */
int or_pagerank(const or_graph* g, int iters, double damp, int dangling_rule, double* rank) {
  const int64_t n = g->n;
  if (iters < 0 || damp < 0.0 || damp > 1.0) return -1;
  if (n == 0) return 0;
  double* r = rank;
  double* nr = (double*)malloc((size_t)n * sizeof(double));
  double* outdeg = (double*)malloc((size_t)n * sizeof(double));
  double* w = (double*)malloc((size_t)n * sizeof(double));
  if (!nr || !outdeg || !w) { free(nr); free(outdeg); free(w); return -3; }
  for (int64_t u = 0; u < n; ++u) outdeg[u] = (double)(g->csr_off[u + 1] - g->csr_off[u]);
  for (int64_t v = 0; v < n; ++v) r[v] = 1.0 / (double)n;
  const double base = (1.0 - damp) / (double)n;
  for (int it = 0; it < iters; ++it) {
    double D = 0.0;
    for (int64_t u = 0; u < n; ++u)
      if (outdeg[u] == 0.0) D += r[u];
    const double spread = dangling_rule == 0 ? D / (double)n : 0.0;
    /* w[u] = r[u] / outdeg[u], the edge weight of every out-edge of u (the
     * same IEEE quotient the edge loop would form per edge, formed once) */
#pragma omp parallel for schedule(static)
    for (int64_t u = 0; u < n; ++u) w[u] = outdeg[u] > 0.0 ? r[u] / outdeg[u] : 0.0;
#pragma omp parallel for schedule(dynamic, 4096)
    for (int64_t v = 0; v < n; ++v) {
      double s = 0.0;
      for (int64_t j = g->csc_off[v]; j < g->csc_off[v + 1]; ++j) {
        const int32_t u = g->csc_idx[j];
        s += w[u];
      }
      nr[v] = base + damp * (s + spread);
    }
    memcpy(r, nr, (size_t)n * sizeof(double));
  }
  free(nr);
  free(outdeg);
  free(w);
  return 0;
}

/* FIFO BFS over out-edges; depth[v] = -1 when unreachable. */
int or_bfs_depth(const or_graph* g, int32_t source, int32_t* depth) {
  const int64_t n = g->n;
  if (source < 0 || source >= n) return -2;
  int32_t* q = (int32_t*)malloc((size_t)n * sizeof(int32_t));
  if (!q) return -3;
  for (int64_t v = 0; v < n; ++v) depth[v] = -1;
  int64_t head = 0, tail = 0;
  depth[source] = 0;
  q[tail++] = source;
  while (head < tail) {
    const int32_t u = q[head++];
    for (int64_t j = g->csr_off[u]; j < g->csr_off[u + 1]; ++j) {
      const int32_t v = g->csr_idx[j];
      if (depth[v] < 0) {
        depth[v] = depth[u] + 1;
        q[tail++] = v;
      }
    }
  }
  free(q);
  return 0;
}

/* The same depths, level by level (level-synchronous, top-down): the
 * frontier F_L = {v : depth(v) = L}; F_{L+1} = the out-neighbours of F_L with
 * no depth yet. Depths are unique, so the order in which a level's vertices
 * are discovered (OpenMP threads racing on a compare-and-swap) changes
 * nothing. For the billion-edge configs, whose FIFO run is minutes per source
 * (BASELINE.md CPU-baseline plan); pinned to or_bfs_depth. */
int or_bfs_depth_levels(const or_graph* g, int32_t source, int32_t* depth) {
  const int64_t n = g->n;
  if (source < 0 || source >= n) return -2;
  int32_t* cur = (int32_t*)malloc((size_t)n * sizeof(int32_t));
  int32_t* nxt = (int32_t*)malloc((size_t)n * sizeof(int32_t));
  if (!cur || !nxt) { free(cur); free(nxt); return -3; }
#pragma omp parallel for schedule(static)
  for (int64_t v = 0; v < n; ++v) depth[v] = -1;
  depth[source] = 0;
  cur[0] = source;
  int64_t ncur = 1;
  for (int32_t level = 0; ncur > 0; ++level) {
    int64_t nnext = 0;
#pragma omp parallel for schedule(dynamic, 64)
    for (int64_t i = 0; i < ncur; ++i) {
      const int32_t u = cur[i];
      for (int64_t j = g->csr_off[u]; j < g->csr_off[u + 1]; ++j) {
        const int32_t v = g->csr_idx[j];
        int32_t unseen = -1;
        if (__atomic_load_n(&depth[v], __ATOMIC_RELAXED) == -1 &&
            __atomic_compare_exchange_n(&depth[v], &unseen, level + 1, 0, __ATOMIC_RELAXED, __ATOMIC_RELAXED)) {
          int64_t at;
#pragma omp atomic capture
          at = nnext++;
          nxt[at] = v;
        }
      }
    }
    int32_t* t = cur;
    cur = nxt;
    nxt = t;
    ncur = nnext;
  }
  free(cur);
  free(nxt);
  return 0;
}

static int has_edge(const or_graph* g, int32_t u, int32_t v) {
  int64_t lo = g->csr_off[u], hi = g->csr_off[u + 1];
  while (lo < hi) {
    const int64_t mid = lo + (hi - lo) / 2;
    if (g->csr_idx[mid] < v) lo = mid + 1;
    else hi = mid;
  }
  return lo < g->csr_off[u + 1] && g->csr_idx[lo] == v;
}

/* Returns 0 if valid; otherwise 1 + the index of the failed rule and sets
 * *bad_vertex:  1 root not self-parent, 2 reachability mismatch,
 * 3 parent out of range, 4 parent edge missing, 5 depth(parent) != depth-1. */
int or_validate_bfs(const or_graph* g, int32_t source, const int32_t* depth,
                    const int32_t* parent, int64_t* bad_vertex) {
  const int64_t n = g->n;
  *bad_vertex = -1;
  if (parent[source] != source) { *bad_vertex = source; return 1; }
  /* every vertex is checked on its own; the smallest failing vertex is reported */
  int64_t first = n;
#pragma omp parallel for schedule(dynamic, 65536) reduction(min : first)
  for (int64_t v = 0; v < n; ++v) {
    if (v == source || v >= first) continue;
    const int32_t p = parent[v];
    int bad = 0;
    if ((p == -1) != (depth[v] == -1)) bad = 1;
    else if (p == -1) bad = 0;
    else if (p < 0 || p >= n) bad = 1;
    else if (!has_edge(g, p, (int32_t)v)) bad = 1;
    else if (depth[p] != depth[v] - 1) bad = 1;
    if (bad && v < first) first = v;
  }
  if (first == n) return 0;
  /* the rule the first failing vertex breaks */
  const int64_t v = first;
  const int32_t p = parent[v];
  *bad_vertex = v;
  if ((p == -1) != (depth[v] == -1)) return 2;
  if (p < 0 || p >= n) return 3;
  if (!has_edge(g, p, (int32_t)v)) return 4;
  return 5;
}

/* Edge count examined by a BFS tree in TEPS terms (R16): sum of outdeg over
 * reached vertices. */
int64_t or_reached_out_edges(const or_graph* g, const int32_t* depth) {
  int64_t s = 0;
#pragma omp parallel for reduction(+ : s)
  for (int64_t v = 0; v < g->n; ++v)
    if (depth[v] >= 0) s += g->csr_off[v + 1] - g->csr_off[v];
  return s;
}

/* PageRankDelta (NEXT #1 of SURVEY §8(f)), fp64, following the GraphIt program
 * P:849-893 (with Alg. PageRankDelta):
 *   Rank = 0, DeltaSum = 0, Delta = 1/V, Frontier = V
 *   for round 1..MaxIter:
 *     DeltaSum[dst] += Delta[src] / OutDegree[src] for every edge (src, dst)
 *       with src in Frontier                        edges.from(frontier) P:862-864
 *     round 1: Delta = d*DeltaSum + (1-d)/V; Rank += Delta; Delta -= 1/V
 *       (the program's order, P:865-868 and Ligra's P:3018-3021 [punt]; the
 *       pseudocode P:440-446 subtracts before adding — reading R17)
 *     later:   Delta = DeltaSum * d; Rank += Delta
 *     DeltaSum = 0; v joins the next frontier iff |Delta[v]| > eps * Rank[v]
 *       (P:869's garbled fabs(Delta[v] > eps*Rank[v]) read as P:874 — R18)
 *   updateVertex runs on every vertex every round (vertices.filter), so a
 *   vertex outside the frontier still takes the deltas it receives.
 * frontier_sizes[k] (optional) = |Frontier| entering round k+1. */
int or_pagerank_delta(const or_graph* g, int iters, double damp, double eps, double* rank,
                      int64_t* frontier_sizes) {
  const int64_t n = g->n;
  if (iters < 0 || damp < 0.0 || damp > 1.0 || eps < 0.0) return -1;
  if (n == 0) return 0;
  double* delta = (double*)malloc((size_t)n * sizeof(double));
  double* dsum = (double*)calloc((size_t)n, sizeof(double));
  unsigned char* inF = (unsigned char*)malloc((size_t)n);
  if (!delta || !dsum || !inF) { free(delta); free(dsum); free(inF); return -3; }
  const double invV = 1.0 / (double)n, base = (1.0 - damp) / (double)n;
  for (int64_t v = 0; v < n; ++v) { rank[v] = 0.0; delta[v] = invV; inF[v] = 1; }
  for (int round = 1; round <= iters; ++round) {
    int64_t fs = 0;
    for (int64_t v = 0; v < n; ++v) fs += inF[v];
    if (frontier_sizes) frontier_sizes[round - 1] = fs;
    /* edge pass, pull form over CSC rows (ascending sources): same sums as the push loop */
#pragma omp parallel for schedule(dynamic, 4096)
    for (int64_t v = 0; v < n; ++v) {
      double s = 0.0;
      for (int64_t j = g->csc_off[v]; j < g->csc_off[v + 1]; ++j) {
        const int32_t u = g->csc_idx[j];
        if (inF[u]) s += delta[u] / (double)(g->csr_off[u + 1] - g->csr_off[u]);
      }
      dsum[v] = s;
    }
    for (int64_t v = 0; v < n; ++v) {
      if (round == 1) {
        delta[v] = damp * dsum[v] + base;
        rank[v] += delta[v];
        delta[v] = delta[v] - invV;
      } else {
        delta[v] = dsum[v] * damp;
        rank[v] += delta[v];
      }
      dsum[v] = 0.0;
      inF[v] = fabs(delta[v]) > eps * rank[v];
    }
  }
  free(delta);
  free(dsum);
  free(inF);
  return 0;
}

/* Connected components by label propagation (or_cc_labels).
 * The paper's CC: IDs[v] = v (init), then rounds of
 *   frontier = edges.from(frontier).apply(updateEdge).modified(IDs)
 * with updateEdge: IDs[dst] min= IDs[src]      P:3440-3472 [punt]
 * ("synchronous label propagation" P:2237; "initially operates on the whole
 * graph and in subsequent iterations only ... the vertices whose data changed"
 * P:2249 [punt]), until the frontier is empty. Every round only lowers labels
 * and a lowered label is pushed on, so the rounds stop exactly at the fixed
 * point
 *   IDs[v] = min { u : u = v or there is a directed path u ->* v }
 * (on a symmetric graph: the smallest vertex of v's connected component).
 * That plain definition is what this function writes out: for u = 0..n-1 in
 * increasing order, every vertex reachable from u along out-edges that has no
 * label yet gets label u (a vertex labelled earlier by some u' < u has all it
 * reaches labelled too, so the walk stops there). Labels are vertex ids. */
int or_cc_labels(const or_graph* g, int32_t* label) {
  const int64_t n = g->n;
  int32_t* q = (int32_t*)malloc((size_t)(n > 0 ? n : 1) * sizeof(int32_t));
  if (!q) return -3;
  for (int64_t v = 0; v < n; ++v) label[v] = -1;
  for (int64_t u = 0; u < n; ++u) {
    if (label[u] >= 0) continue;
    int64_t head = 0, tail = 0;
    label[u] = (int32_t)u;
    q[tail++] = (int32_t)u;
    while (head < tail) {
      const int32_t x = q[head++];
      for (int64_t j = g->csr_off[x]; j < g->csr_off[x + 1]; ++j) {
        const int32_t y = g->csr_idx[j];
        if (label[y] < 0) {
          label[y] = (int32_t)u;
          q[tail++] = y;
        }
      }
    }
  }
  free(q);
  return 0;
}

/* Single-source shortest paths (or_sssp). The paper's SSSP is a frontier-based
 * Bellman-Ford ("an active set-based version of Bellman-Ford"
 * P:2246-2247 [punt]): dist[s] = 0, frontier = {s}, rounds of
 *   frontier = edges.from(frontier).apply(dist[dst] min= dist[src] + w).modified(dist)
 * until empty. With non-negative weights it stops at the shortest-path
 * distances, which is what this function writes out: Dijkstra's algorithm with
 * a binary heap (a textbook routine) over out-edges. w[j] is the weight of CSR
 * edge j (int32 >= 0); dist[v] = -1 when v is unreachable. int64 sums. */
typedef struct {
  int64_t d;
  int32_t v;
} or_heap_item;

static void heap_push(or_heap_item* h, int64_t* size, int64_t d, int32_t v) {
  int64_t i = (*size)++;
  while (i > 0) {
    const int64_t p = (i - 1) / 2;
    if (h[p].d <= d) break;
    h[i] = h[p];
    i = p;
  }
  h[i].d = d;
  h[i].v = v;
}

static or_heap_item heap_pop(or_heap_item* h, int64_t* size) {
  const or_heap_item top = h[0];
  const or_heap_item last = h[--(*size)];
  int64_t i = 0;
  for (;;) {
    int64_t c = 2 * i + 1;
    if (c >= *size) break;
    if (c + 1 < *size && h[c + 1].d < h[c].d) ++c;
    if (last.d <= h[c].d) break;
    h[i] = h[c];
    i = c;
  }
  if (*size > 0) h[i] = last;
  return top;
}

int or_sssp(const or_graph* g, int32_t source, const int32_t* w, int64_t* dist) {
  const int64_t n = g->n;
  if (source < 0 || source >= n) return -2;
  or_heap_item* h = (or_heap_item*)malloc((size_t)(g->m + 1) * sizeof(or_heap_item));
  if (!h) return -3;
  for (int64_t v = 0; v < n; ++v) dist[v] = -1;
  int64_t size = 0;
  dist[source] = 0;
  heap_push(h, &size, 0, source);
  while (size > 0) {
    const or_heap_item it = heap_pop(h, &size);
    if (it.d != dist[it.v]) continue; /* stale entry */
    for (int64_t j = g->csr_off[it.v]; j < g->csr_off[it.v + 1]; ++j) {
      const int32_t y = g->csr_idx[j];
      const int64_t nd = it.d + w[j];
      if (dist[y] < 0 || nd < dist[y]) {
        dist[y] = nd;
        heap_push(h, &size, nd, y);
      }
    }
  }
  free(h);
  return 0;
}
