/*
 * graphgen.c -- seeded synthetic graph generators (input harness only).
 *
 * This module produces the CSR inputs that BOTH the oracle (oracle/) and the
 * CUDA path (paper_2008_11321_b200/) consume.  It contains none of the
 * method's arithmetic (no ADG, no priorities, no coloring): only random
 * sampling and CSR construction.  Its random numbers come from its own
 * counter-based generator (gg_mix below); the splitmix64 tie-break hash of
 * the method is implemented separately, and independently, on each side.
 *
 * The recipes follow BASELINE.json "configs" and SURVEY.md §8(d):
 *   ER G(n,m)       : uniform unordered pairs u != v, distinct, until m edges
 *   R-MAT           : per level one 32-bit draw vs floor(p * 2^32) thresholds,
 *                     no per-level noise, ids relabelled by a Fisher-Yates pi
 *   road-like grid  : W x W grid, each axis edge kept w.p. p_keep, each unit
 *                     square gets one diagonal w.p. p_diag (main/anti by one
 *                     more bit), ids relabelled by pi
 *   Chung-Lu        : w_i = min(wmax, c * ((i+1/2)/n)^(-1/(gamma-1))), c by
 *                     bisection so mean(w) = mean_deg; M = mean_deg/2 * n
 *                     endpoint pairs drawn with an alias table; ids -> pi
 * Every graph is symmetrised, self-loops dropped, duplicates removed, rows
 * sorted ascending, isolated vertices kept.
 *
 * Parallelism: OpenMP; every sample is a pure function of (seed, stream,
 * index), so the output does not depend on the thread count.
 */
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#include <math.h>
#include <omp.h>

#define GG_EXPORT __attribute__((visibility("default")))

/* ---- counter-based RNG (generator-private) ------------------------------ */
static inline uint64_t gg_mix(uint64_t x) {
  uint64_t z = x + 0x9E3779B97F4A7C15ULL;
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ULL;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBULL;
  return z ^ (z >> 31);
}
static inline uint64_t gg_key(uint64_t seed, uint64_t stream) {
  return gg_mix(seed ^ (stream * 0xD6E8FEB86659FD93ULL));
}
static inline uint64_t gg_rand(uint64_t key, uint64_t i) { return gg_mix(key ^ gg_mix(i)); }
/* uniform integer in [0, bound) from a 64-bit draw (multiply-high) */
static inline uint64_t gg_below(uint64_t r, uint64_t bound) {
  return (uint64_t)(((unsigned __int128)r * bound) >> 64);
}
static inline uint32_t gg_thresh32(double p) {
  if (p <= 0.0) return 0;
  if (p >= 1.0) return 0xFFFFFFFFu;
  return (uint32_t)(p * 4294967296.0);
}

enum { S_ER = 1, S_RMAT = 2, S_PERM = 3, S_GRID_H = 4, S_GRID_V = 5, S_GRID_D = 6,
       S_CL = 7 };

/* ---- result handle ------------------------------------------------------ */
typedef struct gg_graph {
  int64_t n, nnz;
  int64_t* off;   /* n+1 */
  int32_t* col;   /* nnz */
} gg_graph;

GG_EXPORT void gg_free(gg_graph* g) {
  if (!g) return;
  free(g->off);
  free(g->col);
  free(g);
}
GG_EXPORT int64_t gg_n(const gg_graph* g) { return g->n; }
GG_EXPORT int64_t gg_nnz(const gg_graph* g) { return g->nnz; }
/* copy into caller-owned arrays (parallel memcpy) */
GG_EXPORT void gg_take(const gg_graph* g, int64_t* off_dst, int32_t* col_dst) {
  memcpy(off_dst, g->off, sizeof(int64_t) * (size_t)(g->n + 1));
  int64_t nnz = g->nnz;
  int nt = omp_get_max_threads();
#pragma omp parallel for schedule(static)
  for (int t = 0; t < nt; ++t) {
    int64_t a = nnz * t / nt, b = nnz * (t + 1) / nt;
    if (b > a) memcpy(col_dst + a, g->col + a, sizeof(int32_t) * (size_t)(b - a));
  }
}

/* ---- CSR construction from an arc-pair list ------------------------------
 * Takes M unordered pairs (u[i], v[i]); pairs with u<0 are skipped, self-loops
 * dropped.  Emits the symmetric, deduplicated, row-sorted CSR. */
static int cmp_i32(const void* a, const void* b) {
  int32_t x = *(const int32_t*)a, y = *(const int32_t*)b;
  return (x > y) - (x < y);
}
static void sort_row(int32_t* a, int64_t len) {
  if (len < 48) {
    for (int64_t i = 1; i < len; ++i) {
      int32_t x = a[i];
      int64_t j = i - 1;
      while (j >= 0 && a[j] > x) { a[j + 1] = a[j]; --j; }
      a[j + 1] = x;
    }
  } else {
    qsort(a, (size_t)len, sizeof(int32_t), cmp_i32);
  }
}

static gg_graph* build_csr(int64_t n, int64_t M, const int32_t* u, const int32_t* v) {
  gg_graph* g = (gg_graph*)calloc(1, sizeof(gg_graph));
  g->n = n;
  int64_t* cnt = (int64_t*)calloc((size_t)n + 1, sizeof(int64_t));
#pragma omp parallel for schedule(static)
  for (int64_t i = 0; i < M; ++i) {
    int32_t a = u[i], b = v[i];
    if (a < 0 || a == b) continue;
#pragma omp atomic
    cnt[a + 1]++;
#pragma omp atomic
    cnt[b + 1]++;
  }
  for (int64_t i = 0; i < n; ++i) cnt[i + 1] += cnt[i];
  int64_t raw = cnt[n];
  int32_t* tmp = (int32_t*)malloc(sizeof(int32_t) * (size_t)(raw > 0 ? raw : 1));
  int64_t* cur = (int64_t*)malloc(sizeof(int64_t) * (size_t)(n > 0 ? n : 1));
  memcpy(cur, cnt, sizeof(int64_t) * (size_t)n);
#pragma omp parallel for schedule(static)
  for (int64_t i = 0; i < M; ++i) {
    int32_t a = u[i], b = v[i];
    if (a < 0 || a == b) continue;
    int64_t pa, pb;
#pragma omp atomic capture
    pa = cur[a]++;
#pragma omp atomic capture
    pb = cur[b]++;
    tmp[pa] = b;
    tmp[pb] = a;
  }
  free(cur);
  int64_t* deg = (int64_t*)calloc((size_t)n + 1, sizeof(int64_t));
#pragma omp parallel for schedule(dynamic, 4096)
  for (int64_t r = 0; r < n; ++r) {
    int32_t* a = tmp + cnt[r];
    int64_t len = cnt[r + 1] - cnt[r];
    sort_row(a, len);
    int64_t k = 0;
    for (int64_t i = 0; i < len; ++i)
      if (k == 0 || a[i] != a[k - 1]) a[k++] = a[i];
    deg[r + 1] = k;
  }
  for (int64_t i = 0; i < n; ++i) deg[i + 1] += deg[i];
  g->nnz = deg[n];
  g->off = deg;
  g->col = (int32_t*)malloc(sizeof(int32_t) * (size_t)(g->nnz > 0 ? g->nnz : 1));
#pragma omp parallel for schedule(dynamic, 4096)
  for (int64_t r = 0; r < n; ++r)
    memcpy(g->col + deg[r], tmp + cnt[r], sizeof(int32_t) * (size_t)(deg[r + 1] - deg[r]));
  free(tmp);
  free(cnt);
  return g;
}

/* Fisher-Yates permutation pi of [0,n) driven by stream S_PERM. */
static int32_t* make_perm(int64_t n, uint64_t seed) {
  int32_t* p = (int32_t*)malloc(sizeof(int32_t) * (size_t)(n > 0 ? n : 1));
  for (int64_t i = 0; i < n; ++i) p[i] = (int32_t)i;
  uint64_t key = gg_key(seed, S_PERM);
  for (int64_t i = n - 1; i >= 1; --i) {
    int64_t j = (int64_t)gg_below(gg_rand(key, (uint64_t)i), (uint64_t)i + 1);
    int32_t t = p[i]; p[i] = p[j]; p[j] = t;
  }
  return p;
}

/* ---- public generators -------------------------------------------------- */

/* Arbitrary edge list (for tests): symmetrise / dedup / drop loops. */
GG_EXPORT gg_graph* gg_from_edges(int64_t n, int64_t M, const int32_t* u, const int32_t* v) {
  return build_csr(n, M, u, v);
}

/* Erdos-Renyi G(n, m): uniform distinct unordered pairs, u != v. */
GG_EXPORT gg_graph* gg_er(int64_t n, int64_t m, uint64_t seed) {
  if (n < 2) return build_csr(n, 0, NULL, NULL);
  int64_t maxm = n * (n - 1) / 2;
  if (m > maxm) m = maxm;
  /* open-addressing set of canonical pairs */
  uint64_t cap = 1;
  while (cap < (uint64_t)(4 * m + 16)) cap <<= 1;
  uint64_t* set = (uint64_t*)malloc(sizeof(uint64_t) * cap);
  memset(set, 0xFF, sizeof(uint64_t) * cap);
  int32_t* eu = (int32_t*)malloc(sizeof(int32_t) * (size_t)(m > 0 ? m : 1));
  int32_t* ev = (int32_t*)malloc(sizeof(int32_t) * (size_t)(m > 0 ? m : 1));
  uint64_t key = gg_key(seed, S_ER);
  int64_t got = 0;
  for (uint64_t i = 0; got < m; ++i) {
    uint64_t r = gg_rand(key, i);
    uint64_t a = ((r & 0xFFFFFFFFULL) * (uint64_t)n) >> 32;
    uint64_t b = ((r >> 32) * (uint64_t)n) >> 32;
    if (a == b) continue;
    if (a > b) { uint64_t t = a; a = b; b = t; }
    uint64_t k = a * (uint64_t)n + b;
    uint64_t h = gg_mix(k) & (cap - 1);
    int dup = 0;
    while (set[h] != ~0ULL) {
      if (set[h] == k) { dup = 1; break; }
      h = (h + 1) & (cap - 1);
    }
    if (dup) continue;
    set[h] = k;
    eu[got] = (int32_t)a;
    ev[got] = (int32_t)b;
    ++got;
  }
  free(set);
  gg_graph* g = build_csr(n, m, eu, ev);
  free(eu);
  free(ev);
  return g;
}

/* R-MAT (Kronecker) graph: 2^scale vertices, edge_factor * 2^scale samples. */
GG_EXPORT gg_graph* gg_rmat(int scale, int64_t edge_factor, double a, double b, double c,
                            uint64_t seed) {
  int64_t n = (int64_t)1 << scale;
  int64_t M = edge_factor * n;
  uint32_t tA = gg_thresh32(a), tAB = gg_thresh32(a + b), tABC = gg_thresh32(a + b + c);
  int32_t* pi = make_perm(n, seed);
  int32_t* eu = (int32_t*)malloc(sizeof(int32_t) * (size_t)M);
  int32_t* ev = (int32_t*)malloc(sizeof(int32_t) * (size_t)M);
  uint64_t key = gg_key(seed, S_RMAT);
  int64_t draws = (scale + 1) / 2;
#pragma omp parallel for schedule(static)
  for (int64_t i = 0; i < M; ++i) {
    uint64_t row = 0, colv = 0;
    for (int64_t d = 0; d < draws; ++d) {
      uint64_t r = gg_rand(key, (uint64_t)i * (uint64_t)draws + (uint64_t)d);
      for (int half = 0; half < 2; ++half) {
        int level = (int)(2 * d + half);
        if (level >= scale) break;
        uint32_t w = half ? (uint32_t)(r >> 32) : (uint32_t)r;
        uint64_t rb, cb;
        if (w < tA) { rb = 0; cb = 0; }
        else if (w < tAB) { rb = 0; cb = 1; }
        else if (w < tABC) { rb = 1; cb = 0; }
        else { rb = 1; cb = 1; }
        row = (row << 1) | rb;
        colv = (colv << 1) | cb;
      }
    }
    eu[i] = pi[row];
    ev[i] = pi[colv];
  }
  free(pi);
  gg_graph* g = build_csr(n, M, eu, ev);
  free(eu);
  free(ev);
  return g;
}

/* Road-like planar graph on a W x W grid. */
GG_EXPORT gg_graph* gg_grid(int64_t W, double p_keep, double p_diag, uint64_t seed) {
  int64_t n = W * W;
  int32_t* pi = make_perm(n, seed);
  int64_t nh = W * (W - 1), nv = (W - 1) * W, nd = (W - 1) * (W - 1);
  int64_t M = nh + nv + nd;
  int32_t* eu = (int32_t*)malloc(sizeof(int32_t) * (size_t)(M > 0 ? M : 1));
  int32_t* ev = (int32_t*)malloc(sizeof(int32_t) * (size_t)(M > 0 ? M : 1));
  uint32_t tk = gg_thresh32(p_keep), td = gg_thresh32(p_diag);
  uint64_t kh = gg_key(seed, S_GRID_H), kv = gg_key(seed, S_GRID_V), kd = gg_key(seed, S_GRID_D);
#pragma omp parallel for schedule(static)
  for (int64_t idx = 0; idx < nh; ++idx) {   /* (i,j)-(i,j+1) */
    int64_t i = idx / (W - 1), j = idx % (W - 1);
    uint64_t r = gg_rand(kh, (uint64_t)idx);
    int keep = (uint32_t)r < tk;
    eu[idx] = keep ? pi[i * W + j] : -1;
    ev[idx] = keep ? pi[i * W + j + 1] : -1;
  }
#pragma omp parallel for schedule(static)
  for (int64_t idx = 0; idx < nv; ++idx) {   /* (i,j)-(i+1,j) */
    int64_t i = idx / W, j = idx % W;
    uint64_t r = gg_rand(kv, (uint64_t)idx);
    int keep = (uint32_t)r < tk;
    eu[nh + idx] = keep ? pi[i * W + j] : -1;
    ev[nh + idx] = keep ? pi[(i + 1) * W + j] : -1;
  }
#pragma omp parallel for schedule(static)
  for (int64_t idx = 0; idx < nd; ++idx) {   /* unit square (i,j) */
    int64_t i = idx / (W - 1), j = idx % (W - 1);
    uint64_t r = gg_rand(kd, (uint64_t)idx);
    int keep = (uint32_t)r < td;
    int anti = (int)((r >> 32) & 1);
    int64_t x = anti ? i * W + j + 1 : i * W + j;
    int64_t y = anti ? (i + 1) * W + j : (i + 1) * W + j + 1;
    eu[nh + nv + idx] = keep ? pi[x] : -1;
    ev[nh + nv + idx] = keep ? pi[y] : -1;
  }
  free(pi);
  gg_graph* g = build_csr(n, M, eu, ev);
  free(eu);
  free(ev);
  return g;
}

/* Chung-Lu power-law graph. */
GG_EXPORT gg_graph* gg_chung_lu(int64_t n, double mean_deg, double gamma, double wmax,
                                uint64_t seed) {
  double* q = (double*)malloc(sizeof(double) * (size_t)n);
  double ex = -1.0 / (gamma - 1.0);
#pragma omp parallel for schedule(static)
  for (int64_t i = 0; i < n; ++i) q[i] = pow(((double)i + 0.5) / (double)n, ex);
  /* bisection on c: mean(min(wmax, c*q_i)) = mean_deg (monotone in c) */
  double lo = 0.0, hi = wmax;
  for (int it = 0; it < 100; ++it) {
    double c = 0.5 * (lo + hi), s = 0.0;
    /* sequential sum: deterministic regardless of thread count */
    for (int64_t i = 0; i < n; ++i) { double w = c * q[i]; s += w < wmax ? w : wmax; }
    if (s / (double)n < mean_deg) lo = c; else hi = c;
  }
  double c = 0.5 * (lo + hi);
  double tot = 0.0;
  for (int64_t i = 0; i < n; ++i) { double w = c * q[i]; q[i] = w < wmax ? w : wmax; tot += q[i]; }
  /* Vose alias table: prob[i] as a 32-bit threshold, alias[i] */
  uint32_t* prob = (uint32_t*)malloc(sizeof(uint32_t) * (size_t)n);
  int32_t* alias = (int32_t*)malloc(sizeof(int32_t) * (size_t)n);
  int32_t* small = (int32_t*)malloc(sizeof(int32_t) * (size_t)n);
  int32_t* large = (int32_t*)malloc(sizeof(int32_t) * (size_t)n);
  int64_t ns = 0, nl = 0;
  for (int64_t i = 0; i < n; ++i) {
    q[i] = q[i] * (double)n / tot;
    if (q[i] < 1.0) small[ns++] = (int32_t)i; else large[nl++] = (int32_t)i;
  }
  while (ns > 0 && nl > 0) {
    int32_t s = small[--ns], l = large[--nl];
    prob[s] = gg_thresh32(q[s]);
    alias[s] = l;
    q[l] = (q[l] + q[s]) - 1.0;
    if (q[l] < 1.0) small[ns++] = l; else large[nl++] = l;
  }
  while (nl > 0) { int32_t l = large[--nl]; prob[l] = 0xFFFFFFFFu; alias[l] = l; }
  while (ns > 0) { int32_t s = small[--ns]; prob[s] = 0xFFFFFFFFu; alias[s] = s; }
  free(small);
  free(large);
  free(q);
  int32_t* pi = make_perm(n, seed);
  int64_t M = (int64_t)(mean_deg * 0.5 * (double)n);
  int32_t* eu = (int32_t*)malloc(sizeof(int32_t) * (size_t)M);
  int32_t* ev = (int32_t*)malloc(sizeof(int32_t) * (size_t)M);
  uint64_t key = gg_key(seed, S_CL);
#pragma omp parallel for schedule(static)
  for (int64_t e = 0; e < M; ++e) {
    int32_t ends[2];
    for (int k = 0; k < 2; ++k) {
      uint64_t r = gg_rand(key, (uint64_t)e * 2 + (uint64_t)k);
      int64_t i = (int64_t)((((r & 0xFFFFFFFFULL)) * (uint64_t)n) >> 32);
      uint32_t coin = (uint32_t)(r >> 32);
      int32_t pick = (coin < prob[i] || prob[i] == 0xFFFFFFFFu) ? (int32_t)i : alias[i];
      ends[k] = pi[pick];
    }
    eu[e] = ends[0];
    ev[e] = ends[1];
  }
  free(prob);
  free(alias);
  free(pi);
  gg_graph* g = build_csr(n, M, eu, ev);
  free(eu);
  free(ev);
  return g;
}
