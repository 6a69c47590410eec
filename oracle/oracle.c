/*
 * oracle.c -- sequential CPU oracle for JP-ADG (arXiv 2008.11321).
 *
 * TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and
 * bench.py's cpu_baseline / --impl reference legs may load this library.
 * The product path (paper_2008_11321_b200/) never links, imports or calls
 * it, and shares no code, header or constant table with it.
 *
 * Plain, slow, obviously correct, single-threaded C.  All arithmetic is
 * integer (the method fixes no floating point: SURVEY.md §8c Q2).  Each
 * function cites the passage of /root/reference/PAPER.md it follows.
 *
 * Readings of the paper:
 *   Q1  threshold uses "<=" (Alg. 1 line R_def; proof 769)
 *   Q2  eps = num/den, test den*D[v]*|U| <= (den+num)*S exactly (128-bit)
 *   Q3  D is the residual degree in G[U]; S = sum of D over U
 *   Q6  rounds are 1-based (Alg. 1 "l = 1")
 *   Q8  later ADG round = higher priority; larger hash wins inside a round
 *   Q9  rho_R(v) = splitmix64(seed XOR v) (first output of a SplitMix64
 *       generator whose state is seed^v); compared unsigned
 *   Q11 colors are 1-based, 0 = uncolored
 *   Q12 isolated vertices count in |U| (Count(U))
 *
 * Pins (tests/test_oracle_*.py): Appendix B worked examples, the ADG and JP
 * certificate characterisations, Lemma 1 / Lemma 4 / Corollary 1 bounds,
 * exact degeneracy, brute-force chromatic number, published SplitMix64
 * output vectors, exhaustive enumeration of all graphs on <= 6 vertices.
 * The choice of hash (Q9) is a convention, not a paper fact: "parity
 * unpinned" for the choice itself.
 */
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

#define ORC_EXPORT __attribute__((visibility("default")))

/* ------------------------------------------------------------------------ */
/* rho_R: SplitMix64.  Written from the published definition:
 *   z = x + 0x9E3779B97F4A7C15; z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9;
 *   z = (z ^ (z >> 27)) * 0x94D049BB133111EB; return z ^ (z >> 31).        */
ORC_EXPORT uint64_t orc_splitmix64(uint64_t x) {
  uint64_t z = x + 0x9E3779B97F4A7C15ULL;
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ULL;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBULL;
  return z ^ (z >> 31);
}

/* ------------------------------------------------------------------------ */
/* ADG -- Algorithm 1.
 *
 *   D = [deg(v_1) ... deg(v_n)];  l = 1;  U = V               (676-677)
 *   while U != {}:                                             (679)
 *     |U| = Count(U);  cnt = Reduce(U) = sum_{v in U} D[v]     (680-681)
 *     delta = cnt/|U|                                          (682)
 *     R = { u in U : D[u] <= (1+eps) * delta }                 (685)
 *     UPDATE(U, R, D): for v in R, u in N_U(v): D[u] -= 1      (686, 692-696)
 *     U = U \ R                                                (687)
 *     rho_ADG(v) = l for v in R                                (688-689)
 *     l = l + 1                                                (690)
 *
 * With eps = num/den the test D[u] <= (1+eps)*cnt/|U| is, multiplied by the
 * positive den*|U|:  den * D[u] * |U| <= (den + num) * cnt, in 128 bits.
 * UPDATE runs before U = U \ R, so (literally) R-R edges are decremented
 * too; those D values are never read again.
 *
 * Returns T (number of rounds), -1 on bad arguments, -2 if a round selects
 * nothing (cannot happen for eps > 0: min degree <= mean).  Optional stats:
 *   stats[0] = T, stats[1] = sum_l |U_l|, stats[2] = X = number of decrements
 *   applied to vertices that survive the round (cross-round edges),
 *   stats[3] = total decrements including R-R ones.
 * Optional per-round arrays (capacity cap): nU[l-1], S[l-1], nR[l-1].       */
ORC_EXPORT int orc_adg(int64_t n, const int64_t* off, const int32_t* col, uint32_t num,
                       uint32_t den, int32_t* round_out, int64_t* stats, int64_t cap,
                       int64_t* per_nU, int64_t* per_S, int64_t* per_nR) {
  if (n < 0 || num == 0 || den == 0) return -1;
  int64_t* D = (int64_t*)malloc(sizeof(int64_t) * (size_t)(n + 1));
  char* inU = (char*)malloc((size_t)n + 1);
  char* inR = (char*)malloc((size_t)n + 1);
  int64_t* U = (int64_t*)malloc(sizeof(int64_t) * (size_t)(n + 1));   /* list of U */
  int64_t sizeU = n;
  for (int64_t v = 0; v < n; ++v) {
    D[v] = off[v + 1] - off[v];
    inU[v] = 1;
    inR[v] = 0;
    U[v] = v;
    round_out[v] = 0;
  }
  int64_t l = 1, sum_active = 0, cross = 0, all_dec = 0;
  while (sizeU > 0) {
    /* Count and Reduce over U (680-681) */
    int64_t countU = 0;
    uint64_t cnt = 0;
    for (int64_t i = 0; i < sizeU; ++i) {
      countU += 1;
      cnt += (uint64_t)D[U[i]];
    }
    sum_active += countU;
    /* R = { u in U : D[u] <= (1+eps) * cnt / |U| }  (685), exact */
    int64_t sizeR = 0;
    for (int64_t i = 0; i < sizeU; ++i) {
      int64_t u = U[i];
      unsigned __int128 lhs = (unsigned __int128)den * (uint64_t)D[u] * (uint64_t)countU;
      unsigned __int128 rhs = ((unsigned __int128)den + num) * cnt;
      if (lhs <= rhs) { inR[u] = 1; ++sizeR; }
    }
    if (sizeR == 0) {   /* impossible by Lemma 1 (the minimum is <= the mean); guard */
      free(D); free(inU); free(inR); free(U);
      return -2;
    }
    if (l - 1 < cap) {
      if (per_nU) per_nU[l - 1] = countU;
      if (per_S) per_S[l - 1] = (int64_t)cnt;
      if (per_nR) per_nR[l - 1] = sizeR;
    }
    /* UPDATE(U, R, D) (692-696): for v in R, for u in N_U(v): DecrementAndFetch(D[u]) */
    for (int64_t i = 0; i < sizeU; ++i) {
      int64_t v = U[i];
      if (!inR[v]) continue;
      for (int64_t e = off[v]; e < off[v + 1]; ++e) {
        int64_t u = col[e];
        if (inU[u]) {
          D[u] -= 1;
          all_dec += 1;
          if (!inR[u]) cross += 1;
        }
      }
    }
    /* U = U \ R (687); rho_ADG(v) = l for v in R (688-689) */
    int64_t k = 0;
    for (int64_t i = 0; i < sizeU; ++i) {
      int64_t v = U[i];
      if (inR[v]) {
        inU[v] = 0;
        inR[v] = 0;
        round_out[v] = (int32_t)l;
      } else {
        U[k++] = v;
      }
    }
    sizeU = k;
    l += 1;   /* (690) */
  }
  free(D);
  free(inU);
  free(inR);
  free(U);
  if (stats) {
    stats[0] = l - 1;
    stats[1] = sum_active;
    stats[2] = cross;
    stats[3] = all_dec;
  }
  return (int)(l - 1);
}

/* ------------------------------------------------------------------------ */
/* ADG-M -- "Degree Median Instead of Degree Average"
 * (analysis 2553-2611).  ADG-M differs from Algorithm 1 only in that
 *   (1) the median degree delta_m of the vertices in U replaces the mean, and
 *   (2) R = { v in U : D[v] <= delta_m }, limited to half the size of U
 *       (+1 if |U| is odd)                                     (2296-2301)
 * and the paper derives delta_m from U sorted by degree with a linear-time
 * integer sort (2286-2294).  Readings (Q19-Q21): U is sorted by
 * (D ascending, id ascending) -- a stable integer sort of U in id order;
 * delta_m is the D of the ceil(|U|/2)-th element of that order (the lower
 * median); the cap keeps the first ceil(|U|/2) vertices of the order.  All of
 * them pass the test D <= delta_m, so R_l is exactly that prefix (the (1+eps)
 * factor of the conference text, 2277, would change nothing under the cap).
 * UPDATE and the rest of the round are Algorithm 1's (692-696, 687-690).
 * Returns T; stats[0] = T, stats[1] = sum_l |U_l|, stats[2] = X.            */
static const int64_t* g_keyD;
static int cmp_deg_id(const void* a, const void* b) {
  int64_t u = *(const int64_t*)a, v = *(const int64_t*)b;
  if (g_keyD[u] != g_keyD[v]) return g_keyD[u] < g_keyD[v] ? -1 : 1;
  return u < v ? -1 : (u > v ? 1 : 0);
}

ORC_EXPORT int orc_adg_m(int64_t n, const int64_t* off, const int32_t* col, int32_t* round_out,
                         int64_t* stats) {
  if (n < 0) return -1;
  int64_t* D = (int64_t*)malloc(sizeof(int64_t) * (size_t)(n + 1));
  char* inU = (char*)malloc((size_t)n + 1);
  char* inR = (char*)malloc((size_t)n + 1);
  int64_t* U = (int64_t*)malloc(sizeof(int64_t) * (size_t)(n + 1));
  int64_t sizeU = n;
  for (int64_t v = 0; v < n; ++v) {
    D[v] = off[v + 1] - off[v];
    inU[v] = 1;
    inR[v] = 0;
    U[v] = v;
    round_out[v] = 0;
  }
  int64_t l = 1, sum_active = 0, cross = 0;
  while (sizeU > 0) {
    sum_active += sizeU;
    /* U in ascending (D, id) order; delta_m = D of the ceil(|U|/2)-th */
    g_keyD = D;
    qsort(U, (size_t)sizeU, sizeof(int64_t), cmp_deg_id);
    const int64_t half = sizeU / 2 + (sizeU % 2);   /* half the size of U, +1 if odd */
    const int64_t delta_m = D[U[half - 1]];
    /* R = { v in U : D[v] <= delta_m }, limited to the first `half` of the order */
    int64_t sizeR = 0;
    for (int64_t i = 0; i < sizeU && sizeR < half; ++i)
      if (D[U[i]] <= delta_m) { inR[U[i]] = 1; ++sizeR; }
    /* UPDATE(U, R, D) (692-696) */
    for (int64_t i = 0; i < sizeU; ++i) {
      int64_t v = U[i];
      if (!inR[v]) continue;
      for (int64_t e = off[v]; e < off[v + 1]; ++e) {
        int64_t u = col[e];
        if (inU[u]) {
          D[u] -= 1;
          if (!inR[u]) cross += 1;
        }
      }
    }
    /* U = U \ R; rho(v) = l for v in R; l += 1 (687-690) */
    int64_t k = 0;
    for (int64_t i = 0; i < sizeU; ++i) {
      int64_t v = U[i];
      if (inR[v]) {
        inU[v] = 0;
        inR[v] = 0;
        round_out[v] = (int32_t)l;
      } else {
        U[k++] = v;
      }
    }
    sizeU = k;
    l += 1;
  }
  free(D);
  free(inU);
  free(inR);
  free(U);
  if (stats) {
    stats[0] = l - 1;
    stats[1] = sum_active;
    stats[2] = cross;
  }
  return (int)(l - 1);
}

/* ------------------------------------------------------------------------ */
/* ADG-O -- the listing "ADG-O, a variant of ADG with optimizations",
 * PAPER.md:2397-2453 (sorting, 2231-2252; fused rank, 2257-2271):
 *
 *   D = [deg(v)];  U = V;  l = 0;  rho(v) = n for all v
 *   while U != {}:
 *     delta = (1/|U|) sum_{v in U} D[v]
 *     PARTITION(U, (1+eps) delta): R = { u in U : D[u] <= (1+eps) delta }
 *     SORT(R, D): increasing D
 *     rho(r_i) = l + i   for r_i in R = [r_0 .. r_{|R|-1}]
 *     U = U \ R
 *     UPDATEandPRIORITIZE: for v in R, w in N(v) with rho(w) > rho(v):
 *         D[w] -= 1; c += 1;  rank(v) = c
 *     l = l + |R|
 *
 * The selection is Algorithm 1's (same exact integer test, Q1/Q2), so the
 * rounds equal ADG's.  Reading Q22: SORT is stable in ascending
 * id, i.e. R is ordered by (D ascending, id ascending).  rho is a total order
 * (a permutation of 0..n-1), so JP needs no tie-break.  Outputs: round_out
 * (1-based round, as Alg. 1), rho_out (int64), rank_out (int64, the number of
 * neighbours with a higher rho = |pred(v)| for JP with rho), drem_out (D at
 * selection time).  Returns T.                                              */
static const int64_t* g_sortD;
static int cmp_r_deg_id(const void* a, const void* b) {
  int64_t u = *(const int64_t*)a, v = *(const int64_t*)b;
  if (g_sortD[u] != g_sortD[v]) return g_sortD[u] < g_sortD[v] ? -1 : 1;
  return u < v ? -1 : (u > v ? 1 : 0);
}

ORC_EXPORT int orc_adg_o(int64_t n, const int64_t* off, const int32_t* col, uint32_t num,
                         uint32_t den, int32_t* round_out, int64_t* rho_out, int64_t* rank_out,
                         int64_t* drem_out) {
  if (n < 0 || num == 0 || den == 0) return -1;
  int64_t* D = (int64_t*)malloc(sizeof(int64_t) * (size_t)(n + 1));
  char* inU = (char*)malloc((size_t)n + 1);
  int64_t* U = (int64_t*)malloc(sizeof(int64_t) * (size_t)(n + 1));
  int64_t* R = (int64_t*)malloc(sizeof(int64_t) * (size_t)(n + 1));
  int64_t sizeU = n;
  for (int64_t v = 0; v < n; ++v) {
    D[v] = off[v + 1] - off[v];
    inU[v] = 1;
    U[v] = v;
    rho_out[v] = n;        /* rho(v) = n: not yet removed */
    round_out[v] = 0;
  }
  int64_t l = 0, it = 1;
  while (sizeU > 0) {
    uint64_t cnt = 0;
    for (int64_t i = 0; i < sizeU; ++i) cnt += (uint64_t)D[U[i]];
    /* PARTITION: R = { u in U : den*D[u]*|U| <= (den+num)*sum D } (exact) */
    int64_t sizeR = 0, k = 0;
    for (int64_t i = 0; i < sizeU; ++i) {
      int64_t u = U[i];
      unsigned __int128 lhs = (unsigned __int128)den * (uint64_t)D[u] * (uint64_t)sizeU;
      unsigned __int128 rhs = ((unsigned __int128)den + num) * cnt;
      if (lhs <= rhs) R[sizeR++] = u;
      else U[k++] = u;
    }
    if (sizeR == 0) { free(D); free(inU); free(U); free(R); return -2; }
    /* SORT(R, D): increasing D, ties by increasing id */
    g_sortD = D;
    qsort(R, (size_t)sizeR, sizeof(int64_t), cmp_r_deg_id);
    for (int64_t i = 0; i < sizeR; ++i) {
      rho_out[R[i]] = l + i;
      round_out[R[i]] = (int32_t)it;
      if (drem_out) drem_out[R[i]] = D[R[i]];
      inU[R[i]] = 0;
    }
    sizeU = k;
    /* UPDATEandPRIORITIZE(D, U, R, rank) */
    for (int64_t i = 0; i < sizeR; ++i) {
      int64_t v = R[i], c = 0;
      for (int64_t e = off[v]; e < off[v + 1]; ++e) {
        int64_t w = col[e];
        if (rho_out[w] > rho_out[v]) {
          D[w] -= 1;
          c += 1;
        }
      }
      if (rank_out) rank_out[v] = c;
    }
    l += sizeR;
    it += 1;
  }
  free(D);
  free(inU);
  free(U);
  free(R);
  return (int)(it - 1);
}

/* JP (Algorithm 3) for a total-order priority rho
 * (int64, larger = higher priority), e.g. rho_ADG-O: sequential greedy in
 * decreasing rho, GetColor (1135-1138) from the already colored preds.     */
static const int64_t* g_rho;
static int cmp_rho_desc(const void* a, const void* b) {
  int64_t u = *(const int64_t*)a, v = *(const int64_t*)b;
  return g_rho[u] > g_rho[v] ? -1 : (g_rho[u] < g_rho[v] ? 1 : 0);
}

ORC_EXPORT int orc_jp_rho(int64_t n, const int64_t* off, const int32_t* col, const int64_t* rho,
                          int32_t* color_out) {
  if (n < 0) return -1;
  int64_t* order = (int64_t*)malloc(sizeof(int64_t) * (size_t)(n + 1));
  for (int64_t v = 0; v < n; ++v) order[v] = v;
  g_rho = rho;
  qsort(order, (size_t)n, sizeof(int64_t), cmp_rho_desc);
  int64_t* stamp = (int64_t*)malloc(sizeof(int64_t) * (size_t)(n + 2));
  for (int64_t i = 0; i < n + 2; ++i) stamp[i] = -1;
  for (int64_t v = 0; v < n; ++v) color_out[v] = 0;
  int32_t K = 0;
  for (int64_t i = 0; i < n; ++i) {
    int64_t v = order[i], npred = 0;
    for (int64_t e = off[v]; e < off[v + 1]; ++e) {
      int64_t u = col[e];
      if (rho[u] > rho[v]) {
        npred += 1;
        stamp[color_out[u]] = i;
      }
    }
    int64_t c = 1;
    while (c <= npred + 1 && stamp[c] == i) ++c;
    color_out[v] = (int32_t)c;
    if (c > K) K = (int32_t)c;
  }
  free(order);
  free(stamp);
  return K;
}

/* ------------------------------------------------------------------------ */
/* DEC-ADG-ITR: DEC-ADG (Algorithm "DEC-ADG",
 * PAPER.md:1346-1369) with SIM-COL changed in its Part 1:
 * "colors are not picked randomly, but we choose the smallest color not in
 * B_v".
 *
 *   C = 0; rho = ADG(G)                      (partitions R(l) = {v : rho(v) = l})
 *   for l = T down to 1:                     (the densest partition first)
 *     B_v = colors of v's neighbours in the colored partitions Q (1366-1368)
 *     SIM-COL-ITR(G(l), B):  U = R(l)
 *       while U != {}:
 *         Part 1: for v in U: C[v] = min({1, 2, ...} \ B_v)
 *         Part 2: for v in U: if some u in N_U(v) has C[u] == C[v]: C[v] = 0
 *         Part 3: for v in U, u in N_U(v): if C[u] > 0: B_v = B_v u {C[u]}
 *         U = U \ {v in U : C[v] > 0}
 *
 * Reading Q23: with Part 1 deterministic, two adjacent vertices
 * with equal B would pick the same color forever (SIM-COL's random choice is
 * what breaks that tie), so Part 2 resets v only for a same-colored active
 * neighbour u of HIGHER priority, h(u) > h(v) with h(x) = splitmix64(seed ^ x)
 * (the tie-break of JP-ADG; ITR resolves conflicts the same way, one endpoint
 * keeping its color).  The highest-priority vertex of U always keeps its color,
 * so every pass fixes at least one vertex.  Reading Q24: ADG runs with the
 * caller's eps (the eps/12 of DEC-ADG's listing is a proof device, 1391-1393).
 * B_v is exactly the set of colors of v's fixed neighbours, so Part 1 is the
 * mex over the neighbours colored so far (earlier partitions and earlier
 * passes).  Returns K; passes_out (optional) receives the total number of
 * SIM-COL passes over all partitions.                                         */
ORC_EXPORT int orc_dec_adg_itr(int64_t n, const int64_t* off, const int32_t* col,
                               const int32_t* round, int32_t T, uint64_t seed,
                               int32_t* color_out, int64_t* passes_out) {
  if (n < 0) return -1;
  int32_t* tent = (int32_t*)malloc(sizeof(int32_t) * (size_t)(n + 1));
  char* active = (char*)malloc((size_t)n + 1);
  int64_t* U = (int64_t*)malloc(sizeof(int64_t) * (size_t)(n + 1));
  int64_t* W = (int64_t*)malloc(sizeof(int64_t) * (size_t)(n + 1));
  int64_t* stamp = (int64_t*)malloc(sizeof(int64_t) * (size_t)(n + 2));
  for (int64_t i = 0; i < n + 2; ++i) stamp[i] = -1;
  for (int64_t v = 0; v < n; ++v) { color_out[v] = 0; active[v] = 0; }
  int32_t K = 0;
  int64_t passes = 0, tick = 0;
  for (int32_t l = T; l >= 1; --l) {
    int64_t sizeU = 0;
    for (int64_t v = 0; v < n; ++v)
      if (round[v] == l) { U[sizeU++] = v; active[v] = 1; }
    while (sizeU > 0) {
      passes += 1;
      /* Part 1: C[v] = smallest color not in B_v (the fixed neighbours' colors) */
      for (int64_t i = 0; i < sizeU; ++i) {
        int64_t v = U[i];
        tick += 1;
        for (int64_t e = off[v]; e < off[v + 1]; ++e) {
          int64_t u = col[e];
          if (color_out[u] > 0 && color_out[u] <= n + 1) stamp[color_out[u]] = tick;
        }
        int32_t c = 1;
        while (stamp[c] == tick) ++c;
        tent[v] = c;
      }
      /* Part 2: reset on a same-colored active neighbour of higher priority (Q23) */
      int64_t k = 0, nw = 0;
      for (int64_t i = 0; i < sizeU; ++i) {
        int64_t v = U[i];
        int keep = 1;
        const uint64_t hv = orc_splitmix64(seed ^ (uint64_t)v);
        for (int64_t e = off[v]; e < off[v + 1] && keep; ++e) {
          int64_t u = col[e];
          if (active[u] && tent[u] == tent[v] && orc_splitmix64(seed ^ (uint64_t)u) > hv) keep = 0;
        }
        if (keep) W[nw++] = v;   /* C[v] stays: v is colored */
        else U[k++] = v;         /* C[v] = 0: v stays in U */
      }
      /* Part 3 and U = U \ {colored}: the colored ones leave U; their colors
       * reach the neighbours' B_v through Part 1's mex over colored neighbours */
      for (int64_t i = 0; i < nw; ++i) {
        const int64_t v = W[i];
        color_out[v] = tent[v];
        active[v] = 0;
        if (tent[v] > K) K = tent[v];
      }
      sizeU = k;
    }
  }
  free(tent);
  free(active);
  free(U);
  free(W);
  free(stamp);
  if (passes_out) *passes_out = passes;
  return K;
}

/* ------------------------------------------------------------------------ */
/* JP priority rho = <rho_ADG, rho_R>, lexicographic (PAPER.md:1073-1078,
 * 1095-1096): u has higher priority than v iff
 *   round[u] > round[v], or round[u] == round[v] and h(u) > h(v),
 * with h(x) = splitmix64(seed ^ x) compared as unsigned 64-bit.              */
static uint64_t g_seed;
static const int32_t* g_round;

static int higher(int64_t u, int64_t v) {
  if (g_round[u] != g_round[v]) return g_round[u] > g_round[v];
  return orc_splitmix64(g_seed ^ (uint64_t)u) > orc_splitmix64(g_seed ^ (uint64_t)v);
}

static int cmp_desc(const void* a, const void* b) {
  int64_t u = *(const int64_t*)a, v = *(const int64_t*)b;
  if (u == v) return 0;
  return higher(u, v) ? -1 : 1;
}

/* JP (Algorithm 3) evaluated as sequential greedy in
 * decreasing priority: every predecessor of v (pred[v] = {u in N(v) :
 * rho(u) > rho(v)}, 1118) precedes v, so when v is reached all of pred[v]
 * is colored and GetColor (1135-1138) returns
 *   min({1, ..., |pred[v]|+1} \ {C[u] : u in pred[v]}).
 * This equals JP's output because JPColor colors v exactly once, after all
 * of pred[v] (Join on count[v], 1130-1133), from pred colors alone.
 *
 * Returns K = max color (0 for n = 0), -1 on bad arguments.  Optional
 * level_out[v] = 1 + max level over pred[v] (the JP DAG depth; J = max).   */
ORC_EXPORT int orc_jp(int64_t n, const int64_t* off, const int32_t* col, const int32_t* round,
                      uint64_t seed, int32_t* color_out, int32_t* level_out, int64_t* J_out) {
  if (n < 0) return -1;
  g_seed = seed;
  g_round = round;
  int64_t* order = (int64_t*)malloc(sizeof(int64_t) * (size_t)(n + 1));
  for (int64_t v = 0; v < n; ++v) order[v] = v;
  qsort(order, (size_t)n, sizeof(int64_t), cmp_desc);
  int64_t* stamp = (int64_t*)malloc(sizeof(int64_t) * (size_t)(n + 2));
  for (int64_t i = 0; i < n + 2; ++i) stamp[i] = -1;
  for (int64_t v = 0; v < n; ++v) color_out[v] = 0;   /* C = [0 0 ... 0] (1115) */
  int32_t K = 0;
  int64_t J = 0;
  for (int64_t i = 0; i < n; ++i) {
    int64_t v = order[i];
    int64_t npred = 0, lvl = 0;
    for (int64_t e = off[v]; e < off[v + 1]; ++e) {
      int64_t u = col[e];
      if (higher(u, v)) {                  /* u in pred[v] */
        npred += 1;
        stamp[color_out[u]] = i;           /* C = C - {C[u]} */
        if (level_out && level_out[u] > lvl) lvl = level_out[u];
      }
    }
    int64_t c = 1;                         /* min of {1..|pred|+1} \ used */
    while (c <= npred + 1 && stamp[c] == i) ++c;
    color_out[v] = (int32_t)c;
    if (c > K) K = (int32_t)c;
    if (level_out) {
      level_out[v] = (int32_t)(lvl + 1);
      if (lvl + 1 > J) J = lvl + 1;
    }
  }
  free(order);
  free(stamp);
  if (J_out) *J_out = J;
  return K;
}

/* ------------------------------------------------------------------------ */
/* Exact degeneracy d: the smallest-last peel of Matula and
 * Beck -- repeatedly remove a vertex of minimum residual degree; d is the
 * largest minimum seen.  Bucket queue, O(n + m).                          */
ORC_EXPORT int64_t orc_degeneracy(int64_t n, const int64_t* off, const int32_t* col) {
  if (n <= 0) return 0;
  int64_t maxdeg = 0;
  int64_t* deg = (int64_t*)malloc(sizeof(int64_t) * (size_t)n);
  for (int64_t v = 0; v < n; ++v) {
    deg[v] = off[v + 1] - off[v];
    if (deg[v] > maxdeg) maxdeg = deg[v];
  }
  /* bucket sort vertices by degree: bin[d] = start of degree-d block */
  int64_t* bin = (int64_t*)calloc((size_t)maxdeg + 2, sizeof(int64_t));
  int64_t* pos = (int64_t*)malloc(sizeof(int64_t) * (size_t)n);
  int64_t* vert = (int64_t*)malloc(sizeof(int64_t) * (size_t)n);
  for (int64_t v = 0; v < n; ++v) bin[deg[v]]++;
  int64_t start = 0;
  for (int64_t d = 0; d <= maxdeg; ++d) { int64_t c = bin[d]; bin[d] = start; start += c; }
  for (int64_t v = 0; v < n; ++v) { pos[v] = bin[deg[v]]; vert[pos[v]] = v; bin[deg[v]]++; }
  for (int64_t d = maxdeg; d >= 1; --d) bin[d] = bin[d - 1];
  bin[0] = 0;
  int64_t dgn = 0;
  for (int64_t i = 0; i < n; ++i) {
    int64_t v = vert[i];            /* a vertex of minimum residual degree */
    if (deg[v] > dgn) dgn = deg[v];
    for (int64_t e = off[v]; e < off[v + 1]; ++e) {
      int64_t u = col[e];
      if (deg[u] > deg[v]) {        /* u not yet removed: move it down one bucket */
        int64_t du = deg[u], pu = pos[u], pw = bin[du], w = vert[pw];
        if (u != w) { pos[u] = pw; vert[pu] = w; pos[w] = pu; vert[pw] = u; }
        bin[du]++;
        deg[u]--;
      }
    }
  }
  free(deg);
  free(bin);
  free(pos);
  free(vert);
  return dgn;
}

/* ------------------------------------------------------------------------ */
/* Brute-force chromatic number (north star): the smallest k
 * for which a backtracking search finds a proper k-coloring.  n <= 16.      */
static int bt(int64_t v, int64_t n, const int64_t* off, const int32_t* col, int k, int* c) {
  if (v == n) return 1;
  for (int x = 1; x <= k; ++x) {
    int ok = 1;
    for (int64_t e = off[v]; e < off[v + 1]; ++e)
      if (col[e] < v && c[col[e]] == x) { ok = 0; break; }
    if (!ok) continue;
    c[v] = x;
    if (bt(v + 1, n, off, col, k, c)) return 1;
    c[v] = 0;
  }
  return 0;
}

ORC_EXPORT int orc_brute_chi(int64_t n, const int64_t* off, const int32_t* col) {
  if (n < 0 || n > 16) return -1;
  if (n == 0) return 0;
  int c[16];
  for (int k = 1; k <= n; ++k) {
    memset(c, 0, sizeof(c));
    if (bt(0, n, off, col, k, c)) return k;
  }
  return (int)n;
}
