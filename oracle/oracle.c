/* TEST INFRASTRUCTURE ONLY — plain-C restatement of the reference hot path,
 * used as the parity checker (see oracle.h). Each function cites the
 * reference file:line it restates. Parity pinned by tests/test_oracle_pins.py
 * (reference KATs + outputs of the reference library built in oracle/_ref).
 */
#include "oracle.h"

#include <stdlib.h>
#include <string.h>

/* ---------------------------------------------------------------- rng.hpp */

uint64_t orc_splitmix64(uint64_t x) { /* rng.hpp:49-54 */
  x += 0x9e3779b97f4a7c15ULL;
  x = (x ^ (x >> 30)) * 0xbf58476d1ce4e5b9ULL;
  x = (x ^ (x >> 27)) * 0x94d049bb133111ebULL;
  return x ^ (x >> 31);
}

/* std::mt19937_64 as pinned by [rand.predef]: w=64 n=312 m=156 r=31 */
void orc_mt_seed(orc_mt* m, uint64_t seed) {
  m->mt[0] = seed;
  for (int i = 1; i < 312; ++i)
    m->mt[i] = 6364136223846793005ULL * (m->mt[i - 1] ^ (m->mt[i - 1] >> 62)) +
               (uint64_t)i;
  m->idx = 312;
}

static void mt_twist(orc_mt* m) {
  for (int i = 0; i < 312; ++i) {
    const uint64_t x = (m->mt[i] & 0xFFFFFFFF80000000ULL) |
                       (m->mt[(i + 1) % 312] & 0x7FFFFFFFULL);
    uint64_t xa = x >> 1;
    if (x & 1) xa ^= 0xB5026F5AA96619E9ULL;
    m->mt[i] = m->mt[(i + 156) % 312] ^ xa;
  }
  m->idx = 0;
}

uint64_t orc_mt_next(orc_mt* m) {
  if (m->idx >= 312) mt_twist(m);
  uint64_t y = m->mt[m->idx++];
  y ^= (y >> 29) & 0x5555555555555555ULL;
  y ^= (y << 17) & 0x71D67FFFEDA60000ULL;
  y ^= (y << 37) & 0xFFF7EEE000000000ULL;
  y ^= y >> 43;
  return y;
}

uint64_t orc_bounded(orc_mt* m, uint64_t n) { /* rng.hpp:21-30 */
  if (n < 2) return 0;
  const uint64_t rem = (UINT64_MAX % n + 1) % n;
  const uint64_t limit = UINT64_MAX - rem;
  uint64_t v;
  do {
    v = orc_mt_next(m);
  } while (v > limit);
  return v % n;
}

double orc_unit(orc_mt* m) { /* rng.hpp:33 */
  return (double)(orc_mt_next(m) >> 11) * 0x1.0p-53;
}

void orc_random_order(int32_t n_recv, uint64_t seed, int32_t* perm) {
  /* schedule.cpp:73-84 + rng.hpp:40-46: Fisher-Yates from the top over
   * recv_ids() in ascending order; rank i goes to recvs[i]. */
  orc_mt m;
  orc_mt_seed(&m, seed);
  for (int32_t i = 0; i < n_recv; ++i) perm[i] = i;
  for (int64_t i = n_recv; i > 1; --i) {
    const int64_t j = (int64_t)orc_bounded(&m, (uint64_t)i);
    const int32_t t = perm[i - 1];
    perm[i - 1] = perm[j];
    perm[j] = t;
  }
}

/* ------------------------------------------------------- properties.cpp */

static int32_t* recv_columns(const orc_graph* g, int32_t* n_recv,
                             int32_t** col_op) {
  int32_t* col = (int32_t*)malloc(sizeof(int32_t) * (size_t)(g->n ? g->n : 1));
  int32_t r = 0;
  for (int32_t i = 0; i < g->n; ++i) col[i] = g->kind[i] == ORC_RECV ? r++ : -1;
  *n_recv = r;
  if (col_op) {
    *col_op = (int32_t*)malloc(sizeof(int32_t) * (size_t)(r ? r : 1));
    for (int32_t i = 0; i < g->n; ++i)
      if (col[i] >= 0) (*col_op)[col[i]] = i;
  }
  return col;
}

int32_t orc_dep_words(const orc_graph* g) {
  int32_t r = 0;
  for (int32_t i = 0; i < g->n; ++i) r += g->kind[i] == ORC_RECV;
  return (r + 63) / 64 > 0 ? (r + 63) / 64 : 1;
}

static int32_t* topo(const orc_graph* g) {
  int32_t* order = (int32_t*)malloc(sizeof(int32_t) * (size_t)(g->n + 1));
  int32_t* missing = (int32_t*)malloc(sizeof(int32_t) * (size_t)(g->n + 1));
  int32_t tail = 0;
  for (int32_t i = 0; i < g->n; ++i) {
    missing[i] = g->pred_off[i + 1] - g->pred_off[i];
    if (!missing[i]) order[tail++] = i;
  }
  for (int32_t h = 0; h < tail; ++h) {
    const int32_t v = order[h];
    for (int32_t e = g->succ_off[v]; e < g->succ_off[v + 1]; ++e)
      if (--missing[g->succ_idx[e]] == 0) order[tail++] = g->succ_idx[e];
  }
  free(missing);
  return order;
}

void orc_dependencies(const orc_graph* g, uint64_t* bits) {
  /* properties.cpp:19-66: dep[v] = union of dep over preds, plus v itself
   * when v is a recv. Set union is order-independent, so any topological
   * order gives the reference's sets. */
  const int32_t w = orc_dep_words(g);
  int32_t nr;
  int32_t* col = recv_columns(g, &nr, NULL);
  int32_t* order = topo(g);
  memset(bits, 0, sizeof(uint64_t) * (size_t)w * (size_t)g->n);
  for (int32_t k = 0; k < g->n; ++k) {
    const int32_t v = order[k];
    uint64_t* row = bits + (size_t)v * (size_t)w;
    for (int32_t e = g->pred_off[v]; e < g->pred_off[v + 1]; ++e) {
      const uint64_t* pr = bits + (size_t)g->pred_idx[e] * (size_t)w;
      for (int32_t q = 0; q < w; ++q) row[q] |= pr[q];
    }
    if (col[v] >= 0) row[col[v] >> 6] |= 1ULL << (col[v] & 63);
  }
  free(order);
  free(col);
}

void orc_properties(const orc_graph* g, const uint8_t* outstanding, int mode,
                    int64_t* M, int64_t* P, int64_t* Mplus) {
  const int32_t w = orc_dep_words(g);
  int32_t nr;
  int32_t* col_op;
  int32_t* col = recv_columns(g, &nr, &col_op);
  uint64_t* bits = (uint64_t*)malloc(sizeof(uint64_t) * (size_t)w * (size_t)(g->n ? g->n : 1));
  uint64_t* out = (uint64_t*)calloc((size_t)w, sizeof(uint64_t));
  orc_dependencies(g, bits);
  for (int32_t c = 0; c < nr; ++c)
    if (outstanding[c]) out[c >> 6] |= 1ULL << (c & 63);
  /* properties.cpp:82-87: M = outstanding communication among deps */
  for (int32_t v = 0; v < g->n; ++v) {
    int64_t m = 0;
    const uint64_t* row = bits + (size_t)v * (size_t)w;
    for (int32_t q = 0; q < w; ++q) {
      uint64_t x = row[q] & out[q];
      while (x) {
        const int b = __builtin_ctzll(x);
        m += g->dur[col_op[q * 64 + b]];
        x &= x - 1;
      }
    }
    M[v] = m;
  }
  for (int32_t c = 0; c < nr; ++c)
    if (outstanding[c]) {
      P[c] = 0;
      Mplus[c] = ORC_INF;
    }
  /* properties.cpp:92-107 */
  for (int32_t v = 0; v < g->n; ++v) {
    if (col[v] >= 0 && outstanding[col[v]]) continue;
    const uint64_t* row = bits + (size_t)v * (size_t)w;
    int64_t cnt = 0;
    int32_t only = -1;
    for (int32_t q = 0; q < w; ++q) {
      const uint64_t x = row[q] & out[q];
      if (x && only < 0) only = q * 64 + __builtin_ctzll(x);
      cnt += __builtin_popcountll(x);
    }
    if (cnt == 0) continue;
    if (cnt == 1) {
      P[only] += g->dur[v];
      if (mode == 1 && M[v] < Mplus[only]) Mplus[only] = M[v];
    } else {
      for (int32_t q = 0; q < w; ++q) {
        uint64_t x = row[q] & out[q];
        while (x) {
          const int32_t c = q * 64 + __builtin_ctzll(x);
          if (M[v] < Mplus[c]) Mplus[c] = M[v];
          x &= x - 1;
        }
      }
    }
  }
  free(out);
  free(bits);
  free(col_op);
  free(col);
}

/* --------------------------------------------------------- schedule.cpp */

int orc_precedes(int32_t a_id, int64_t a_p, int64_t a_m, int64_t a_mp,
                 int32_t b_id, int64_t b_p, int64_t b_m, int64_t b_mp) {
  /* schedule.cpp:12-19; ORC_INF encodes nullopt, which sorts last exactly
   * like duration_less (properties.hpp:27-32) */
  const int64_t ab = b_p < a_m ? b_p : a_m;
  const int64_t ba = a_p < b_m ? a_p : b_m;
  if (ab != ba) return ab < ba;
  if (a_mp < b_mp) return 1;
  if (b_mp < a_mp) return 0;
  return a_id < b_id;
}

static int cmp_i64(const void* a, const void* b) {
  const int64_t x = *(const int64_t*)a, y = *(const int64_t*)b;
  return (x > y) - (x < y);
}

int orc_tic(const orc_graph* g, int mode, int32_t* prio) {
  /* schedule.cpp:21-42: general oracle (time_oracle.cpp:86-91), all recvs
   * outstanding, dense rank of M+ ascending with nullopt last. */
  int32_t nr;
  int32_t* col = recv_columns(g, &nr, NULL);
  int64_t* unit = (int64_t*)malloc(sizeof(int64_t) * (size_t)(g->n ? g->n : 1));
  for (int32_t v = 0; v < g->n; ++v) unit[v] = g->kind[v] == ORC_RECV ? 1 : 0;
  orc_graph gu = *g;
  gu.dur = unit;
  uint8_t* out = (uint8_t*)malloc((size_t)(nr ? nr : 1));
  memset(out, 1, (size_t)(nr ? nr : 1));
  int64_t* M = (int64_t*)malloc(sizeof(int64_t) * (size_t)(g->n ? g->n : 1));
  int64_t* P = (int64_t*)malloc(sizeof(int64_t) * (size_t)(nr ? nr : 1));
  int64_t* Mp = (int64_t*)malloc(sizeof(int64_t) * (size_t)(nr ? nr : 1));
  orc_properties(&gu, out, mode, M, P, Mp);
  int64_t* vals = (int64_t*)malloc(sizeof(int64_t) * (size_t)(nr ? nr : 1));
  memcpy(vals, Mp, sizeof(int64_t) * (size_t)nr);
  qsort(vals, (size_t)nr, sizeof(int64_t), cmp_i64);
  int32_t u = 0;
  for (int32_t i = 0; i < nr; ++i)
    if (i == 0 || vals[i] != vals[u - 1]) vals[u++] = vals[i];
  for (int32_t c = 0; c < nr; ++c) {
    int32_t lo = 0, hi = u;
    while (lo < hi) {
      const int32_t mid = (lo + hi) / 2;
      if (vals[mid] < Mp[c]) lo = mid + 1; else hi = mid;
    }
    prio[c] = lo;
  }
  free(vals); free(Mp); free(P); free(M); free(out); free(unit); free(col);
  return u == nr;
}

void orc_tac(const orc_graph* g, int32_t* prio) {
  /* schedule.cpp:44-71, amended properties every round (default argument,
   * properties.hpp:59), left fold in ascending id order. */
  int32_t nr;
  int32_t* col_op;
  int32_t* col = recv_columns(g, &nr, &col_op);
  uint8_t* out = (uint8_t*)malloc((size_t)(nr ? nr : 1));
  memset(out, 1, (size_t)(nr ? nr : 1));
  int64_t* M = (int64_t*)malloc(sizeof(int64_t) * (size_t)(g->n ? g->n : 1));
  int64_t* P = (int64_t*)malloc(sizeof(int64_t) * (size_t)(nr ? nr : 1));
  int64_t* Mp = (int64_t*)malloc(sizeof(int64_t) * (size_t)(nr ? nr : 1));
  for (int32_t next = 0; next < nr; ++next) {
    orc_properties(g, out, 1, M, P, Mp);
    int32_t best = -1;
    for (int32_t c = 0; c < nr; ++c) {
      if (!out[c]) continue;
      if (best < 0 || orc_precedes(c, P[c], M[col_op[c]], Mp[c], best, P[best],
                                   M[col_op[best]], Mp[best]))
        best = c;
    }
    prio[best] = next;
    out[best] = 0;
  }
  free(Mp); free(P); free(M); free(out); free(col_op); free(col);
}

void orc_tac_incremental(const orc_graph* g, int32_t* prio) {
  /* with recvs as roots, cnt/M/xr only change on the
   * retired recv's descendants; amended M+ = min of M over direct succs. */
  const int32_t w = orc_dep_words(g);
  int32_t nr;
  int32_t* col_op;
  int32_t* col = recv_columns(g, &nr, &col_op);
  uint64_t* bits = (uint64_t*)malloc(sizeof(uint64_t) * (size_t)w * (size_t)(g->n ? g->n : 1));
  orc_dependencies(g, bits);
  int32_t* cnt = (int32_t*)calloc((size_t)(g->n + 1), sizeof(int32_t));
  int64_t* M = (int64_t*)calloc((size_t)(g->n + 1), sizeof(int64_t));
  int32_t* xr = (int32_t*)calloc((size_t)(g->n + 1), sizeof(int32_t));
  int64_t* P = (int64_t*)calloc((size_t)(nr + 1), sizeof(int64_t));
  uint8_t* out = (uint8_t*)malloc((size_t)(nr + 1));
  memset(out, 1, (size_t)(nr + 1));
  for (int32_t v = 0; v < g->n; ++v) {
    const uint64_t* row = bits + (size_t)v * (size_t)w;
    for (int32_t q = 0; q < w; ++q) {
      uint64_t x = row[q];
      while (x) {
        const int32_t c = q * 64 + __builtin_ctzll(x);
        cnt[v]++;
        M[v] += g->dur[col_op[c]];
        xr[v] ^= c;
        x &= x - 1;
      }
    }
    if (col[v] < 0 && cnt[v] == 1) P[xr[v]] += g->dur[v];
  }
  for (int32_t next = 0; next < nr; ++next) {
    int32_t best = -1;
    int64_t bp = 0, bm = 0, bmp = 0;
    for (int32_t c = 0; c < nr; ++c) {
      if (!out[c]) continue;
      const int32_t r = col_op[c];
      int64_t mp = ORC_INF;
      for (int32_t e = g->succ_off[r]; e < g->succ_off[r + 1]; ++e)
        if (M[g->succ_idx[e]] < mp) mp = M[g->succ_idx[e]];
      if (best < 0 || orc_precedes(c, P[c], M[r], mp, best, bp, bm, bmp)) {
        best = c;
        bp = P[c];
        bm = M[r];
        bmp = mp;
      }
    }
    prio[best] = next;
    out[best] = 0;
    const int64_t t = g->dur[col_op[best]];
    for (int32_t v = 0; v < g->n; ++v) {
      if (col[v] >= 0) continue;
      if (!((bits[(size_t)v * (size_t)w + (best >> 6)] >> (best & 63)) & 1)) continue;
      cnt[v]--;
      M[v] -= t;
      xr[v] ^= best;
      if (cnt[v] == 1) P[xr[v]] += g->dur[v];
    }
  }
  free(out); free(P); free(xr); free(M); free(cnt); free(bits); free(col_op);
  free(col);
}

void orc_tac_rows(const orc_graph* g, int32_t* prio) {
  /* The same SURVEY A.1 incremental TAC as orc_tac_incremental, with the
   * dependency closure kept per ROW instead of per op: a non-recv op whose
   * predecessors all sit in one non-recv row shares that row's set (its
   * dep set is the union of its predecessors', properties.cpp:44-58), so
   * cnt/M/xr are per row and a row's ops are weighed together when its cnt
   * drops to one. Retire walks a column-major (recv x row) bitset. Needed
   * where the op-level closure is 12.5 GB and the retire loop O(V) per round
   * (config 5's top point: 10^6 ops / 10^5 recvs); checked against
   * orc_tac_incremental and orc_tac in tests/test_oracle_pins.py. */
  const int32_t n = g->n;
  int32_t nr;
  int32_t* col_op;
  int32_t* col = recv_columns(g, &nr, &col_op);
  const int32_t w = (nr + 63) / 64;
  int32_t* order = (int32_t*)malloc(sizeof(int32_t) * (size_t)(n ? n : 1));
  int32_t* miss = (int32_t*)malloc(sizeof(int32_t) * (size_t)(n ? n : 1));
  int32_t head = 0, tail = 0;
  for (int32_t v = 0; v < n; ++v)
    if ((miss[v] = g->pred_off[v + 1] - g->pred_off[v]) == 0) order[tail++] = v;
  while (head < tail) {
    const int32_t v = order[head++];
    for (int32_t e = g->succ_off[v]; e < g->succ_off[v + 1]; ++e)
      if (--miss[g->succ_idx[e]] == 0) order[tail++] = g->succ_idx[e];
  }
  /* row of every op: recvs -> -1 (their set is {own column}); a non-recv op
   * aliases the row of its predecessors when they all share one non-recv
   * row, else opens a new row = OR of its predecessors' sets. */
  int32_t* row = (int32_t*)malloc(sizeof(int32_t) * (size_t)(n ? n : 1));
  size_t cap = 1024, nrows = 0;
  uint64_t* rbits = (uint64_t*)calloc(cap * (size_t)(w ? w : 1), sizeof(uint64_t));
  for (int32_t h = 0; h < tail; ++h) {
    const int32_t v = order[h];
    if (col[v] >= 0) { row[v] = -1; continue; }
    int32_t same = -2;
    for (int32_t e = g->pred_off[v]; e < g->pred_off[v + 1]; ++e) {
      const int32_t p = g->pred_idx[e], rp = row[p];
      if (rp < 0 || (same != -2 && same != rp)) { same = -1; break; }
      same = rp;
    }
    if (same >= 0) { row[v] = same; continue; }
    if (nrows == cap) {
      rbits = (uint64_t*)realloc(rbits, sizeof(uint64_t) * 2 * cap * (size_t)(w ? w : 1));
      memset(rbits + cap * (size_t)w, 0, sizeof(uint64_t) * cap * (size_t)w);
      cap *= 2;
    }
    uint64_t* dst = rbits + nrows * (size_t)w;
    for (int32_t e = g->pred_off[v]; e < g->pred_off[v + 1]; ++e) {
      const int32_t p = g->pred_idx[e];
      if (row[p] < 0) {
        dst[col[p] >> 6] |= 1ULL << (col[p] & 63);
      } else {
        const uint64_t* src = rbits + (size_t)row[p] * (size_t)w;
        for (int32_t q = 0; q < w; ++q) dst[q] |= src[q];
      }
    }
    row[v] = (int32_t)nrows++;
  }
  const size_t R_ = nrows, rw = (R_ + 63) / 64;
  int64_t* wt = (int64_t*)calloc(R_ + 1, sizeof(int64_t));
  int32_t* cnt = (int32_t*)calloc(R_ + 1, sizeof(int32_t));
  int64_t* M = (int64_t*)calloc(R_ + 1, sizeof(int64_t));
  int32_t* xr = (int32_t*)calloc(R_ + 1, sizeof(int32_t));
  int64_t* P = (int64_t*)calloc((size_t)nr + 1, sizeof(int64_t));
  uint64_t* cbits = (uint64_t*)calloc((size_t)(nr ? nr : 1) * (rw ? rw : 1), sizeof(uint64_t));
  for (int32_t v = 0; v < n; ++v)
    if (row[v] >= 0) wt[row[v]] += g->dur[v];
  for (size_t r = 0; r < R_; ++r) {
    const uint64_t* b = rbits + r * (size_t)w;
    for (int32_t q = 0; q < w; ++q) {
      uint64_t x = b[q];
      while (x) {
        const int32_t c = q * 64 + __builtin_ctzll(x);
        cnt[r]++;
        M[r] += g->dur[col_op[c]];
        xr[r] ^= c;
        cbits[(size_t)c * rw + (r >> 6)] |= 1ULL << (r & 63);
        x &= x - 1;
      }
    }
    if (cnt[r] == 1) P[xr[r]] += wt[r];
  }
  free(rbits);
  uint8_t* out = (uint8_t*)malloc((size_t)nr + 1);
  memset(out, 1, (size_t)nr + 1);
  for (int32_t next = 0; next < nr; ++next) {
    int32_t best = -1;
    int64_t bp = 0, bm = 0, bmp = 0;
    for (int32_t c = 0; c < nr; ++c) {
      if (!out[c]) continue;
      const int32_t r = col_op[c];
      int64_t mp = ORC_INF;
      for (int32_t e = g->succ_off[r]; e < g->succ_off[r + 1]; ++e) {
        const int32_t s = row[g->succ_idx[e]];
        if (s >= 0 && M[s] < mp) mp = M[s];
      }
      const int64_t m = g->dur[r]; /* an outstanding recv's own M */
      if (best < 0 || orc_precedes(c, P[c], m, mp, best, bp, bm, bmp)) {
        best = c;
        bp = P[c];
        bm = m;
        bmp = mp;
      }
    }
    prio[best] = next;
    out[best] = 0;
    const int64_t t = g->dur[col_op[best]];
    const uint64_t* cb = cbits + (size_t)best * rw;
    for (size_t q = 0; q < rw; ++q) {
      uint64_t x = cb[q];
      while (x) {
        const size_t r = q * 64 + (size_t)__builtin_ctzll(x);
        cnt[r]--;
        M[r] -= t;
        xr[r] ^= best;
        if (cnt[r] == 1) P[xr[r]] += wt[r];
        x &= x - 1;
      }
    }
  }
  free(out); free(cbits); free(P); free(xr); free(M); free(cnt); free(wt);
  free(row); free(miss); free(order); free(col_op); free(col);
}

/* --------------------------------------------------------------- sim.cpp */

typedef struct { int32_t* v; int32_t n, cap; } ivec;
static void iv_push(ivec* a, int32_t x) {
  if (a->n == a->cap) {
    a->cap = a->cap ? 2 * a->cap : 8;
    a->v = (int32_t*)realloc(a->v, sizeof(int32_t) * (size_t)a->cap);
  }
  a->v[a->n++] = x;
}
static int cmp_i32(const void* a, const void* b) {
  const int32_t x = *(const int32_t*)a, y = *(const int32_t*)b;
  return (x > y) - (x < y);
}

typedef struct {
  const orc_graph* g;
  const int32_t* prio;
} rank_ctx;
static const rank_ctx* g_rank_ctx;
static int cmp_rank(const void* a, const void* b) { /* sim.cpp:100-104 */
  const int32_t x = *(const int32_t*)a, y = *(const int32_t*)b;
  const int32_t px = g_rank_ctx->prio[x], py = g_rank_ctx->prio[y];
  if (px != py) return px < py ? -1 : 1;
  return (x > y) - (x < y);
}

#define SALT 0x9e3779b97f4a7c15ULL /* sim.cpp:14 */

int orc_simulate(const orc_graph* g, const int32_t* prio, int gated,
                 uint64_t choice_seed, double noise, int64_t* makespan,
                 int64_t* violations, int64_t* start, int64_t* end) {
  const int32_t n = g->n, nres = g->n_res;
  int32_t* gate = (int32_t*)malloc(sizeof(int32_t) * (size_t)(n + 1));
  int32_t* orig = (int32_t*)malloc(sizeof(int32_t) * (size_t)(n + 1));
  uint8_t* forced = (uint8_t*)calloc((size_t)(n + 1), 1);
  int64_t* st = (int64_t*)malloc(sizeof(int64_t) * (size_t)(n + 1));
  int64_t* en = (int64_t*)malloc(sizeof(int64_t) * (size_t)(n + 1));
  for (int32_t i = 0; i < n; ++i) gate[i] = orig[i] = -1;

  /* sim.cpp:90-115: dense per-channel ranks from (priority, id); noise
   * swaps from one stream shared by all channels, in resource order. */
  orc_mt noise_rng;
  orc_mt_seed(&noise_rng, orc_splitmix64(choice_seed ^ SALT));
  int32_t* ranked = (int32_t*)malloc(sizeof(int32_t) * (size_t)(n + 1));
  rank_ctx rc = {g, prio};
  g_rank_ctx = &rc;
  for (int32_t r = 0; r < nres; ++r) {
    if (!g->res_channel[r]) continue;
    int32_t k = 0;
    for (int32_t i = 0; i < n; ++i)
      if (g->res[i] == r && prio[i] >= 0) ranked[k++] = i;
    qsort(ranked, (size_t)k, sizeof(int32_t), cmp_rank);
    for (int32_t p = 0; p < k; ++p) orig[ranked[p]] = p;
    if (!gated) continue;
    if (noise > 0.0)
      for (int32_t p = 1; p < k; ++p)
        if (orc_unit(&noise_rng) < noise) {
          const int32_t t = ranked[p - 1];
          ranked[p - 1] = ranked[p];
          ranked[p] = t;
        }
    for (int32_t p = 0; p < k; ++p) gate[ranked[p]] = p;
  }

  orc_mt choice;
  orc_mt_seed(&choice, choice_seed);
  int32_t* missing = (int32_t*)malloc(sizeof(int32_t) * (size_t)(n + 1));
  ivec* queue = (ivec*)calloc((size_t)(nres + 1), sizeof(ivec));
  ivec* comp = (ivec*)calloc((size_t)(nres + 1), sizeof(ivec));
  int32_t* running = (int32_t*)malloc(sizeof(int32_t) * (size_t)(nres + 1));
  int64_t* run_end = (int64_t*)calloc((size_t)(nres + 1), sizeof(int64_t));
  int64_t* counter = (int64_t*)calloc((size_t)(nres + 1), sizeof(int64_t));
  int32_t* cands = (int32_t*)malloc(sizeof(int32_t) * (size_t)(n + 1));
  for (int32_t i = 0; i < n; ++i) {
    missing[i] = g->pred_off[i + 1] - g->pred_off[i];
    if (!missing[i]) iv_push(&queue[g->res[i]], i);
  }
  for (int32_t r = 0; r < nres; ++r) running[r] = -1;
  int64_t t = 0, n_forced = 0;
  int32_t finished = 0;
  int rc_status = 0;

#define ADMITTED(i) \
  (!gated || gate[i] < 0 || forced[i] || (int64_t)gate[i] <= counter[g->res[i]])

  while (finished < n) {
    int progress = 1;
    while (progress) {
      progress = 0;
      for (int32_t r = 0; r < nres; ++r) { /* try_start, sim.cpp:163-192 */
        if (running[r] >= 0 || queue[r].n == 0) continue;
        ivec* q = &queue[r];
        qsort(q->v, (size_t)q->n, sizeof(int32_t), cmp_i32);
        int32_t best = -1;
        for (int32_t k = 0; k < q->n; ++k) {
          const int32_t i = q->v[k];
          if (prio[i] < 0 || !ADMITTED(i)) continue;
          if (best < 0 || prio[i] < best) best = prio[i];
        }
        int32_t nc = 0;
        for (int32_t k = 0; k < q->n; ++k) {
          const int32_t i = q->v[k];
          if (prio[i] < 0) cands[nc++] = i;
          else if (ADMITTED(i) && prio[i] == best) cands[nc++] = i;
        }
        if (nc == 0) continue;
        const int32_t pick =
            nc == 1 ? cands[0] : cands[orc_bounded(&choice, (uint64_t)nc)];
        int32_t k = 0;
        while (q->v[k] != pick) ++k;
        memmove(q->v + k, q->v + k + 1, sizeof(int32_t) * (size_t)(q->n - k - 1));
        q->n--;
        running[r] = pick;
        run_end[r] = t + g->dur[pick];
        st[pick] = t;
        en[pick] = run_end[r];
        progress = 1;
      }
      /* complete_ending_now, sim.cpp:144-161 */
      for (int32_t r = 0; r < nres; ++r) {
        if (running[r] < 0 || run_end[r] != t) continue;
        const int32_t i = running[r];
        running[r] = -1;
        ++finished;
        progress = 1;
        if (prio[i] >= 0 && g->res_channel[r]) {
          counter[r]++;
          iv_push(&comp[r], orig[i]);
        }
        for (int32_t e = g->succ_off[i]; e < g->succ_off[i + 1]; ++e) {
          const int32_t w = g->succ_idx[e];
          if (--missing[w] == 0) iv_push(&queue[g->res[w]], w);
        }
      }
    }
    if (finished == n) break;
    int any = 0;
    int64_t next_t = INT64_MAX;
    for (int32_t r = 0; r < nres; ++r)
      if (running[r] >= 0) {
        any = 1;
        if (run_end[r] < next_t) next_t = run_end[r];
      }
    if (!any) { /* forced release, sim.cpp:211-229 */
      int32_t victim = -1;
      for (int32_t r = 0; r < nres; ++r)
        for (int32_t k = 0; k < queue[r].n; ++k) {
          const int32_t i = queue[r].v[k];
          if (gate[i] < 0 || ADMITTED(i)) continue;
          if (victim < 0 || gate[i] < gate[victim] ||
              (gate[i] == gate[victim] && i < victim))
            victim = i;
        }
      if (victim < 0) {
        rc_status = 2;
        break;
      }
      forced[victim] = 1;
      n_forced++;
      continue;
    }
    t = next_t;
    for (int32_t r = 0; r < nres; ++r) {
      if (running[r] < 0 || run_end[r] != t) continue;
      const int32_t i = running[r];
      running[r] = -1;
      ++finished;
      if (prio[i] >= 0 && g->res_channel[r]) {
        counter[r]++;
        iv_push(&comp[r], orig[i]);
      }
      for (int32_t e = g->succ_off[i]; e < g->succ_off[i + 1]; ++e) {
        const int32_t w = g->succ_idx[e];
        if (--missing[w] == 0) iv_push(&queue[g->res[w]], w);
      }
    }
  }
#undef ADMITTED
  if (rc_status == 0) {
    int64_t m = 0, inv = 0;
    for (int32_t i = 0; i < n; ++i) if (en[i] > m) m = en[i];
    for (int32_t r = 0; r < nres; ++r) /* sim.cpp:247-255 */
      for (int32_t a = 0; a < comp[r].n; ++a)
        for (int32_t b = a + 1; b < comp[r].n; ++b)
          if (comp[r].v[a] > comp[r].v[b]) inv++;
    *makespan = m;
    *violations = inv + n_forced;
    if (start) memcpy(start, st, sizeof(int64_t) * (size_t)n);
    if (end) memcpy(end, en, sizeof(int64_t) * (size_t)n);
  }
  for (int32_t r = 0; r < nres; ++r) {
    free(queue[r].v);
    free(comp[r].v);
  }
  free(cands); free(counter); free(run_end); free(running); free(comp);
  free(queue); free(missing); free(ranked); free(en); free(st); free(forced);
  free(orig); free(gate);
  return rc_status;
}
