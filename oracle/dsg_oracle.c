/*
 * dsg_oracle.c — TEST INFRASTRUCTURE ONLY (the parity checker, never the
 * product).  Plain-C restatement of the reference max-load DP over ideals:
 *
 *   exact rationals          /root/reference/proj/src/rational.cpp:34-157
 *   NodeSet ops / lex / hash /root/reference/proj/src/graph.cpp:14-88
 *   Graph adjacency          /root/reference/proj/src/graph.cpp:132-158
 *   reachability_within      /root/reference/proj/src/graph.cpp:291-345
 *   is_contiguous            /root/reference/proj/src/graph.cpp:349-363
 *   combine_interleaving     /root/reference/proj/src/graph.cpp:457-467
 *   enumerate_impl           /root/reference/proj/src/ideals.cpp:14-75
 *   RatAccum / BlockTracker  /root/reference/proj/src/dp_solver.cpp:16-98
 *   replicated_load          /root/reference/proj/src/dp_solver.cpp:100-108
 *   MaxloadDp                /root/reference/proj/src/dp_solver.cpp:116-383
 *
 * Same visit orders as the reference (bitset index order, adjacency in edge
 * insertion order, DFS candidate order), so it reproduces the reference's
 * tie-breaking too, not only its optimum.  Pinned against the compiled
 * reference (oracle/_ref) and the committed golden vectors in tests/golden.
 */
#include "dsg_oracle.h"

#include <setjmp.h>
#include <stdarg.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>
#include <time.h>

typedef __int128 i128;

/* ------------------------------------------------------------------ ctx */

typedef struct {
  jmp_buf jb;
  int status;
  char msg[256];
  int64_t budget_limit;
  void** allocs;
  size_t n_allocs, cap_allocs;
} ctx_t;

static void ctx_fail(ctx_t* c, int status, const char* fmt, ...) {
  c->status = status;
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(c->msg, sizeof c->msg, fmt, ap);
  va_end(ap);
  longjmp(c->jb, 1);
}

static void* ctx_track(ctx_t* c, void* p) {
  if (!p) ctx_fail(c, DSG_INVALID, "out of host memory");
  if (c->n_allocs == c->cap_allocs) {
    size_t nc = c->cap_allocs ? 2 * c->cap_allocs : 64;
    void** na = (void**)realloc(c->allocs, nc * sizeof(void*));
    if (!na) {
      free(p);
      c->status = DSG_INVALID;
      snprintf(c->msg, sizeof c->msg, "out of host memory");
      longjmp(c->jb, 1);
    }
    c->allocs = na;
    c->cap_allocs = nc;
  }
  c->allocs[c->n_allocs++] = p;
  return p;
}

static void* cmalloc(ctx_t* c, size_t n) { return ctx_track(c, malloc(n && n < ((size_t)1 << 48) ? n : 1)); }
static void* ccalloc(ctx_t* c, size_t n, size_t s) {
  return ctx_track(c, calloc(n ? n : 1, s ? s : 1));
}
/* realloc of a tracked pointer: replace its slot */
static void* crealloc(ctx_t* c, void* p, size_t n) {
  if (!p) return cmalloc(c, n);
  void* q = realloc(p, n ? n : 1);
  if (!q) ctx_fail(c, DSG_INVALID, "out of host memory");
  for (size_t i = c->n_allocs; i-- > 0;) {
    if (c->allocs[i] == p) {
      c->allocs[i] = q;
      return q;
    }
  }
  return ctx_track(c, q);
}

static void ctx_free_all(ctx_t* c) {
  for (size_t i = 0; i < c->n_allocs; ++i) free(c->allocs[i]);
  free(c->allocs);
  c->allocs = NULL;
  c->n_allocs = c->cap_allocs = 0;
}

/* ------------------------------------------------------------ rationals */
/* rational.cpp:34-157 */

typedef struct {
  int64_t num, den; /* den == 0: +infinity (num 1) */
} rat;

static const rat RAT_ZERO = {0, 1};
static const rat RAT_INF = {1, 0};

static int rat_inf(rat a) { return a.den == 0; }

static i128 gcd128(i128 a, i128 b) {
  if (a < 0) a = -a;
  if (b < 0) b = -b;
  while (b != 0) {
    i128 t = a % b;
    a = b;
    b = t;
  }
  return a;
}

static int64_t narrow(ctx_t* c, i128 x) {
  if (x > (i128)INT64_MAX || x < (i128)INT64_MIN)
    ctx_fail(c, DSG_OVERFLOW, "rational overflow");
  return (int64_t)x;
}

static rat make_reduced(ctx_t* c, i128 num, i128 den) {
  if (den == 0) {
    if (num <= 0) ctx_fail(c, DSG_INVALID, "invalid rational");
    return RAT_INF;
  }
  if (den < 0) {
    den = -den;
    num = -num;
  }
  i128 g = gcd128(num, den);
  if (g > 1) {
    num /= g;
    den /= g;
  }
  rat r = {narrow(c, num), narrow(c, den)};
  return r;
}

static rat rat_from(ctx_t* c, dsg_rat x) {
  if (x.den == 0) {
    if (x.num <= 0) ctx_fail(c, DSG_INVALID, "invalid rational");
    return RAT_INF;
  }
  return make_reduced(c, x.num, x.den);
}

static rat rat_add(ctx_t* c, rat a, rat b) {
  if (rat_inf(a) || rat_inf(b)) return RAT_INF;
  return make_reduced(c, (i128)a.num * b.den + (i128)b.num * a.den,
                      (i128)a.den * b.den);
}

static rat rat_sub(ctx_t* c, rat a, rat b) {
  if (rat_inf(b)) ctx_fail(c, DSG_INVALID, "subtracting infinity");
  if (rat_inf(a)) return a;
  return make_reduced(c, (i128)a.num * b.den - (i128)b.num * a.den,
                      (i128)a.den * b.den);
}

static rat rat_mul(ctx_t* c, rat a, rat b) {
  if (rat_inf(a) || rat_inf(b)) {
    if ((!rat_inf(a) && a.num == 0) || (!rat_inf(b) && b.num == 0))
      ctx_fail(c, DSG_INVALID, "0 * infinity");
    if (a.num < 0 || b.num < 0) ctx_fail(c, DSG_INVALID, "negative * infinity");
    return RAT_INF;
  }
  return make_reduced(c, (i128)a.num * b.num, (i128)a.den * b.den);
}

static rat rat_div(ctx_t* c, rat a, rat b) {
  if (rat_inf(b)) ctx_fail(c, DSG_INVALID, "dividing by infinity");
  if (b.num == 0) ctx_fail(c, DSG_INVALID, "division by zero");
  if (rat_inf(a)) {
    if (b.num < 0) ctx_fail(c, DSG_INVALID, "infinity / negative");
    return a;
  }
  return make_reduced(c, (i128)a.num * b.den, (i128)a.den * b.num);
}

static int rat_lt(rat a, rat b) {
  if (rat_inf(a)) return 0;
  if (rat_inf(b)) return 1;
  return (i128)a.num * b.den < (i128)b.num * a.den;
}
static int rat_eq(rat a, rat b) { return a.num == b.num && a.den == b.den; }
static rat rat_max(rat a, rat b) { return rat_lt(a, b) ? b : a; }
static rat rat_int(int64_t v) {
  rat r = {v, 1};
  return r;
}

/* -------------------------------------------------------------- bitsets */

typedef uint64_t word;

static int bs_has(const word* s, int v) { return (int)((s[v >> 6] >> (v & 63)) & 1u); }
static void bs_set(word* s, int v) { s[v >> 6] |= (word)1 << (v & 63); }
static void bs_clr(word* s, int v) { s[v >> 6] &= ~((word)1 << (v & 63)); }

/* graph.cpp:81-88 (FNV-1a over words) */
static uint64_t bs_hash(const word* s, int W) {
  uint64_t h = 1469598103934665603ull;
  for (int i = 0; i < W; ++i) {
    h ^= s[i];
    h *= 1099511628211ull;
  }
  return h;
}

/* graph.cpp:62-72: the set containing the smallest differing index first */
static int bs_lex_less(const word* a, const word* b, int W) {
  for (int i = 0; i < W; ++i) {
    word diff = a[i] ^ b[i];
    if (diff) {
      word lowest = diff & (~diff + 1);
      return (a[i] & lowest) != 0;
    }
  }
  return 0;
}

static int bs_empty(const word* s, int W) {
  for (int i = 0; i < W; ++i)
    if (s[i]) return 0;
  return 1;
}

/* ---------------------------------------------------------------- graph */

typedef struct {
  int n;
  int W;
  int32_t* id;
  rat *cpu, *acc, *comm, *mem;
  uint8_t* bw;
  int32_t* pair_id; /* external id or DSG_NO_PAIR */
  /* CSR adjacency in edge insertion order (graph.cpp:145-157) */
  int *out_off, *out_adj, *in_off, *in_adj;         /* real */
  int *oall_off, *oall_adj, *iall_off, *iall_adj;   /* real + artificial */
} graph_t;

static int find_index(const graph_t* g, int32_t id) {
  /* first occurrence wins (graph.cpp:137-140); linear scan is fine here */
  for (int i = 0; i < g->n; ++i)
    if (g->id[i] == id) return i;
  return -1;
}

static void build_csr(ctx_t* c, int n, int m, const int* from, const int* to,
                      int** off_out, int** adj_out) {
  int* off = (int*)ccalloc(c, (size_t)n + 1, sizeof(int));
  int* adj = (int*)cmalloc(c, sizeof(int) * (size_t)(m ? m : 1));
  for (int e = 0; e < m; ++e) off[from[e] + 1]++;
  for (int i = 0; i < n; ++i) off[i + 1] += off[i];
  int* fill = (int*)cmalloc(c, sizeof(int) * (size_t)(n ? n : 1));
  for (int i = 0; i < n; ++i) fill[i] = off[i];
  for (int e = 0; e < m; ++e) adj[fill[from[e]]++] = to[e];
  *off_out = off;
  *adj_out = adj;
}

static void load_graph(ctx_t* c, const dsg_graph* dg, graph_t* g) {
  memset(g, 0, sizeof *g);
  int n = dg->n_nodes;
  if (n < 0) ctx_fail(c, DSG_INVALID, "negative node count");
  g->n = n;
  g->W = (n + 63) / 64;
  g->id = (int32_t*)cmalloc(c, sizeof(int32_t) * (size_t)(n ? n : 1));
  g->cpu = (rat*)cmalloc(c, sizeof(rat) * (size_t)(n ? n : 1));
  g->acc = (rat*)cmalloc(c, sizeof(rat) * (size_t)(n ? n : 1));
  g->comm = (rat*)cmalloc(c, sizeof(rat) * (size_t)(n ? n : 1));
  g->mem = (rat*)cmalloc(c, sizeof(rat) * (size_t)(n ? n : 1));
  g->bw = (uint8_t*)ccalloc(c, (size_t)n, 1);
  g->pair_id = (int32_t*)cmalloc(c, sizeof(int32_t) * (size_t)(n ? n : 1));
  for (int i = 0; i < n; ++i) {
    g->id[i] = dg->ids[i];
    g->cpu[i] = rat_from(c, dg->cpu_time[i]);
    g->acc[i] = rat_from(c, dg->acc_time[i]);
    g->comm[i] = rat_from(c, dg->comm_time[i]);
    g->mem[i] = rat_from(c, dg->mem_size[i]);
    g->bw[i] = dg->is_backward ? (dg->is_backward[i] != 0) : 0;
    g->pair_id[i] = dg->forward_pair ? dg->forward_pair[i] : DSG_NO_PAIR;
  }
  int mr = dg->n_edges, ma = dg->n_artificial;
  int* rf = (int*)cmalloc(c, sizeof(int) * (size_t)(mr + 1));
  int* rt = (int*)cmalloc(c, sizeof(int) * (size_t)(mr + 1));
  int* af = (int*)cmalloc(c, sizeof(int) * (size_t)(mr + ma + 1));
  int* at = (int*)cmalloc(c, sizeof(int) * (size_t)(mr + ma + 1));
  int nr = 0, na = 0;
  for (int e = 0; e < mr; ++e) {
    int f = find_index(g, dg->edge_from[e]), t = find_index(g, dg->edge_to[e]);
    if (f < 0 || t < 0) continue;
    rf[nr] = f;
    rt[nr] = t;
    ++nr;
    af[na] = f;
    at[na] = t;
    ++na;
  }
  for (int e = 0; e < ma; ++e) {
    int f = find_index(g, dg->art_from[e]), t = find_index(g, dg->art_to[e]);
    if (f < 0 || t < 0) continue;
    af[na] = f;
    at[na] = t;
    ++na;
  }
  build_csr(c, n, nr, rf, rt, &g->out_off, &g->out_adj);
  build_csr(c, n, nr, rt, rf, &g->in_off, &g->in_adj);
  build_csr(c, n, na, af, at, &g->oall_off, &g->oall_adj);
  build_csr(c, n, na, at, af, &g->iall_off, &g->iall_adj);
}

#define FOR_ADJ(off, adj, v, w) \
  for (int _k = (off)[v], w; _k < (off)[(v) + 1] && ((w = (adj)[_k]), 1); ++_k)

/* ---------------------------------------------------- ideal enumeration */
/* ideals.cpp:14-75 + IdealIndex::ordinal_of graph.cpp:386-393 */

typedef struct {
  int W;
  int64_t count, cap;
  word* bits; /* count * W */
  /* open-addressing ordinal lookup keyed by the NodeSet */
  int64_t* table;
  int64_t tcap;
  int64_t* level_off;
  int n_levels;
} index_t;

static word* idx_at(const index_t* ix, int64_t ord) { return ix->bits + (size_t)ord * ix->W; }

static void idx_table_insert(index_t* ix, int64_t ord) {
  uint64_t h = bs_hash(idx_at(ix, ord), ix->W);
  int64_t m = ix->tcap - 1;
  int64_t p = (int64_t)(h & (uint64_t)m);
  while (ix->table[p] >= 0) p = (p + 1) & m;
  ix->table[p] = ord;
}

static int64_t idx_ordinal_of(const index_t* ix, const word* s) {
  uint64_t h = bs_hash(s, ix->W);
  int64_t m = ix->tcap - 1;
  int64_t p = (int64_t)(h & (uint64_t)m);
  while (ix->table[p] >= 0) {
    if (memcmp(idx_at(ix, ix->table[p]), s, sizeof(word) * ix->W) == 0) return ix->table[p];
    p = (p + 1) & m;
  }
  return -1;
}

static int g_sort_W; /* qsort has no context argument */
static int cmp_lex(const void* a, const void* b) {
  const word* x = (const word*)a;
  const word* y = (const word*)b;
  if (bs_lex_less(x, y, g_sort_W)) return -1;
  if (bs_lex_less(y, x, g_sort_W)) return 1;
  return 0;
}

static void idx_push(ctx_t* c, index_t* ix, const word* s) {
  if (ix->count == ix->cap) {
    ix->cap = ix->cap ? ix->cap * 2 : 64;
    ix->bits = (word*)crealloc(c, ix->bits, sizeof(word) * (size_t)ix->cap * ix->W);
  }
  memcpy(idx_at(ix, ix->count), s, sizeof(word) * ix->W);
  ix->count++;
}

static void enumerate_impl(ctx_t* c, const graph_t* g, const word* within,
                           int64_t budget, index_t* ix) {
  int W = g->W;
  memset(ix, 0, sizeof *ix);
  ix->W = W;
  word* empty = (word*)ccalloc(c, (size_t)W, sizeof(word));
  idx_push(c, ix, empty);
  int levels_cap = g->n + 2;
  ix->level_off = (int64_t*)cmalloc(c, sizeof(int64_t) * (size_t)(levels_cap + 1));
  ix->level_off[0] = 0;
  ix->n_levels = 0;

  int* eligible = (int*)cmalloc(c, sizeof(int) * (size_t)(g->n + 1));
  int n_el = 0;
  for (int v = 0; v < g->n; ++v)
    if (!within || bs_has(within, v)) eligible[n_el++] = v;

  int64_t lvl_begin = 0, lvl_end = 1;
  word* next = NULL;
  int64_t next_n = 0, next_cap = 0;
  /* hash set over `next` (seen hashes + equality scan, ideals.cpp:49-63);
   * an exact open-addressing set gives the same dedup result. */
  int64_t* seen = NULL;
  int64_t seen_cap = 0;
  word* grown = (word*)cmalloc(c, sizeof(word) * (size_t)W);
  word* base = (word*)cmalloc(c, sizeof(word) * (size_t)W);
  while (lvl_end > lvl_begin) {
    ix->level_off[++ix->n_levels] = lvl_end;
    next_n = 0;
    if (seen_cap < 1024) {
      seen_cap = 1024;
      seen = (int64_t*)crealloc(c, seen, sizeof(int64_t) * (size_t)seen_cap);
    }
    for (int64_t i = 0; i < seen_cap; ++i) seen[i] = -1;
    for (int64_t ord = lvl_begin; ord < lvl_end; ++ord) {
      memcpy(base, idx_at(ix, ord), sizeof(word) * W);
      for (int e = 0; e < n_el; ++e) {
        int v = eligible[e];
        if (bs_has(base, v)) continue;
        int closed = 1;
        FOR_ADJ(g->iall_off, g->iall_adj, v, u) {
          if (within && !bs_has(within, u)) continue;
          if (!bs_has(base, u)) {
            closed = 0;
            break;
          }
        }
        if (!closed) continue;
        memcpy(grown, base, sizeof(word) * W);
        bs_set(grown, v);
        /* dedup */
        uint64_t h = bs_hash(grown, W);
        int64_t m = seen_cap - 1;
        int64_t p = (int64_t)(h & (uint64_t)m);
        int dup = 0;
        while (seen[p] >= 0) {
          if (memcmp(next + (size_t)seen[p] * W, grown, sizeof(word) * W) == 0) {
            dup = 1;
            break;
          }
          p = (p + 1) & m;
        }
        if (dup) continue;
        if (next_n == next_cap) {
          next_cap = next_cap ? 2 * next_cap : 64;
          next = (word*)crealloc(c, next, sizeof(word) * (size_t)next_cap * W);
        }
        memcpy(next + (size_t)next_n * W, grown, sizeof(word) * W);
        seen[p] = next_n;
        ++next_n;
        if (2 * next_n > seen_cap) { /* rehash */
          seen_cap *= 4;
          seen = (int64_t*)crealloc(c, seen, sizeof(int64_t) * (size_t)seen_cap);
          for (int64_t i = 0; i < seen_cap; ++i) seen[i] = -1;
          for (int64_t i = 0; i < next_n; ++i) {
            uint64_t hh = bs_hash(next + (size_t)i * W, W);
            int64_t mm = seen_cap - 1, q = (int64_t)(hh & (uint64_t)mm);
            while (seen[q] >= 0) q = (q + 1) & mm;
            seen[q] = i;
          }
        }
      }
    }
    /* std::sort(next, lex_less) — elements are distinct, so any correct
     * sort yields the same order (ideals.cpp:66) */
    g_sort_W = W;
    if (next_n > 1) qsort(next, (size_t)next_n, sizeof(word) * W, cmp_lex);
    lvl_begin = lvl_end;
    for (int64_t i = 0; i < next_n; ++i) {
      if (ix->count >= budget) { /* ideals.cpp:69 */
        c->budget_limit = budget;
        ctx_fail(c, DSG_BUDGET, "ideal budget %lld exceeded", (long long)budget);
      }
      idx_push(c, ix, next + (size_t)i * W);
    }
    lvl_end = ix->count;
  }
  /* ordinal lookup table */
  ix->tcap = 16;
  while (ix->tcap < 2 * ix->count + 2) ix->tcap *= 2;
  ix->table = (int64_t*)cmalloc(c, sizeof(int64_t) * (size_t)ix->tcap);
  for (int64_t i = 0; i < ix->tcap; ++i) ix->table[i] = -1;
  for (int64_t i = 0; i < ix->count; ++i) idx_table_insert(ix, i);
}

/* ------------------------------------------------------- reachability */
/* graph.cpp:291-345 (within variant), 349-363 */

typedef struct {
  int n, stride;
  word* from;
  word* to;
} reach_t;

static void reachability_within(ctx_t* c, const graph_t* g, const word* within,
                                reach_t* r) {
  int n = g->n;
  r->n = n;
  r->stride = (n + 63) / 64;
  r->from = (word*)ccalloc(c, (size_t)n * r->stride + 1, sizeof(word));
  r->to = (word*)ccalloc(c, (size_t)n * r->stride + 1, sizeof(word));
  int* indeg = (int*)ccalloc(c, (size_t)n + 1, sizeof(int));
  int* order = (int*)cmalloc(c, sizeof(int) * (size_t)(n + 1));
  int* ready = (int*)cmalloc(c, sizeof(int) * (size_t)(n + 1));
  int n_order = 0, n_ready = 0;
  for (int v = 0; v < n; ++v) {
    if (!bs_has(within, v)) continue;
    FOR_ADJ(g->oall_off, g->oall_adj, v, w) {
      if (bs_has(within, w)) ++indeg[w];
    }
  }
  for (int v = n - 1; v >= 0; --v)
    if (bs_has(within, v) && indeg[v] == 0) ready[n_ready++] = v;
  while (n_ready > 0) {
    int v = ready[--n_ready];
    order[n_order++] = v;
    FOR_ADJ(g->oall_off, g->oall_adj, v, w) {
      if (bs_has(within, w) && --indeg[w] == 0) ready[n_ready++] = w;
    }
  }
  for (int i = n_order - 1; i >= 0; --i) {
    int u = order[i];
    word* ru = r->from + (size_t)u * r->stride;
    bs_set(ru, u);
    FOR_ADJ(g->oall_off, g->oall_adj, u, w) {
      if (!bs_has(within, w)) continue;
      const word* rw = r->from + (size_t)w * r->stride;
      for (int k = 0; k < r->stride; ++k) ru[k] |= rw[k];
    }
  }
  for (int u = 0; u < n; ++u) {
    if (!bs_has(within, u)) continue;
    const word* ru = r->from + (size_t)u * r->stride;
    for (int w = 0; w < n; ++w)
      if (bs_has(ru, w)) bs_set(r->to + (size_t)w * r->stride, u);
  }
}

static int is_contiguous(const reach_t* r, const word* s, word* tmp_from, word* tmp_to) {
  int S = r->stride;
  memset(tmp_from, 0, sizeof(word) * S);
  memset(tmp_to, 0, sizeof(word) * S);
  for (int u = 0; u < r->n; ++u) {
    if (!bs_has(s, u)) continue;
    const word* rf = r->from + (size_t)u * S;
    const word* rt = r->to + (size_t)u * S;
    for (int k = 0; k < S; ++k) {
      tmp_from[k] |= rf[k];
      tmp_to[k] |= rt[k];
    }
  }
  for (int k = 0; k < S; ++k)
    if ((tmp_from[k] & tmp_to[k]) & ~s[k]) return 0;
  return 1;
}

/* ---------------------------------------------------------- DP engine */

typedef struct {
  rat finite;
  int inf_count;
} accum_t;

static void accum_add(ctx_t* c, accum_t* a, rat r) {
  if (rat_inf(r)) ++a->inf_count;
  else a->finite = rat_add(c, a->finite, r);
}
static void accum_sub(ctx_t* c, accum_t* a, rat r) {
  if (rat_inf(r)) --a->inf_count;
  else a->finite = rat_sub(c, a->finite, r);
}
static rat accum_total(const accum_t* a) { return a->inf_count > 0 ? RAT_INF : a->finite; }

typedef struct {
  const graph_t* g;
  int* into_c;
  uint8_t* in_c;
  accum_t comm_in, comm_out;
  rat proc, cpu, mem;
  int unsupported;
  word* bw_members;
} tracker_t;

static int outdeg(const graph_t* g, int v) { return g->out_off[v + 1] - g->out_off[v]; }

/* dp_solver.cpp:50-68 */
static void tracker_add(ctx_t* c, tracker_t* t, int x) {
  const graph_t* g = t->g;
  FOR_ADJ(g->in_off, g->in_adj, x, u) {
    int old = t->into_c[u]++;
    if (t->in_c[u]) {
      if (old + 1 == outdeg(g, u)) accum_sub(c, &t->comm_out, g->comm[u]);
    } else if (old == 0) {
      accum_add(c, &t->comm_in, g->comm[u]);
    }
  }
  if (t->into_c[x] > 0) accum_sub(c, &t->comm_in, g->comm[x]);
  t->in_c[x] = 1;
  if (t->into_c[x] < outdeg(g, x)) accum_add(c, &t->comm_out, g->comm[x]);
  if (!rat_inf(g->acc[x])) t->proc = rat_add(c, t->proc, g->acc[x]);
  else ++t->unsupported;
  t->cpu = rat_add(c, t->cpu, g->cpu[x]);
  t->mem = rat_add(c, t->mem, g->mem[x]);
  if (g->bw[x]) bs_set(t->bw_members, x);
}

/* dp_solver.cpp:70-88 */
static void tracker_remove(ctx_t* c, tracker_t* t, int x) {
  const graph_t* g = t->g;
  if (g->bw[x]) bs_clr(t->bw_members, x);
  t->mem = rat_sub(c, t->mem, g->mem[x]);
  t->cpu = rat_sub(c, t->cpu, g->cpu[x]);
  if (!rat_inf(g->acc[x])) t->proc = rat_sub(c, t->proc, g->acc[x]);
  else --t->unsupported;
  if (t->into_c[x] < outdeg(g, x)) accum_sub(c, &t->comm_out, g->comm[x]);
  t->in_c[x] = 0;
  if (t->into_c[x] > 0) accum_add(c, &t->comm_in, g->comm[x]);
  FOR_ADJ(g->in_off, g->in_adj, x, u) {
    int old = t->into_c[u]--;
    if (t->in_c[u]) {
      if (old == outdeg(g, u)) accum_add(c, &t->comm_out, g->comm[u]);
    } else if (old == 1) {
      accum_sub(c, &t->comm_in, g->comm[u]);
    }
  }
}

/* graph.cpp:457-467 */
static rat combine(ctx_t* c, rat in, rat proc, rat out, int mode) {
  switch (mode) {
    case DSG_INTERLEAVE_SUM:
      return rat_add(c, rat_add(c, in, proc), out);
    case DSG_INTERLEAVE_HALF_DUPLEX_MAX:
      return rat_max(proc, rat_add(c, in, out));
    case DSG_INTERLEAVE_FULL_DUPLEX_MAX:
      return rat_max(proc, rat_max(in, out));
  }
  return RAT_ZERO;
}

typedef struct {
  int prev;
  int8_t kind; /* 0 none, 1 acc, 2 cpu, 3 waste acc, 4 waste cpu */
  int16_t repl;
} backptr_t;

typedef struct {
  ctx_t* c;
  const graph_t* g;
  int training, replication;
  int K, L;
  rat mem_limit;
  int interleaving;
  int has_bandwidth;
  rat bandwidth;
  int repl_combine;
  word* universe;
  index_t index;
  int** paired_bw; /* fw dense idx -> list, terminated by -1 */
  int* paired_cnt;
  int has_bw_reach;
  reach_t bw_reach;
  rat* dp;
  backptr_t* bp;
  int64_t* stamp;
  int64_t deadline_tick;
  int has_deadline;
  struct timespec deadline;
  int64_t pairs;
  word *tmp_a, *tmp_b;
} dp_t;

static size_t cell(const dp_t* d, int64_t ord, int k, int l) {
  return ((size_t)ord * (d->K + 1) + k) * (d->L + 1) + l;
}

/* dp_solver.cpp:172-178 */
static void check_deadline(dp_t* d) {
  if (!d->has_deadline) return;
  if ((++d->deadline_tick & 1023) != 0) return;
  struct timespec now;
  clock_gettime(CLOCK_MONOTONIC, &now);
  if (now.tv_sec > d->deadline.tv_sec ||
      (now.tv_sec == d->deadline.tv_sec && now.tv_nsec > d->deadline.tv_nsec))
    ctx_fail(d->c, DSG_DEADLINE, "time limit reached");
}

/* dp_solver.cpp:180-193 */
static void monotone_pass(dp_t* d, int64_t ord) {
  for (int k = 0; k <= d->K; ++k) {
    for (int l = 0; l <= d->L; ++l) {
      size_t here = cell(d, ord, k, l);
      if (k > 0 && rat_lt(d->dp[cell(d, ord, k - 1, l)], d->dp[here])) {
        d->dp[here] = d->dp[cell(d, ord, k - 1, l)];
        backptr_t b = {(int)ord, 3, 1};
        d->bp[here] = b;
      }
      if (l > 0 && rat_lt(d->dp[cell(d, ord, k, l - 1)], d->dp[here])) {
        d->dp[here] = d->dp[cell(d, ord, k, l - 1)];
        backptr_t b = {(int)ord, 4, 1};
        d->bp[here] = b;
      }
    }
  }
}

/* dp_solver.cpp:90-97 */
static rat acc_load(dp_t* d, const tracker_t* t) {
  if (t->unsupported > 0 || rat_lt(d->mem_limit, t->mem)) return RAT_INF;
  rat in = accum_total(&t->comm_in), out = accum_total(&t->comm_out);
  if (rat_inf(in) || rat_inf(out)) return RAT_INF;
  return combine(d->c, in, t->proc, out, d->interleaving);
}

/* dp_solver.cpp:100-108 */
static rat replicated_load(dp_t* d, rat base, rat block_mem, int r) {
  if (r <= 1 || rat_inf(base)) return base;
  ctx_t* c = d->c;
  rat divided = rat_div(c, base, rat_int(r));
  rat sync = rat_div(c, rat_mul(c, rat_int(r - 1), block_mem),
                     rat_mul(c, rat_int(r), d->bandwidth));
  return d->repl_combine == DSG_REPL_SUM ? rat_add(c, divided, sync)
                                         : rat_max(divided, sync);
}

/* dp_solver.cpp:197-233 */
static void apply_candidate(dp_t* d, int64_t ord, int64_t sub, const tracker_t* t) {
  check_deadline(d);
  d->pairs++;
  if (d->training && d->has_bw_reach && !bs_empty(t->bw_members, d->g->W) &&
      !is_contiguous(&d->bw_reach, t->bw_members, d->tmp_a, d->tmp_b))
    return;
  rat acc_base = acc_load(d, t);
  rat cpu_load = t->cpu;
  for (int k = 0; k <= d->K; ++k) {
    for (int l = 0; l <= d->L; ++l) {
      rat* target = &d->dp[cell(d, ord, k, l)];
      if (k >= 1 && !rat_inf(acc_base)) {
        int max_r = d->replication ? k : 1;
        for (int r = 1; r <= max_r; ++r) {
          rat rest = d->dp[cell(d, sub, k - r, l)];
          if (rat_inf(rest)) continue;
          rat load = replicated_load(d, acc_base, t->mem, r);
          rat val = rat_max(rest, load);
          if (rat_lt(val, *target)) {
            *target = val;
            backptr_t b = {(int)sub, 1, (int16_t)r};
            d->bp[cell(d, ord, k, l)] = b;
          }
        }
      }
      if (l >= 1) {
        rat rest = d->dp[cell(d, sub, k, l - 1)];
        if (!rat_inf(rest)) {
          rat val = rat_max(rest, cpu_load);
          if (rat_lt(val, *target)) {
            *target = val;
            backptr_t b = {(int)sub, 2, 1};
            d->bp[cell(d, ord, k, l)] = b;
          }
        }
      }
    }
  }
}

static void push_block_nodes(dp_t* d, tracker_t* t, int fw, int add) {
  if (add) {
    tracker_add(d->c, t, fw);
    if (d->training)
      for (int i = 0; i < d->paired_cnt[fw]; ++i) tracker_add(d->c, t, d->paired_bw[fw][i]);
  } else {
    if (d->training)
      for (int i = d->paired_cnt[fw] - 1; i >= 0; --i) tracker_remove(d->c, t, d->paired_bw[fw][i]);
    tracker_remove(d->c, t, fw);
  }
}

typedef struct {
  int* cand;
  int n_cand;
  int next;
  int removed;
} frame_t;

/* dp_solver.cpp:256-317 */
static void walk_subideals(dp_t* d, int64_t ord, tracker_t* t, word* current, int* out_cnt,
                           frame_t* stack, int* cand_pool) {
  const graph_t* g = d->g;
  int W = g->W;
  ctx_t* c = d->c;
  /* reset tracker */
  memset(t->into_c, 0, sizeof(int) * (size_t)g->n);
  memset(t->in_c, 0, (size_t)g->n);
  t->comm_in.finite = RAT_ZERO;
  t->comm_in.inf_count = 0;
  t->comm_out = t->comm_in;
  t->proc = t->cpu = t->mem = RAT_ZERO;
  t->unsupported = 0;
  memset(t->bw_members, 0, sizeof(word) * W);

  memcpy(current, idx_at(&d->index, ord), sizeof(word) * W);
  int pool_top = 0;
  int* initial = cand_pool + pool_top;
  int n_init = 0;
  for (int v = 0; v < g->n; ++v) {
    if (!bs_has(current, v)) continue;
    int cnt = 0;
    FOR_ADJ(g->oall_off, g->oall_adj, v, w) {
      if (bs_has(current, w)) ++cnt;
    }
    out_cnt[v] = cnt;
    if (cnt == 0) initial[n_init++] = v;
  }
  pool_top += n_init;
  int depth = 0;
  stack[0].cand = initial;
  stack[0].n_cand = n_init;
  stack[0].next = 0;
  stack[0].removed = -1;
  depth = 1;
  while (depth > 0) {
    frame_t* f = &stack[depth - 1];
    if (f->next < f->n_cand) {
      int v = f->cand[f->next++];
      bs_clr(current, v);
      int64_t sub = idx_ordinal_of(&d->index, current);
      if (sub < 0) ctx_fail(c, DSG_LOGIC, "sub-ideal lookup failed");
      if (d->stamp[sub] == ord) {
        bs_set(current, v);
        continue;
      }
      d->stamp[sub] = ord;
      int* child = cand_pool + pool_top;
      int n_child = 0;
      for (int i = 0; i < f->n_cand; ++i)
        if (f->cand[i] != v) child[n_child++] = f->cand[i];
      FOR_ADJ(g->iall_off, g->iall_adj, v, u) {
        if (bs_has(current, u) && --out_cnt[u] == 0) child[n_child++] = u;
      }
      pool_top += n_child;
      push_block_nodes(d, t, v, 1);
      apply_candidate(d, ord, sub, t);
      frame_t* nf = &stack[depth++];
      nf->cand = child;
      nf->n_cand = n_child;
      nf->next = 0;
      nf->removed = v;
    } else {
      int v = f->removed;
      pool_top -= f->n_cand;
      if (depth == 1) pool_top = 0;
      --depth;
      if (v >= 0) {
        push_block_nodes(d, t, v, 0);
        FOR_ADJ(g->iall_off, g->iall_adj, v, u) {
          if (bs_has(current, u)) ++out_cnt[u];
        }
        bs_set(current, v);
      }
    }
  }
}

static void set_deadline(dp_t* d, const dsg_options* o) {
  d->has_deadline = 0;
  if (!o || !(o->deadline_seconds > 0)) return;
  d->has_deadline = 1;
  clock_gettime(CLOCK_MONOTONIC, &d->deadline);
  double s = o->deadline_seconds;
  long sec = (long)s;
  long ns = (long)((s - (double)sec) * 1e9);
  d->deadline.tv_sec += sec;
  d->deadline.tv_nsec += ns;
  if (d->deadline.tv_nsec >= 1000000000L) {
    d->deadline.tv_sec += 1;
    d->deadline.tv_nsec -= 1000000000L;
  }
}

static void fill_result_rat(dsg_rat* out, rat r) {
  out->num = r.num;
  out->den = r.den;
}

static double now_ms(void) {
  struct timespec t;
  clock_gettime(CLOCK_MONOTONIC, &t);
  return (double)t.tv_sec * 1e3 + (double)t.tv_nsec * 1e-6;
}

static void solve(ctx_t* c, int mode, const dsg_graph* dg, const dsg_config* cfg,
                  const dsg_options* opt, dsg_result* res) {
  double t0 = now_ms();
  graph_t g;
  load_graph(c, dg, &g);
  dp_t d;
  memset(&d, 0, sizeof d);
  d.c = c;
  d.g = &g;
  d.training = mode == DSG_MODE_TRAINING;
  d.replication = mode == DSG_MODE_REPLICATED;
  d.K = cfg->accelerators;
  d.L = cfg->cpus;
  d.mem_limit = rat_from(c, cfg->memory_limit);
  d.interleaving = cfg->interleaving;
  d.has_bandwidth = cfg->has_bandwidth;
  if (cfg->has_bandwidth) d.bandwidth = rat_from(c, cfg->bandwidth);
  d.repl_combine = cfg->replication_combine;
  int W = g.W;
  if (mode == DSG_MODE_REPLICATED) { /* dp_solver.cpp:397-405 */
    if (!cfg->has_bandwidth) ctx_fail(c, DSG_MISSING_BANDWIDTH, "replication requires a bandwidth value");
    for (int i = 0; i < g.n; ++i)
      if (g.bw[i]) ctx_fail(c, DSG_INVALID, "replicated solve expects an inference graph");
  }
  /* MaxloadDp ctor, dp_solver.cpp:133-166 */
  if (d.K + d.L < 1) ctx_fail(c, DSG_INVALID, "need at least one device");
  if (d.replication && !d.has_bandwidth) ctx_fail(c, DSG_MISSING_BANDWIDTH, "replication requires a bandwidth value");
  d.universe = (word*)ccalloc(c, (size_t)W + 1, sizeof(word));
  d.paired_cnt = (int*)ccalloc(c, (size_t)g.n + 1, sizeof(int));
  d.paired_bw = (int**)ccalloc(c, (size_t)g.n + 1, sizeof(int*));
  if (d.training) {
    for (int v = 0; v < g.n; ++v)
      if (!g.bw[v]) bs_set(d.universe, v);
    for (int b = 0; b < g.n; ++b) {
      if (!g.bw[b]) continue;
      if (g.pair_id[b] == DSG_NO_PAIR)
        ctx_fail(c, DSG_INVALID,
                 "training solve requires every backward node to be paired "
                 "(run preprocessing first)");
      int f = find_index(&g, g.pair_id[b]);
      if (f < 0) ctx_fail(c, DSG_INVALID, "forward_pair references missing node");
      d.paired_cnt[f]++;
    }
    for (int v = 0; v < g.n; ++v)
      d.paired_bw[v] = (int*)cmalloc(c, sizeof(int) * (size_t)(d.paired_cnt[v] + 1));
    int* fill = (int*)ccalloc(c, (size_t)g.n + 1, sizeof(int));
    for (int b = 0; b < g.n; ++b) {
      if (!g.bw[b]) continue;
      int f = find_index(&g, g.pair_id[b]);
      d.paired_bw[f][fill[f]++] = b;
    }
    word* bw = (word*)ccalloc(c, (size_t)W + 1, sizeof(word));
    for (int v = 0; v < g.n; ++v)
      if (g.bw[v]) bs_set(bw, v);
    if (!bs_empty(bw, W)) {
      d.has_bw_reach = 1;
      reachability_within(c, &g, bw, &d.bw_reach);
    }
  } else {
    for (int v = 0; v < g.n; ++v) bs_set(d.universe, v);
  }
  int64_t budget = opt ? opt->ideal_budget : DSG_DEFAULT_IDEAL_BUDGET;
  double t1 = now_ms();
  enumerate_impl(c, &g, d.universe, budget, &d.index);
  double t2 = now_ms();
  set_deadline(&d, opt);

  /* run(), dp_solver.cpp:319-382 */
  int64_t I = d.index.count;
  size_t cells = (size_t)I * (d.K + 1) * (d.L + 1);
  d.dp = (rat*)cmalloc(c, sizeof(rat) * cells);
  d.bp = (backptr_t*)cmalloc(c, sizeof(backptr_t) * cells);
  for (size_t i = 0; i < cells; ++i) {
    d.dp[i] = RAT_INF;
    backptr_t b = {-1, 0, 1};
    d.bp[i] = b;
  }
  d.stamp = (int64_t*)cmalloc(c, sizeof(int64_t) * (size_t)I);
  for (int64_t i = 0; i < I; ++i) d.stamp[i] = -1;
  tracker_t t;
  memset(&t, 0, sizeof t);
  t.g = &g;
  t.into_c = (int*)ccalloc(c, (size_t)g.n + 1, sizeof(int));
  t.in_c = (uint8_t*)ccalloc(c, (size_t)g.n + 1, 1);
  t.bw_members = (word*)ccalloc(c, (size_t)W + 1, sizeof(word));
  word* current = (word*)ccalloc(c, (size_t)W + 1, sizeof(word));
  int* out_cnt = (int*)ccalloc(c, (size_t)g.n + 1, sizeof(int));
  frame_t* stack = (frame_t*)ccalloc(c, (size_t)g.n + 2, sizeof(frame_t));
  /* a DFS path has depth <= |I|; frames hold <= n candidates plus in-degree
   * additions, so pool <= (n + 1) * (n + max indegree + 1) */
  size_t pool = (size_t)(g.n + 2) * (size_t)(g.n + g.iall_off[g.n] + 2);
  int* cand_pool = (int*)cmalloc(c, sizeof(int) * pool);
  d.tmp_a = (word*)ccalloc(c, (size_t)W + 1, sizeof(word));
  d.tmp_b = (word*)ccalloc(c, (size_t)W + 1, sizeof(word));

  d.dp[cell(&d, 0, 0, 0)] = RAT_ZERO;
  monotone_pass(&d, 0);
  for (int64_t ord = 1; ord < I; ++ord) {
    walk_subideals(&d, ord, &t, current, out_cnt, stack, cand_pool);
    monotone_pass(&d, ord);
  }
  int64_t full = I - 1;
  rat best = d.dp[cell(&d, full, d.K, d.L)];
  res->n_ideals = I;
  res->n_pairs = d.pairs;
  res->n_levels = d.index.n_levels;
  if (rat_inf(best)) ctx_fail(c, DSG_INFEASIBLE, "no feasible assignment exists");
  int bk = d.K, bl = d.L;
  for (int total = 0; total <= d.K + d.L; ++total) {
    int found = 0;
    int klo = total - d.L > 0 ? total - d.L : 0;
    int khi = d.K < total ? d.K : total;
    for (int k = klo; k <= khi; ++k) {
      int l = total - k;
      if (rat_eq(d.dp[cell(&d, full, k, l)], best)) {
        bk = k;
        bl = l;
        found = 1;
        break;
      }
    }
    if (found) break;
  }
  /* traceback, dp_solver.cpp:353-380 */
  int max_blocks = d.K + d.L + 1;
  dsg_block* blocks = (dsg_block*)calloc((size_t)max_blocks, sizeof(dsg_block));
  int* members = (int*)malloc(sizeof(int) * (size_t)(g.n + 1));
  int n_blocks = 0, n_members = 0;
  int64_t ord = full;
  int k = bk, l = bl;
  while (!(ord == 0 && k == 0 && l == 0)) {
    backptr_t b = d.bp[cell(&d, ord, k, l)];
    if (b.kind == 0) {
      free(blocks);
      free(members);
      ctx_fail(c, DSG_LOGIC, "dp reconstruction stuck");
    }
    if (b.kind == 3) {
      --k;
      continue;
    }
    if (b.kind == 4) {
      --l;
      continue;
    }
    const word* a = idx_at(&d.index, ord);
    const word* p = idx_at(&d.index, b.prev);
    dsg_block* blk = &blocks[n_blocks++];
    blk->cpu = b.kind == 2;
    blk->repl = b.repl;
    blk->offset = n_members;
    for (int v = 0; v < g.n; ++v) {
      if (bs_has(a, v) && !bs_has(p, v)) {
        members[n_members++] = v;
        if (d.training)
          for (int i = 0; i < d.paired_cnt[v]; ++i) members[n_members++] = d.paired_bw[v][i];
      }
    }
    blk->n_members = n_members - blk->offset;
    if (b.kind == 1) k -= b.repl;
    else --l;
    ord = b.prev;
  }
  double t3 = now_ms();
  fill_result_rat(&res->objective, best);
  res->best_k = bk;
  res->best_l = bl;
  res->n_blocks = n_blocks;
  res->blocks = blocks;
  res->members = members;
  res->value_bits = 0;
  res->denominator = 0;
  res->t_prepare_ms = t1 - t0;
  res->t_enumerate_ms = t2 - t1;
  res->t_dp_ms = t3 - t2;
  res->t_total_ms = t3 - t0;
  if (opt && (opt->flags & DSG_FLAG_KEEP_TABLES)) {
    res->words = W;
    res->ideal_bits = (uint64_t*)malloc(sizeof(word) * (size_t)I * W + 1);
    memcpy(res->ideal_bits, d.index.bits, sizeof(word) * (size_t)I * W);
  }
}

int dsgo_dp_solve(int32_t mode, const dsg_graph* graph, const dsg_config* config,
                  const dsg_options* options, dsg_result* result) {
  memset(result, 0, sizeof *result);
  ctx_t c;
  memset(&c, 0, sizeof c);
  if (setjmp(c.jb) == 0) {
    solve(&c, mode, graph, config, options, result);
    c.status = DSG_OK;
  } else {
    result->budget_limit = c.budget_limit;
  }
  result->status = c.status;
  memcpy(result->message, c.msg, sizeof result->message);
  ctx_free_all(&c);
  return c.status;
}

void dsgo_result_free(dsg_result* r) {
  if (!r) return;
  free(r->blocks);
  free(r->members);
  free(r->ideal_bits);
  free(r->dp_values);
  r->blocks = NULL;
  r->members = NULL;
  r->ideal_bits = NULL;
  r->dp_values = NULL;
}

int dsgo_enumerate_ideals(const dsg_graph* graph, const uint8_t* within, int64_t budget,
                          const dsg_options* options, dsg_ideals* out) {
  (void)options;
  memset(out, 0, sizeof *out);
  ctx_t c;
  memset(&c, 0, sizeof c);
  if (setjmp(c.jb) == 0) {
    double t0 = now_ms();
    graph_t g;
    load_graph(&c, graph, &g);
    word* w = NULL;
    if (within) {
      w = (word*)ccalloc(&c, (size_t)g.W + 1, sizeof(word));
      for (int v = 0; v < g.n; ++v)
        if (within[v]) bs_set(w, v);
    }
    index_t ix;
    enumerate_impl(&c, &g, w, budget, &ix);
    out->count = ix.count;
    out->words = g.W;
    out->bits = (uint64_t*)malloc(sizeof(word) * (size_t)ix.count * g.W + 1);
    memcpy(out->bits, ix.bits, sizeof(word) * (size_t)ix.count * g.W);
    out->n_levels = ix.n_levels;
    out->level_offsets = (int64_t*)malloc(sizeof(int64_t) * (size_t)(ix.n_levels + 1));
    memcpy(out->level_offsets, ix.level_off, sizeof(int64_t) * (size_t)ix.n_levels);
    out->level_offsets[ix.n_levels] = ix.count;
    out->t_ms = now_ms() - t0;
    c.status = DSG_OK;
  } else {
    out->budget_limit = c.budget_limit;
  }
  out->status = c.status;
  memcpy(out->message, c.msg, sizeof out->message);
  ctx_free_all(&c);
  return c.status;
}

void dsgo_ideals_free(dsg_ideals* out) {
  if (!out) return;
  free(out->bits);
  free(out->level_offsets);
  out->bits = NULL;
  out->level_offsets = NULL;
}
