/*
 * tm_oracle.c — CPU restatement of the reference mining semantics.
 *
 * TEST INFRASTRUCTURE ONLY.  This file is the *checker* for the B200 path:
 * only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline /
 * `--impl reference` leg may load it.  The product library
 * (paper_2604_12241_b200/csrc) never links or calls it.
 *
 * It restates, per trigger edge e = (u -> v, t) with window [t - delta, t]
 * (closed, by timestamp only; pkg/docs/pattern_grammar.md:56-60), the column
 * formulas of the reference:
 *   fan / degree     kernels.py:290-303  (batch_fan_degree), :62-101
 *   cycle_2/3/4      kernels.py:306-345  (batch_cycle)
 *   sg_count         kernels.py:348-376  (batch_scatter_gather)
 *   stack_count      kernels.py:379-402  (batch_stack)
 *   cycle_5..8, gs   generic interpreter engine.py:516-562 / 325-430 run on
 *                    the SURVEY.md Appendix B DSL (set_cardinality per
 *                    binding, engine.py:462-464; source_count :483-485)
 * Conventions restated from kernels.py:9-13 and txgraph.py:113-170:
 * adjacency runs sorted by (time, edge id); self-loops never appear in any
 * iteration; windowed stage outputs are DISTINCT node sets
 * (kernels.py:45-59 np.unique).
 *
 * Its data structures are deliberately plain: int64 everywhere, a per-node
 * adjacency sorted by (time, eid) (what txgraph.py builds with np.lexsort)
 * plus a per-node copy sorted by (nbr, time) used to answer "is there an
 * a->b edge inside the window" by bisection.  Distinct sets are built by
 * sort + unique, as np.unique does.  Parity of this file against the
 * reference itself is pinned by tests/test_oracle_golden.py on fixtures the
 * reference generated (tests/golden/make_golden.py).
 *
 * Threads: trigger ranges are handed out in chunks to `n_threads` pthreads;
 * results are independent of the thread count (disjoint rows).
 */
#include <pthread.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

/* family codes — same meaning as the product header, restated here so the
 * checker does not depend on product headers */
enum { OF_FAN = 1, OF_DEGREE = 2, OF_CYCLE = 3, OF_SG = 4, OF_GS = 5, OF_STACK = 6 };

typedef struct {
  int64_t n_nodes, n_edges;
  const int64_t *src, *dst, *time;
  /* dir 0 = in, 1 = out; adjacency sorted by (time, eid) */
  int64_t *ptr[2];
  int64_t *nbr[2];
  int64_t *tim[2];
  int64_t *eid[2];
  /* same runs re-sorted by (nbr, time): existence probes */
  int64_t *pnbr[2];
  int64_t *ptim[2];
  int64_t max_deg;
} og_graph;

typedef struct {
  int32_t family, endpoint, direction, exclude_trigger, cycle_len, min_size;
  int64_t delta;
} og_plan;

/* ---------------------------------------------------------------- build */

typedef struct { int64_t key1, key2, a, b; } quad;

static int cmp_quad(const void *x, const void *y) {
  const quad *p = (const quad *)x, *q = (const quad *)y;
  if (p->key1 != q->key1) return p->key1 < q->key1 ? -1 : 1;
  if (p->key2 != q->key2) return p->key2 < q->key2 ? -1 : 1;
  return 0;
}

static int build_dir(og_graph *g, int dir) {
  const int64_t n = g->n_nodes, e = g->n_edges;
  const int64_t *owner = dir ? g->src : g->dst;
  const int64_t *other = dir ? g->dst : g->src;
  int64_t *ptr = calloc((size_t)n + 1, sizeof(int64_t));
  int64_t *nbr = malloc(sizeof(int64_t) * (size_t)(e ? e : 1));
  int64_t *tim = malloc(sizeof(int64_t) * (size_t)(e ? e : 1));
  int64_t *eid = malloc(sizeof(int64_t) * (size_t)(e ? e : 1));
  int64_t *pnbr = malloc(sizeof(int64_t) * (size_t)(e ? e : 1));
  int64_t *ptim = malloc(sizeof(int64_t) * (size_t)(e ? e : 1));
  int64_t *fill = malloc(sizeof(int64_t) * (size_t)(n ? n : 1));
  if (!ptr || !nbr || !tim || !eid || !pnbr || !ptim || !fill) return -1;
  for (int64_t i = 0; i < e; ++i) ptr[owner[i] + 1]++;
  for (int64_t x = 0; x < n; ++x) ptr[x + 1] += ptr[x];
  memcpy(fill, ptr, sizeof(int64_t) * (size_t)n);
  for (int64_t i = 0; i < e; ++i) { /* eid order => ties stay eid-ascending */
    int64_t p = fill[owner[i]]++;
    eid[p] = i;
  }
  int64_t maxd = 0;
  quad *buf = NULL;
  size_t cap = 0;
  for (int64_t x = 0; x < n; ++x) {
    int64_t a = ptr[x], b = ptr[x + 1], d = b - a;
    if (d > maxd) maxd = d;
    if ((size_t)d > cap) { cap = (size_t)d; free(buf); buf = malloc(sizeof(quad) * cap); if (!buf) return -1; }
    for (int64_t j = 0; j < d; ++j) {
      int64_t id = eid[a + j];
      buf[j].key1 = g->time[id]; buf[j].key2 = id; buf[j].a = other[id]; buf[j].b = id;
    }
    qsort(buf, (size_t)d, sizeof(quad), cmp_quad); /* (time, eid): txgraph.py:135-136 */
    for (int64_t j = 0; j < d; ++j) { eid[a + j] = buf[j].b; nbr[a + j] = buf[j].a; tim[a + j] = buf[j].key1; }
    for (int64_t j = 0; j < d; ++j) { buf[j].key1 = nbr[a + j]; buf[j].key2 = tim[a + j]; }
    qsort(buf, (size_t)d, sizeof(quad), cmp_quad); /* (nbr, time) */
    for (int64_t j = 0; j < d; ++j) { pnbr[a + j] = buf[j].key1; ptim[a + j] = buf[j].key2; }
  }
  free(buf);
  free(fill);
  g->ptr[dir] = ptr; g->nbr[dir] = nbr; g->tim[dir] = tim; g->eid[dir] = eid;
  g->pnbr[dir] = pnbr; g->ptim[dir] = ptim;
  if (maxd > g->max_deg) g->max_deg = maxd;
  return 0;
}

void og_free(og_graph *g) {
  if (!g) return;
  for (int d = 0; d < 2; ++d) {
    free(g->ptr[d]); free(g->nbr[d]); free(g->tim[d]); free(g->eid[d]);
    free(g->pnbr[d]); free(g->ptim[d]);
  }
  free(g);
}

og_graph *og_build(int64_t n_nodes, int64_t n_edges, const int64_t *src, const int64_t *dst,
                   const int64_t *time) {
  og_graph *g = calloc(1, sizeof(og_graph));
  if (!g) return NULL;
  g->n_nodes = n_nodes; g->n_edges = n_edges; g->src = src; g->dst = dst; g->time = time;
  if (build_dir(g, 0) || build_dir(g, 1)) { og_free(g); return NULL; }
  return g;
}

/* export the (time, eid)-sorted CSR for CSR parity checks */
void og_export(const og_graph *g, int dir, int64_t *ptr, int64_t *nbr, int64_t *tim, int64_t *eid) {
  memcpy(ptr, g->ptr[dir], sizeof(int64_t) * (size_t)(g->n_nodes + 1));
  memcpy(nbr, g->nbr[dir], sizeof(int64_t) * (size_t)g->n_edges);
  memcpy(tim, g->tim[dir], sizeof(int64_t) * (size_t)g->n_edges);
  memcpy(eid, g->eid[dir], sizeof(int64_t) * (size_t)g->n_edges);
}

/* ---------------------------------------------------------------- queries */

static int64_t lower_t(const int64_t *t, int64_t a, int64_t b, int64_t x) { /* first t >= x */
  while (a < b) { int64_t m = a + (b - a) / 2; if (t[m] < x) a = m + 1; else b = m; }
  return a;
}
static int64_t upper_t(const int64_t *t, int64_t a, int64_t b, int64_t x) { /* first t > x */
  while (a < b) { int64_t m = a + (b - a) / 2; if (t[m] <= x) a = m + 1; else b = m; }
  return a;
}

/* number of (owner=x, nbr=y) entries of direction dir with time in [lo, hi] */
static int64_t pair_count(const og_graph *g, int dir, int64_t x, int64_t y, int64_t lo, int64_t hi) {
  const int64_t *pn = g->pnbr[dir], *pt = g->ptim[dir];
  int64_t a = g->ptr[dir][x], b = g->ptr[dir][x + 1];
  /* range of nbr == y */
  int64_t l = a, r = b;
  while (l < r) { int64_t m = l + (r - l) / 2; if (pn[m] < y) l = m + 1; else r = m; }
  int64_t s = l; r = b;
  while (l < r) { int64_t m = l + (r - l) / 2; if (pn[m] <= y) l = m + 1; else r = m; }
  int64_t e = l;
  return upper_t(pt, s, e, hi) - lower_t(pt, s, e, lo);
}

static int edge_in_window(const og_graph *g, int64_t a, int64_t b, int64_t lo, int64_t hi) {
  return pair_count(g, 1, a, b, lo, hi) > 0; /* a's out-run, neighbour b */
}

/* windowed edge count, self-loops excluded (kernels.py:62-74) */
static int64_t windowed_edges(const og_graph *g, int dir, int64_t x, int64_t lo, int64_t hi) {
  int64_t a = g->ptr[dir][x], b = g->ptr[dir][x + 1];
  const int64_t *t = g->tim[dir];
  int64_t n = upper_t(t, a, b, hi) - lower_t(t, a, b, lo);
  return n - pair_count(g, dir, x, x, lo, hi);
}

static int cmp_i64(const void *x, const void *y) {
  int64_t a = *(const int64_t *)x, b = *(const int64_t *)y;
  return a < b ? -1 : (a > b);
}

/* sorted distinct windowed neighbours of x, self-loops and ex0/ex1 dropped
 * (kernels.py:45-59 windowed_nodes + the callers' explicit exclusions) */
static int64_t windowed_nodes(const og_graph *g, int dir, int64_t x, int64_t lo, int64_t hi,
                              int64_t ex0, int64_t ex1, int64_t *out) {
  int64_t a = g->ptr[dir][x], b = g->ptr[dir][x + 1];
  const int64_t *t = g->tim[dir], *nb = g->nbr[dir];
  int64_t s = lower_t(t, a, b, lo), e = upper_t(t, a, b, hi), n = 0;
  for (int64_t j = s; j < e; ++j) {
    int64_t y = nb[j];
    if (y == x || y == ex0 || y == ex1) continue;
    out[n++] = y;
  }
  qsort(out, (size_t)n, sizeof(int64_t), cmp_i64);
  int64_t m = 0;
  for (int64_t j = 0; j < n; ++j)
    if (m == 0 || out[m - 1] != out[j]) out[m++] = out[j];
  return m;
}

static int contains(const int64_t *set, int64_t n, int64_t y) {
  int64_t l = 0, r = n;
  while (l < r) { int64_t m = l + (r - l) / 2; if (set[m] < y) l = m + 1; else r = m; }
  return l < n && set[l] == y;
}

typedef struct {
  int64_t *buf[8]; /* scratch sets, each max_deg long */
} scratch;

/* cycle_k, k >= 4: Appendix A — chains a1..a_{k-3} from v, closing set
 * C = (N+(a_last) ∩ N-(u)) \ {v, a1..a_{last-1}}, |C| added when >= K.
 * cycle_4 (kernels.py:328-343) is the k = 4 instance. */
static int64_t cycle_dfs(const og_graph *g, scratch *sc, int depth, int chain, int64_t *path,
                         int64_t u, int64_t v, const int64_t *closers, int64_t n_closers,
                         int64_t lo, int64_t hi, int64_t K) {
  int64_t last = path[depth - 1];
  if (depth == chain) {
    int64_t c = 0;
    for (int64_t i = 0; i < n_closers; ++i) {
      int64_t w = closers[i]; /* closers = N-(u) \ {v} */
      int skip = 0;
      for (int j = 0; j < depth - 1; ++j) if (path[j] == w) { skip = 1; break; }
      if (skip || w == last) continue;
      if (edge_in_window(g, last, w, lo, hi)) ++c;
    }
    return c >= K ? c : 0;
  }
  int64_t *nxt = sc->buf[2 + depth];
  int64_t n = windowed_nodes(g, 1, last, lo, hi, u, v, nxt);
  int64_t total = 0;
  for (int64_t i = 0; i < n; ++i) {
    int64_t a = nxt[i];
    int skip = 0;
    for (int j = 0; j < depth - 1; ++j) if (path[j] == a) { skip = 1; break; }
    if (skip) continue;
    path[depth] = a;
    total += cycle_dfs(g, sc, depth + 1, chain, path, u, v, closers, n_closers, lo, hi, K);
  }
  return total;
}

static int64_t eval(const og_graph *g, const og_plan *p, int64_t e, scratch *sc) {
  const int64_t u = g->src[e], v = g->dst[e], t = g->time[e];
  const int64_t lo = t - p->delta, hi = t;
  const int64_t K = p->min_size;
  switch (p->family) {
    case OF_FAN:
    case OF_DEGREE: { /* kernels.py:290-303 */
      int64_t x = p->endpoint ? v : u;
      int64_t c = windowed_edges(g, p->direction, x, lo, hi);
      if (p->exclude_trigger && u != v) c -= 1;
      if (K > 1 && c < K) c = 0;
      return c;
    }
    case OF_CYCLE: {
      if (u == v) return 0; /* kernels.py:315 */
      if (p->cycle_len == 2) { /* kernels.py:320-322 */
        int64_t raw = edge_in_window(g, v, u, lo, hi) ? 1 : 0;
        return raw >= K ? raw : 0;
      }
      int64_t *cl = sc->buf[0];
      if (p->cycle_len == 3) { /* kernels.py:323-327: |N+(v)\{u} ∩ N-(u)| */
        int64_t n = windowed_nodes(g, 0, u, lo, hi, u, v, cl); /* v is never in N+(v) */
        int64_t raw = 0;
        for (int64_t i = 0; i < n; ++i) if (edge_in_window(g, v, cl[i], lo, hi)) ++raw;
        return raw >= K ? raw : 0;
      }
      int64_t nc = windowed_nodes(g, 0, u, lo, hi, v, v, cl); /* closers.discard(v) */
      if (nc == 0) return 0;
      int64_t *a1 = sc->buf[1];
      int64_t n1 = windowed_nodes(g, 1, v, lo, hi, u, u, a1); /* m != u */
      int64_t path[8];
      int64_t total = 0;
      for (int64_t i = 0; i < n1; ++i) {
        path[0] = a1[i];
        total += cycle_dfs(g, sc, 1, p->cycle_len - 3, path, u, v, cl, nc, lo, hi, K);
      }
      return total;
    }
    case OF_SG: { /* kernels.py:348-376 */
      int64_t *src = sc->buf[0], *gat = sc->buf[1], *mids = sc->buf[2];
      int64_t ns = windowed_nodes(g, 0, u, lo, hi, u, v, src);
      if (ns == 0) return 0;
      int64_t ng = windowed_nodes(g, 0, v, lo, hi, v, v, gat);
      int64_t count = 0;
      for (int64_t i = 0; i < ns; ++i) {
        int64_t s = src[i], hits = 0;
        if (windowed_edges(g, 1, s, lo, hi) < ng) {
          int64_t nm = windowed_nodes(g, 1, s, lo, hi, s, s, mids);
          for (int64_t j = 0; j < nm; ++j) hits += contains(gat, ng, mids[j]);
        } else {
          for (int64_t j = 0; j < ng; ++j) hits += (gat[j] != s) && edge_in_window(g, s, gat[j], lo, hi);
        }
        if (hits >= K) ++count;
      }
      return count;
    }
    case OF_GS: { /* Appendix B: #{d in N+(v)\{u} : |N-(d) ∩ N+(u)| >= K} */
      int64_t *ds = sc->buf[0], *md = sc->buf[1];
      int64_t nd = windowed_nodes(g, 1, v, lo, hi, u, u, ds);
      int64_t count = 0;
      for (int64_t i = 0; i < nd; ++i) {
        int64_t d = ds[i], hits = 0;
        int64_t nm = windowed_nodes(g, 0, d, lo, hi, d, d, md);
        for (int64_t j = 0; j < nm; ++j) hits += (md[j] != u) && edge_in_window(g, u, md[j], lo, hi);
        if (hits >= K) ++count;
      }
      return count;
    }
    case OF_STACK: { /* kernels.py:379-402 */
      int64_t *b0 = sc->buf[0];
      int64_t a = windowed_nodes(g, 0, u, lo, hi, u, v, b0);
      if (a < K || a == 0) return 0;
      int64_t c = windowed_nodes(g, 1, v, lo, hi, v, u, b0);
      if (c < K || c == 0) return 0;
      return a * c;
    }
    default:
      return INT64_MIN;
  }
}

typedef struct {
  const og_graph *g;
  const og_plan *plans;
  int n_plans;
  int64_t lo, hi;
  int64_t *out;
  int64_t next;
  pthread_mutex_t mu;
  int err;
} job;

static void *worker(void *arg) {
  job *jb = (job *)arg;
  scratch sc;
  int64_t cap = jb->g->max_deg + 1;
  for (int i = 0; i < 8; ++i) {
    sc.buf[i] = malloc(sizeof(int64_t) * (size_t)cap);
    if (!sc.buf[i]) { jb->err = 1; return NULL; }
  }
  const int64_t chunk = 256;
  for (;;) {
    pthread_mutex_lock(&jb->mu);
    int64_t a = jb->next;
    jb->next += chunk;
    pthread_mutex_unlock(&jb->mu);
    if (a >= jb->hi) break;
    int64_t b = a + chunk < jb->hi ? a + chunk : jb->hi;
    for (int64_t e = a; e < b; ++e)
      for (int c = 0; c < jb->n_plans; ++c)
        jb->out[(e - jb->lo) * jb->n_plans + c] = eval(jb->g, &jb->plans[c], e, &sc);
  }
  for (int i = 0; i < 8; ++i) free(sc.buf[i]);
  return NULL;
}

/* rows [lo, hi) x n_plans, C-order; returns 0 on success */
int og_mine(const og_graph *g, const og_plan *plans, int n_plans, int64_t lo, int64_t hi,
            int64_t *out, int n_threads) {
  if (!g || lo < 0 || hi > g->n_edges || lo > hi) return -1;
  for (int c = 0; c < n_plans; ++c) {
    if (plans[c].family < OF_FAN || plans[c].family > OF_STACK) return -2;
    if (plans[c].family == OF_CYCLE && (plans[c].cycle_len < 2 || plans[c].cycle_len > 8)) return -2;
  }
  job jb = {g, plans, n_plans, lo, hi, out, lo, PTHREAD_MUTEX_INITIALIZER, 0};
  if (n_threads < 1) n_threads = 1;
  if (n_threads > 256) n_threads = 256;
  pthread_t th[256];
  for (int i = 0; i < n_threads; ++i) pthread_create(&th[i], NULL, worker, &jb);
  for (int i = 0; i < n_threads; ++i) pthread_join(th[i], NULL);
  return jb.err ? -3 : 0;
}
