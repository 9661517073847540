// tm_mine.cu — per-trigger pattern-count kernels for sm_100a.
//
// Reference semantics (trigger attribution, window [t - delta, t] closed,
// self-loops never iterated, windowed stage outputs are distinct node sets):
//   FAN / DEGREE     kernels.py:290-303   (+ single-edge defs :81-101)
//   CYCLE 2/3/4      kernels.py:306-345
//   SG               kernels.py:348-376
//   STACK            kernels.py:379-402
//   CYCLE 5..8, GS   generic interpreter engine.py:516-562 on SURVEY.md
//                    Appendix B (per-binding set_cardinality :462-464,
//                    source_count :483-485)
//
// Work balancing for power-law hubs (the reference has none: equal
// contiguous ranges per worker, engine.py:681-682) — three tiers:
//
//   k_mine_light   one THREAD per trigger edge, all columns.  Windows come
//                  from bisection of the time-ranked CSR; set columns iterate
//                  the SMALLER windowed slice and test the other side with
//                  one pair-index bisection; distinct-ness is an O(1)
//                  pair-predecessor test.  Each trigger carries a work
//                  budget; a trigger that would exceed it is appended to the
//                  heavy queue (warp-aggregated atomic) and left to ...
//   k_mine_heavy   one WARP per heavy trigger: each column's outer slice is
//                  spread over the lanes.  Outer slices longer than
//                  kOuterSplit, and — inside cycle_k's depth-first chain
//                  enumeration — every node whose windowed out-slice is
//                  longer than kDeepSplit, are not walked serially but cut
//                  into range TASKS of kTaskSpan entries, appended to a task
//                  queue and ...
//   k_mine_tasks   one WARP per task, lane per slice entry, launched in
//                  rounds (a task only spawns tasks one level deeper, so
//                  <= 5 rounds for cycle_8).  Partial counts are combined
//                  with atomicAdd on the int64 output cell, which the heavy
//                  kernel initialized with its own partial.
// Every count is an integer sum over disjoint pieces, so the result is
// exactly the reference's regardless of the split.
#include "tm_internal.cuh"

namespace tmb {
namespace {

constexpr int kLightThreads = 256;
constexpr int kHeavyThreads = 256;
constexpr int kLightBudget = 768;  // slice entries + probes per light trigger
constexpr int kOuterSplit = 512;   // heavy row: outer slices above this become tasks
constexpr int kDeepSplit = 64;     // chain nodes with wider windows become tasks
constexpr int kTaskSpan = 128;     // entries per task (4 per lane)
constexpr int kMaxChain = 5;       // cycle_8: a1..a5

struct Win {
  int a, b;
  __device__ __forceinline__ int len() const { return b - a; }
};

__device__ __forceinline__ int lb_u32(const uint32_t *__restrict__ r, int a, int b, uint32_t x) {
  while (a < b) {
    int m = (a + b) >> 1;
    if (__ldg(r + m) < x) a = m + 1; else b = m;
  }
  return a;
}
__device__ __forceinline__ int ub_u32(const uint32_t *__restrict__ r, int a, int b, uint32_t x) {
  while (a < b) {
    int m = (a + b) >> 1;
    if (__ldg(r + m) <= x) a = m + 1; else b = m;
  }
  return a;
}
__device__ __forceinline__ int lb_u64(const uint64_t *__restrict__ k, int a, int b, uint64_t x) {
  while (a < b) {
    int m = (a + b) >> 1;
    if (__ldg(k + m) < x) a = m + 1; else b = m;
  }
  return a;
}

struct Ctx {
  const DevGraph &g;
  int u, v;
  uint32_t lo, hi;  // window in rank space
};

// windowed slice of x's dir-run: rank in [lo, hi]   (kernels.py:268-276)
__device__ __forceinline__ Win window(const Ctx &c, int dir, int x) {
  const int a = __ldg(c.g.ptr[dir] + x), b = __ldg(c.g.ptr[dir] + x + 1);
  const int wa = lb_u32(c.g.rnk[dir], a, b, c.lo);
  return {wa, ub_u32(c.g.rnk[dir], wa, b, c.hi)};
}

// self-loops of x inside the window (kernels.py:279-287): pair run (x, x)
__device__ __forceinline__ int loops_in_window(const Ctx &c, int x) {
  if (!__ldg(c.g.loop + x)) return 0;
  const int a = __ldg(c.g.ptr[1] + x), b = __ldg(c.g.ptr[1] + x + 1);
  const uint64_t base = (uint64_t)(uint32_t)x << c.g.rank_bits;
  return lb_u64(c.g.pkey[1], a, b, base + c.hi + 1) - lb_u64(c.g.pkey[1], a, b, base + c.lo);
}

// is there an edge a -> b inside the window?  bisection of the shorter of
// a's out pair-run and b's in pair-run
__device__ __forceinline__ bool has_edge(const Ctx &c, int a, int b) {
  const int oa = __ldg(c.g.ptr[1] + a), ob = __ldg(c.g.ptr[1] + a + 1);
  const int ia = __ldg(c.g.ptr[0] + b), ib = __ldg(c.g.ptr[0] + b + 1);
  int s, e, dir;
  uint32_t other;
  if (ob - oa <= ib - ia) { s = oa; e = ob; dir = 1; other = (uint32_t)b; }
  else { s = ia; e = ib; dir = 0; other = (uint32_t)a; }
  if (s == e) return false;
  const uint64_t base = (uint64_t)other << c.g.rank_bits;
  const int q = lb_u64(c.g.pkey[dir], s, e, base + c.lo);
  return q < e && __ldg(c.g.pkey[dir] + q) <= base + c.hi;
}

// CSR entry j (neighbour n) of the run starting at seg is the first
// occurrence of n inside the window  <=>  its pair predecessor is another
// neighbour or lies before the window (np.unique, kernels.py:59)
__device__ __forceinline__ bool first_in_window(const Ctx &c, int dir, int seg, int j, int n) {
  const int q = __ldg(c.g.c2p[dir] + j);
  if (q == seg) return true;
  const uint64_t prev = __ldg(c.g.pkey[dir] + q - 1);
  const int rb = c.g.rank_bits;
  return (uint32_t)(prev >> rb) != (uint32_t)n ||
         (uint32_t)(prev & ((1ull << rb) - 1)) < c.lo;
}

__device__ __forceinline__ long long warp_sum(long long x) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) x += __shfl_xor_sync(0xffffffffu, x, o);
  return x;
}

// budget of the light (thread-per-trigger) tier; unlimited elsewhere
struct Budget {
  int left;
  bool blown;
  __device__ __forceinline__ bool take(int n) {
    if (n > left) { blown = true; return false; }
    left -= n;
    return true;
  }
};

// ------------------------------------------------------------ task queue

struct Task {
  int32_t row;   // trigger row (relative to lo); < 0 = empty slot
  int8_t col;    // plan index
  int8_t level;  // slice level: 0 = the trigger's own slice, L = out-slice of a_L
  int8_t side;   // cycle_3: 0 = iterate N+(v), 1 = iterate N-(u)
  int8_t pad;
  int32_t a, b;  // CSR range of the slice piece
  int32_t path[kMaxChain];
};

struct Emitter {
  Task *q;
  int32_t *count;
  int32_t cap;
  int32_t row;
  int32_t col;
  bool on;
  // cut [a, b) into kTaskSpan pieces; false (caller walks it serially) when
  // emission is off or the queue is full
  __device__ bool emit(int level, int side, const int *path, int a, int b) const {
    if (!on) return false;
    const int n = (b - a + kTaskSpan - 1) / kTaskSpan;
    const int base = atomicAdd(count, n);
    if (base + n > cap) {
      for (int k = base; k < cap; ++k) q[k].row = -1;  // holes stay empty
      return false;
    }
    for (int k = 0; k < n; ++k) {
      Task t;
      t.row = row;
      t.col = (int8_t)col;
      t.level = (int8_t)level;
      t.side = (int8_t)side;
      t.pad = 0;
      t.a = a + k * kTaskSpan;
      t.b = min(b, t.a + kTaskSpan);
#pragma unroll
      for (int i = 0; i < kMaxChain; ++i) t.path[i] = i < level ? path[i] : -1;
      q[base + k] = t;
    }
    return true;
  }
};

// ---------------------------------------------------------- families

// FAN / DEGREE (kernels.py:290-303)
__device__ __forceinline__ long long col_fan_degree(const Ctx &c, const DevPlan &p) {
  const int x = p.endpoint ? c.v : c.u;
  const Win w = window(c, p.direction, x);
  long long n = w.len() - loops_in_window(c, x);
  if (p.exclude_trigger && c.u != c.v) n -= 1;
  if (p.min_size > 1 && n < p.min_size) n = 0;
  return n;
}

// cycle_2 = [u != v and v -> u in window] (kernels.py:320-322)
__device__ __forceinline__ long long col_cycle2(const Ctx &c, const DevPlan &p) {
  if (c.u == c.v) return 0;
  long long raw = has_edge(c, c.v, c.u) ? 1 : 0;
  return raw >= p.min_size ? raw : 0;
}

// distinct windowed neighbours of x in dir over CSR range [ja, jb) with
// stride, excluding x (self-loops) and ex
__device__ long long distinct_range(const Ctx &c, int dir, int x, int ex, int ja, int jb,
                                    int stride) {
  const int seg = __ldg(c.g.ptr[dir] + x);
  long long n = 0;
  for (int j = ja; j < jb; j += stride) {
    const int y = __ldg(c.g.nbr[dir] + j);
    if (y == x || y == ex) continue;
    n += first_in_window(c, dir, seg, j, y);
  }
  return n;
}

// cycle_3 entry (kernels.py:323-327): side 0 walks N+(v)\{u} testing m -> u,
// side 1 walks N-(u)\{v} testing v -> m
__device__ __forceinline__ int c3_entry(const Ctx &c, int side, int j) {
  if (side == 0) {
    const int m = __ldg(c.g.nbr[1] + j);
    if (m == c.v || m == c.u || !first_in_window(c, 1, __ldg(c.g.ptr[1] + c.v), j, m)) return 0;
    return has_edge(c, m, c.u);
  }
  const int m = __ldg(c.g.nbr[0] + j);
  if (m == c.u || m == c.v || !first_in_window(c, 0, __ldg(c.g.ptr[0] + c.u), j, m)) return 0;
  return has_edge(c, c.v, m);
}

// |N^{dx}(x) ∩ N^{dy}(y)|, early exit at K (sg: x = s out, y = v in;
// gs: x = d in, y = u out).  x and y are never members (no self-loops).
__device__ int inner_hits(const Ctx &c, int x, int dx, int y, int dy, int K, Budget *bud) {
  const Win wx = window(c, dx, x), wy = window(c, dy, y);
  int hits = 0;
  if (wx.len() <= wy.len()) {
    if (bud && !bud->take(2 * wx.len())) return 0;
    const int seg = __ldg(c.g.ptr[dx] + x);
    for (int j = wx.a; j < wx.b && hits < K; ++j) {
      const int m = __ldg(c.g.nbr[dx] + j);
      if (m == x || m == y || !first_in_window(c, dx, seg, j, m)) continue;
      hits += dy ? has_edge(c, y, m) : has_edge(c, m, y);
    }
  } else {
    if (bud && !bud->take(2 * wy.len())) return 0;
    const int seg = __ldg(c.g.ptr[dy] + y);
    for (int j = wy.a; j < wy.b && hits < K; ++j) {
      const int m = __ldg(c.g.nbr[dy] + j);
      if (m == y || m == x || !first_in_window(c, dy, seg, j, m)) continue;
      hits += dx ? has_edge(c, x, m) : has_edge(c, m, x);
    }
  }
  return hits;
}

// sg entry: s = CSR in-entry j of u; #{s : |N+(s) ∩ N-(v)| >= K} (kernels.py:358-375)
__device__ __forceinline__ int sg_entry(const Ctx &c, int K, int j, Budget *bud) {
  const int s = __ldg(c.g.nbr[0] + j);
  if (s == c.u || s == c.v || !first_in_window(c, 0, __ldg(c.g.ptr[0] + c.u), j, s)) return 0;
  return inner_hits(c, s, 1, c.v, 0, K, bud) >= K;
}

// gs entry: d = CSR out-entry j of v; #{d : |N-(d) ∩ N+(u)| >= K} (Appendix B)
__device__ __forceinline__ int gs_entry(const Ctx &c, int K, int j, Budget *bud) {
  const int d = __ldg(c.g.nbr[1] + j);
  if (d == c.v || d == c.u || !first_in_window(c, 1, __ldg(c.g.ptr[1] + c.v), j, d)) return 0;
  return inner_hits(c, d, 0, c.u, 1, K, bud) >= K;
}

// closing set size for a chain ending at `a`:
//   |(N+(a) ∩ N-(u)) \ {v, path[0..np-1]}|   (Appendix A cycle_k; cycle_4
//   kernels.py:330-341 for np = 0).
__device__ int close_count(const Ctx &c, int a, const int *path, int np, const Win &wu,
                           Budget *bud) {
  const Win wa = window(c, 1, a);
  int cnt = 0;
  if (wa.len() <= wu.len()) {
    if (bud && !bud->take(2 * wa.len())) return 0;
    const int seg = __ldg(c.g.ptr[1] + a);
    for (int j = wa.a; j < wa.b; ++j) {
      const int m = __ldg(c.g.nbr[1] + j);
      if (m == a || m == c.u || m == c.v) continue;
      bool dup = false;
      for (int i = 0; i < np; ++i) dup |= (path[i] == m);
      if (dup || !first_in_window(c, 1, seg, j, m)) continue;
      cnt += has_edge(c, m, c.u);
    }
  } else {
    if (bud && !bud->take(2 * wu.len())) return 0;
    const int seg = __ldg(c.g.ptr[0] + c.u);
    for (int j = wu.a; j < wu.b; ++j) {
      const int w = __ldg(c.g.nbr[0] + j);
      if (w == c.u || w == c.v || w == a) continue;
      bool dup = false;
      for (int i = 0; i < np; ++i) dup |= (path[i] == w);
      if (dup || !first_in_window(c, 0, seg, j, w)) continue;
      cnt += has_edge(c, a, w);
    }
  }
  return cnt;
}

// cycle_k, k = 4..8, chains a1..a_{chain}, chain = k - 3:
//   a1 in N+(v)\{u};  a_i in N+(a_{i-1}) \ {u, v, a1..a_{i-2}};
//   each chain adds |C| = close_count(a_chain) when |C| >= K.
// Enumerates the entries j in [ja, jb) (stride `stride`) of the level-L0
// slice (owner v for L0 = 0, else path[L0-1]) and everything below them,
// depth-first.  A node whose window exceeds kDeepSplit is handed to the
// emitter as tasks instead of being walked (when emission is on).
__device__ long long cycle_dfs(const Ctx &c, int K, int chain, int *path, int L0, int ja, int jb,
                               int stride, const Win &wu, Budget *bud, const Emitter &em) {
  int pos[kMaxChain], end[kMaxChain], seg[kMaxChain];
  long long total = 0;
  int L = L0;
  pos[L] = ja;
  end[L] = jb;
  seg[L] = __ldg(c.g.ptr[1] + (L == 0 ? c.v : path[L - 1]));
  while (L >= L0) {
    const int j = pos[L];
    if (j >= end[L]) { --L; continue; }
    pos[L] = j + (L == L0 ? stride : 1);
    const int owner = L == 0 ? c.v : path[L - 1];
    const int a = __ldg(c.g.nbr[1] + j);
    if (a == owner || a == c.u || a == c.v) continue;
    bool dup = false;
    for (int i = 0; i + 1 < L; ++i) dup |= (path[i] == a);
    if (dup || !first_in_window(c, 1, seg[L], j, a)) continue;
    if (L == chain - 1) {
      const int cc = close_count(c, a, path, L, wu, bud);
      if (bud && bud->blown) return 0;
      if (cc >= K) total += cc;
      continue;
    }
    path[L] = a;
    const Win w = window(c, 1, a);
    if (w.len() > kDeepSplit && em.emit(L + 1, 0, path, w.a, w.b)) continue;
    if (bud && !bud->take(w.len())) return 0;
    ++L;
    pos[L] = w.a;
    end[L] = w.b;
    seg[L] = __ldg(c.g.ptr[1] + a);
  }
  return total;
}

// ------------------------------------------------------------- tier 1

// full column, one thread, budgeted
__device__ long long eval_light(const Ctx &c, const DevPlan &p, Budget &bud, const Emitter &off) {
  switch (p.family) {
    case TM_FAN:
    case TM_DEGREE: return col_fan_degree(c, p);
    case TM_CYCLE: {
      if (p.cycle_len == 2) return col_cycle2(c, p);
      if (c.u == c.v) return 0;
      if (p.cycle_len == 3) {
        const Win wv = window(c, 1, c.v), wu = window(c, 0, c.u);
        if (wv.len() == 0 || wu.len() == 0) return 0;
        const int side = wv.len() <= wu.len() ? 0 : 1;
        const Win w = side ? wu : wv;
        if (!bud.take(2 * w.len())) return 0;
        long long raw = 0;
        for (int j = w.a; j < w.b; ++j) raw += c3_entry(c, side, j);
        return raw >= p.min_size ? raw : 0;
      }
      const Win wu = window(c, 0, c.u);
      if (wu.len() == 0) return 0;
      const Win wv = window(c, 1, c.v);
      if (!bud.take(wv.len())) return 0;
      int path[kMaxChain];
      return cycle_dfs(c, p.min_size, p.cycle_len - 3, path, 0, wv.a, wv.b, 1, wu, &bud, off);
    }
    case TM_SG: {
      const Win w = window(c, 0, c.u);
      if (!bud.take(w.len())) return 0;
      long long n = 0;
      for (int j = w.a; j < w.b; ++j) {
        n += sg_entry(c, p.min_size, j, &bud);
        if (bud.blown) return 0;
      }
      return n;
    }
    case TM_GS: {
      const Win w = window(c, 1, c.v);
      if (!bud.take(w.len())) return 0;
      long long n = 0;
      for (int j = w.a; j < w.b; ++j) {
        n += gs_entry(c, p.min_size, j, &bud);
        if (bud.blown) return 0;
      }
      return n;
    }
    case TM_STACK: {  // kernels.py:379-402
      const Win wa = window(c, 0, c.u);
      if (!bud.take(wa.len())) return 0;
      const long long a = distinct_range(c, 0, c.u, c.v, wa.a, wa.b, 1);
      if (a == 0 || a < p.min_size) return 0;
      const Win wc = window(c, 1, c.v);
      if (!bud.take(wc.len())) return 0;
      const long long d = distinct_range(c, 1, c.v, c.u, wc.a, wc.b, 1);
      if (d == 0 || d < p.min_size) return 0;
      return a * d;
    }
    default: return 0;
  }
}

__global__ void __launch_bounds__(kLightThreads) k_mine_light(
    const DevGraph g, const DevPlans plans, int64_t lo, int64_t n_rows, long long *__restrict__ out,
    int32_t *__restrict__ heavy_q, int32_t *__restrict__ heavy_n) {
  const int64_t row = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  bool heavy = false;
  if (row < n_rows) {
    const int e = (int)(lo + row);
    const int u = __ldg(g.e_src + e), v = __ldg(g.e_dst + e);
    const uint32_t r = __ldg(g.e_rank + e);
    Budget bud{kLightBudget, false};
    const Emitter off{nullptr, nullptr, 0, 0, 0, false};
    long long *o = out + row * plans.n;
    for (int ci = 0; ci < plans.n; ++ci) {
      const DevPlan p = plans.p[ci];
      const Ctx c{g, u, v, __ldg(p.lo_tab + r), r};
      const long long val = eval_light(c, p, bud, off);
      if (bud.blown) { heavy = true; break; }
      o[ci] = val;
    }
  }
  // warp-aggregated append of heavy triggers
  const unsigned m = __ballot_sync(0xffffffffu, heavy);
  if (m) {
    const int lane = threadIdx.x & 31;
    int base = 0;
    if (lane == __ffs(m) - 1) base = atomicAdd(heavy_n, __popc(m));
    base = __shfl_sync(0xffffffffu, base, __ffs(m) - 1);
    if (heavy) heavy_q[base + __popc(m & ((1u << lane) - 1))] = (int32_t)row;
  }
}

// ------------------------------------------------------------- tier 2

// warp-uniform emission of a level-0 slice: lane 0 emits, all lanes agree
__device__ __forceinline__ bool warp_emit(const Emitter &em, const int *path, const Win &w) {
  int ok = 0;
  if ((threadIdx.x & 31) == 0) ok = em.emit(0, 0, path, w.a, w.b) ? 1 : 0;
  return __shfl_sync(0xffffffffu, ok, 0) != 0;
}

// one warp, one heavy trigger, one column: returns the warp's partial (all
// lanes hold it); pieces beyond kOuterSplit / kDeepSplit are emitted
__device__ long long eval_heavy(const Ctx &c, const DevPlan &p, const Emitter &em) {
  const int lane = threadIdx.x & 31;
  switch (p.family) {
    case TM_FAN:
    case TM_DEGREE: return col_fan_degree(c, p);
    case TM_CYCLE: {
      if (p.cycle_len == 2) return col_cycle2(c, p);
      if (c.u == c.v) return 0;
      if (p.cycle_len == 3) {
        const Win wv = window(c, 1, c.v), wu = window(c, 0, c.u);
        if (wv.len() == 0 || wu.len() == 0) return 0;
        const int side = wv.len() <= wu.len() ? 0 : 1;
        const Win w = side ? wu : wv;
        // the threshold applies to the count, so the whole count must be
        // one piece: walk it with the warp (no task split)
        long long raw = 0;
        for (int j = w.a + lane; j < w.b; j += 32) raw += c3_entry(c, side, j);
        raw = warp_sum(raw);
        return raw >= p.min_size ? raw : 0;
      }
      const Win wu = window(c, 0, c.u);
      if (wu.len() == 0) return 0;
      const Win wv = window(c, 1, c.v);
      int path[kMaxChain];
      if (wv.len() > kOuterSplit && warp_emit(em, path, wv)) return 0;
      return warp_sum(cycle_dfs(c, p.min_size, p.cycle_len - 3, path, 0, wv.a + lane, wv.b, 32, wu,
                                nullptr, em));
    }
    case TM_SG: {
      const Win w = window(c, 0, c.u);
      int path[1];
      if (w.len() > kOuterSplit && warp_emit(em, path, w)) return 0;
      long long n = 0;
      for (int j = w.a + lane; j < w.b; j += 32) n += sg_entry(c, p.min_size, j, nullptr);
      return warp_sum(n);
    }
    case TM_GS: {
      const Win w = window(c, 1, c.v);
      int path[1];
      if (w.len() > kOuterSplit && warp_emit(em, path, w)) return 0;
      long long n = 0;
      for (int j = w.a + lane; j < w.b; j += 32) n += gs_entry(c, p.min_size, j, nullptr);
      return warp_sum(n);
    }
    case TM_STACK: {
      const Win wa = window(c, 0, c.u);
      const long long a = warp_sum(distinct_range(c, 0, c.u, c.v, wa.a + lane, wa.b, 32));
      if (a == 0 || a < p.min_size) return 0;
      const Win wc = window(c, 1, c.v);
      const long long d = warp_sum(distinct_range(c, 1, c.v, c.u, wc.a + lane, wc.b, 32));
      if (d == 0 || d < p.min_size) return 0;
      return a * d;
    }
    default: return 0;
  }
}

struct Queues {
  Task *q;
  int32_t *count;
  int32_t cap;
};

__global__ void __launch_bounds__(kHeavyThreads) k_mine_heavy(
    const DevGraph g, const DevPlans plans, int64_t lo, long long *__restrict__ out,
    const int32_t *__restrict__ heavy_q, const int32_t *__restrict__ heavy_n, Queues tq) {
  const int n = *heavy_n;
  const int warps = gridDim.x * (blockDim.x >> 5);
  for (int i = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5); i < n; i += warps) {
    const int row = heavy_q[i];
    const int e = (int)(lo + row);
    const int u = __ldg(g.e_src + e), v = __ldg(g.e_dst + e);
    const uint32_t r = __ldg(g.e_rank + e);
    long long *o = out + (int64_t)row * plans.n;
    for (int ci = 0; ci < plans.n; ++ci) {
      const DevPlan p = plans.p[ci];
      const Ctx c{g, u, v, __ldg(p.lo_tab + r), r};
      const Emitter em{tq.q, tq.count, tq.cap, row, ci, true};
      const long long val = eval_heavy(c, p, em);
      if ((threadIdx.x & 31) == 0) o[ci] = val;
    }
  }
}

// ------------------------------------------------------------- tier 3

__global__ void __launch_bounds__(kHeavyThreads) k_mine_tasks(
    const DevGraph g, const DevPlans plans, int64_t lo, long long *__restrict__ out, Queues in,
    Queues next) {
  const int n = min(*in.count, in.cap);
  const int warps = gridDim.x * (blockDim.x >> 5);
  const int lane = threadIdx.x & 31;
  for (int i = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5); i < n; i += warps) {
    const Task t = in.q[i];
    if (t.row < 0) continue;
    const int e = (int)(lo + t.row);
    const int u = __ldg(g.e_src + e), v = __ldg(g.e_dst + e);
    const uint32_t r = __ldg(g.e_rank + e);
    const DevPlan p = plans.p[t.col];
    const Ctx c{g, u, v, __ldg(p.lo_tab + r), r};
    const Emitter em{next.q, next.count, next.cap, t.row, t.col, true};
    long long part = 0;
    if (p.family == TM_SG) {
      for (int j = t.a + lane; j < t.b; j += 32) part += sg_entry(c, p.min_size, j, nullptr);
    } else if (p.family == TM_GS) {
      for (int j = t.a + lane; j < t.b; j += 32) part += gs_entry(c, p.min_size, j, nullptr);
    } else if (p.family == TM_CYCLE && p.cycle_len >= 4) {
      const Win wu = window(c, 0, c.u);
      int path[kMaxChain];
#pragma unroll
      for (int k = 0; k < kMaxChain; ++k) path[k] = t.path[k];
      part = cycle_dfs(c, p.min_size, p.cycle_len - 3, path, t.level, t.a + lane, t.b, 32, wu,
                       nullptr, em);
    }
    part = warp_sum(part);
    if (lane == 0 && part) atomicAdd(reinterpret_cast<unsigned long long *>(out + (int64_t)t.row * plans.n + t.col),
                                     (unsigned long long)part);
  }
}

// lo_tab[r] = lower_bound(uniq_time, uniq_time[r] - delta)
__global__ void k_lo_table(const int64_t *__restrict__ uniq, int64_t R, long long delta,
                           uint32_t *__restrict__ lo_tab) {
  const int64_t r = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (r >= R) return;
  const long long t = uniq[r];
  int64_t a = 0, b = r;  // answer <= r since delta >= 0
  if (t >= LLONG_MIN + delta) {
    const long long x = t - delta;
    while (a < b) {
      int64_t m = (a + b) >> 1;
      if (__ldg(uniq + m) < x) a = m + 1; else b = m;
    }
  }
  lo_tab[r] = (uint32_t)a;
}

}  // namespace
}  // namespace tmb

using namespace tmb;

extern "C" int tm_mine(tm_graph *g, const tm_plan_desc *plans, int n_plans, int64_t lo, int64_t hi,
                       int64_t *out, int out_on_device, void *stream) {
  if (!g) return fail(TM_E_BAD_ARG, "graph is NULL");
  if (n_plans < 0 || n_plans > kMaxPlans)
    return fail(TM_E_BAD_ARG, "n_plans must be in [0, " + std::to_string(kMaxPlans) + "]");
  if (n_plans > 0 && !plans) return fail(TM_E_BAD_ARG, "plans is NULL");
  if (lo < 0 || hi < lo || hi > g->n_edges) return fail(TM_E_BAD_ARG, "bad trigger range");
  const int64_t rows = hi - lo;
  if (rows > 0 && n_plans > 0 && !out) return fail(TM_E_BAD_ARG, "out is NULL");
  for (int i = 0; i < n_plans; ++i) {
    const tm_plan_desc &p = plans[i];
    if (p.family < TM_FAN || p.family > TM_STACK)
      return fail(TM_E_UNSUPPORTED_PLAN, "plan " + std::to_string(i) + ": unknown family");
    if (p.family == TM_CYCLE && (p.cycle_len < 2 || p.cycle_len > 8))
      return fail(TM_E_UNSUPPORTED_PLAN, "plan " + std::to_string(i) + ": cycle length must be 2..8");
    if (p.min_size < 1) return fail(TM_E_BAD_ARG, "plan " + std::to_string(i) + ": min_size < 1");
    if (p.delta < 0) return fail(TM_E_BAD_ARG, "plan " + std::to_string(i) + ": negative delta");
    if ((p.family == TM_FAN || p.family == TM_DEGREE) &&
        ((p.endpoint != 0 && p.endpoint != 1) || (p.direction != 0 && p.direction != 1)))
      return fail(TM_E_BAD_ARG, "plan " + std::to_string(i) + ": bad endpoint/direction");
  }
  g->last = tm_mine_stats{};
  g->prof_pending = false;
  g->last.triggers = rows;
  g->last.light_ms = g->last.heavy_ms = -1.f;
  if (rows == 0 || n_plans == 0) return TM_OK;
  TM_CUDA(cudaSetDevice(g->device));
  cudaStream_t s = stream ? static_cast<cudaStream_t>(stream) : g->stream;
  const int64_t launches0 = tm_kernel_launch_count();

  // distinct deltas -> window lower-bound tables
  int64_t deltas[kMaxPlans];
  int slot_of[kMaxPlans];
  int nd = 0;
  for (int i = 0; i < n_plans; ++i) {
    int k = 0;
    while (k < nd && deltas[k] != plans[i].delta) ++k;
    if (k == nd) deltas[nd++] = plans[i].delta;
    slot_of[i] = k;
  }
  const int64_t R = g->n_ranks;
  int rc;
  if ((rc = g->lo_tabs.ensure(sizeof(uint32_t) * (size_t)(R > 0 ? R : 1) * nd))) return rc;
  for (int k = 0; k < nd; ++k) {
    k_lo_table<<<grid_for(R, 256), 256, 0, s>>>(g->uniq_time.as<int64_t>(), R, deltas[k],
                                                g->lo_tabs.as<uint32_t>() + (size_t)k * R);
    TM_LAUNCHED("k_lo_table");
  }
  DevPlans dp{};
  dp.n = n_plans;
  int rounds = 0;
  for (int i = 0; i < n_plans; ++i) {
    const tm_plan_desc &p = plans[i];
    dp.p[i] = DevPlan{p.family, p.endpoint, p.direction, p.exclude_trigger, p.cycle_len,
                      p.min_size, g->lo_tabs.as<uint32_t>() + (size_t)slot_of[i] * R};
    if (!(p.family == TM_FAN || p.family == TM_DEGREE ||
          (p.family == TM_CYCLE && p.cycle_len == 2)))
      dp.needs_sets = 1;
    // task rounds: level-0 pieces (sg/gs/cycle) + one per deeper chain level
    if (p.family == TM_SG || p.family == TM_GS) rounds = std::max(rounds, 1);
    if (p.family == TM_CYCLE && p.cycle_len >= 4) rounds = std::max(rounds, p.cycle_len - 3);
  }

  long long *d_out;
  if (out_on_device) {
    d_out = reinterpret_cast<long long *>(out);
  } else {
    if ((rc = g->out_scratch.ensure(sizeof(long long) * (size_t)rows * n_plans))) return rc;
    d_out = g->out_scratch.as<long long>();
  }
  // counters: [0] heavy rows, [1..2] task queues A/B
  const int64_t task_cap = std::min<int64_t>(std::max<int64_t>(1 << 20, rows / 2), 1 << 24);
  if ((rc = g->heavy_n.ensure(sizeof(int32_t) * 4)) ||
      (rc = g->heavy_q.ensure(sizeof(int32_t) * (size_t)rows)) ||
      (rc = g->tasks.ensure(sizeof(Task) * (size_t)task_cap * 2)))
    return rc;
  int32_t *cnt = g->heavy_n.as<int32_t>();
  TM_CUDA(cudaMemsetAsync(cnt, 0, sizeof(int32_t) * 4, s));
  Queues qa{g->tasks.as<Task>(), cnt + 1, (int32_t)task_cap};
  Queues qb{g->tasks.as<Task>() + task_cap, cnt + 2, (int32_t)task_cap};

  const DevGraph dg = g->dev();
  g->prof_pending = g->prof;
  if (g->prof) TM_CUDA(cudaEventRecord(g->ev[0], s));
  k_mine_light<<<grid_for(rows, kLightThreads), kLightThreads, 0, s>>>(dg, dp, lo, rows, d_out,
                                                                      g->heavy_q.as<int32_t>(), cnt);
  TM_LAUNCHED("k_mine_light");
  if (g->prof) TM_CUDA(cudaEventRecord(g->ev[1], s));
  if (dp.needs_sets) {
    const int grid = 148 * (2048 / kHeavyThreads);
    k_mine_heavy<<<grid, kHeavyThreads, 0, s>>>(dg, dp, lo, d_out, g->heavy_q.as<int32_t>(), cnt, qa);
    TM_LAUNCHED("k_mine_heavy");
    for (int r = 0; r < rounds; ++r) {
      TM_CUDA(cudaMemsetAsync(qb.count, 0, sizeof(int32_t), s));
      k_mine_tasks<<<grid, kHeavyThreads, 0, s>>>(dg, dp, lo, d_out, qa, qb);
      TM_LAUNCHED("k_mine_tasks");
      std::swap(qa, qb);
    }
  }
  if (g->prof) TM_CUDA(cudaEventRecord(g->ev[2], s));
  if (!out_on_device) {
    TM_CUDA(cudaMemcpyAsync(out, d_out, sizeof(long long) * (size_t)rows * n_plans,
                            cudaMemcpyDeviceToHost, s));
    int32_t nh = 0;
    TM_CUDA(cudaMemcpyAsync(&nh, cnt, sizeof(int32_t), cudaMemcpyDeviceToHost, s));
    TM_CUDA(cudaStreamSynchronize(s));
    g->last.heavy_triggers = nh;
  } else {
    g->last.heavy_triggers = -1;  // not read back on the async path
  }
  g->last.kernel_launches = tm_kernel_launch_count() - launches0;
  return TM_OK;
}

extern "C" int tm_last_mine_stats(tm_graph *g, tm_mine_stats *stats) {
  if (!g || !stats) return fail(TM_E_BAD_ARG, "NULL argument");
  if (g->prof_pending) {
    TM_CUDA(cudaSetDevice(g->device));
    TM_CUDA(cudaEventSynchronize(g->ev[2]));
    TM_CUDA(cudaEventElapsedTime(&g->last.light_ms, g->ev[0], g->ev[1]));
    TM_CUDA(cudaEventElapsedTime(&g->last.heavy_ms, g->ev[1], g->ev[2]));
    g->prof_pending = false;
  }
  *stats = g->last;
  return TM_OK;
}

extern "C" int tm_set_profiling(tm_graph *g, int on) {
  if (!g) return fail(TM_E_BAD_ARG, "NULL graph");
  TM_CUDA(cudaSetDevice(g->device));
  for (int i = 0; i < 3; ++i)
    if (!g->ev[i]) TM_CUDA(cudaEventCreate(&g->ev[i]));
  g->prof = on != 0;
  return TM_OK;
}
