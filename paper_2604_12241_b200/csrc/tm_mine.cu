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
//   k_mine_light   one THREAD per trigger edge, all columns.  The trigger's
//                  four windows are bisected once per delta group; set
//                  columns iterate the SMALLER windowed slice and test the
//                  other side with one pair-index bisection; distinct-ness is
//                  an O(1) pair-predecessor test.  Each trigger carries a
//                  work budget; a trigger that would exceed it is appended to
//                  the heavy queue (warp-aggregated atomic) and left to ...
//   k_mine_heavy   one WARP per heavy trigger: each column's outer slice is
//                  spread over the lanes.  Outer slices longer than
//                  kOuterSplit, and — inside cycle_k's depth-first chain
//                  enumeration — every node whose windowed out-slice is
//                  longer than kDeepSplit, are not walked serially but cut
//                  into range TASKS of kTaskSpan entries, appended to a task
//                  queue and ...
//   k_mine_tasks   one WARP per task, lane per slice entry, launched in
//                  rounds (a task only spawns tasks deeper in the chain, so
//                  <= 5 rounds for cycle_8).  Partial counts are combined
//                  with atomicAdd on the int64 output cell, which the heavy
//                  kernel initialized with its own partial.
// Every count is an integer sum over disjoint pieces, so the result is
// exactly the reference's regardless of the split.
//
// The chain enumeration is a compile-time-depth template (chain_level<CHAIN,
// L>) so the path and loop state stay in registers; kernel parameters are
// __grid_constant__ so taking their address does not spill them to local
// memory.
#include "tm_internal.cuh"

namespace tmb {
namespace {

constexpr int kLightThreads = 128;
constexpr int kHeavyThreads = 256;
constexpr int kLightBudget = 96;   // default slice entries + probes per light trigger
constexpr int kOuterSplit = 512;   // heavy row: outer slices above this become tasks
constexpr int kDeepSplit = 64;     // chain nodes with wider windows become tasks
constexpr int kTaskSpan = 128;     // entries per task (4 per lane)
constexpr int kMaxChain = 5;       // cycle_8: a1..a5
constexpr int kStageCols = 16;     // light rows staged in smem up to this many columns

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
  const DevGraph &g;  // a __grid_constant__ kernel parameter
  int u, v;
  uint32_t lo, hi;    // window in rank space
  Win wui, wuo, wvi, wvo;  // trigger windows, see fill_windows
};

// windowed slice of x's dir-run: rank in [lo, hi]   (kernels.py:268-276).
// Runs of <= kSmallRun entries (most accounts) are read with independent
// loads and counted in registers — one memory round trip instead of two
// dependent bisections; longer runs bisect.
#ifndef TM_SMALL_RUN  // 0: always bisect (measured faster, see profiles/)
#define TM_SMALL_RUN 0
#endif
constexpr int kSmallRun = TM_SMALL_RUN;
__device__ __forceinline__ Win window(const Ctx &c, int dir, int x) {
  const int a = __ldg(c.g.ptr[dir] + x), b = __ldg(c.g.ptr[dir] + x + 1);
  const uint32_t *r = c.g.rnk[dir];
  if (kSmallRun > 0 && b - a <= kSmallRun) {
    int below = 0, upto = 0;
#pragma unroll
    for (int i = 0; i < kSmallRun; ++i) {
      if (a + i < b) {
        const uint32_t t = __ldg(r + a + i);
        below += t < c.lo;
        upto += t <= c.hi;
      }
    }
    return {a + below, a + upto};
  }
  const int wa = lb_u32(r, a, b, c.lo);
  return {wa, ub_u32(r, wa, b, c.hi)};
}

// the trigger-endpoint windows a plan group needs (DevPlan::need bits:
// 1 u-in, 2 u-out, 4 v-in, 8 v-out) — bisected once per trigger and delta
__device__ __forceinline__ void fill_windows(Ctx &c, int need) {
  if (need & 1) c.wui = window(c, 0, c.u);
  if (need & 2) c.wuo = window(c, 1, c.u);
  if (need & 4) c.wvi = window(c, 0, c.v);
  if (need & 8) c.wvo = window(c, 1, c.v);
}

// self-loops of x inside the window (kernels.py:279-287): pair run (x, x)
__device__ __forceinline__ int loops_in_window(const Ctx &c, int x) {
  if (!__ldg(c.g.loop + x)) return 0;
  const int a = __ldg(c.g.ptr[1] + x), b = __ldg(c.g.ptr[1] + x + 1);
  const uint64_t base = (uint64_t)(uint32_t)x << c.g.rank_bits;
  return lb_u64(c.g.pkey[1], a, b, base + c.hi + 1) - lb_u64(c.g.pkey[1], a, b, base + c.lo);
}

// CSR entry j is the first occurrence of its neighbour inside the window
// (np.unique, kernels.py:59): the previous entry with the same (owner, nbr)
// lies before lo (prev = rank + 1, 0 = none)
__device__ __forceinline__ bool first_in_window(const Ctx &c, int dir, int j) {
  return __ldg(c.g.prev[dir] + j) <= c.lo;
}

// does x's dir-window w contain neighbour n?  Windows are time-local and
// short: scan them; fall back to a pair-run bisection when w is wide.
#ifndef TM_SCAN_WIN
#define TM_SCAN_WIN 16
#endif
constexpr int kScanWin = TM_SCAN_WIN;
__device__ __forceinline__ bool exists_in(const Ctx &c, int dir, int x, const Win &w, int n) {
  if (w.len() <= kScanWin) {
    bool hit = false;
    for (int j = w.a; j < w.b && !hit; ++j) hit = __ldg(c.g.nbr[dir] + j) == n;
    return hit;
  }
  const int s = __ldg(c.g.ptr[dir] + x), e = __ldg(c.g.ptr[dir] + x + 1);
  const uint64_t base = (uint64_t)(uint32_t)n << c.g.rank_bits;
  const int q = lb_u64(c.g.pkey[dir], s, e, base + c.lo);
  return q < e && __ldg(c.g.pkey[dir] + q) <= base + c.hi;
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
  int8_t pad0, pad1;
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
  // emission is off or the queue is full.  Path by value: no address taken.
  __device__ bool emit(int level, int p0, int p1, int p2, int p3, int p4, int a, int b) const {
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
      t.pad0 = t.pad1 = 0;
      t.a = a + k * kTaskSpan;
      t.b = min(b, t.a + kTaskSpan);
      t.path[0] = p0; t.path[1] = p1; t.path[2] = p2; t.path[3] = p3; t.path[4] = p4;
      q[base + k] = t;
    }
    return true;
  }
};

// ---------------------------------------------------------- families

// FAN / DEGREE (kernels.py:290-303)
__device__ __forceinline__ long long col_fan_degree(const Ctx &c, const DevPlan &p) {
  const int x = p.endpoint ? c.v : c.u;
  const Win w = p.endpoint ? (p.direction ? c.wvo : c.wvi) : (p.direction ? c.wuo : c.wui);
  long long n = w.len() - loops_in_window(c, x);
  if (p.exclude_trigger && c.u != c.v) n -= 1;
  if (p.min_size > 1 && n < p.min_size) n = 0;
  return n;
}

// cycle_2 = [u != v and v -> u in window] (kernels.py:320-322)
__device__ __forceinline__ long long col_cycle2(const Ctx &c, const DevPlan &p) {
  if (c.u == c.v) return 0;
  long long raw = exists_in(c, 1, c.v, c.wvo, c.u) ? 1 : 0;
  return raw >= p.min_size ? raw : 0;
}

// distinct windowed neighbours of x in dir over CSR range [ja, jb) with
// stride, excluding x (self-loops) and ex
__device__ __forceinline__ long long distinct_range(const Ctx &c, int dir, int x, int ex, int ja,
                                                    int jb, int stride) {
  long long n = 0;
#pragma unroll 4
  for (int j = ja; j < jb; j += stride) {
    const int y = __ldg(c.g.nbr[dir] + j);
    if (y == x || y == ex) continue;
    n += first_in_window(c, dir, j);
  }
  return n;
}

// |N^{dx}(x) ∩ N^{dy}(y)|, early exit at K (sg: x = s out, y = v in;
// gs: x = d in, y = u out).  x and y are never members (no self-loops).
__device__ __forceinline__ int inner_hits(const Ctx &c, int x, int dx, int y, int dy,
                                          const Win &wy, int K, Budget *bud) {
  const Win wx = window(c, dx, x);
  const bool walk_x = wx.len() <= wy.len();
  const Win w = walk_x ? wx : wy;
  if (bud && !bud->take(2 * w.len())) return 0;
  const int owner = walk_x ? x : y, other = walk_x ? y : x;
  const int d = walk_x ? dx : dy, od = walk_x ? dy : dx;
  const Win ow = walk_x ? wy : wx;
  int hits = 0;
  for (int j = w.a; j < w.b && hits < K; ++j) {
    const int m = __ldg(c.g.nbr[d] + j);
    if (m == owner || m == other || !first_in_window(c, d, j)) continue;
    hits += exists_in(c, od, other, ow, m);
  }
  return hits;
}

// sg entry: s = CSR in-entry j of u; #{s : |N+(s) ∩ N-(v)| >= K} (kernels.py:358-375)
__device__ __forceinline__ int sg_entry(const Ctx &c, int K, int seg_u, int j, Budget *bud) {
  const int s = __ldg(c.g.nbr[0] + j);
  if (s == c.u || s == c.v || !first_in_window(c, 0, j)) return 0;
  return inner_hits(c, s, 1, c.v, 0, c.wvi, K, bud) >= K;
}

// gs entry: d = CSR out-entry j of v; #{d : |N-(d) ∩ N+(u)| >= K} (Appendix B)
__device__ __forceinline__ int gs_entry(const Ctx &c, int K, int seg_v, int j, Budget *bud) {
  const int d = __ldg(c.g.nbr[1] + j);
  if (d == c.v || d == c.u || !first_in_window(c, 1, j)) return 0;
  return inner_hits(c, d, 0, c.u, 1, c.wuo, K, bud) >= K;
}

// closing set size for a chain ending at `a` with NP earlier chain nodes:
//   |(N+(a) ∩ N-(u)) \ {v, path[0..NP-1]}|   (Appendix A cycle_k; cycle_4
//   kernels.py:330-341 for NP = 0).
template <int NP>
__device__ __forceinline__ int close_count(const Ctx &c, int a, const int (&path)[kMaxChain],
                                           Budget *bud) {
  const Win wa = window(c, 1, a);
  const bool walk_a = wa.len() <= c.wui.len();
  const Win w = walk_a ? wa : c.wui;
  if (bud && !bud->take(2 * w.len())) return 0;
  const int d = walk_a ? 1 : 0;
  int cnt = 0;
  for (int j = w.a; j < w.b; ++j) {
    const int m = __ldg(c.g.nbr[d] + j);
    if (m == a || m == c.u || m == c.v) continue;
    bool dup = false;
#pragma unroll
    for (int i = 0; i < NP; ++i) dup |= (path[i] == m);
    if (dup || !first_in_window(c, d, j)) continue;
    cnt += walk_a ? exists_in(c, 0, c.u, c.wui, m) : exists_in(c, 1, a, wa, m);
  }
  return cnt;
}

// Fused cycle group: every CYCLE column (length 3..8) of one delta shares
// one depth-first chain enumeration.  Depth d = chain length (number of
// intermediate accounts a1..a_d); cycle_{d+3} is closed at depth d:
//   a1 in N+(v)\{u};  a_i in N+(a_{i-1}) \ {u, v, a1..a_{i-2}};
//   each chain adds |C| = close_count(a_d) when |C| >= K_{d+3}
//   (depth 0: a = v, C = N+(v) ∩ N-(u) \ {u, v} = cycle_3, kernels.py:323-327;
//   depth 1: cycle_4, kernels.py:328-343; depths 2..5: cycle_5..8, Appendix A).
// Level L enumerates the entries j in [ja, jb) (stride) of the out-slice of
// its owner (v for L = 0, else a_L = path[L-1]); the chosen node is a_{L+1}
// at depth L+1.  A node whose window exceeds kDeepSplit is handed to the
// emitter as tasks instead of being walked (when emission is on).
struct CycAcc {
  long long d[kMaxChain + 1];
};

template <int MAXD, int L>
__device__ __forceinline__ void chain_level(const Ctx &c, const CycGroup &cg,
                                            int (&path)[kMaxChain], int ja, int jb, int stride,
                                            CycAcc &acc, Budget *bud, const Emitter &em) {
  const int owner = L == 0 ? c.v : path[L > 0 ? L - 1 : 0];
  for (int j = ja; j < jb; j += stride) {
    const int a = __ldg(c.g.nbr[1] + j);
    if (a == owner || a == c.u || a == c.v) continue;
    bool dup = false;
#pragma unroll
    for (int i = 0; i + 1 < L; ++i) dup |= (path[i] == a);
    if (dup || !first_in_window(c, 1, j)) continue;
    if (cg.mask & (1 << (L + 1))) {
      const int cc = close_count<L>(c, a, path, bud);
      if (bud && bud->blown) return;
      if (cc >= cg.k[L + 1]) acc.d[L + 1] += cc;
    }
    if constexpr (L + 1 < MAXD) {
      path[L] = a;
      const Win w = window(c, 1, a);
      if (w.len() > kDeepSplit &&
          em.emit(L + 1, path[0], path[1], path[2], path[3], path[4], w.a, w.b))
        continue;
      if (bud && !bud->take(w.len())) return;
      chain_level<MAXD, L + 1>(c, cg, path, w.a, w.b, 1, acc, bud, em);
      if (bud && bud->blown) return;
    }
  }
}

// runtime (max depth, start level) -> template instance
__device__ __forceinline__ void cycle_chain(const Ctx &c, const CycGroup &cg, int L0,
                                            const int (&path0)[kMaxChain], int ja, int jb,
                                            int stride, CycAcc &acc, Budget *bud,
                                            const Emitter &em) {
  int path[kMaxChain] = {path0[0], path0[1], path0[2], path0[3], path0[4]};
  switch (cg.maxd * 8 + L0) {
#define TM_CHAIN_CASE(C_, L_) \
  case C_ * 8 + L_: chain_level<C_, L_>(c, cg, path, ja, jb, stride, acc, bud, em); return;
    TM_CHAIN_CASE(1, 0)
    TM_CHAIN_CASE(2, 0) TM_CHAIN_CASE(2, 1)
    TM_CHAIN_CASE(3, 0) TM_CHAIN_CASE(3, 1) TM_CHAIN_CASE(3, 2)
    TM_CHAIN_CASE(4, 0) TM_CHAIN_CASE(4, 1) TM_CHAIN_CASE(4, 2) TM_CHAIN_CASE(4, 3)
    TM_CHAIN_CASE(5, 0) TM_CHAIN_CASE(5, 1) TM_CHAIN_CASE(5, 2) TM_CHAIN_CASE(5, 3)
    TM_CHAIN_CASE(5, 4)
#undef TM_CHAIN_CASE
    default: return;
  }
}

// depth-0 close (cycle_3) of a group, uniform across lanes
__device__ __forceinline__ long long cycle3_of(const Ctx &c, const CycGroup &cg, Budget *bud) {
  if (!(cg.mask & 1)) return 0;
  const int path[kMaxChain] = {-1, -1, -1, -1, -1};
  const int cc = close_count<0>(c, c.v, path, bud);
  return cc >= cg.k[0] ? cc : 0;
}

// ------------------------------------------------------------- tier 1

// cycle group in one thread (budgeted): acc.d[d] = column of length d + 3
__device__ __forceinline__ void eval_cycle_group_light(const Ctx &c, const CycGroup &cg, CycAcc &acc,
                                                       Budget &bud, const Emitter &off) {
#pragma unroll
  for (int d = 0; d <= kMaxChain; ++d) acc.d[d] = 0;
  if (c.u == c.v || c.wui.len() == 0 || c.wvo.len() == 0) return;
  acc.d[0] = cycle3_of(c, cg, &bud);
  if (bud.blown || cg.maxd == 0) return;
  if (!bud.take(c.wvo.len())) return;
  const int path[kMaxChain] = {-1, -1, -1, -1, -1};
  cycle_chain(c, cg, 0, path, c.wvo.a, c.wvo.b, 1, acc, &bud, off);
}

// full column, one thread, budgeted
__device__ __forceinline__ long long eval_light(const Ctx &c, const DevPlan &p, Budget &bud,
                                                const Emitter &off) {
  switch (p.family) {
    case TM_FAN:
    case TM_DEGREE: return col_fan_degree(c, p);
    case TM_CYCLE:  // cycle_2 only; lengths >= 3 go through eval_cycle_group
      return col_cycle2(c, p);
    case TM_SG: {
      const Win w = c.wui;
      if (!bud.take(w.len())) return 0;
      const int seg = __ldg(c.g.ptr[0] + c.u);
      long long n = 0;
      for (int j = w.a; j < w.b; ++j) {
        n += sg_entry(c, p.min_size, seg, j, &bud);
        if (bud.blown) return 0;
      }
      return n;
    }
    case TM_GS: {
      const Win w = c.wvo;
      if (!bud.take(w.len())) return 0;
      const int seg = __ldg(c.g.ptr[1] + c.v);
      long long n = 0;
      for (int j = w.a; j < w.b; ++j) {
        n += gs_entry(c, p.min_size, seg, j, &bud);
        if (bud.blown) return 0;
      }
      return n;
    }
    case TM_STACK: {  // kernels.py:379-402
      if (!bud.take(c.wui.len())) return 0;
      const long long a = distinct_range(c, 0, c.u, c.v, c.wui.a, c.wui.b, 1);
      if (a == 0 || a < p.min_size) return 0;
      if (!bud.take(c.wvo.len())) return 0;
      const long long d = distinct_range(c, 1, c.v, c.u, c.wvo.a, c.wvo.b, 1);
      if (d == 0 || d < p.min_size) return 0;
      return a * d;
    }
    default: return 0;
  }
}

__global__ void __launch_bounds__(kLightThreads) k_mine_light(
    const __grid_constant__ DevGraph g, const __grid_constant__ DevPlans plans, int64_t lo,
    int64_t n_rows, long long *__restrict__ out, int32_t *__restrict__ heavy_q,
    int32_t *__restrict__ heavy_n, int budget) {
  extern __shared__ long long stage[];  // per warp [32][plans.n] when plans.n <= kStageCols
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int64_t wrow0 = (int64_t)blockIdx.x * blockDim.x + warp * 32;
  const int64_t row = wrow0 + lane;
  const int C = plans.n;
  const bool staged = C <= kStageCols;
  long long *wstage = stage + (size_t)warp * 32 * C;
  bool heavy = false;
  if (row < n_rows) {
    const int e = (int)(lo + row);
    const int u = __ldg(g.e_src + e), v = __ldg(g.e_dst + e);
    const uint32_t r = __ldg(g.e_rank + e);
    Budget bud{budget, false};
    const Emitter off{nullptr, nullptr, 0, 0, 0, false};
    Ctx c{g, u, v, 0u, r, {}, {}, {}, {}};
    const uint32_t *cur = nullptr;
    long long *o = staged ? wstage + lane * C : out + row * C;
    for (int ci = 0; ci < C; ++ci) {
      const DevPlan &p = plans.p[ci];
      if (p.lo_tab != cur) {  // new delta group: its windows, once
        cur = p.lo_tab;
        c.lo = __ldg(cur + r);
        fill_windows(c, p.need_group);
      }
      if (p.family == TM_CYCLE && p.cycle_len >= 3) {
        if (p.cyc.lead) {  // one fused enumeration writes every member column
          CycAcc acc;
          eval_cycle_group_light(c, p.cyc, acc, bud, off);
          if (bud.blown) { heavy = true; break; }
#pragma unroll
          for (int d = 0; d <= kMaxChain; ++d)
            if (p.cyc.mask & (1 << d)) o[p.cyc.col[d]] = acc.d[d];
        }
        continue;
      }
      const long long val = eval_light(c, p, bud, off);
      if (bud.blown) { heavy = true; break; }
      o[ci] = val;
    }
  }
  if (staged) {  // coalesced write-back of the warp's 32 rows (no block barrier)
    __syncwarp();
    const int64_t left = n_rows - wrow0;
    const int nrow = left < 32 ? (int)(left > 0 ? left : 0) : 32;
    long long *dst = out + wrow0 * C;
    for (int i = lane; i < nrow * C; i += 32) dst[i] = wstage[i];
  }
  // warp-aggregated append of heavy triggers (their rows are rewritten by
  // k_mine_heavy)
  const unsigned m = __ballot_sync(0xffffffffu, heavy);
  if (m) {
    int base = 0;
    if (lane == __ffs(m) - 1) base = atomicAdd(heavy_n, __popc(m));
    base = __shfl_sync(0xffffffffu, base, __ffs(m) - 1);
    if (heavy) heavy_q[base + __popc(m & ((1u << lane) - 1))] = (int32_t)row;
  }
}

// ------------------------------------------------------------- tier 2

// warp-uniform emission of a level-0 slice: lane 0 emits, all lanes agree
__device__ __forceinline__ bool warp_emit(const Emitter &em, const Win &w) {
  int ok = 0;
  if ((threadIdx.x & 31) == 0) ok = em.emit(0, -1, -1, -1, -1, -1, w.a, w.b) ? 1 : 0;
  return __shfl_sync(0xffffffffu, ok, 0) != 0;
}

// one warp, one heavy trigger, one column: returns the warp's partial (all
// lanes hold it); pieces beyond kOuterSplit / kDeepSplit are emitted
__device__ long long eval_heavy(const Ctx &c, const DevPlan &p, const Emitter &em) {
  const int lane = threadIdx.x & 31;
  switch (p.family) {
    case TM_FAN:
    case TM_DEGREE: return col_fan_degree(c, p);
    case TM_CYCLE:  // cycle_2 only; lengths >= 3 go through the group path
      return col_cycle2(c, p);
    case TM_SG: {
      if (c.wui.len() > kOuterSplit && warp_emit(em, c.wui)) return 0;
      const int seg = __ldg(c.g.ptr[0] + c.u);
      long long n = 0;
      for (int j = c.wui.a + lane; j < c.wui.b; j += 32) n += sg_entry(c, p.min_size, seg, j, nullptr);
      return warp_sum(n);
    }
    case TM_GS: {
      if (c.wvo.len() > kOuterSplit && warp_emit(em, c.wvo)) return 0;
      const int seg = __ldg(c.g.ptr[1] + c.v);
      long long n = 0;
      for (int j = c.wvo.a + lane; j < c.wvo.b; j += 32) n += gs_entry(c, p.min_size, seg, j, nullptr);
      return warp_sum(n);
    }
    case TM_STACK: {
      const long long a = warp_sum(distinct_range(c, 0, c.u, c.v, c.wui.a + lane, c.wui.b, 32));
      if (a == 0 || a < p.min_size) return 0;
      const long long d = warp_sum(distinct_range(c, 1, c.v, c.u, c.wvo.a + lane, c.wvo.b, 32));
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
    const __grid_constant__ DevGraph g, const __grid_constant__ DevPlans plans, int64_t lo,
    long long *__restrict__ out, const int32_t *__restrict__ heavy_q,
    const int32_t *__restrict__ heavy_n, Queues tq) {
  const int n = *heavy_n;
  const int warps = gridDim.x * (blockDim.x >> 5);
  const int lane = threadIdx.x & 31;
  for (int i = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5); i < n; i += warps) {
    const int row = heavy_q[i];
    const int e = (int)(lo + row);
    const int u = __ldg(g.e_src + e), v = __ldg(g.e_dst + e);
    const uint32_t r = __ldg(g.e_rank + e);
    long long *o = out + (int64_t)row * plans.n;
    for (int ci = 0; ci < plans.n; ++ci) {
      const DevPlan &p = plans.p[ci];
      Ctx c{g, u, v, __ldg(p.lo_tab + r), r, {}, {}, {}, {}};
      fill_windows(c, p.need);
      const Emitter em{tq.q, tq.count, tq.cap, row, ci, true};
      if (p.family == TM_CYCLE && p.cycle_len >= 3) {
        if (!p.cyc.lead) continue;
        // cycle group: depth 0 (cycle_3) uniform; chains spread over lanes,
        // wide nodes / a wide first slice become tasks
        CycAcc acc;
#pragma unroll
        for (int d = 0; d <= kMaxChain; ++d) acc.d[d] = 0;
        if (c.u != c.v && c.wui.len() > 0 && c.wvo.len() > 0) {
          acc.d[0] = cycle3_of(c, p.cyc, nullptr);
          if (p.cyc.maxd > 0 && !(c.wvo.len() > kOuterSplit && warp_emit(em, c.wvo))) {
            const int path[kMaxChain] = {-1, -1, -1, -1, -1};
            cycle_chain(c, p.cyc, 0, path, c.wvo.a + lane, c.wvo.b, 32, acc, nullptr, em);
          }
        }
#pragma unroll
        for (int d = 1; d <= kMaxChain; ++d) acc.d[d] = warp_sum(acc.d[d]);
        if (lane == 0) {
#pragma unroll
          for (int d = 0; d <= kMaxChain; ++d)
            if (p.cyc.mask & (1 << d)) o[p.cyc.col[d]] = acc.d[d];
        }
        continue;
      }
      const long long val = eval_heavy(c, p, em);
      if (lane == 0) o[ci] = val;
    }
  }
}

// ------------------------------------------------------------- tier 3

__global__ void __launch_bounds__(kHeavyThreads) k_mine_tasks(
    const __grid_constant__ DevGraph g, const __grid_constant__ DevPlans plans, int64_t lo,
    long long *__restrict__ out, Queues in, Queues next) {
  const int n = min(*in.count, in.cap);
  const int warps = gridDim.x * (blockDim.x >> 5);
  const int lane = threadIdx.x & 31;
  for (int i = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5); i < n; i += warps) {
    const Task t = in.q[i];
    if (t.row < 0) continue;
    const int e = (int)(lo + t.row);
    const int u = __ldg(g.e_src + e), v = __ldg(g.e_dst + e);
    const uint32_t r = __ldg(g.e_rank + e);
    const DevPlan &p = plans.p[t.col];
    Ctx c{g, u, v, __ldg(p.lo_tab + r), r, {}, {}, {}, {}};
    fill_windows(c, p.need);
    const Emitter em{next.q, next.count, next.cap, t.row, t.col, true};
    long long part = 0;
    if (p.family == TM_SG) {
      const int seg = __ldg(g.ptr[0] + u);
      for (int j = t.a + lane; j < t.b; j += 32) part += sg_entry(c, p.min_size, seg, j, nullptr);
    } else if (p.family == TM_GS) {
      const int seg = __ldg(g.ptr[1] + v);
      for (int j = t.a + lane; j < t.b; j += 32) part += gs_entry(c, p.min_size, seg, j, nullptr);
    } else if (p.family == TM_CYCLE) {  // group lead: per-depth partials
      const int path[kMaxChain] = {t.path[0], t.path[1], t.path[2], t.path[3], t.path[4]};
      CycAcc acc;
#pragma unroll
      for (int d = 0; d <= kMaxChain; ++d) acc.d[d] = 0;
      cycle_chain(c, p.cyc, t.level, path, t.a + lane, t.b, 32, acc, nullptr, em);
#pragma unroll
      for (int d = 1; d <= kMaxChain; ++d) {
        const long long s = warp_sum(acc.d[d]);
        if (lane == 0 && s)
          atomicAdd(reinterpret_cast<unsigned long long *>(out + (int64_t)t.row * plans.n + p.cyc.col[d]),
                    (unsigned long long)s);
      }
      continue;
    }
    part = warp_sum(part);
    if (lane == 0 && part)
      atomicAdd(reinterpret_cast<unsigned long long *>(out + (int64_t)t.row * plans.n + t.col),
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

// pipeline depth; TM_CHUNKS (1..4) overrides it for tuning sweeps
static int pipeline_chunks(int64_t rows) {
  static int forced = [] {
    const char *e = getenv("TM_CHUNKS");
    const int v = e ? atoi(e) : 0;
    return v >= 1 && v <= kMaxChunks ? v : 0;
  }();
  if (forced) return forced;
  (void)rows;
  return 1;  // measured: overlap loses to the extra per-chunk tail rounds at HI-Small
}

// side stream + events of the chunk pipeline (created once per graph)
static int ensure_pipeline(tm_graph *g) {
  if (g->side) return TM_OK;
  TM_CUDA(cudaStreamCreateWithFlags(&g->side, cudaStreamNonBlocking));
  TM_CUDA(cudaEventCreateWithFlags(&g->ev_fork, cudaEventDisableTiming));
  TM_CUDA(cudaEventCreateWithFlags(&g->ev_join, cudaEventDisableTiming));
  for (int i = 0; i < 3; ++i) TM_CUDA(cudaEventCreate(&g->ev[i]));
  for (int c = 0; c < kMaxChunks; ++c)
    for (int i = 0; i < 4; ++i) TM_CUDA(cudaEventCreate(&g->pev[c][i]));
  return TM_OK;
}

// light-tier work budget; TM_LIGHT_BUDGET overrides it for tuning sweeps
static int light_budget() {
  static int b = [] {
    const char *e = getenv("TM_LIGHT_BUDGET");
    const int v = e ? atoi(e) : 0;
    return v > 0 ? v : kLightBudget;
  }();
  return b;
}

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
  g->last.light_ms = g->last.heavy_ms = g->last.total_ms = -1.f;
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
  auto need_of = [](const tm_plan_desc &p) -> int {
    switch (p.family) {
      case TM_FAN:
      case TM_DEGREE: return 1 << (2 * p.endpoint + p.direction);
      case TM_CYCLE: return p.cycle_len == 2 ? 8 : (1 | 8);
      case TM_SG: return 1 | 4;
      case TM_GS: return 8 | 2;
      case TM_STACK: return 1 | 8;
      default: return 0;
    }
  };
  int rounds = 0;
  for (int i = 0; i < n_plans; ++i) {
    const tm_plan_desc &p = plans[i];
    dp.p[i] = DevPlan{p.family, p.endpoint, p.direction, p.exclude_trigger, p.cycle_len,
                      p.min_size, need_of(p), 0, g->lo_tabs.as<uint32_t>() + (size_t)slot_of[i] * R};
    if (!(p.family == TM_FAN || p.family == TM_DEGREE ||
          (p.family == TM_CYCLE && p.cycle_len == 2)))
      dp.needs_sets = 1;
    // task rounds: level-0 pieces (sg/gs/cycle) + one per deeper chain level
    if (p.family == TM_SG || p.family == TM_GS) rounds = std::max(rounds, 1);
    if (p.family == TM_CYCLE && p.cycle_len >= 4) rounds = std::max(rounds, p.cycle_len - 3);
  }
  // fused cycle groups: CYCLE columns of length >= 3 sharing a delta
  for (int i = 0; i < n_plans; ++i) {
    if (!(plans[i].family == TM_CYCLE && plans[i].cycle_len >= 3)) continue;
    CycGroup cg{};
    int lead = -1;
    for (int k = 0; k < n_plans; ++k) {
      if (!(plans[k].family == TM_CYCLE && plans[k].cycle_len >= 3) || slot_of[k] != slot_of[i]) continue;
      const int d = plans[k].cycle_len - 3;
      if (cg.mask & (1 << d)) continue;  // duplicate length: first column owns it
      if (lead < 0) lead = k;
      cg.mask |= 1 << d;
      cg.k[d] = plans[k].min_size;
      cg.col[d] = (int8_t)k;
      cg.maxd = std::max(cg.maxd, d);
    }
    cg.lead = (lead == i) ? 1 : 0;
    const int d = plans[i].cycle_len - 3;
    if (cg.col[d] != i) {  // duplicate of an earlier same-length column: own group
      CycGroup solo{};
      solo.mask = 1 << d;
      solo.k[d] = plans[i].min_size;
      solo.col[d] = (int8_t)i;
      solo.maxd = d;
      solo.lead = 1;
      cg = solo;
    }
    dp.p[i].cyc = cg;
  }

  for (int i = 0; i < n_plans; ++i) {  // union of needs per delta group
    int m = 0;
    for (int k = 0; k < n_plans; ++k)
      if (slot_of[k] == slot_of[i]) m |= dp.p[k].need;
    dp.p[i].need_group = m;
  }

  long long *d_out;
  if (out_on_device) {
    d_out = reinterpret_cast<long long *>(out);
  } else {
    if ((rc = g->out_scratch.ensure(sizeof(long long) * (size_t)rows * n_plans))) return rc;
    d_out = g->out_scratch.as<long long>();
  }
  // Pipeline: the trigger range is cut into `nch` chunks; chunk i's light
  // kernel runs on stream s while chunk i-1's heavy + task kernels run on the
  // graph's side stream, so the warp-level tail work overlaps the
  // thread-level bulk of the next chunk.  Rows of different chunks are
  // disjoint; every chunk has its own heavy-queue slice and counter, the task
  // queues are reused in side-stream order.
  const int nch = pipeline_chunks(rows);
  const int64_t task_cap = std::min<int64_t>(std::max<int64_t>(1 << 20, rows / 2), 1 << 24);
  if ((rc = g->heavy_n.ensure(sizeof(int32_t) * (kMaxChunks + 2))) ||
      (rc = g->heavy_q.ensure(sizeof(int32_t) * (size_t)rows)) ||
      (rc = g->tasks.ensure(sizeof(Task) * (size_t)task_cap * 2)))
    return rc;
  if ((rc = ensure_pipeline(g))) return rc;
  int32_t *cnt = g->heavy_n.as<int32_t>();  // [0..kMaxChunks) heavy rows, then task queues A/B
  TM_CUDA(cudaMemsetAsync(cnt, 0, sizeof(int32_t) * (kMaxChunks + 2), s));
  Queues qa{g->tasks.as<Task>(), cnt + kMaxChunks, (int32_t)task_cap};
  Queues qb{g->tasks.as<Task>() + task_cap, cnt + kMaxChunks + 1, (int32_t)task_cap};
  cudaStream_t s2 = g->side;
  TM_CUDA(cudaEventRecord(g->ev_fork, s));
  TM_CUDA(cudaStreamWaitEvent(s2, g->ev_fork, 0));

  const DevGraph dg = g->dev();
  g->prof_pending = g->prof;
  g->prof_chunks = nch;
  if (g->prof) TM_CUDA(cudaEventRecord(g->ev[0], s));
  const size_t smem = n_plans <= kStageCols ? sizeof(long long) * kLightThreads * n_plans : 0;
  const int heavy_grid = 148 * (2048 / kHeavyThreads);
  const int64_t per = (rows + nch - 1) / nch;
  for (int ch = 0; ch < nch; ++ch) {
    const int64_t r0 = std::min<int64_t>(rows, ch * per), r1 = std::min<int64_t>(rows, r0 + per);
    if (r1 <= r0) continue;
    int32_t *hq = g->heavy_q.as<int32_t>() + r0;
    if (g->prof) TM_CUDA(cudaEventRecord(g->pev[ch][0], s));
    k_mine_light<<<grid_for(r1 - r0, kLightThreads), kLightThreads, smem, s>>>(
        dg, dp, lo + r0, r1 - r0, d_out + r0 * n_plans, hq, cnt + ch, light_budget());
    TM_LAUNCHED("k_mine_light");
    TM_CUDA(cudaEventRecord(g->pev[ch][1], s));
    if (!dp.needs_sets) continue;
    TM_CUDA(cudaStreamWaitEvent(s2, g->pev[ch][1], 0));
    if (g->prof) TM_CUDA(cudaEventRecord(g->pev[ch][2], s2));
    TM_CUDA(cudaMemsetAsync(qa.count, 0, sizeof(int32_t), s2));
    k_mine_heavy<<<heavy_grid, kHeavyThreads, 0, s2>>>(dg, dp, lo + r0, d_out + r0 * n_plans, hq,
                                                       cnt + ch, qa);
    TM_LAUNCHED("k_mine_heavy");
    Queues a = qa, b = qb;
    for (int r = 0; r < rounds; ++r) {
      TM_CUDA(cudaMemsetAsync(b.count, 0, sizeof(int32_t), s2));
      k_mine_tasks<<<heavy_grid, kHeavyThreads, 0, s2>>>(dg, dp, lo + r0, d_out + r0 * n_plans, a, b);
      TM_LAUNCHED("k_mine_tasks");
      std::swap(a, b);
    }
    if (g->prof) TM_CUDA(cudaEventRecord(g->pev[ch][3], s2));
  }
  TM_CUDA(cudaEventRecord(g->ev_join, s2));
  TM_CUDA(cudaStreamWaitEvent(s, g->ev_join, 0));
  if (g->prof) TM_CUDA(cudaEventRecord(g->ev[2], s));
  if (!out_on_device) {
    TM_CUDA(cudaMemcpyAsync(out, d_out, sizeof(long long) * (size_t)rows * n_plans,
                            cudaMemcpyDeviceToHost, s));
    int32_t nh[kMaxChunks] = {0, 0, 0, 0};
    TM_CUDA(cudaMemcpyAsync(nh, cnt, sizeof(nh), cudaMemcpyDeviceToHost, s));
    TM_CUDA(cudaStreamSynchronize(s));
    g->last.heavy_triggers = (int64_t)nh[0] + nh[1] + nh[2] + nh[3];
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
    float lt = 0.f, ht = 0.f, x = 0.f;
    for (int ch = 0; ch < g->prof_chunks; ++ch) {
      if (cudaEventElapsedTime(&x, g->pev[ch][0], g->pev[ch][1]) == cudaSuccess) lt += x;
      if (cudaEventElapsedTime(&x, g->pev[ch][2], g->pev[ch][3]) == cudaSuccess) ht += x;
    }
    cudaGetLastError();  // chunks without heavy work leave their events unrecorded
    g->last.light_ms = lt;
    g->last.heavy_ms = ht;
    TM_CUDA(cudaEventElapsedTime(&g->last.total_ms, g->ev[0], g->ev[2]));
    g->prof_pending = false;
  }
  *stats = g->last;
  return TM_OK;
}

extern "C" int tm_set_profiling(tm_graph *g, int on) {
  if (!g) return fail(TM_E_BAD_ARG, "NULL graph");
  TM_CUDA(cudaSetDevice(g->device));
  int rc;
  if ((rc = ensure_pipeline(g))) return rc;
  g->prof = on != 0;
  return TM_OK;
}
