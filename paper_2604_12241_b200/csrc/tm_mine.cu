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
// Execution model (work balancing for power-law hubs, kernels.py has none —
// it splits contiguous ranges per worker, engine.py:681-682):
//   k_mine_light   one THREAD per trigger edge.  Windows come from bisection
//                  of the time-ranked CSR; set columns iterate the SMALLER of
//                  the two windowed slices and test membership of the other
//                  side with one pair-index bisection; distinct-ness is an O(1)
//                  pair-predecessor test.  Every trigger has a work budget; a
//                  trigger that would exceed it (hub slices, cycle fan-out)
//                  is appended to the heavy queue with a warp-aggregated
//                  atomic and its row is left to ...
//   k_mine_heavy   one WARP per queued trigger: the outer iteration of every
//                  set column is spread over the 32 lanes, inner work stays
//                  per lane, counts are combined with __shfl_xor_sync.
// Both kernels share one templated implementation (ThreadGrp / WarpGrp), so
// the light and heavy paths cannot drift apart.
#include "tm_internal.cuh"

namespace tmb {
namespace {

constexpr int kLightThreads = 256;
constexpr int kHeavyThreads = 256;
constexpr int kLightBudget = 768;  // slice entries + probes per light trigger

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

// ------------------------------------------------------------- groups

struct ThreadGrp {
  static constexpr bool kCoop = false;
  __device__ __forceinline__ int lane() const { return 0; }
  __device__ __forceinline__ int width() const { return 1; }
  __device__ __forceinline__ long long sum(long long x) const { return x; }
};

struct WarpGrp {
  static constexpr bool kCoop = true;
  __device__ __forceinline__ int lane() const { return threadIdx.x & 31; }
  __device__ __forceinline__ int width() const { return 32; }
  __device__ __forceinline__ long long sum(long long x) const {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) x += __shfl_xor_sync(0xffffffffu, x, o);
    return x;
  }
};

struct Budget {
  int left;
  bool blown;
  __device__ __forceinline__ bool take(int n) {
    if (n > left) { blown = true; return false; }
    left -= n;
    return true;
  }
};

template <class G> __device__ __forceinline__ bool spend(Budget &bud, int n) {
  if (G::kCoop) return true;
  return bud.take(n);
}

// |distinct windowed neighbours of x in dir| excluding x (self-loops) and ex
template <class G>
__device__ long long count_distinct(const G &grp, const Ctx &c, int dir, int x, int ex,
                                    Budget &bud) {
  const Win w = window(c, dir, x);
  if (!spend<G>(bud, w.len())) return 0;
  const int seg = __ldg(c.g.ptr[dir] + x);
  long long n = 0;
  for (int j = w.a + grp.lane(); j < w.b; j += grp.width()) {
    const int y = __ldg(c.g.nbr[dir] + j);
    if (y == x || y == ex) continue;
    n += first_in_window(c, dir, seg, j, y);
  }
  return grp.sum(n);
}

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

// cycle_3 = |N+(v)\{u} ∩ N-(u)| (kernels.py:323-327)
template <class G>
__device__ long long col_cycle3(const G &grp, const Ctx &c, const DevPlan &p, Budget &bud) {
  if (c.u == c.v) return 0;
  const Win wv = window(c, 1, c.v), wu = window(c, 0, c.u);
  if (wv.len() == 0 || wu.len() == 0) return 0;
  long long raw = 0;
  if (wv.len() <= wu.len()) {
    if (!spend<G>(bud, 2 * wv.len())) return 0;
    const int seg = __ldg(c.g.ptr[1] + c.v);
    for (int j = wv.a + grp.lane(); j < wv.b; j += grp.width()) {
      const int m = __ldg(c.g.nbr[1] + j);
      if (m == c.v || m == c.u || !first_in_window(c, 1, seg, j, m)) continue;
      raw += has_edge(c, m, c.u);
    }
  } else {
    if (!spend<G>(bud, 2 * wu.len())) return 0;
    const int seg = __ldg(c.g.ptr[0] + c.u);
    for (int j = wu.a + grp.lane(); j < wu.b; j += grp.width()) {
      const int m = __ldg(c.g.nbr[0] + j);
      if (m == c.u || m == c.v || !first_in_window(c, 0, seg, j, m)) continue;
      raw += has_edge(c, c.v, m);
    }
  }
  raw = grp.sum(raw);
  return raw >= p.min_size ? raw : 0;
}

// closing set size for a chain ending at `a`:
//   |(N+(a) ∩ N-(u)) \ {v, path[0..np-1]}|   (Appendix A cycle_k, cycle_4
//   kernels.py:330-341 for np = 0).  Sequential per lane.
__device__ int close_count(const Ctx &c, int a, const int *path, int np, const Win &wu,
                           Budget &bud, bool coop) {
  const Win wa = window(c, 1, a);
  int cnt = 0;
  if (wa.len() <= wu.len()) {
    if (!coop && !bud.take(2 * wa.len())) return 0;
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
    if (!coop && !bud.take(2 * wu.len())) return 0;
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

// cycle_k, k = 4..8: chains a1..a_{k-3}, a1 in N+(v)\{u},
// a_i in N+(a_{i-1}) \ {u, v, a1..a_{i-2}}, each chain adds |C| when
// |C| >= K (per-binding threshold).  Iterative DFS; level 0 is spread over
// the group's lanes.
template <class G>
__device__ long long col_cycle_k(const G &grp, const Ctx &c, const DevPlan &p, Budget &bud) {
  if (c.u == c.v) return 0;
  const Win wu = window(c, 0, c.u);
  if (wu.len() == 0) return 0;
  const Win wv = window(c, 1, c.v);
  if (!spend<G>(bud, wv.len())) return 0;
  const int chain = p.cycle_len - 3;  // 1..5
  int path[5], pos[5], end[5], seg[5];
  long long total = 0;
  int L = 0;
  pos[0] = wv.a + grp.lane();
  end[0] = wv.b;
  seg[0] = __ldg(c.g.ptr[1] + c.v);
  while (L >= 0) {
    const int j = pos[L];
    if (j >= end[L]) { --L; continue; }
    pos[L] = j + (L == 0 ? grp.width() : 1);
    const int owner = L == 0 ? c.v : path[L - 1];
    const int a = __ldg(c.g.nbr[1] + j);
    if (a == owner || a == c.u || a == c.v) continue;
    bool dup = false;
    for (int i = 0; i + 1 < L; ++i) dup |= (path[i] == a);
    if (dup || !first_in_window(c, 1, seg[L], j, a)) continue;
    if (L == chain - 1) {
      const int cc = close_count(c, a, path, L, wu, bud, G::kCoop);
      if (!G::kCoop && bud.blown) return 0;
      if (cc >= p.min_size) total += cc;
    } else {
      path[L] = a;
      ++L;
      const Win w = window(c, 1, a);
      if (!spend<G>(bud, w.len())) return 0;
      pos[L] = w.a;
      end[L] = w.b;
      seg[L] = __ldg(c.g.ptr[1] + a);
    }
  }
  return grp.sum(total);
}

// inner count of sg / gs: |N^{dx}(x) ∩ N^{dy}(y)|, early exit at K.
// sg: x = s (out), y = v (in);  gs: x = d (in), y = u (out).
// x and y themselves are never members (no self-loops in either set).
__device__ int inner_hits(const Ctx &c, int x, int dx, int y, int dy, int K, Budget &bud,
                          bool coop) {
  const Win wx = window(c, dx, x), wy = window(c, dy, y);
  int hits = 0;
  // iterate the shorter side; probe the other with has_edge in the right
  // orientation (dir 1 = out: x -> m, dir 0 = in: m -> x)
  if (wx.len() <= wy.len()) {
    if (!coop && !bud.take(2 * wx.len())) return 0;
    const int seg = __ldg(c.g.ptr[dx] + x);
    for (int j = wx.a; j < wx.b && hits < K; ++j) {
      const int m = __ldg(c.g.nbr[dx] + j);
      if (m == x || m == y || !first_in_window(c, dx, seg, j, m)) continue;
      hits += dy ? has_edge(c, y, m) : has_edge(c, m, y);
    }
  } else {
    if (!coop && !bud.take(2 * wy.len())) return 0;
    const int seg = __ldg(c.g.ptr[dy] + y);
    for (int j = wy.a; j < wy.b && hits < K; ++j) {
      const int m = __ldg(c.g.nbr[dy] + j);
      if (m == y || m == x || !first_in_window(c, dy, seg, j, m)) continue;
      hits += dx ? has_edge(c, x, m) : has_edge(c, m, x);
    }
  }
  return hits;
}

// sg_count = #{s in N-(u)\{u,v} : |N+(s) ∩ N-(v)| >= K}  (kernels.py:348-376)
template <class G>
__device__ long long col_sg(const G &grp, const Ctx &c, const DevPlan &p, Budget &bud) {
  const Win wu = window(c, 0, c.u);
  if (wu.len() == 0) return 0;
  if (!spend<G>(bud, wu.len())) return 0;
  const int seg = __ldg(c.g.ptr[0] + c.u);
  long long cnt = 0;
  for (int j = wu.a + grp.lane(); j < wu.b; j += grp.width()) {
    const int s = __ldg(c.g.nbr[0] + j);
    if (s == c.u || s == c.v || !first_in_window(c, 0, seg, j, s)) continue;
    const int h = inner_hits(c, s, 1, c.v, 0, p.min_size, bud, G::kCoop);
    if (!G::kCoop && bud.blown) return 0;
    cnt += (h >= p.min_size);
  }
  return grp.sum(cnt);
}

// gs_count = #{d in N+(v)\{u} : |N-(d) ∩ N+(u)| >= K}  (Appendix B)
template <class G>
__device__ long long col_gs(const G &grp, const Ctx &c, const DevPlan &p, Budget &bud) {
  const Win wv = window(c, 1, c.v);
  if (wv.len() == 0) return 0;
  if (!spend<G>(bud, wv.len())) return 0;
  const int seg = __ldg(c.g.ptr[1] + c.v);
  long long cnt = 0;
  for (int j = wv.a + grp.lane(); j < wv.b; j += grp.width()) {
    const int d = __ldg(c.g.nbr[1] + j);
    if (d == c.v || d == c.u || !first_in_window(c, 1, seg, j, d)) continue;
    const int h = inner_hits(c, d, 0, c.u, 1, p.min_size, bud, G::kCoop);
    if (!G::kCoop && bud.blown) return 0;
    cnt += (h >= p.min_size);
  }
  return grp.sum(cnt);
}

// stack = a*c if a >= K and c >= K; a = |N-(u)\{u,v}|, c = |N+(v)\{u,v}|
// (kernels.py:379-402)
template <class G>
__device__ long long col_stack(const G &grp, const Ctx &c, const DevPlan &p, Budget &bud) {
  const long long a = count_distinct(grp, c, 0, c.u, c.v, bud);
  if (a == 0 || a < p.min_size) return 0;
  const long long d = count_distinct(grp, c, 1, c.v, c.u, bud);
  if (d == 0 || d < p.min_size) return 0;
  return a * d;
}

template <class G>
__device__ long long eval_column(const G &grp, const Ctx &c, const DevPlan &p, Budget &bud) {
  switch (p.family) {
    case TM_FAN:
    case TM_DEGREE: return col_fan_degree(c, p);
    case TM_CYCLE:
      if (p.cycle_len == 2) return col_cycle2(c, p);
      if (p.cycle_len == 3) return col_cycle3(grp, c, p, bud);
      return col_cycle_k(grp, c, p, bud);
    case TM_SG: return col_sg(grp, c, p, bud);
    case TM_GS: return col_gs(grp, c, p, bud);
    case TM_STACK: return col_stack(grp, c, p, bud);
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
    const ThreadGrp grp;
    long long *o = out + row * plans.n;
    for (int ci = 0; ci < plans.n; ++ci) {
      const DevPlan p = plans.p[ci];
      const Ctx c{g, u, v, __ldg(p.lo_tab + r), r};
      const long long val = eval_column(grp, c, p, bud);
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

__global__ void __launch_bounds__(kHeavyThreads) k_mine_heavy(
    const DevGraph g, const DevPlans plans, int64_t lo, long long *__restrict__ out,
    const int32_t *__restrict__ heavy_q, const int32_t *__restrict__ heavy_n) {
  const int n = *heavy_n;
  const int warps = gridDim.x * (blockDim.x >> 5);
  const WarpGrp grp;
  for (int i = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5); i < n; i += warps) {
    const int64_t row = heavy_q[i];
    const int e = (int)(lo + row);
    const int u = __ldg(g.e_src + e), v = __ldg(g.e_dst + e);
    const uint32_t r = __ldg(g.e_rank + e);
    Budget bud{0x7fffffff, false};
    long long *o = out + row * plans.n;
    for (int ci = 0; ci < plans.n; ++ci) {
      const DevPlan p = plans.p[ci];
      const Ctx c{g, u, v, __ldg(p.lo_tab + r), r};
      const long long val = eval_column(grp, c, p, bud);
      if (grp.lane() == 0) o[ci] = val;
    }
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
  for (int i = 0; i < n_plans; ++i) {
    const tm_plan_desc &p = plans[i];
    dp.p[i] = DevPlan{p.family, p.endpoint, p.direction, p.exclude_trigger, p.cycle_len,
                      p.min_size, g->lo_tabs.as<uint32_t>() + (size_t)slot_of[i] * R};
    if (!(p.family == TM_FAN || p.family == TM_DEGREE ||
          (p.family == TM_CYCLE && p.cycle_len == 2)))
      dp.needs_sets = 1;
  }

  long long *d_out;
  if (out_on_device) {
    d_out = reinterpret_cast<long long *>(out);
  } else {
    if ((rc = g->out_scratch.ensure(sizeof(long long) * (size_t)rows * n_plans))) return rc;
    d_out = g->out_scratch.as<long long>();
  }
  if ((rc = g->heavy_n.ensure(sizeof(int32_t) * 2)) ||
      (rc = g->heavy_q.ensure(sizeof(int32_t) * (size_t)rows)))
    return rc;
  TM_CUDA(cudaMemsetAsync(g->heavy_n.p, 0, sizeof(int32_t), s));

  const DevGraph dg = g->dev();
  g->prof_pending = g->prof;
  if (g->prof) TM_CUDA(cudaEventRecord(g->ev[0], s));
  k_mine_light<<<grid_for(rows, kLightThreads), kLightThreads, 0, s>>>(
      dg, dp, lo, rows, d_out, g->heavy_q.as<int32_t>(), g->heavy_n.as<int32_t>());
  TM_LAUNCHED("k_mine_light");
  if (g->prof) TM_CUDA(cudaEventRecord(g->ev[1], s));
  if (dp.needs_sets) {
    k_mine_heavy<<<148 * 8, kHeavyThreads, 0, s>>>(dg, dp, lo, d_out, g->heavy_q.as<int32_t>(),
                                                   g->heavy_n.as<int32_t>());
    TM_LAUNCHED("k_mine_heavy");
  }
  if (g->prof) TM_CUDA(cudaEventRecord(g->ev[2], s));
  if (!out_on_device) {
    TM_CUDA(cudaMemcpyAsync(out, d_out, sizeof(long long) * (size_t)rows * n_plans,
                            cudaMemcpyDeviceToHost, s));
    int32_t nh = 0;
    TM_CUDA(cudaMemcpyAsync(&nh, g->heavy_n.p, sizeof(int32_t), cudaMemcpyDeviceToHost, s));
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
