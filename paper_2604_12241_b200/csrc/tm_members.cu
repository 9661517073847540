// tm_members.cu — members attribution on the GPU.
//
// Reference: engine._mine_range members branch (engine.py:629-640) over the
// generic interpreter's instances (_EmissionState engine.py:433-513,
// pattern_grammar.md:116-122).  Every instance found at trigger e is the
// SET of edges that bound it — the trigger plus every windowed adjacency
// entry (parallel edges included) admitting each bound node.  It is counted
// only at its temporally last member, (timestamp, edge id) order, and then
// adds 1 to the row of every member edge, so contributions land on rows
// outside the trigger range: the output is a full (n_edges x C) block that
// this kernel ADDS into.
//
// Instances per family (trigger e = u -> v, window [t - delta, t]):
//   FAN / DEGREE  {e, f} per windowed entry f (f = e for a degree slice
//                 holding the trigger), when the entry count reaches K
//   CYCLE_2       {e} + leg(v->u)
//   CYCLE_k       {e} + legs v->a1 -> ... -> a_d -> c -> u per closing c,
//                 when the binding's closing set reaches K
//   SG            per source s with |M| >= K: {e} + leg(s->u) +
//                 legs s->m, m->v for every m in M (one instance)
//   GS            per destination d with |M| >= K: {e} + leg(v->d) +
//                 legs m->d, u->m for every m in M
//   STACK         per (a, c) in A x C when |A|, |C| >= K: {e} + leg(a->u) +
//                 leg(v->c); aggregated: a->u edges add |C_ok|, v->c edges
//                 add |A_ok|, e adds |A_ok| * |C_ok|
// where leg(x->y) = every x->y edge inside the window (a contiguous run of
// the pair index).  "Last member" means no member edge has the trigger's
// timestamp and a larger edge id (every member lies in [t - delta, t]).
// One warp per trigger; the outer loop of each family is spread over lanes.
#include "tm_device.cuh"

namespace tmb {
namespace {

using namespace dev;

constexpr int kMemThreads = 256;

struct Leg {
  const uint64_t *k;
  const int32_t *pe;
  int q0, q1;
};

// every x -> y edge inside the window: a run of the shorter pair index
__device__ __forceinline__ Leg leg_of(const Ctx &c, int x, int y) {
  const int xs = __ldg(c.g.ptr[1] + x), xe = __ldg(c.g.ptr[1] + x + 1);
  const int ys = __ldg(c.g.ptr[0] + y), ye = __ldg(c.g.ptr[0] + y + 1);
  const bool from_x = xe - xs <= ye - ys;
  const int d = from_x ? 1 : 0;
  const uint64_t base = (uint64_t)(uint32_t)(from_x ? y : x) << c.g.rank_bits;
  const int s = from_x ? xs : ys, e = from_x ? xe : ye;
  const int q0 = lb_u64(c.g.pkey[d], s, e, base + c.lo);
  const int q1 = lb_u64(c.g.pkey[d], q0, e, base + c.hi + 1);
  return Leg{c.g.pkey[d], c.g.peid[d], q0, q1};
}

// does the leg hold an edge after the trigger (same timestamp, larger id)?
// The run is sorted by (rank, eid): only its last slot can be.
__device__ __forceinline__ bool leg_late(const Ctx &c, const Leg &l, int e) {
  if (l.q1 <= l.q0) return false;
  const uint32_t rk = (uint32_t)(__ldg(l.k + l.q1 - 1) & ((1ull << c.g.rank_bits) - 1));
  return rk == c.hi && __ldg(l.pe + l.q1 - 1) > e;
}

__device__ __forceinline__ void add_row(long long *out, int C, int col, int eid, long long w) {
  atomicAdd(reinterpret_cast<unsigned long long *>(out + (int64_t)eid * C + col), (unsigned long long)w);
}

__device__ __forceinline__ void leg_add(const Leg &l, long long *out, int C, int col, long long w,
                                        int skip) {
  for (int q = l.q0; q < l.q1; ++q) {
    const int ed = __ldg(l.pe + q);
    if (ed != skip) add_row(out, C, col, ed, w);
  }
}

// FAN / DEGREE: instances {e, f}
__device__ void m_fan_degree(const Ctx &c, int e, const DevPlan &p, long long *out, int C, int col) {
  const int lane = threadIdx.x & 31;
  const int x = p.endpoint ? c.v : c.u, d = p.direction;
  const Win w = window(c, d, x);
  long long iters = w.len() - loops_in_window(c, x);
  if (p.exclude_trigger && c.u != c.v) iters -= 1;
  if (iters < p.min_size || iters <= 0) return;
  long long mine = 0;
  for (int j = w.a + lane; j < w.b; j += 32) {
    const int n = __ldg(c.g.nbr[d] + j);
    if (n == x) continue;  // self-loops never iterate
    const int f = __ldg(c.g.eid[d] + j);
    if (f == e) {
      if (!p.exclude_trigger) ++mine;  // instance {e}
      continue;
    }
    const uint32_t rf = __ldg(c.g.rnk[d] + j);
    if (rf < c.hi || f < e) {  // f before e (rf <= hi inside the window)
      ++mine;
      add_row(out, C, col, f, 1);
    }
  }
  mine = warp_sum(mine);
  if (lane == 0 && mine) add_row(out, C, col, e, mine);
}

// CYCLE_2: {e} + leg(v -> u)
__device__ void m_cycle2(const Ctx &c, int e, const DevPlan &p, long long *out, int C, int col) {
  if ((threadIdx.x & 31) != 0 || c.u == c.v || p.min_size > 1) return;
  const Leg l = leg_of(c, c.v, c.u);
  if (l.q1 <= l.q0 || leg_late(c, l, e)) return;
  add_row(out, C, col, e, 1);
  leg_add(l, out, C, col, 1, -1);
}

// closing set of chain node a (after NP earlier chain nodes in path)
template <bool EMIT>
__device__ int m_close(const Ctx &c, int a, const int *path, int np, int e, long long *out, int C,
                       int col, long long *n_ok) {
  const Win wa = window(c, 1, a);
  const bool walk_a = wa.len() <= c.wui.len();
  const Win w = walk_a ? wa : c.wui;
  const int d = walk_a ? 1 : 0;
  int cnt = 0;
  for (int j = w.a; j < w.b; ++j) {
    const int m = __ldg(c.g.nbr[d] + j);
    if (m == a || m == c.u || m == c.v) continue;
    bool dup = false;
    for (int i = 0; i < np; ++i) dup |= (path[i] == m);
    if (dup || !first_in_window(c, d, j)) continue;
    if (!(walk_a ? exists_in(c, 0, c.u, c.wui, m) : exists_in(c, 1, a, wa, m))) continue;
    ++cnt;
    if (EMIT) {  // instance legs a -> m, m -> u
      const Leg l1 = leg_of(c, a, m), l2 = leg_of(c, m, c.u);
      if (leg_late(c, l1, e) || leg_late(c, l2, e)) continue;
      ++*n_ok;
      leg_add(l1, out, C, col, 1, -1);
      leg_add(l2, out, C, col, 1, -1);
    }
  }
  return cnt;
}

// CYCLE_k (k >= 3): chain bindings a1..a_d, d = k - 3 (d = 0: cycle_3, a = v)
__device__ void m_cycle(const Ctx &c, int e, const DevPlan &p, long long *out, int C, int col) {
  const int lane = threadIdx.x & 31;
  if (c.u == c.v || c.wui.len() == 0) return;
  const int chain = p.cycle_len - 3;
  const int K = p.min_size;
  long long mine = 0;  // instances counted for e by this lane
  if (chain == 0) {
    if (lane != 0) return;
    int path[kMaxChain];
    if (m_close<false>(c, c.v, path, 0, e, out, C, col, nullptr) < K) return;
    long long ok = 0;
    m_close<true>(c, c.v, path, 0, e, out, C, col, &ok);
    if (ok) add_row(out, C, col, e, ok);
    return;
  }
  // depth-first over chains; level 0 (a1) spread over lanes
  int path[kMaxChain], pos[kMaxChain], end[kMaxChain];
  const Win wv = c.wvo;
  int L = 0;
  pos[0] = wv.a + lane;
  end[0] = wv.b;
  while (L >= 0) {
    const int j = pos[L];
    if (j >= end[L]) { --L; continue; }
    pos[L] = j + (L == 0 ? 32 : 1);
    const int owner = L == 0 ? c.v : path[L - 1];
    const int a = __ldg(c.g.nbr[1] + j);
    if (a == owner || a == c.u || a == c.v) continue;
    bool dup = false;
    for (int i = 0; i + 1 < L; ++i) dup |= (path[i] == a);
    if (dup || !first_in_window(c, 1, j)) continue;
    path[L] = a;
    if (L + 1 < chain) {
      const Win w = window(c, 1, a);
      ++L;
      pos[L] = w.a;
      end[L] = w.b;
      continue;
    }
    // binding a1..a_chain complete: closing set of a = path[chain-1]
    if (m_close<false>(c, a, path, chain - 1, e, out, C, col, nullptr) < K) continue;
    bool late = leg_late(c, leg_of(c, c.v, path[0]), e);
    for (int i = 0; i + 1 < chain && !late; ++i) late = leg_late(c, leg_of(c, path[i], path[i + 1]), e);
    if (late) continue;
    long long ok = 0;
    m_close<true>(c, a, path, chain - 1, e, out, C, col, &ok);
    if (!ok) continue;
    mine += ok;  // chain legs belong to every valid closing instance
    leg_add(leg_of(c, c.v, path[0]), out, C, col, ok, -1);
    for (int i = 0; i + 1 < chain; ++i) leg_add(leg_of(c, path[i], path[i + 1]), out, C, col, ok, -1);
  }
  mine = warp_sum(mine);
  if (lane == 0 && mine) add_row(out, C, col, e, mine);
}

// SG / GS: one instance per qualifying source s / destination d.
//   sg: x = s (outer, u's in-slice), hub side: legs s->u, s->m, m->v
//   gs: x = d (outer, v's out-slice), legs v->d, m->d, u->m
template <bool SG>
__device__ void m_sg_gs(const Ctx &c, int e, const DevPlan &p, long long *out, int C, int col) {
  const int lane = threadIdx.x & 31;
  const int K = p.min_size;
  const Win wo = SG ? c.wui : c.wvo;         // outer slice
  const int od = SG ? 0 : 1;                 // its direction
  const Win wy = SG ? c.wvi : c.wuo;         // the other side of the intersection
  long long mine = 0;
  for (int j = wo.a + lane; j < wo.b; j += 32) {
    const int x = __ldg(c.g.nbr[od] + j);
    if (x == c.u || x == c.v || !first_in_window(c, od, j)) continue;
    // M = N+(s) ∩ N-(v)  (sg)   |   N-(d) ∩ N+(u)  (gs)
    const int dx = SG ? 1 : 0, y = SG ? c.v : c.u, dy = SG ? 0 : 1;
    const Win wx = window(c, dx, x);
    const bool walk_x = wx.len() <= wy.len();
    const Win w = walk_x ? wx : wy;
    const int d = walk_x ? dx : dy, odir = walk_x ? dy : dx, other = walk_x ? y : x;
    const Win ow = walk_x ? wy : wx;
    int msize = 0;
    for (int k = w.a; k < w.b; ++k) {
      const int m = __ldg(c.g.nbr[d] + k);
      if (m == x || m == y || !first_in_window(c, d, k)) continue;
      msize += exists_in(c, odir, other, ow, m);
    }
    if (msize < K || msize == 0) continue;
    // the instance: bound leg + two legs per m; check, then add
    const Leg lb = SG ? leg_of(c, x, c.u) : leg_of(c, c.v, x);
    bool late = leg_late(c, lb, e);
    for (int pass = 0; pass < 2 && !late; ++pass) {
      for (int k = w.a; k < w.b && !late; ++k) {
        const int m = __ldg(c.g.nbr[d] + k);
        if (m == x || m == y || !first_in_window(c, d, k)) continue;
        if (!exists_in(c, odir, other, ow, m)) continue;
        // sg: s->m (dup of s->u when m == u), m->v (holds e when m == u)
        // gs: m->d (dup of v->d when m == v), u->m (holds e when m == v)
        const int dupn = SG ? c.u : c.v;
        const Leg l1 = SG ? leg_of(c, x, m) : leg_of(c, m, x);
        const Leg l2 = SG ? leg_of(c, m, c.v) : leg_of(c, c.u, m);
        if (pass == 0) {
          late = (m != dupn && leg_late(c, l1, e)) || leg_late(c, l2, e);
        } else {
          if (m != dupn) leg_add(l1, out, C, col, 1, -1);
          leg_add(l2, out, C, col, 1, e);
        }
      }
      if (pass == 0 && !late) leg_add(lb, out, C, col, 1, -1);
    }
    if (!late) ++mine;
  }
  mine = warp_sum(mine);
  if (lane == 0 && mine) add_row(out, C, col, e, mine);
}

// STACK: A x C instances, aggregated
__device__ void m_stack(const Ctx &c, int e, const DevPlan &p, long long *out, int C, int col) {
  const int lane = threadIdx.x & 31;
  long long na = 0, nc = 0, oka = 0, okc = 0;
  for (int j = c.wui.a + lane; j < c.wui.b; j += 32) {
    const int a = __ldg(c.g.nbr[0] + j);
    if (a == c.u || a == c.v || !first_in_window(c, 0, j)) continue;
    ++na;
    oka += !leg_late(c, leg_of(c, a, c.u), e);
  }
  for (int j = c.wvo.a + lane; j < c.wvo.b; j += 32) {
    const int x = __ldg(c.g.nbr[1] + j);
    if (x == c.v || x == c.u || !first_in_window(c, 1, j)) continue;
    ++nc;
    okc += !leg_late(c, leg_of(c, c.v, x), e);
  }
  na = warp_sum(na); nc = warp_sum(nc); oka = warp_sum(oka); okc = warp_sum(okc);
  if (na == 0 || nc == 0 || na < p.min_size || nc < p.min_size || oka == 0 || okc == 0) return;
  for (int j = c.wui.a + lane; j < c.wui.b; j += 32) {
    const int a = __ldg(c.g.nbr[0] + j);
    if (a == c.u || a == c.v || !first_in_window(c, 0, j)) continue;
    const Leg l = leg_of(c, a, c.u);
    if (!leg_late(c, l, e)) leg_add(l, out, C, col, okc, -1);
  }
  for (int j = c.wvo.a + lane; j < c.wvo.b; j += 32) {
    const int x = __ldg(c.g.nbr[1] + j);
    if (x == c.v || x == c.u || !first_in_window(c, 1, j)) continue;
    const Leg l = leg_of(c, c.v, x);
    if (!leg_late(c, l, e)) leg_add(l, out, C, col, oka, -1);
  }
  if (lane == 0) add_row(out, C, col, e, oka * okc);
}

__global__ void __launch_bounds__(kMemThreads) k_members(const __grid_constant__ DevGraph g,
                                                         const __grid_constant__ DevPlans P, int64_t lo,
                                                         int64_t n_rows, long long *__restrict__ out) {
  const int warps = gridDim.x * (blockDim.x >> 5);
  for (int64_t i = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5); i < n_rows; i += warps) {
    const int e = (int)(lo + i);
    const uint32_t r = __ldg(g.e_rank + e);
    const int u = __ldg(g.e_src + e), v = __ldg(g.e_dst + e);
    for (int ci = 0; ci < P.n; ++ci) {
      const DevPlan &p = P.p[ci];
      const DevGroup &gr = P.gr[p.group];
      Ctx c{g, u, v, __ldg(gr.lo_tab + r), r, {}, {}, {}, {}};
      c.wui = window(c, 0, u);
      c.wuo = window(c, 1, u);
      c.wvi = window(c, 0, v);
      c.wvo = window(c, 1, v);
      switch (p.family) {
        case TM_FAN:
        case TM_DEGREE: m_fan_degree(c, e, p, out, P.n, ci); break;
        case TM_CYCLE:
          if (p.cycle_len == 2) m_cycle2(c, e, p, out, P.n, ci);
          else m_cycle(c, e, p, out, P.n, ci);
          break;
        case TM_SG: m_sg_gs<true>(c, e, p, out, P.n, ci); break;
        case TM_GS: m_sg_gs<false>(c, e, p, out, P.n, ci); break;
        case TM_STACK: m_stack(c, e, p, out, P.n, ci); break;
        default: break;
      }
      __syncwarp();
    }
  }
}

__global__ void k_lo_table_m(const int64_t *__restrict__ uniq, int64_t R, long long delta,
                             uint32_t *__restrict__ lo_tab) {
  const int64_t r = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (r >= R) return;
  const long long t = uniq[r];
  int64_t a = 0, b = r;
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

extern "C" int tm_mine_members(tm_graph *g, const tm_plan_desc *plans, int n_plans, int64_t lo,
                               int64_t hi, int64_t *out, int out_on_device, void *stream) {
  if (!g) return fail(TM_E_BAD_ARG, "graph is NULL");
  if (n_plans < 0 || n_plans > kMaxPlans)
    return fail(TM_E_BAD_ARG, "n_plans must be in [0, " + std::to_string(kMaxPlans) + "]");
  if (n_plans > 0 && !plans) return fail(TM_E_BAD_ARG, "plans is NULL");
  if (lo < 0 || hi < lo || hi > g->n_edges) return fail(TM_E_BAD_ARG, "bad trigger range");
  const int64_t E = g->n_edges;
  if (E > 0 && n_plans > 0 && !out) return fail(TM_E_BAD_ARG, "out is NULL");
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
  g->last.triggers = hi - lo;
  g->last.light_ms = g->last.heavy_ms = g->last.total_ms = -1.f;
  g->prof_pending = false;
  if (n_plans == 0 || E == 0) return TM_OK;
  TM_CUDA(cudaSetDevice(g->device));
  cudaStream_t s = stream ? static_cast<cudaStream_t>(stream) : g->stream;
  TM_CUDA(g->begin(s));  // the shared scratch below may still be in use by the previous call
  const int64_t launches0 = tm_kernel_launch_count();
  DevPlans dp{};
  dp.n = n_plans;
  int64_t deltas[kMaxPlans];
  for (int i = 0; i < n_plans; ++i) {
    int k = 0;
    while (k < dp.ngroups && deltas[k] != plans[i].delta) ++k;
    if (k == dp.ngroups) {
      if (dp.ngroups == kMaxGroups) return fail(TM_E_UNSUPPORTED_PLAN, "too many distinct deltas");
      deltas[dp.ngroups++] = plans[i].delta;
    }
    const tm_plan_desc &p = plans[i];
    dp.p[i] = DevPlan{p.family, p.endpoint, p.direction, p.exclude_trigger, p.cycle_len, p.min_size, k};
  }
  const int64_t R = g->n_ranks;
  int rc;
  if ((rc = g->lo_tabs.ensure_pooled(sizeof(uint32_t) * (size_t)(R > 0 ? R : 1) * dp.ngroups, s, g->stream)))
    return rc;
  for (int k = 0; k < dp.ngroups; ++k) {
    dp.gr[k].lo_tab = g->lo_tabs.as<uint32_t>() + (size_t)k * R;
    k_lo_table_m<<<grid_for(R, 256), 256, 0, s>>>(g->uniq_time.as<int64_t>(), R, deltas[k],
                                                  g->lo_tabs.as<uint32_t>() + (size_t)k * R);
    TM_LAUNCHED("k_lo_table_m");
  }
  long long *d_out;
  const size_t bytes = sizeof(long long) * (size_t)E * n_plans;
  if (out_on_device) {
    d_out = reinterpret_cast<long long *>(out);  // accumulated into
  } else {
    if ((rc = g->out_scratch.ensure_pooled(bytes, s, g->stream))) return rc;
    d_out = g->out_scratch.as<long long>();
    TM_CUDA(cudaMemsetAsync(d_out, 0, bytes, s));
  }
  if (hi > lo) {
    k_members<<<148 * 8, kMemThreads, 0, s>>>(g->dev(), dp, lo, hi - lo, d_out);
    TM_LAUNCHED("k_members");
  }
  if (!out_on_device) {
    TM_CUDA(cudaMemcpyAsync(out, d_out, bytes, cudaMemcpyDeviceToHost, s));
    TM_CUDA(cudaStreamSynchronize(s));
  }
  TM_CUDA(g->end(s));
  g->last.kernel_launches = tm_kernel_launch_count() - launches0;
  return TM_OK;
}
