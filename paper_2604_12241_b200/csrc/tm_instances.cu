// tm_instances.cu — instance records on the GPU (mine(..., collect_instances=True)).
//
// Reference: engine._mine_range with collect=True (engine.py:629-645) runs
// every plan through the generic interpreter and records one
// InstanceRecord(pattern, trigger_edge, member_edges, member_nodes) per
// instance _EmissionState finds at a trigger (engine.py:455-513), whatever
// the attribution.  The instances are those of tm_members.cu:
//   FAN / DEGREE  {e, f} per windowed entry f, nodes {u, v, nbr(f)}
//   CYCLE_2       {e} + leg(v->u), nodes {u, v}
//   CYCLE_k       {e} + legs v->a1..a_d->c->u, nodes {u, v, a1..a_d, c}
//   SG            {e} + leg(s->u) + legs s->m, m->v (m in M), nodes {u,v,s} + M
//   GS            {e} + leg(v->d) + legs m->d, u->m (m in M), nodes {u,v,d} + M
//   STACK         {e} + leg(a->u) + leg(v->c), nodes {u, v, a, c}
// Records are written as int32 streams [plan, trigger, n_edges, n_nodes,
// edges..., nodes...] in two passes (sizes -> 64-bit offsets -> writes), one
// thread per trigger; the host dedups / sorts each record as the reference
// does (frozenset -> sorted tuple, then sort by (pattern, trigger, edges)).
// Instance lists are a small-graph feature (a HI-Small fan_out column alone
// has 2e10 instances); the total is bounded by TM_E_OVERFLOW.
#include "tm_device.cuh"

namespace tmb {
namespace {

using namespace dev;

// count (W = false) or write (W = true) the records of one trigger
struct Rec {
  int32_t *buf;  // write cursor (W) or null
  long long n;   // int32 words used
  template <bool W>
  __device__ __forceinline__ void put(int32_t x) {
    if (W) buf[n] = x;
    ++n;
  }
};

// the x -> y edges inside the window: a pair-index run
struct Leg {
  const int32_t *pe;
  int q0, q1;
  __device__ __forceinline__ int len() const { return q1 - q0; }
};

__device__ __forceinline__ Leg leg_of(const Ctx &c, int x, int y) {
  const int xs = __ldg(c.g.ptr[1] + x), xe = __ldg(c.g.ptr[1] + x + 1);
  const int ys = __ldg(c.g.ptr[0] + y), ye = __ldg(c.g.ptr[0] + y + 1);
  const bool from_x = xe - xs <= ye - ys;
  const int d = from_x ? 1 : 0;
  const uint64_t base = (uint64_t)(uint32_t)(from_x ? y : x) << c.g.rank_bits;
  const int s = from_x ? xs : ys, e = from_x ? xe : ye;
  const int q0 = lb_u64(c.g.pkey[d], s, e, base + c.lo);
  const int q1 = lb_u64(c.g.pkey[d], q0, e, base + c.hi + 1);
  return Leg{c.g.peid[d], q0, q1};
}

template <bool W>
__device__ __forceinline__ void put_leg(Rec &r, const Leg &l) {
  for (int q = l.q0; q < l.q1; ++q) r.put<W>(__ldg(l.pe + q));
}

// record header; the edge and node counts are patched after the lists
template <bool W>
__device__ __forceinline__ long long open_rec(Rec &r, int plan, int e) {
  const long long at = r.n;
  r.put<W>(plan);
  r.put<W>(e);
  r.put<W>(0);
  r.put<W>(0);
  return at;
}
template <bool W>
__device__ __forceinline__ void close_rec(Rec &r, long long at, int ne, int nn) {
  if (W) {
    r.buf[at + 2] = ne;
    r.buf[at + 3] = nn;
  }
}

// members of C (closing set of a, after np chain nodes in path): calls f(m)
template <class F>
__device__ __forceinline__ int for_close(const Ctx &c, int a, const int *path, int np, F &&f) {
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
    f(m);
  }
  return cnt;
}

template <bool W>
__device__ void rec_trigger(const Ctx &c, int e, int ci, const DevPlan &p, Rec &r) {
  const int u = c.u, v = c.v, K = p.min_size;
  switch (p.family) {
    case TM_FAN:
    case TM_DEGREE: {
      const int x = p.endpoint ? v : u, d = p.direction;
      const Win w = window(c, d, x);
      long long iters = w.len() - loops_in_window(c, x);
      if (p.exclude_trigger && u != v) iters -= 1;
      if (iters < K || iters <= 0) return;
      for (int j = w.a; j < w.b; ++j) {
        const int n = __ldg(c.g.nbr[d] + j);
        if (n == x) continue;
        const int f = __ldg(c.g.eid[d] + j);
        if (f == e && p.exclude_trigger) continue;
        const long long at = open_rec<W>(r, ci, e);
        r.put<W>(e);
        if (f != e) r.put<W>(f);
        r.put<W>(u);
        r.put<W>(v);
        r.put<W>(n);
        close_rec<W>(r, at, f != e ? 2 : 1, 3);
      }
      return;
    }
    case TM_CYCLE: {
      if (u == v) return;
      if (p.cycle_len == 2) {
        if (K > 1) return;
        const Leg l = leg_of(c, v, u);
        if (l.len() == 0) return;
        const long long at = open_rec<W>(r, ci, e);
        r.put<W>(e);
        put_leg<W>(r, l);
        r.put<W>(u);
        r.put<W>(v);
        close_rec<W>(r, at, 1 + l.len(), 2);
        return;
      }
      if (c.wui.len() == 0) return;
      const int chain = p.cycle_len - 3;
      int path[kMaxChain], pos[kMaxChain], end[kMaxChain];
      auto emit_close = [&](int a, int np) {
        // binding complete at a (a = v for cycle_3): one record per closing m
        if (for_close(c, a, path, np, [](int) {}) < K) return;
        for_close(c, a, path, np, [&](int m) {
          const long long at = open_rec<W>(r, ci, e);
          int ne = 1;
          r.put<W>(e);
          if (chain > 0) {
            const Leg l0 = leg_of(c, v, path[0]);
            put_leg<W>(r, l0);
            ne += l0.len();
            for (int i = 0; i + 1 < chain; ++i) {
              const Leg li = leg_of(c, path[i], path[i + 1]);
              put_leg<W>(r, li);
              ne += li.len();
            }
          }
          const Leg l1 = leg_of(c, a, m), l2 = leg_of(c, m, u);
          put_leg<W>(r, l1);
          put_leg<W>(r, l2);
          ne += l1.len() + l2.len();
          r.put<W>(u);
          r.put<W>(v);
          for (int i = 0; i < chain; ++i) r.put<W>(path[i]);
          r.put<W>(m);
          close_rec<W>(r, at, ne, 3 + chain);
        });
      };
      if (chain == 0) {
        emit_close(v, 0);
        return;
      }
      int L = 0;
      pos[0] = c.wvo.a;
      end[0] = c.wvo.b;
      while (L >= 0) {
        const int j = pos[L];
        if (j >= end[L]) { --L; continue; }
        pos[L] = j + 1;
        const int owner = L == 0 ? v : path[L - 1];
        const int a = __ldg(c.g.nbr[1] + j);
        if (a == owner || a == u || a == v) continue;
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
        emit_close(a, chain - 1);
      }
      return;
    }
    case TM_SG:
    case TM_GS: {
      const bool sg = p.family == TM_SG;
      const Win wo = sg ? c.wui : c.wvo;
      const int od = sg ? 0 : 1;
      const Win wy = sg ? c.wvi : c.wuo;
      for (int jo = wo.a; jo < wo.b; ++jo) {
        const int x = __ldg(c.g.nbr[od] + jo);
        if (x == u || x == v || !first_in_window(c, od, jo)) continue;
        const int dx = sg ? 1 : 0, y = sg ? v : u, dy = sg ? 0 : 1;
        const Win wx = window(c, dx, x);
        const bool walk_x = wx.len() <= wy.len();
        const Win w = walk_x ? wx : wy;
        const int d = walk_x ? dx : dy, odir = walk_x ? dy : dx, other = walk_x ? y : x;
        const Win ow = walk_x ? wy : wx;
        auto each_m = [&](auto &&f) {
          int n = 0;
          for (int k = w.a; k < w.b; ++k) {
            const int m = __ldg(c.g.nbr[d] + k);
            if (m == x || m == y || !first_in_window(c, d, k)) continue;
            if (!exists_in(c, odir, other, ow, m)) continue;
            ++n;
            f(m);
          }
          return n;
        };
        const int msize = each_m([](int) {});
        if (msize < K || msize == 0) continue;
        const long long at = open_rec<W>(r, ci, e);
        int ne = 1;
        r.put<W>(e);
        const Leg lb = sg ? leg_of(c, x, u) : leg_of(c, v, x);
        put_leg<W>(r, lb);
        ne += lb.len();
        each_m([&](int m) {  // duplicates (m = u / m = v) are removed on the host
          const Leg l1 = sg ? leg_of(c, x, m) : leg_of(c, m, x);
          const Leg l2 = sg ? leg_of(c, m, v) : leg_of(c, u, m);
          put_leg<W>(r, l1);
          put_leg<W>(r, l2);
          ne += l1.len() + l2.len();
        });
        r.put<W>(u);
        r.put<W>(v);
        r.put<W>(x);
        each_m([&](int m) { r.put<W>(m); });
        close_rec<W>(r, at, ne, 3 + msize);
      }
      return;
    }
    case TM_STACK: {
      long long na = 0, nc = 0;
      for (int j = c.wui.a; j < c.wui.b; ++j) {
        const int a = __ldg(c.g.nbr[0] + j);
        na += !(a == u || a == v) && first_in_window(c, 0, j);
      }
      for (int j = c.wvo.a; j < c.wvo.b; ++j) {
        const int x = __ldg(c.g.nbr[1] + j);
        nc += !(x == v || x == u) && first_in_window(c, 1, j);
      }
      if (na == 0 || nc == 0 || na < K || nc < K) return;
      for (int j = c.wui.a; j < c.wui.b; ++j) {
        const int a = __ldg(c.g.nbr[0] + j);
        if (a == u || a == v || !first_in_window(c, 0, j)) continue;
        const Leg la = leg_of(c, a, u);
        for (int k = c.wvo.a; k < c.wvo.b; ++k) {
          const int x = __ldg(c.g.nbr[1] + k);
          if (x == v || x == u || !first_in_window(c, 1, k)) continue;
          const Leg lc = leg_of(c, v, x);
          const long long at = open_rec<W>(r, ci, e);
          r.put<W>(e);
          put_leg<W>(r, la);
          put_leg<W>(r, lc);
          r.put<W>(u);
          r.put<W>(v);
          r.put<W>(a);
          r.put<W>(x);
          close_rec<W>(r, at, 1 + la.len() + lc.len(), 4);
        }
      }
      return;
    }
    default:
      return;
  }
}

template <bool W>
__global__ void k_instances(const __grid_constant__ DevGraph g, const __grid_constant__ DevPlans P,
                            int64_t lo, int64_t n_rows, unsigned long long *__restrict__ size,
                            int32_t *__restrict__ buf) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n_rows) return;
  const int e = (int)(lo + i);
  const uint32_t r = __ldg(g.e_rank + e);
  const int u = __ldg(g.e_src + e), v = __ldg(g.e_dst + e);
  Rec rec{W ? buf + size[i] : nullptr, 0};
  for (int ci = 0; ci < P.n; ++ci) {
    const DevPlan &p = P.p[ci];
    Ctx c{g, u, v, __ldg(P.gr[p.group].lo_tab + r), r, {}, {}, {}, {}};
    fill_windows(c, 1 | 2 | 4 | 8);
    rec_trigger<W>(c, e, ci, p, rec);
  }
  if (!W) size[i] = (unsigned long long)rec.n;
}

__global__ void k_lo_table_i(const int64_t *__restrict__ uniq, int64_t R, long long delta,
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

extern "C" int tm_collect_instances(tm_graph *g, const tm_plan_desc *plans, int n_plans, int64_t lo,
                                    int64_t hi, int64_t *out_words) {
  if (!g || !out_words) return fail(TM_E_BAD_ARG, "NULL argument");
  *out_words = 0;
  if (n_plans < 0 || n_plans > kMaxPlans || (n_plans > 0 && !plans))
    return fail(TM_E_BAD_ARG, "bad plans");
  if (lo < 0 || hi < lo || hi > g->n_edges) return fail(TM_E_BAD_ARG, "bad trigger range");
  for (int i = 0; i < n_plans; ++i) {
    const tm_plan_desc &p = plans[i];
    if (p.family < TM_FAN || p.family > TM_STACK ||
        (p.family == TM_CYCLE && (p.cycle_len < 2 || p.cycle_len > 8)))
      return fail(TM_E_UNSUPPORTED_PLAN, "plan " + std::to_string(i) + ": unsupported");
    if (p.min_size < 1 || p.delta < 0) return fail(TM_E_BAD_ARG, "plan " + std::to_string(i) + ": bad K / delta");
  }
  const int64_t rows = hi - lo;
  g->inst_words = 0;
  if (rows == 0 || n_plans == 0) return TM_OK;
  TM_CUDA(cudaSetDevice(g->device));
  cudaStream_t s = g->stream;
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
  TM_CUDA(g->begin(s));
  if ((rc = g->lo_tabs.ensure_pooled(sizeof(uint32_t) * (size_t)(R > 0 ? R : 1) * dp.ngroups, s, g->stream)))
    return rc;
  for (int k = 0; k < dp.ngroups; ++k) {
    dp.gr[k].lo_tab = g->lo_tabs.as<uint32_t>() + (size_t)k * R;
    k_lo_table_i<<<grid_for(R, 256), 256, 0, s>>>(g->uniq_time.as<int64_t>(), R, deltas[k],
                                                  g->lo_tabs.as<uint32_t>() + (size_t)k * R);
    TM_LAUNCHED("k_lo_table_i");
  }
  DevBuf size;
  if ((rc = size.ensure_on(sizeof(unsigned long long) * (size_t)(rows + 1), s))) return rc;
  const DevGraph dg = g->dev();
  k_instances<false><<<grid_for(rows, 128), 128, 0, s>>>(dg, dp, lo, rows, size.as<unsigned long long>(),
                                                         nullptr);
  TM_LAUNCHED("k_instances<count>");
  TM_CUDA(cudaMemsetAsync(size.as<unsigned long long>() + rows, 0, sizeof(unsigned long long), s));
  if ((rc = scan_u64_exclusive(size.as<unsigned long long>(), rows + 1, s))) return rc;
  unsigned long long total = 0;
  TM_CUDA(cudaMemcpyAsync(&total, size.as<unsigned long long>() + rows, 8, cudaMemcpyDeviceToHost, s));
  TM_CUDA(cudaStreamSynchronize(s));
  if (total > (1ull << 33)) return fail(TM_E_OVERFLOW, "instance records exceed 32 GiB");
  if ((rc = g->inst_buf.ensure(sizeof(int32_t) * (size_t)(total ? total : 1)))) return rc;
  k_instances<true><<<grid_for(rows, 128), 128, 0, s>>>(dg, dp, lo, rows, size.as<unsigned long long>(),
                                                        g->inst_buf.as<int32_t>());
  TM_LAUNCHED("k_instances<write>");
  TM_CUDA(cudaStreamSynchronize(s));
  g->inst_words = (int64_t)total;
  *out_words = (int64_t)total;
  return TM_OK;
}

extern "C" int tm_fetch_instances(tm_graph *g, int32_t *dst, int64_t n_words) {
  if (!g || (!dst && n_words > 0) || n_words > g->inst_words) return fail(TM_E_BAD_ARG, "bad argument");
  if (n_words == 0) return TM_OK;
  TM_CUDA(cudaSetDevice(g->device));
  TM_CUDA(cudaMemcpyAsync(dst, g->inst_buf.p, sizeof(int32_t) * (size_t)n_words, cudaMemcpyDeviceToHost,
                          g->stream));
  TM_CUDA(cudaStreamSynchronize(g->stream));
  return TM_OK;
}
