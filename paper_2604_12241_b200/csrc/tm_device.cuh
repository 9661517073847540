// tm_device.cuh — device-side set primitives shared by the mining kernels
// (tm_mine.cu: trigger attribution, tm_members.cu: members attribution).
// See tm_internal.cuh for the graph layout they read.
#pragma once

#include "tm_internal.cuh"

namespace tmb {
namespace dev {

// Work counters for tools/work_profile.py (build with -DTM_COUNTERS=1; a
// no-op otherwise).  Each translation unit has its own copy.
#ifndef TM_COUNTERS
#define TM_COUNTERS 0
#endif
enum CtrId {
  kCtrTrig, kCtrUWalk, kCtrUItem, kCtrVWalk, kCtrVItem, kCtrWin, kCtrBisect32, kCtrScanCall,
  kCtrScanLoad, kCtrPairCall, kCtrBisect64, kCtrInnerCall, kCtrInnerWalk, kCtrChain1, kCtrChain2,
  kCtrChain3, kCtrChain4, kCtrCloseCall, kCtrCloseWalk, kCtrDomTask, kCtrChainTask, kCtrFirst,
  kCtrInnerSkip, kCtrPull, kCtrQueueFull, kCtrSlotFull, kCtrUsefulOver, kCtrBloomOver, kCtrChainOver, kCtrN
};
#if TM_COUNTERS
static __device__ unsigned long long tm_ctr[kCtrN];
#define TM_CNT(i, n) atomicAdd(&::tmb::dev::tm_ctr[(i)], (unsigned long long)(n))
#else
#define TM_CNT(i, n) ((void)0)
#endif

struct Win {
  int a, b;
  __device__ __forceinline__ int len() const { return b - a; }
};

__device__ __forceinline__ int lb_u32(const uint32_t *__restrict__ r, int a, int b, uint32_t x) {
  while (a < b) {
    TM_CNT(kCtrBisect32, 1);
    int m = (a + b) >> 1;
    if (__ldg(r + m) < x) a = m + 1; else b = m;
  }
  return a;
}
__device__ __forceinline__ int ub_u32(const uint32_t *__restrict__ r, int a, int b, uint32_t x) {
  while (a < b) {
    TM_CNT(kCtrBisect32, 1);
    int m = (a + b) >> 1;
    if (__ldg(r + m) <= x) a = m + 1; else b = m;
  }
  return a;
}
__device__ __forceinline__ int lb_u64(const uint64_t *__restrict__ k, int a, int b, uint64_t x) {
  while (a < b) {
    TM_CNT(kCtrBisect64, 1);
    int m = (a + b) >> 1;
    if (__ldg(k + m) < x) a = m + 1; else b = m;
  }
  return a;
}

struct Ctx {
  const DevGraph &g;  // a __grid_constant__ kernel parameter (global or slab view)
  int u, v;
  uint32_t lo, hi;    // window in rank space
  Win wui, wuo, wvi, wvo;  // trigger windows (u-in, u-out, v-in, v-out)
  int64_t soff = 0;   // slab view: row of the trigger's slab in the offset table
};

// Galloping upper bounds measured slower on HI-Small (4.73 -> 5.25 ms/step,
// tools/sweep_budget.py A/B): kept off, selectable for other graphs.
#ifndef TM_UB_GALLOP
#define TM_UB_GALLOP 0
#endif
#ifndef TM_SCAN4
#define TM_SCAN4 1  // measured: HI-Small -4 %, HI-Medium -3 %
#endif
#ifndef TM_VEC_SCAN
#define TM_VEC_SCAN 0  // measured: HI-Large warp kernel 70.2 -> 73.6 ms (more bytes per probe)
#endif
#ifndef TM_WIN_PAR
#define TM_WIN_PAR 1  // measured: HI-Medium -3 %
#endif
#ifndef TM_WIN4
#define TM_WIN4 0  // trigger windows: one joint bisection loop for all four (A/B)
#endif


// first index in [s, e) with r > x, galloping forward from s: windows are
// short, so this is usually one load of a line the lower bound just touched
__device__ __forceinline__ int ub_gallop(const uint32_t *__restrict__ r, int s, int e, uint32_t x) {
  if (s >= e || __ldg(r + s) > x) return s;
  int lo = s, step = 1;  // r[lo] <= x
  while (lo + step < e && __ldg(r + lo + step) <= x) {
    lo += step;
    step <<= 1;
  }
  return ub_u32(r, lo + 1, min(lo + step, e), x);
}

// Runs of at most kShortRun entries can be counted with independent loads of
// the whole run — one round trip — instead of a bisection (two or three
// dependent round trips for 2..4 entries).  Measured slower: the extra load
// instructions cost more than the round trips they save (off by default).
#ifndef TM_SHORT_RUN
#define TM_SHORT_RUN 0  // measured: 4 -> HI-Large warp kernel 70.3 -> 89.9 ms, 8 -> 97.6 (more load instructions lose)
#endif
constexpr int kShortRun = TM_SHORT_RUN;

// Runs of at most 4 entries (nearly every run of a slab view) can be counted
// from the aligned 16-byte block(s) holding them — one or two vector loads,
// one round trip — instead of a bisection (device buffers are padded, so a
// block may reach past the array end).  Measured much slower: the kernel is
// bound by the sectors it moves, and the bisection touches fewer.
#ifndef TM_VEC_RUN
#define TM_VEC_RUN 0  // measured: HI-Large warp kernel 70.2 -> 106.3 ms
#endif
__device__ __forceinline__ void count_block(const uint4 q, int base, int a, int b, uint32_t lo, uint32_t hi,
                                            int &l, int &u) {
  const uint32_t v[4] = {q.x, q.y, q.z, q.w};
#pragma unroll
  for (int k = 0; k < 4; ++k) {
    const int i = base + k;
    if (i >= a && i < b) {
      l += v[k] < lo;
      u += v[k] <= hi;
    }
  }
}

// window [lo, hi] (rank space) of the rank-sorted run [a, b) of r
__device__ __forceinline__ Win window_of_run(const uint32_t *__restrict__ r, int a, int b, uint32_t lo,
                                             uint32_t hi) {
#if TM_VEC_RUN
  if (b - a <= 4) {
    int l = a, u = a;
    if (b > a) {
      const int a4 = a & ~3;
      const uint4 q0 = __ldg(reinterpret_cast<const uint4 *>(r + a4));
      if (b > a4 + 4) {
        const uint4 q1 = __ldg(reinterpret_cast<const uint4 *>(r + a4 + 4));
        count_block(q1, a4 + 4, a, b, lo, hi, l, u);
      }
      count_block(q0, a4, a, b, lo, hi, l, u);
    }
    return {l, u};
  }
#endif
  if (b - a <= kShortRun) {
    int l = a, u = a;
#pragma unroll
    for (int k = 0; k < kShortRun; ++k) {
      if (a + k < b) {
        const uint32_t x = __ldg(r + a + k);
        l += x < lo;
        u += x <= hi;
      }
    }
    return {l, u};
  }
#if TM_WIN_PAR
  // both bounds bisected at once: two independent load chains in flight
  int l0 = a, l1 = b, u0 = a, u1 = b;
  while (l0 < l1 || u0 < u1) {
    if (l0 < l1) {
      const int m = (l0 + l1) >> 1;
      if (__ldg(r + m) < lo) l0 = m + 1; else l1 = m;
    }
    if (u0 < u1) {
      const int m = (u0 + u1) >> 1;
      if (__ldg(r + m) <= hi) u0 = m + 1; else u1 = m;
    }
  }
  return {l0, u0};
#else
  const int wa = lb_u32(r, a, b, lo);
#if TM_UB_GALLOP
  return {wa, ub_gallop(r, wa, b, hi)};
#else
  return {wa, ub_u32(r, wa, b, hi)};
#endif
#endif
}

// windowed slice of x's dir-run: rank in [lo, hi]   (kernels.py:268-276)
// run [ptr[x], ptr[x+1]) of node x (two loads of one sector; an 8-byte load
// of even nodes' pairs would need even slab-row offsets)
__device__ __forceinline__ int2 run_of(const int32_t *__restrict__ pt, int x) {
  return make_int2(__ldg(pt + x), __ldg(pt + x + 1));
}

__device__ __forceinline__ Win window(const Ctx &c, int dir, int x) {
  TM_CNT(kCtrWin, 1);
  const int2 ab = run_of(c.g.ptr[dir] + c.soff, x);
  return window_of_run(c.g.rnk[dir], ab.x, ab.y, c.lo, c.hi);
}

// trigger windows a delta group needs (bits: 1 u-in, 2 u-out, 4 v-in, 8 v-out).
// All run bounds are loaded first, then every short run in one round of
// independent loads; only long runs (hubs) bisect.
__device__ __forceinline__ void fill_windows(Ctx &c, int need) {
  int a[4], b[4];
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    const int dir = i & 1, x = (i >> 1) ? c.v : c.u;
    const bool on = (need >> i) & 1;
    const int2 ab = on ? run_of(c.g.ptr[dir] + c.soff, x) : make_int2(0, 0);
    a[i] = ab.x;
    b[i] = ab.y;
  }
  Win w[4];
#if TM_WIN4
  // the four windows bisected together: up to 8 independent chains in flight
  int l0[4], l1[4], u0[4], u1[4];
#pragma unroll
  for (int i = 0; i < 4; ++i) l0[i] = u0[i] = a[i], l1[i] = u1[i] = b[i];
  bool more = true;
  while (more) {
    more = false;
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      const uint32_t *__restrict__ r = c.g.rnk[i & 1];
      if (l0[i] < l1[i]) {
        const int m = (l0[i] + l1[i]) >> 1;
        if (__ldg(r + m) < c.lo) l0[i] = m + 1; else l1[i] = m;
        more |= l0[i] < l1[i];
      }
      if (u0[i] < u1[i]) {
        const int m = (u0[i] + u1[i]) >> 1;
        if (__ldg(r + m) <= c.hi) u0[i] = m + 1; else u1[i] = m;
        more |= u0[i] < u1[i];
      }
    }
  }
  c.wui = Win{l0[0], u0[0]};
  c.wuo = Win{l0[1], u0[1]};
  c.wvi = Win{l0[2], u0[2]};
  c.wvo = Win{l0[3], u0[3]};
  return;
#endif
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    const uint32_t *__restrict__ r = c.g.rnk[i & 1];
    int l = a[i], u = a[i];
#pragma unroll
    for (int k = 0; k < kShortRun; ++k) {
      if (b[i] - a[i] <= kShortRun && a[i] + k < b[i]) {
        const uint32_t x = __ldg(r + a[i] + k);
        l += x < c.lo;
        u += x <= c.hi;
      }
    }
    w[i] = Win{l, u};
  }
#pragma unroll
  for (int i = 0; i < 4; ++i)
    if (b[i] - a[i] > kShortRun) w[i] = window_of_run(c.g.rnk[i & 1], a[i], b[i], c.lo, c.hi);
  c.wui = w[0];
  c.wuo = w[1];
  c.wvi = w[2];
  c.wvo = w[3];
}

// self-loops of x inside the window (kernels.py:279-287): pair run (x, x);
// has_loop = loop[x] when the caller already holds it
__device__ __forceinline__ int loops_in_window(const Ctx &c, int x, int has_loop = -1) {
  if (has_loop < 0) has_loop = __ldg(c.g.loop + x);
  if (!has_loop) return 0;
  const int a = __ldg(c.g.gptr[1] + x), b = __ldg(c.g.gptr[1] + x + 1);
  const uint64_t base = (uint64_t)(uint32_t)x << c.g.rank_bits;
  return lb_u64(c.g.pkey[1], a, b, base + c.hi + 1) - lb_u64(c.g.pkey[1], a, b, base + c.lo);
}

// CSR entry j is the first occurrence of its neighbour inside the window
// (np.unique, kernels.py:59): the previous entry with the same (owner, nbr)
// lies before lo (prev = rank + 1, 0 = none)
__device__ __forceinline__ bool first_in_window(const Ctx &c, int dir, int j) {
  TM_CNT(kCtrFirst, 1);
  return (uint32_t)__ldg(c.g.np[dir] + j).y <= c.lo;
}

// (neighbour, prev) of CSR slot j in one 8-byte load: the walkers read both
// for every entry (membership test + np.unique dedup)
__device__ __forceinline__ int2 slot_np(const Ctx &c, int dir, int j) {
  TM_CNT(kCtrFirst, 1);
  return __ldg(c.g.np[dir] + j);
}
__device__ __forceinline__ bool first_of(const Ctx &c, int2 sl) { return (uint32_t)sl.y <= c.lo; }

// does x's dir-window w contain neighbour n?  Windows are time-local and
// short: scan them.  A wide w (a hub) is answered by one bisection of the
// SHORTER pair run: x's dir run keyed by n, or n's opposite run keyed by x
// (n in N^dir(x)  <=>  x in N^{1-dir}(n)).
#ifndef TM_SCAN_WIN
#define TM_SCAN_WIN 16
#endif
constexpr int kScanWin = TM_SCAN_WIN;

// is n in x's dir-window?  x's run is [xs, xe): one bisection of the SHORTER
// pair run — x's dir run keyed by n, or n's opposite run keyed by x
// (n in N^dir(x)  <=>  x in N^{1-dir}(n)).  Needs no window of x.
__device__ __forceinline__ bool exists_pair(const Ctx &c, int dir, int x, int xs, int xe, int n) {
  TM_CNT(kCtrPairCall, 1);
  const int ns = __ldg(c.g.gptr[dir ^ 1] + n), ne = __ldg(c.g.gptr[dir ^ 1] + n + 1);
  const bool from_x = xe - xs <= ne - ns;
  const uint64_t *k = c.g.pkey[from_x ? dir : dir ^ 1];
  const int s = from_x ? xs : ns, e = from_x ? xe : ne;
  const uint64_t base = (uint64_t)(uint32_t)(from_x ? n : x) << c.g.rank_bits;
  const int q = lb_u64(k, s, e, base + c.lo);
  return q < e && __ldg(k + q) <= base + c.hi;
}

// is n among the entries of window w of direction dir?  (short windows)
__device__ __forceinline__ bool scan_for(const Ctx &c, int dir, const Win &w, int n) {
  TM_CNT(kCtrScanCall, 1);
  bool hit = false;
#if TM_VEC_SCAN
  // two 16-byte loads (four entries) per round trip, from the even-aligned
  // block holding w.a (device buffers are padded past their end)
  const int2 *__restrict__ nb = c.g.np[dir];
  for (int j = w.a & ~1; j < w.b && !hit; j += 4) {
    TM_CNT(kCtrScanLoad, 1);
    const int4 p0 = __ldg(reinterpret_cast<const int4 *>(nb + j));
    const int4 p1 = j + 2 < w.b ? __ldg(reinterpret_cast<const int4 *>(nb + j + 2)) : make_int4(-1, 0, -1, 0);
    hit = (j >= w.a && p0.x == n) | (j + 1 < w.b && p0.z == n) | (p1.x == n && j + 2 < w.b) |
          (p1.z == n && j + 3 < w.b);
  }
#elif TM_SCAN4
  // four independent loads per round trip (the early exit only every 4)
  const int2 *__restrict__ nb = c.g.np[dir];
  for (int j = w.a; j < w.b && !hit; j += 4) {
    TM_CNT(kCtrScanLoad, 1);
    const int x0 = __ldg(nb + j).x;
    const int x1 = j + 1 < w.b ? __ldg(nb + j + 1).x : -1;
    const int x2 = j + 2 < w.b ? __ldg(nb + j + 2).x : -1;
    const int x3 = j + 3 < w.b ? __ldg(nb + j + 3).x : -1;
    hit = (x0 == n) | (x1 == n) | (x2 == n) | (x3 == n);
  }
#else
  for (int j = w.a; j < w.b && !hit; ++j) {
    TM_CNT(kCtrScanLoad, 1);
    hit = __ldg(c.g.np[dir] + j).x == n;
  }
#endif
  return hit;
}

#ifndef TM_SLAB_PROBE
#define TM_SLAB_PROBE 1
#endif

// does x's dir-window w contain neighbour n?  Windows are time-local and
// short: scan them.  A wide w (a hub): in a slab view n's opposite window
// (x in N^{1-dir}(n)) is a short slab run — scan that; else (or when that is
// wide too) one bisection of the shorter pair-index run.
// code-size switches (A/B): out-of-line copies of the widest helpers shrink
// the hot code (the kernels show instruction-fetch stalls), but measured
// slower — inner_hits out of line: HI-Large warp kernel 70.1 -> 90.8 ms
#ifndef TM_NOINLINE_PROBE
#define TM_NOINLINE_PROBE 0
#endif
#if TM_NOINLINE_PROBE
#define TM_PROBE_ATTR __noinline__
#else
#define TM_PROBE_ATTR __forceinline__
#endif
__device__ TM_PROBE_ATTR bool exists_in(const Ctx &c, int dir, int x, const Win &w, int n) {
  if (w.len() <= kScanWin) return scan_for(c, dir, w, n);
#if TM_SLAB_PROBE
  if (c.g.ptr[dir ^ 1] != c.g.gptr[dir ^ 1]) {
    const Win wn = window(c, dir ^ 1, n);
    if (wn.len() <= kScanWin) return scan_for(c, dir ^ 1, wn, x);
  }
#endif
  return exists_pair(c, dir, x, __ldg(c.g.gptr[dir] + x), __ldg(c.g.gptr[dir] + x + 1), n);
}

// n in N^dir(x) for a wide x (a hub, pair-index run [xs, xe)): in a slab
// view n's opposite window is usually a few L2-resident entries — scan it
// for x; else one bisection of the shorter pair-index run
__device__ __forceinline__ bool exists_hub(const Ctx &c, int dir, int x, int xs, int xe, int n) {
#if TM_SLAB_PROBE
  if (c.g.ptr[dir ^ 1] != c.g.gptr[dir ^ 1]) {
    const Win wn = window(c, dir ^ 1, n);
    if (wn.len() <= kScanWin) return scan_for(c, dir ^ 1, wn, x);
  }
#endif
  return exists_pair(c, dir, x, xs, xe, n);
}

__device__ __forceinline__ long long warp_sum(long long x) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) x += __shfl_xor_sync(0xffffffffu, x, o);
  return x;
}

}  // namespace dev
}  // namespace tmb
