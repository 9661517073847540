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
// Work decomposition (the reference splits contiguous trigger ranges per
// worker, engine.py:681-682, and walks each trigger serially):
//
// Every set column of a trigger e = (u -> v) is a sum over the distinct
// neighbours of one of two windowed slices of e:
//   U items  m in N-(u) \ {u, v}:  stack's a, cycle_3 (m in N+(v)),
//            sg (|N+(m) ∩ N-(v)| >= K)
//   V items  m in N+(v) \ {u, v}:  stack's c, gs (|N-(m) ∩ N+(u)| >= K),
//            cycle_4..8 (chains a1 = m -> a2 -> ... closing into N-(u))
//
//   k_mine_warp    one warp = 32 triggers.  Each lane bisects its trigger's
//                  four windows and computes FAN / DEGREE / cycle_2.  The
//                  warp then FLATTENS the U items of all 32 triggers into one
//                  list and deals it round-robin to its lanes (exclusive scan
//                  of the slice lengths + a 5-step search of the owner), then
//                  the V items — so a lane's cost no longer depends on its own
//                  trigger's hub degree.  Item contributions go to the staged
//                  output rows in shared memory with atomics; rows leave in
//                  one coalesced write.
//   task queue     a trigger slice longer than kDomSplit is not walked by the
//                  warp but emitted as DOMAIN tasks of kTaskSpan entries; a
//                  chain node whose out-window is longer than kDeepSplit is
//                  emitted as a CHAIN task.  k_mine_tasks (one warp per task,
//                  lane per entry) runs them in rounds — a task only spawns
//                  deeper chain tasks — adding partial counts to the int64
//                  output with atomicAdd.  stack's a * c and cycle_3's
//                  threshold need the whole count: split rows keep a, c and
//                  the raw cycle_3 count in a scratch slot that
//                  k_mine_finalize turns into the column values.
// Every count is an integer sum over disjoint pieces, so the result is
// exactly the reference's regardless of the split.
#include "tm_device.cuh"

namespace tmb {
namespace {

#ifndef TM_WARP_THREADS
#define TM_WARP_THREADS 64  // measured: 64 > 128 > 32 (profiles/)
#endif
constexpr int kThreads = TM_WARP_THREADS;  // k_mine_warp block
constexpr int kWarps = kThreads / 32;
#ifndef TM_TASK_THREADS
#define TM_TASK_THREADS 256
#endif
#ifndef TM_TASK_MINB
#define TM_TASK_MINB 4
#endif
constexpr int kTaskThreads = TM_TASK_THREADS;
#ifndef TM_DOM_SPLIT
#define TM_DOM_SPLIT 128  // swept 64..512 with TM_DEEP_SPLIT 4..128
#endif
#ifndef TM_DEEP_SPLIT
#define TM_DEEP_SPLIT 8  // short windows (mean in-window degree <= 2); long ones use 64
#endif
constexpr int kDomSplit = TM_DOM_SPLIT;    // a trigger slice above this becomes domain tasks
constexpr int kDeepSplit = TM_DEEP_SPLIT;  // CycGroup::deep_split for short windows
constexpr int kTaskSpan = 128;       // entries per task (4 per lane)
constexpr int kLvlDomU = 8, kLvlDomV = 9;  // Task::level of domain tasks
constexpr int kLvlPullV = 10;  // Task::level: gs + cycles of a hub v expanded from u's side
// V-item parts (Task::pad0 of domain V tasks): stack's c, gs, cycles
constexpr int kVStack = 1, kVGs = 2, kVCyc = 4, kVAll = 7;
constexpr int kPullFlag = 32;  // Task::level bit: a whole wide window to expand backwards
constexpr int kHostPieces = 8;     // host-output pieces overlapped with their D2H (tm_graph::piece_ev)

using namespace dev;

// ------------------------------------------------------------ task queue

struct Task {
  int32_t row;   // trigger row (relative to lo); < 0 = empty slot
  int8_t grp;    // delta group
  int8_t level;  // 1..4: chain slice of a_level; kLvlDomU / kLvlDomV: trigger slice
  int8_t pad0, pad1;  // pad0: V-item parts of a domain V task (kV*)
  int32_t a, b;  // CSR range of the slice piece
  int32_t path[kMaxChain];  // chain a1..a_level; domain tasks: path[0] = scratch slot
};

// Backward-layer filters of the trigger a task works for (task kernel; see
// TaskBloom): the chain walk skips nodes that cannot reach u in time
struct TaskBloom;

// A depth-1 chain node a1 = m of a trigger whose descent (chains a2.. of
// cycle_5+) the trigger kernel defers: the deep, rare enumeration (0.08
// depth-2 nodes per trigger at HI-Large) would otherwise keep its registers
// allocated in the hot kernel.  k_mine_chains runs the records, one thread
// each.
struct ChainRec {
  int32_t row, a1, wa, wb, grp;  // trigger row, a1, a1's out-window entries
  int32_t ua, ub;                // the trigger's u-in window (every close reads it)
};
struct ChainQ {
  ChainRec *rec;
  unsigned long long *count;
  unsigned long long cap;
  unsigned int *overflow;  // set when a deferred descent found no room (the call is re-run inline)
};

struct Queue {
  Task *q;
  unsigned long long *count;  // 64-bit: reservations past a full queue cannot wrap it
  int32_t cap;
  const TaskBloom *bloom;  // null: no filtering (warp kernel, small windows)
  ChainQ chains;           // trigger kernel: deferred chain descents (rec null: none)
};

// warp-aggregated reservation of one record per calling lane
__device__ __forceinline__ bool push_chain(const ChainQ &cq, int row, int grp, int a1, int wa, int wb,
                                           const Win &ui) {
  if (!cq.rec) return false;
  const unsigned m = __activemask();
  const int lane = threadIdx.x & 31, leader = __ffs(m) - 1;
  unsigned long long base = 0;
  if (lane == leader) base = atomicAdd(cq.count, (unsigned long long)__popc(m));
  base = __shfl_sync(m, base, leader);
  const unsigned long long k = base + (unsigned long long)__popc(m & ((1u << lane) - 1));
  if (k >= cq.cap) return false;
  cq.rec[k] = ChainRec{row, a1, wa, wb, grp, ui.a, ui.b};
  return true;
}

// Bloom filters of the backward layers B_2..B_5 (B_1 = N-(u) \ {u, v},
// B_{k+1} = N-(B_k) \ {u, v}, windowed): a node at depth j that closes at
// depth d lies in B_{2+d-j}, so a chain walk over a hub window (long delta:
// millions of chain nodes) tests each candidate against the layers its
// depth needs before reading its window.  No false negatives, so the walk
// stays exact; a layer that could not be built completely is "all".
constexpr int kBloomLayers = 4;    // B_2 .. B_5
constexpr int kBloomWords = 256;   // 8192 bits per layer
#ifndef TM_BLOOM_LIST
#define TM_BLOOM_LIST 4096
#endif
constexpr int kBloomList = TM_BLOOM_LIST;  // members of one layer kept to build the next (global scratch)
constexpr int kInPlace = 4096;     // a filtered pull task walks windows up to this long itself
constexpr int kBloomMin = 64;      // tasks over narrower windows do not build filters
struct TaskBloom {
  uint32_t w[kBloomLayers][kBloomWords];
  int32_t valid;  // bit k-2: layer B_k complete
  int32_t n[2];   // list fill counters (ping-pong)
};
__device__ __forceinline__ uint32_t bloom_bit(int x) { return ((uint32_t)x * 0x9E3779B1u) >> 19; }
__device__ __forceinline__ bool bloom_has(const uint32_t *w, int x) {
  const uint32_t b = bloom_bit(x);
  return (w[b >> 5] >> (b & 31)) & 1u;
}

#ifndef TM_WARM_ROLL  // 1: the trigger kernel's short per-column loops stay rolled (smaller code)
#define TM_WARM_ROLL 1
#endif
#if TM_WARM_ROLL
#define TM_WARM_ROLLED _Pragma("unroll 1")
#else
#define TM_WARM_ROLLED
#endif
#ifndef TM_EMIT_NOINLINE  // 1: task emission out of line (cold: 0.006 tasks per trigger)
#define TM_EMIT_NOINLINE 0
#endif
#if TM_EMIT_NOINLINE
#define TM_EMIT_ATTR __noinline__
#else
#define TM_EMIT_ATTR
#endif
// reserve n slots of the queue, or none (-1).  The count is 64-bit, so the
// increments of reservations that fail past a full queue cannot wrap it into
// a small (or negative) index; a failed reservation that straddles the end
// marks its slots below the capacity empty (the consumer reads min(count,
// cap) slots).  A plain atomicAdd: a CAS loop serialized the many emitters
// of a long-window step (HI-Large cycles: 2.7x slower).
__device__ __forceinline__ int reserve(const Queue &qu, int n) {
  const unsigned long long cap = (unsigned long long)qu.cap;
  if (*(volatile unsigned long long *)qu.count >= cap) return -1;
  const unsigned long long base = atomicAdd(qu.count, (unsigned long long)n);
  if (base + (unsigned long long)n > cap) {
#pragma unroll 1  // cold path: keep it out of the hot kernels' instruction footprint
    for (unsigned long long k = base; k < cap; ++k) qu.q[k].row = -1;  // holes stay empty
    return -1;
  }
  return (int)base;
}

// cut [a, b) into kTaskSpan pieces; false (caller walks it itself) when the
// queue is full — the walk is slower but exact and still on the GPU
__device__ TM_EMIT_ATTR bool emit(const Queue &qu, int row, int grp, int level, int p0, int p1, int p2, int p3,
                     int p4, int a, int b, int parts = kVAll) {
  const int n = (b - a + kTaskSpan - 1) / kTaskSpan;
  TM_CNT(level >= kLvlDomU ? kCtrDomTask : kCtrChainTask, n);
  const int base = reserve(qu, n);
  if (base < 0) {
    TM_CNT(kCtrQueueFull, 1);
    return false;
  }
#pragma unroll 1
  for (int k = 0; k < n; ++k) {
    Task t;
    t.row = row;
    t.grp = (int8_t)grp;
    t.level = (int8_t)level;
    t.pad0 = (int8_t)parts;
    t.pad1 = 0;
    t.a = a + k * kTaskSpan;
    t.b = min(b, t.a + kTaskSpan);
    t.path[0] = p0; t.path[1] = p1; t.path[2] = p2; t.path[3] = p3; t.path[4] = p4;
    qu.q[base + k] = t;
  }
  return true;
}

// one task for the whole range [a, b) (a pull task): false when the queue is full
__device__ TM_EMIT_ATTR bool emit_whole(const Queue &qu, int row, int grp, int level, const int (&path)[kMaxChain],
                           int a, int b) {
  TM_CNT(kCtrChainTask, 1);
  const int k = reserve(qu, 1);
  if (k < 0) {
    TM_CNT(kCtrQueueFull, 1);
    return false;
  }
  Task t;
  t.row = row;
  t.grp = (int8_t)grp;
  t.level = (int8_t)level;
  t.pad0 = t.pad1 = 0;
  t.a = a;
  t.b = b;
#pragma unroll
  for (int i = 0; i < kMaxChain; ++i) t.path[i] = path[i];
  qu.q[k] = t;
  return true;
}

// ------------------------------------------------------------ set helpers

// distinct-neighbour intersection |N^{dx}(x) ∩ N^{dy}(y)| \ {x, y}, early
// exit at K (sg: x = s out, y = v in; gs: x = d in, y = u out).  x and y are
// never members (no self-loops).  f >= 0 is a node known to be in the
// intersection and not in {x, y} (sg: u, gs: v, when u != v — the trigger
// and the item edge put it there): it counts without a probe and the walks
// skip it.  Since f is one of y's window entries, no more than wy.len()
// nodes can hit, which often settles the column before x's window is read.
// A wide run of x (a sender hub) is not bisected when y's window is short:
// y's side is walked and each node probed in the pair index instead.
constexpr int kLazyRun = 32;
#ifndef TM_NOINLINE_INNER
#define TM_NOINLINE_INNER 0
#endif
#if TM_NOINLINE_INNER
#define TM_INNER_ATTR __noinline__
#else
#define TM_INNER_ATTR __forceinline__
#endif
__device__ TM_INNER_ATTR int inner_hits(const Ctx &c, int x, int dx, int y, int dy,
                                          const Win &wy, int K, int f) {
  int hits = f >= 0 ? 1 : 0;
  TM_CNT(kCtrInnerCall, 1);
  if (hits >= K || wy.len() < K) {
    TM_CNT(kCtrInnerSkip, 1);
    return hits;
  }
  const int32_t *pt = c.g.ptr[dx] + c.soff;  // x's run (slab view: its slab run)
  const int2 xr = run_of(pt, x);
  const int xa = xr.x, xb = xr.y;
  if (xb - xa > kLazyRun && wy.len() <= kLazyRun) {
    const int xs = __ldg(c.g.gptr[dx] + x), xe = __ldg(c.g.gptr[dx] + x + 1);  // pair-index run
    for (int j = wy.a; j < wy.b && hits < K; ++j) {
      TM_CNT(kCtrInnerWalk, 1);
      const int2 sl = slot_np(c, dy, j);
      const int m = sl.x;
      if (m == x || m == y || m == f || !first_of(c, sl)) continue;
      hits += exists_hub(c, dx, x, xs, xe, m);
    }
    return hits;
  }
  const int wa = lb_u32(c.g.rnk[dx], xa, xb, c.lo);
  const Win wx{wa, ub_u32(c.g.rnk[dx], wa, xb, c.hi)};
  TM_CNT(kCtrWin, 1);
  const bool walk_x = wx.len() <= wy.len();
  const Win w = walk_x ? wx : wy;
  const int other = walk_x ? y : x;
  const int d = walk_x ? dx : dy, od = walk_x ? dy : dx;
  const Win ow = walk_x ? wy : wx;
  for (int j = w.a; j < w.b && hits < K; ++j) {
    TM_CNT(kCtrInnerWalk, 1);
    const int2 sl = slot_np(c, d, j);
    const int m = sl.x;
    if (m == x || m == y || m == f || !first_of(c, sl)) continue;
    hits += exists_in(c, od, other, ow, m);
  }
  return hits;
}

// closing set of a chain ending at `a` with NP earlier chain nodes:
//   |(N+(a) ∩ N-(u)) \ {v, path[0..NP-1]}|   (Appendix A cycle_k; cycle_4
//   kernels.py:330-341 for NP = 0)
template <int NP>
__device__ __forceinline__ int close_count(const Ctx &c, int a, const Win &wa,
                                           const int (&path)[kMaxChain]) {
  const bool walk_a = wa.len() <= c.wui.len();
  const Win w = walk_a ? wa : c.wui;
  const int d = walk_a ? 1 : 0;
  int cnt = 0;
  TM_CNT(kCtrCloseCall, 1);
  for (int j = w.a; j < w.b; ++j) {
    TM_CNT(kCtrCloseWalk, 1);
    const int2 sl = slot_np(c, d, j);
    const int m = sl.x;
    if (m == a || m == c.u || m == c.v) continue;
    bool dup = false;
#pragma unroll
    for (int i = 0; i < NP; ++i) dup |= (path[i] == m);
    if (dup || !first_of(c, sl)) continue;
    cnt += walk_a ? exists_in(c, 0, c.u, c.wui, m) : exists_in(c, 1, a, wa, m);
  }
  return cnt;
}

// per-depth close: add |C| to every cycle column closing at depth d whose
// min_size it reaches (per-binding threshold, engine.py:462-464)
struct CycAcc {
  long long e[kMaxCyc];
};

__device__ __forceinline__ void close_at(const CycGroup &cg, int d, int cc, CycAcc &acc) {
#pragma unroll
  for (int e = 0; e < kMaxCyc; ++e)
    if (e < cg.n && cg.depth[e] == d && cc >= cg.k[e]) acc.e[e] += cc;
}

// Chains a1..a_d of the cycle group (d <= MAXD):
//   a1 in N+(v)\{u};  a_i in N+(a_{i-1}) \ {u, v, a1..a_{i-2}};
//   cycle_{d+3} closes at depth d.
// Level L chooses a_{L+1} among the out-neighbours of a_L = path[L-1]
// (L >= 1; level 0 is the V item loop): either the window entries [ja, jb)
// of a_L's out-run, or — for a wide a_L (a sender hub) — the candidate list
// `cand[ja..jb)` of useful nodes (see useful_nodes), each probed for
// a_L -> a.  Every level has ONE call site of the next, so the inlined
// template tree stays linear in the depth.
#ifndef TM_BCAP
#define TM_BCAP 48  // tests build a tiny-cap variant to exercise the overflow paths
#endif
constexpr int kBCap = TM_BCAP;

// Backward sets: every chain that contributes reaches u inside the window,
// so a node at depth j closing at depth d >= j lies in B_{2+d-j}, where
// B_1 = N-(u) \ {u, v} and B_{k+1} = N-(B_k) \ {u, v} (windowed, distinct).
// They are supersets of the useful choices — pruning with them skips only
// chains that add nothing — and small when in-degrees are.
__device__ __forceinline__ bool bset_add(int *node, int from, int &n, int m) {
  for (int i = from; i < n; ++i)
    if (node[i] == m) return true;
  if (n == kBCap) return false;
  node[n++] = m;
  return true;
}

// the useful depth-J nodes (layers 2 + d - J for the closing depths d >= J
// in mask), or -1 when a set overflows.  Out of line: it runs for wide
// chain nodes only and keeps its arrays off the walkers' registers.
__device__ __noinline__ int useful_nodes(const DevGraph &g, int64_t soff, int u, int v, uint32_t lo,
                                         uint32_t hi, int wa, int wb, int mask, int maxd, int J, int *use) {
  const Ctx c{g, u, v, lo, hi, {wa, wb}, {}, {}, {}, soff};
  const int H = 2 + maxd - J;  // deepest layer any useful depth-J node can be in
  int node[kBCap], lend[kMaxChain + 3];
  int n = 0;
  lend[0] = 0;
  for (int j = wa; j < wb; ++j) {  // B_1
    const int m = __ldg(g.np[0] + j).x;
    if (m == u || m == v || !first_in_window(c, 0, j)) continue;
    if (!bset_add(node, 0, n, m)) return TM_CNT(kCtrUsefulOver, 1), -1;
  }
  lend[1] = n;
  for (int k = 2; k <= H; ++k) {
    for (int i = lend[k - 2]; i < lend[k - 1]; ++i) {
      const Win w = window(c, 0, node[i]);
      if (w.len() > kBCap) return TM_CNT(kCtrUsefulOver, 1), -1;
      for (int j = w.a; j < w.b; ++j) {
        const int m = __ldg(g.np[0] + j).x;
        if (m == u || m == v || !first_in_window(c, 0, j)) continue;
        if (!bset_add(node, lend[k - 1], n, m)) return TM_CNT(kCtrUsefulOver, 1), -1;
      }
    }
    lend[k] = n;
  }
  int nu = 0;
  for (int d = J; d <= maxd; ++d) {
    if (!(mask & (1 << d))) continue;
    const int k = 2 + d - J;
    for (int i = lend[k - 1]; i < lend[k]; ++i)
      if (!bset_add(use, 0, nu, node[i])) return TM_CNT(kCtrUsefulOver, 1), -1;
  }
  return nu;
}

// candidates for depth J under a wide window w of path[J-2]: true and
// (ja, jb, cand) set when the backward sets are much smaller than w
__device__ __forceinline__ bool pull_candidates(const Ctx &c, const CycGroup &cg, int maxd, int J,
                                                const Win &w, int *use, int &ja, int &jb) {
  const int nu = useful_nodes(c.g, c.soff, c.u, c.v, c.lo, c.hi, c.wui.a, c.wui.b, cg.mask, maxd, J, use);
  if (nu < 0 || nu * 4 > w.len()) return false;
  TM_CNT(kCtrPull, 1);
  ja = 0;
  jb = nu;
  return true;
}

template <int L, bool PI>
__device__ __forceinline__ void chain_level(const Ctx &c, const CycGroup &cg, int row, int grp,
                                            int (&path)[kMaxChain], int ja, int jb, const int *cand,
                                            CycAcc &acc, const Queue &qu);

// a_{L+1} = a chosen (all exclusions checked): close at depth L + 1, descend.
// A wide a: PI (task kernel) expands it backwards in place, or splits it
// into chain tasks; the warp kernel hands the whole window to a pull task,
// keeping its walkers lean.  The deepest level is cg.maxd at run time: one
// instantiation per level serves every cycle length (code size: the kernels
// were bound by instruction-cache misses with one tree per maxd).
template <int L, bool PI>
__device__ __forceinline__ void chain_pick(const Ctx &c, const CycGroup &cg, int row, int grp,
                                           int (&path)[kMaxChain], int a, CycAcc &acc,
                                           const Queue &qu) {
  TM_CNT(kCtrChain1 + L, 1);
  const Win w = window(c, 1, a);  // a's out-window: closes and descends
  if (cg.mask & (1 << (L + 1))) close_at(cg, L + 1, close_count<L>(c, a, w, path), acc);
  if constexpr (L + 1 < kMaxChain) {
    if (L + 1 >= cg.maxd) return;
    path[L] = a;
    int ja = w.a, jb = w.b;
    const int *cand = nullptr;
    int use[kBCap];
    if (w.len() > cg.deep_split) {
      if constexpr (PI) {
        if (pull_candidates(c, cg, cg.maxd, L + 2, w, use, ja, jb)) cand = use;
        else if (emit(qu, row, grp, L + 1, path[0], path[1], path[2], path[3], path[4], w.a, w.b)) return;
      } else {
        if (emit_whole(qu, row, grp, (L + 1) | kPullFlag, path, w.a, w.b)) return;
      }
    }
    chain_level<L + 1, PI>(c, cg, row, grp, path, ja, jb, cand, acc, qu);
  }
}

template <int L, bool PI>
__device__ __forceinline__ void chain_level(const Ctx &c, const CycGroup &cg, int row, int grp,
                                            int (&path)[kMaxChain], int ja, int jb, const int *cand,
                                            CycAcc &acc, const Queue &qu) {
  const int owner = path[L - 1];
  int os = 0, oe = 0;
  if (cand) {
    os = __ldg(c.g.gptr[1] + owner);  // pair-index run of the owner
    oe = __ldg(c.g.gptr[1] + owner + 1);
  }
  // layers a depth-(L+1) node must meet: B_{1+d-L} for closing depths d
  int need = 0;
  bool filter = false;
  if constexpr (PI) {
    if (qu.bloom) {
      for (int d = L + 1; d <= cg.maxd; ++d) {
        if (!(cg.mask & (1 << d))) continue;
        const int k = 1 + d - L;
        if (k - 2 < kBloomLayers && ((qu.bloom->valid >> (k - 2)) & 1)) need |= 1 << (k - 2);
        else need |= 1 << kBloomLayers;  // not filtered
      }
      filter = !(need >> kBloomLayers);
    }
  }
  for (int j = ja; j < jb; ++j) {
    const int2 sl = cand ? make_int2(cand[j], 0) : slot_np(c, 1, j);
    const int a = sl.x;
    if (a == owner || a == c.u || a == c.v) continue;
    if constexpr (PI) {
      if (filter) {
        bool hit = false;
#pragma unroll
        for (int k = 0; k < kBloomLayers; ++k)
          if ((need >> k) & 1) hit |= bloom_has(qu.bloom->w[k], a);
        if (!hit) continue;
      }
    }
    bool dup = false;
#pragma unroll
    for (int i = 0; i + 1 < L; ++i) dup |= (path[i] == a);
    if (dup || !(cand ? exists_hub(c, 1, owner, os, oe, a) : first_of(c, sl))) continue;
    chain_pick<L, PI>(c, cg, row, grp, path, a, acc, qu);
  }
}

// cycles through chain node a1 = m (a V item), depths 1..maxd
template <bool PI>
__device__ __forceinline__ void cycles_a1(const Ctx &c, const CycGroup &cg, int row, int grp,
                                          int (&path)[kMaxChain], const Win &w, CycAcc &acc,
                                          const Queue &qu) {
  int ja = w.a, jb = w.b;
  const int *cand = nullptr;
  int use[kBCap];
  if (w.len() > cg.deep_split) {
    if constexpr (PI) {
      if (pull_candidates(c, cg, cg.maxd, 2, w, use, ja, jb)) cand = use;
      else if (emit(qu, row, grp, 1, path[0], -1, -1, -1, -1, w.a, w.b)) return;
    } else {
      if (emit_whole(qu, row, grp, 1 | kPullFlag, path, w.a, w.b)) return;
    }
  }
  chain_level<1, PI>(c, cg, row, grp, path, ja, jb, cand, acc, qu);
}

// DEFER (trigger kernel only): the descent below a1 is not enumerated here —
// a narrow a1 becomes a chain record (k_mine_chains), a wide one a pull
// task.  If a queue is full the record is dropped and the call's overflow
// word set: tm_mine then runs the call again with DEFER off (the inline
// enumeration), so no count is ever lost.
template <bool PI, bool DEFER = false>
__device__ __forceinline__ void cycles_from_a1(const Ctx &c, const CycGroup &cg, int row, int grp,
                                               int m, CycAcc &acc, const Queue &qu) {
  int path[kMaxChain] = {m, -1, -1, -1, -1};
  const Win w = window(c, 1, m);
  if (cg.mask & 2) close_at(cg, 1, close_count<0>(c, m, w, path), acc);
  if (cg.maxd < 2 || w.len() == 0) return;
  if constexpr (DEFER) {
    if (!(w.len() <= cg.deep_split ? push_chain(qu.chains, row, grp, m, w.a, w.b, c.wui)
                                   : emit_whole(qu, row, grp, 1 | kPullFlag, path, w.a, w.b)))
      TM_CNT(kCtrChainOver, 1), atomicOr(qu.chains.overflow, 1u);
  } else {
    cycles_a1<PI>(c, cg, row, grp, path, w, acc, qu);
  }
}

// a chain task resumes at level L with a1..a_L given (entries [ja, jb) of
// a_L's window, or of a candidate list)
__device__ __forceinline__ void cycles_resume(const Ctx &c, const CycGroup &cg, int row, int grp,
                                              int L, const int (&p0)[kMaxChain], int ja, int jb,
                                              const int *cand, CycAcc &acc, const Queue &qu) {
  int path[kMaxChain] = {p0[0], p0[1], p0[2], p0[3], p0[4]};
  if (L < 1 || L >= cg.maxd) return;
  switch (L) {
    case 1: chain_level<1, true>(c, cg, row, grp, path, ja, jb, cand, acc, qu); return;
    case 2: chain_level<2, true>(c, cg, row, grp, path, ja, jb, cand, acc, qu); return;
    case 3: chain_level<3, true>(c, cg, row, grp, path, ja, jb, cand, acc, qu); return;
    default: chain_level<4, true>(c, cg, row, grp, path, ja, jb, cand, acc, qu); return;
  }
}

// ------------------------------------------------------------ items
//
// A Sink receives the contributions of one item of row `owner`:
//   col(ci, v)  additive column value      sa() / sc()  stack a / c     c3()  cycle_3 raw

template <class Sink>
__device__ __forceinline__ void u_item_sl(const Ctx &c, const DevPlans &P, const DevGroup &gr, const int2 sl,
                                          Sink &sk);
template <class Sink>
__device__ __forceinline__ void u_item(const Ctx &c, const DevPlans &P, const DevGroup &gr, int j,
                                       Sink &sk) {
  u_item_sl(c, P, gr, slot_np(c, 0, j), sk);
}
template <class Sink>
__device__ __forceinline__ void u_item_sl(const Ctx &c, const DevPlans &P, const DevGroup &gr, const int2 sl,
                                          Sink &sk) {
  const int m = sl.x;
  TM_CNT(kCtrUWalk, 1);
  if (m == c.u || m == c.v || !first_of(c, sl)) return;
  TM_CNT(kCtrUItem, 1);
  if (gr.has_stack) sk.sa();
  if ((gr.cyc.mask & 1) && c.u != c.v && exists_in(c, 1, c.v, c.wvo, m)) sk.c3();
  for (int i = 0; i < gr.n_sg; ++i) {  // sg: source m (kernels.py:365-374)
    const int ci = gr.sg_col[i], K = P.p[ci].min_size;
    if (inner_hits(c, m, 1, c.v, 0, c.wvi, K, c.u != c.v ? c.u : -1) >= K) sk.col(ci, 1);
  }
}

// V item m (a distinct node of N+(v) \ {u, v}); parts: kV* bits
template <bool PI, class Sink, bool DEFER = false>
__device__ __forceinline__ void v_node(const Ctx &c, const DevPlans &P, const DevGroup &gr, int grp,
                                       int row, int m, Sink &sk, const Queue &qu, int parts) {
  TM_CNT(kCtrVItem, 1);
  if (gr.has_stack && (parts & kVStack)) sk.sc();
  for (int i = 0; i < gr.n_gs && (parts & kVGs); ++i) {  // gs: destination m (Appendix B)
    const int ci = gr.gs_col[i], K = P.p[ci].min_size;
    if (inner_hits(c, m, 0, c.u, 1, c.wuo, K, c.u != c.v ? c.v : -1) >= K) sk.col(ci, 1);
  }
  if ((parts & kVCyc) && gr.cyc.maxd >= 1 && c.u != c.v && c.wui.len() > 0) {
    CycAcc acc;
#pragma unroll
    for (int e = 0; e < kMaxCyc; ++e) acc.e[e] = 0;
    cycles_from_a1<PI, DEFER>(c, gr.cyc, row, grp, m, acc, qu);
#pragma unroll
    for (int e = 0; e < kMaxCyc; ++e)
      if (e < gr.cyc.n && acc.e[e]) sk.col(gr.cyc.col[e], acc.e[e]);
  }
}

// the trigger's windows: own windows from the group's tables, the rest bisected
__device__ __forceinline__ void trigger_windows(Ctx &c, const DevGroup &gr, int e) {
  int need = gr.need;
  if (gr.own[1]) need &= ~2;
  if (gr.own[0]) need &= ~4;
  fill_windows(c, need);
  if (gr.own[1] && (gr.need & 2)) {
    const int2 w = __ldg(gr.own[1] + e);
    c.wuo = Win{w.x, w.y};
  }
  if (gr.own[0] && (gr.need & 4)) {
    const int2 w = __ldg(gr.own[0] + e);
    c.wvi = Win{w.x, w.y};
  }
}

// ------------------------------------------------------------ k_mine_warp

struct WarpShared {
  int rowid[32];
  int u[32], v[32];
  uint32_t lo[32], hi[32];
  Win wui[32], wuo[32], wvi[32], wvo[32];
  int excl[32];
  int sa[32], sc[32];
  int c3[32];  // cycle_3 raw count (low bits) | V-item parts the warp walks << kPartsShift
  int slab[32];  // slab of the trigger (slab view of the group)
};
constexpr int kPartsShift = 28;  // c3 counts stay far below 2^28 (an in-window degree)

struct SmemSink {  // contributions of row `owner` into the warp's shared state
  WarpShared &ws;
  long long *stage;  // [32][S] staged columns
  const int8_t *slot;
  int owner, S;
  __device__ __forceinline__ void col(int ci, long long v) {
    atomicAdd(reinterpret_cast<unsigned long long *>(stage + owner * S + slot[ci]), (unsigned long long)v);
  }
  __device__ __forceinline__ void sa() { atomicAdd(&ws.sa[owner], 1); }
  __device__ __forceinline__ void sc() { atomicAdd(&ws.sc[owner], 1); }
  __device__ __forceinline__ void c3() { atomicAdd(&ws.c3[owner], 1); }
};

__device__ __forceinline__ Ctx ctx_of(const DevGroup &gr, const WarpShared &ws, int o) {
  return Ctx{gr.view, ws.u[o], ws.v[o], ws.lo[o], ws.hi[o], ws.wui[o], ws.wuo[o], ws.wvi[o], ws.wvo[o],
             (int64_t)ws.slab[o] * gr.stride};
}

// slab of rank r in the group's view (0 in the global view)
__device__ __forceinline__ int slab_of(const DevGroup &gr, uint32_t r) {
  return gr.slab_of ? (int)__ldg(gr.slab_of + r) : 0;
}

// owner lane of flattened item k: the last lane whose exclusive prefix <= k
__device__ __forceinline__ int owner_of(const WarpShared &ws, int k) {
  int o = 0;
#pragma unroll
  for (int step = 16; step > 0; step >>= 1)
    if (ws.excl[o + step] <= k) o += step;
  return o;
}

// items of slice length `len` per lane, flattened over the warp: every item
// is processed once by `f(owner lane, index within the owner's slice)`
template <class F>
__device__ __forceinline__ void flat_for(WarpShared &ws, int lane, int len, F &&f) {
  int incl = len;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const int y = __shfl_up_sync(0xffffffffu, incl, o);
    if (lane >= o) incl += y;
  }
  const int total = __shfl_sync(0xffffffffu, incl, 31);
  ws.excl[lane] = incl - len;
  __syncwarp();
  for (int base = 0; base < total; base += 32) {
    const int k = base + lane;
    if (k < total) {
      const int o = owner_of(ws, k);
      f(o, k - ws.excl[o]);
    }
  }
  __syncwarp();
}

#ifndef TM_WARP_MINB  // min resident blocks per SM for k_mine_warp (register cap)
#define TM_WARP_MINB 16  // 64 registers at 64 threads: measured best
#endif
#ifndef TM_WARP_MINB_DEFER  // the same with deferred chain descents (48 registers, no spills)
#define TM_WARP_MINB_DEFER 20
#endif
#ifndef TM_ONE_GROUP  // 1: calls with one delta group run a kernel instance whose group is
#define TM_ONE_GROUP 1   // P.gr[0] at compile time (constant-bank operands instead of indexed loads)
#endif
// one block's 64 triggers (virtual block vb of the call)
template <bool DEFER, bool ONE>
__device__ __forceinline__ void mine_block(const DevGraph &g, const DevPlans &P, int64_t lo, int64_t n_rows,
                                           long long *__restrict__ out, const Queue &qu,
                                           int32_t *__restrict__ split_rows, int32_t *__restrict__ split_n,
                                           int32_t *__restrict__ scratch, int4 *__restrict__ split_win,
                                           int32_t split_cap, const int32_t *__restrict__ order, int64_t vb,
                                           long long *stage_all, WarpShared *wsh) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  WarpShared &ws = wsh[warp];
  const int C = P.n, S = P.n_stage;
  long long *stage = stage_all + (size_t)warp * 32 * S;
  const int64_t wrow0 = vb * kThreads + warp * 32;
  const int64_t pos = wrow0 + lane;  // position in processing order
  const bool valid = pos < n_rows;
  // trigger order: edge-id order, or (full range only) `order` = the
  // out-CSR slots, so a warp's triggers share sources and their windows
  const int64_t row = valid ? (order ? (int64_t)__ldg(order + pos) : pos) : pos;
  ws.rowid[lane] = (int)row;
  int u = 0, v = 0;
  uint32_t r = 0;
  if (valid) {
    const int e = (int)(lo + row);
    u = __ldg(g.e_src + e);
    v = __ldg(g.e_dst + e);
    r = __ldg(g.e_rank + e);
  }
  TM_WARM_ROLLED
  for (int i = 0; i < S; ++i) stage[lane * S + i] = 0;
  if (valid) TM_CNT(kCtrTrig, 1);
  long long *orow = out + row * C;  // the lane's own row (valid lanes only)

  const int ngroups = ONE ? 1 : P.ngroups;
  for (int gi = 0; gi < ngroups; ++gi) {
    const DevGroup &gr = P.gr[ONE ? 0 : gi];
    int slab = 0;
    uint32_t wlo = 1u;
    if (valid) {
      if (gr.lo_slab) {
        const int2 ls = __ldg(gr.lo_slab + row);
        wlo = (uint32_t)ls.x;
        slab = ls.y;
      } else {
        slab = slab_of(gr, r);
        wlo = __ldg(gr.lo_tab + r);
      }
    }
    Ctx c{gr.view, u, v, wlo, r, {}, {}, {}, {}, (int64_t)slab * gr.stride};
    // self-loop flags issued before the window searches they do not depend on
    const int loop_u = valid ? (int)__ldg(g.loop + u) : 0, loop_v = valid ? (int)__ldg(g.loop + v) : 0;
    if (valid) trigger_windows(c, gr, (int)row);
    // per-lane columns: fan / degree (kernels.py:290-303), cycle_2 (:320-322)
    if (valid) {
      TM_WARM_ROLLED
      for (int i = 0; i < gr.n_lane; ++i) {
        const int d = gr.lane_d[i], ci = d & 0xff;
        const long long k = gr.lane_k[i];
        if (d & kLaneCyc2) {
          const long long raw = (u != v && exists_in(c, 1, v, c.wvo, u)) ? 1 : 0;
          orow[ci] = raw >= k ? raw : 0LL;
        } else {
          const bool ep = (d >> 10) & 1, dir = (d >> 11) & 1;
          const Win w = ep ? (dir ? c.wvo : c.wvi) : (dir ? c.wuo : c.wui);
          long long n = w.len() - loops_in_window(c, ep ? v : u, ep ? loop_v : loop_u);
          if (((d >> 12) & 1) && u != v) n -= 1;
          if (k > 1 && n < k) n = 0;
          orow[ci] = n;
        }
      }
    }
    if (!gr.udom && !gr.vdom) continue;
    ws.u[lane] = u; ws.v[lane] = v; ws.lo[lane] = c.lo; ws.hi[lane] = c.hi; ws.slab[lane] = slab;
    ws.wui[lane] = c.wui; ws.wuo[lane] = c.wuo; ws.wvi[lane] = c.wvi; ws.wvo[lane] = c.wvo;
    ws.sa[lane] = ws.sc[lane] = 0;
    int vparts = kVAll;
    // slices too long for the warp become domain tasks
    int ulen = (valid && gr.udom) ? c.wui.len() : 0;
    int vlen = (valid && gr.vdom) ? c.wvo.len() : 0;
    int slot = -1;
    if (ulen > kDomSplit || vlen > kDomSplit) {
      if (gr.has_stack || (gr.cyc.mask & 1)) {
        slot = atomicAdd(split_n, 1);
        if (slot >= split_cap) {
          slot = -2;  // no scratch left: the warp walks the slices itself
          TM_CNT(kCtrSlotFull, 1);
        } else {
          split_rows[2 * slot] = (int)row;
          split_rows[2 * slot + 1] = gi;
          // the trigger's windows, read back by its tasks (no re-search
          // of hub runs per task)
          split_win[2 * slot] = make_int4(c.wui.a, c.wui.b, c.wuo.a, c.wuo.b);
          split_win[2 * slot + 1] = make_int4(c.wvi.a, c.wvi.b, c.wvo.a, c.wvo.b);
        }
      }
      if (slot != -2) {
        if (ulen > kDomSplit && emit(qu, (int)row, gi, kLvlDomU, slot, -1, -1, -1, -1, c.wui.a, c.wui.b))
          ulen = 0;
        if (vlen > kDomSplit) {
          // a hub v: gs and cycles go to one pull task (expanded from u's
          // side, which is small); stack's c is a cheap distinct count the
          // domain tasks stream.  Any emission that fails is walked here.
          const bool pullable = gr.n_gs > 0 || gr.cyc.maxd >= 1;
          int parts = kVAll;
          if (pullable) {
            const int path[kMaxChain] = {slot, -1, -1, -1, -1};
            if (emit_whole(qu, (int)row, gi, kLvlPullV, path, c.wvo.a, c.wvo.b)) parts = gr.has_stack ? kVStack : 0;
          }
          if (parts && emit(qu, (int)row, gi, kLvlDomV, slot, -1, -1, -1, -1, c.wvo.a, c.wvo.b, parts)) parts = 0;
          if (!parts) vlen = 0;
          vparts = parts;
        }
      }
    }
    ws.c3[lane] = vparts << kPartsShift;
    __syncwarp();
    flat_for(ws, lane, ulen, [&](int o, int k) {
      const Ctx co = ctx_of(gr, ws, o);
      SmemSink sk{ws, stage, P.slot, o, S};
      u_item(co, P, gr, co.wui.a + k, sk);
    });
    flat_for(ws, lane, vlen, [&](int o, int k) {
      const Ctx co = ctx_of(gr, ws, o);
      SmemSink sk{ws, stage, P.slot, o, S};
      const int j = co.wvo.a + k;
      const int2 sl = slot_np(co, 1, j);
      const int m = sl.x;
      TM_CNT(kCtrVWalk, 1);
      if (m == co.u || m == co.v || !first_of(co, sl)) return;
      v_node<false, SmemSink, DEFER>(co, P, gr, gi, ws.rowid[o], m, sk, qu, ws.c3[o] >> kPartsShift);
    });
    // whole-count columns: stack a * c (kernels.py:379-402), cycle_3 threshold
    if (valid) {
      const long long a = ws.sa[lane], d = ws.sc[lane], c3 = ws.c3[lane] & ((1 << kPartsShift) - 1);
      if (slot >= 0) {
        scratch[3 * slot] = (int)a;
        scratch[3 * slot + 1] = (int)d;
        scratch[3 * slot + 2] = (int)c3;
      }
      TM_WARM_ROLLED
      for (int i = 0; i < gr.n_end; ++i) {
        const int dd = gr.end_d[i], ci = dd & 0xff;
        const long long k = gr.end_k[i];
        if (dd & kLaneStack)
          orow[ci] = (a > 0 && d > 0 && a >= k && d >= k) ? a * d : 0LL;
        else
          orow[ci] = c3 >= k ? c3 : 0LL;
      }
    }
    __syncwarp();
  }
  __syncwarp();
  if (order) {  // permuted rows: each lane writes its own
    if (valid)
#pragma unroll 1
      for (int i = 0; i < S; ++i) orow[P.slot_col[i]] = stage[lane * S + i];
    return;
  }
  const int64_t left = n_rows - wrow0;
  const int nrow = left < 32 ? (int)(left > 0 ? left : 0) : 32;
  long long *dst = out + wrow0 * C;
  if (S == 0) return;
  // staged cells i = r * S + k, dealt 32 at a time; (r, k) advanced
  // incrementally instead of dividing by the runtime S
  const int dq = 32 / S, dr = 32 % S;
  int r0 = lane / S, k0 = lane % S;
  TM_WARM_ROLLED
  for (int i = lane; i < nrow * S; i += 32) {
    dst[r0 * C + P.slot_col[k0]] = stage[i];
    r0 += dq;
    k0 += dr;
    if (k0 >= S) k0 -= S, ++r0;
  }
}

// The trigger kernel.  gate != null (the rescue pass): a small grid that
// exits at once unless the deferred pass overflowed; virtual blocks are
// strided over the grid, so the rescue needs no full-size launch.
template <bool DEFER, bool ONE>
__global__ void __launch_bounds__(kThreads, DEFER ? TM_WARP_MINB_DEFER : TM_WARP_MINB) k_mine_warp(
    const __grid_constant__ DevGraph g, const __grid_constant__ DevPlans P, int64_t lo,
    int64_t n_rows, long long *__restrict__ out, Queue qu, int32_t *__restrict__ split_rows,
    int32_t *__restrict__ split_n, int32_t *__restrict__ scratch, int4 *__restrict__ split_win,
    int32_t split_cap, const int32_t *__restrict__ order, const unsigned int *__restrict__ gate) {
  if (gate && *(volatile const unsigned int *)gate == 0) return;  // rescue pass not needed
  extern __shared__ long long stage_all[];  // [warp][32][S]: the staged (item) columns only —
                                            // shared memory left unused is L1 for the walkers
  __shared__ WarpShared wsh[kWarps];
  const int64_t nvb = (n_rows + kThreads - 1) / kThreads;
  for (int64_t vb = blockIdx.x; vb < nvb; vb += gridDim.x) {
    mine_block<DEFER, ONE>(g, P, lo, n_rows, out, qu, split_rows, split_n, scratch, split_win, split_cap, order, vb,
                      stage_all, wsh);
    if (vb + gridDim.x < nvb) __syncthreads();  // the next virtual block re-uses the shared state
  }
}

// ------------------------------------------------------------ tasks

struct GlobalSink {  // contributions of one task item, straight to global memory
  long long *orow;
  int32_t *scr;  // scratch slot of the row (stack a, c, cycle_3 raw)
  __device__ __forceinline__ void col(int ci, long long v) {
    atomicAdd(reinterpret_cast<unsigned long long *>(orow + ci), (unsigned long long)v);
  }
  __device__ __forceinline__ void sa() { atomicAdd(scr, 1); }
  __device__ __forceinline__ void sc() { atomicAdd(scr + 1, 1); }
  __device__ __forceinline__ void c3() { atomicAdd(scr + 2, 1); }
};

// gs of a trigger whose v is a hub, from u's side: with threshold K >= 2, d
// counts when 1 (v itself) + #{n in N+(u) \ {u, v, d} : n -> d} >= K, so
// the candidates are the 2-hop out-neighbourhood of u, enumerated (lane 0)
// when small and each probed for v -> d.  False: declined (walk instead).
__device__ __forceinline__ bool pull_gs(const Ctx &c, const DevPlans &P, const DevGroup &gr, int vs, int ve,
                                        int lane, long long *orow) {
  bool ok = c.u != c.v && c.wuo.len() <= 32;
  for (int i = 0; i < gr.n_gs; ++i) ok &= P.p[gr.gs_col[i]].min_size >= 2;
  constexpr int kPairs = 128;
  if (ok && lane == 0) {
    int pd[kPairs], np = 0;
    for (int j = c.wuo.a; j < c.wuo.b && ok; ++j) {
      const int n = __ldg(c.g.np[1] + j).x;
      if (n == c.u || n == c.v || !first_in_window(c, 1, j)) continue;
      const Win w = window(c, 1, n);
      if (np + w.len() > kPairs) {
        ok = false;
        break;
      }
      for (int k = w.a; k < w.b; ++k) {
        const int d = __ldg(c.g.np[1] + k).x;
        if (d == c.u || d == c.v || d == n || !first_in_window(c, 1, k)) continue;
        pd[np++] = d;
      }
    }
    if (ok) {
      long long cnt[kMaxPlans] = {};
      for (int i = 0; i < np; ++i) {
        bool seen = false;
        for (int q = 0; q < i && !seen; ++q) seen = pd[q] == pd[i];
        if (seen) continue;
        int hits = 2;  // v, and the n of this first occurrence
        for (int q = i + 1; q < np; ++q) hits += pd[q] == pd[i];
        bool member = false, probed = false;
        for (int gi = 0; gi < gr.n_gs; ++gi) {
          if (hits < P.p[gr.gs_col[gi]].min_size) continue;
          if (!probed) member = exists_hub(c, 1, c.v, vs, ve, pd[i]), probed = true;
          if (member) ++cnt[gi];
        }
      }
      for (int gi = 0; gi < gr.n_gs; ++gi)
        if (cnt[gi])
          atomicAdd(reinterpret_cast<unsigned long long *>(orow + gr.gs_col[gi]), (unsigned long long)cnt[gi]);
    }
  }
  return __shfl_sync(0xffffffffu, ok, 0);
}

// the task's backward-layer filters B_2..B_top, built by the warp: lanes
// split the previous layer's members (B_1 = u's in-window), expand their
// in-windows, set bits and list the members for the next layer (global
// ping-pong lists); a layer whose list overflows ends the build
__device__ void build_bloom(const Ctx &c, TaskBloom &B, int lane, int top, int *list0, int *list1) {
  __syncwarp();  // lanes may still be reading the previous task's filters
  for (int i = lane; i < kBloomLayers * kBloomWords; i += 32) (&B.w[0][0])[i] = 0u;
  if (lane == 0) {
    B.valid = 0;
    B.n[0] = B.n[1] = 0;
  }
  __syncwarp();
  int *lists[2] = {list0, list1};
  for (int k = 2; k <= top && k - 2 < kBloomLayers; ++k) {
    const int src = k & 1, dst = src ^ 1;  // layer k-1's list -> layer k's list
    const int nsrc = k == 2 ? c.wui.len() : min(B.n[src], kBloomList);
    bool over = false;
    for (int i = lane; i < nsrc; i += 32) {
      int m1;
      if (k == 2) {
        const int2 sl = slot_np(c, 0, c.wui.a + i);
        m1 = sl.x;
        if (m1 == c.u || m1 == c.v || !first_of(c, sl)) continue;
      } else {
        m1 = lists[src][i];
      }
      const Win w = window(c, 0, m1);
      for (int q = w.a; q < w.b; ++q) {
        const int2 s2 = slot_np(c, 0, q);
        const int m2 = s2.x;
        if (m2 == c.u || m2 == c.v || !first_of(c, s2)) continue;
        const uint32_t b = bloom_bit(m2);
        atomicOr(&B.w[k - 2][b >> 5], 1u << (b & 31));
        const int idx = atomicAdd(&B.n[dst], 1);
        if (idx < kBloomList) lists[dst][idx] = m2;
        else over = true, TM_CNT(kCtrBloomOver, 1);
      }
    }
    over = __any_sync(0xffffffffu, over);
    __syncwarp();
    if (lane == 0) {
      B.valid |= 1 << (k - 2);  // B_k itself is complete (its bits are all set)
      B.n[src] = 0;             // the list just consumed becomes the next output
    }
    __syncwarp();
    if (over) break;  // B_k's member list is incomplete: no deeper layer
  }
}

// ---------------------------------------------------------------- TMA staging
// TM_TMA_TASKS=1 (A/B of the north star's "shared-memory staging of hub
// adjacency"): a domain task's piece of the hub window (<= kTaskSpan (nbr,
// prev) entries) is brought into the warp's shared buffer by one
// cp.async.bulk (TMA bulk copy, mbarrier completion) issued by lane 0, and
// the lanes walk it from shared memory instead of one coalesced global load
// per 32 entries.
#ifndef TM_TMA_TASKS
#define TM_TMA_TASKS 0
#endif
constexpr int kStageEntries = kTaskSpan + 2;  // + even alignment of the start
__device__ __forceinline__ uint32_t smem_addr(const void *p) {
  return (uint32_t)__cvta_generic_to_shared(p);
}
__device__ __forceinline__ void mbar_init(uint64_t *bar) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;\n" ::"r"(smem_addr(bar)));
  asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
}
// lane 0: arm the barrier with the byte count and start the bulk copy
__device__ __forceinline__ void bulk_load(void *dst, const void *src, uint32_t bytes, uint64_t *bar) {
  asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");  // earlier generic reads of dst
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(smem_addr(bar)), "r"(bytes)
               : "memory");
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];\n" ::"r"(
          smem_addr(dst)),
      "l"(src), "r"(bytes), "r"(smem_addr(bar))
      : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t *bar, uint32_t phase) {
  asm volatile(
      "{\n .reg .pred p;\n"
      "TM_WAIT_%=:\n mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
      " @!p bra TM_WAIT_%=;\n}\n" ::"r"(smem_addr(bar)),
      "r"(phase)
      : "memory");
}

// Task kinds (one warp per task):
//   kLvlDomU / kLvlDomV   a piece of a trigger's U / V slice, lane per entry
//   kLvlPullV             a hub v's whole N+(v): gs from u's side (pull_gs),
//                         cycles through the useful a1 only (the depth-1
//                         backward sets), each probed for v -> a1 — declined
//                         parts go back to the queue as domain V tasks
//   level | kPullFlag     a wide chain node's whole window: its useful
//                         nodes, or chain tasks for the next round
//   level 1..4            a piece of a chain node's window
// Each kind feeds ONE call site of the item / chain code below.
// MODE 0: every task kind, chain descents inline (calls without deferral
// and the rescue pass); MODE 1: the item kinds (domain U / V, pull-V) with
// their chain descents deferred to records (no chain code in this kernel:
// fewer registers, no Bloom build); MODE 2: the chain kinds only.
template <int MODE, bool ONE = false>
__global__ void __launch_bounds__(kTaskThreads, TM_TASK_MINB) k_mine_tasks(
    const __grid_constant__ DevGraph g, const __grid_constant__ DevPlans P, int64_t lo,
    long long *__restrict__ out, int32_t *__restrict__ scratch, Queue in, Queue next_q,
    int32_t *__restrict__ bloom_lists, const int4 *__restrict__ split_win,
    const unsigned int *__restrict__ gate) {
  if (gate && *(volatile const unsigned int *)gate == 0) return;
  const int n = (int)min(*in.count, (unsigned long long)in.cap);
  const int warps = gridDim.x * (blockDim.x >> 5);
  const int lane = threadIdx.x & 31;
  __shared__ TaskBloom blooms[kTaskThreads / 32];
  TaskBloom &bloom = blooms[threadIdx.x >> 5];
#if TM_TMA_TASKS
  __shared__ __align__(128) int2 stage_np[kTaskThreads / 32][kStageEntries];
  __shared__ __align__(8) uint64_t stage_bar[kTaskThreads / 32];
  int2 *sbuf = stage_np[threadIdx.x >> 5];
  uint64_t *sbar = &stage_bar[threadIdx.x >> 5];
  uint32_t sphase = 0;
  if (lane == 0) mbar_init(sbar);
  __syncwarp();
#endif
  const int gwarp = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  int *blist0 = bloom_lists + (size_t)gwarp * 2 * kBloomList, *blist1 = blist0 + kBloomList;
  for (int i = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5); i < n; i += warps) {
    const Task t = in.q[i];
    if (t.row < 0) continue;
    const bool item_task = t.level == kLvlDomU || t.level == kLvlDomV || t.level == kLvlPullV;
    if ((MODE == 1 && !item_task) || (MODE == 2 && item_task)) continue;
    const int e = (int)(lo + t.row);
    const DevGroup &gr = P.gr[ONE ? 0 : t.grp];
    const uint32_t r = __ldg(g.e_rank + e);
    Ctx c{gr.view, __ldg(g.e_src + e), __ldg(g.e_dst + e), __ldg(gr.lo_tab + r), r, {}, {}, {}, {},
          (int64_t)slab_of(gr, r) * gr.stride};
    if (item_task && t.path[0] >= 0) {  // a split row: the trigger kernel stored its windows
      const int4 w0 = __ldg(split_win + 2 * t.path[0]), w1 = __ldg(split_win + 2 * t.path[0] + 1);
      c.wui = Win{w0.x, w0.y};
      c.wuo = Win{w0.z, w0.w};
      c.wvi = Win{w1.x, w1.y};
      c.wvo = Win{w1.z, w1.w};
    } else if (!item_task) {  // chain tasks close into u's in-window only
      c.wui = window(c, 0, c.u);
    } else {
      trigger_windows(c, gr, t.row);
    }
    // chain walks of this task get the trigger's backward-layer filters
    Queue next = next_q;
    const bool chains = MODE != 1 && t.level != kLvlDomU && !(t.level == kLvlDomV && !(t.pad0 & kVCyc));
    // (narrow windows are cheaper to walk than the filters are to build)
    if (chains && gr.cyc.maxd >= 2 && c.u != c.v && c.wui.len() > 0 && t.b - t.a > kBloomMin) {
      // layers up to the one a depth-1 node needs for the deepest close
      build_bloom(c, bloom, lane, 1 + gr.cyc.maxd, blist0, blist1);
      next.bloom = &bloom;
    }
    long long *orow = out + (int64_t)t.row * P.n;
    int use[kBCap];
    if constexpr (MODE != 2) {
    if (t.level == kLvlDomU) {
      GlobalSink sk{orow, scratch + 3 * (t.path[0] >= 0 ? t.path[0] : 0)};
#if TM_TMA_TASKS
      const int a2 = t.a & ~1;
      __syncwarp();  // every lane is done with the previous piece
      if (lane == 0)
        bulk_load(sbuf, c.g.np[0] + a2, (uint32_t)(((t.b - a2) * 8 + 15) & ~15), sbar);
      mbar_wait(sbar, sphase);
      sphase ^= 1;
      for (int j = t.a + lane; j < t.b; j += 32) u_item_sl(c, P, gr, sbuf[j - a2], sk);
#else
      for (int j = t.a + lane; j < t.b; j += 32) u_item(c, P, gr, j, sk);
#endif
    } else if (t.level == kLvlDomV || t.level == kLvlPullV) {
      GlobalSink sk{orow, scratch + 3 * (t.path[0] >= 0 ? t.path[0] : 0)};
      int parts = t.pad0, ja = t.a, jb = t.b;
      const int *cand = nullptr;
      const int vs = __ldg(g.gptr[1] + c.v), ve = __ldg(g.gptr[1] + c.v + 1);  // v's pair-index run
      if (t.level == kLvlPullV) {
        int redo = 0;
        parts = 0;
        if (gr.n_gs > 0 && !pull_gs(c, P, gr, vs, ve, lane, orow)) redo |= kVGs;
        const CycGroup &cg = gr.cyc;
        if (cg.maxd >= 1 && c.u != c.v && c.wui.len() > 0) {
          const int nu = useful_nodes(c.g, c.soff, c.u, c.v, c.lo, c.hi, c.wui.a, c.wui.b, cg.mask, cg.maxd, 1,
                                      use);
          if (nu < 0 || nu * 4 > t.b - t.a) {
            redo |= kVCyc;
          } else {
            cand = use;
            ja = 0;
            jb = nu;
            parts = kVCyc;
          }
        }
        if (redo) {
          bool ok = false;
          // with filters built, a moderate window is walked here rather than
          // rebuilding the filters in every domain task; wide ones are split
          if (lane == 0 && !(next.bloom && (redo & kVCyc) && t.b - t.a <= kInPlace))
            ok = emit(next, t.row, t.grp, kLvlDomV, t.path[0], -1, -1, -1, -1, t.a, t.b, redo);
          if (!__shfl_sync(0xffffffffu, ok, 0)) {  // queue full: this warp walks the declined parts too
            if (cand) {
              for (int j = t.a + lane; j < t.b; j += 32) {
                const int m = __ldg(c.g.np[1] + j).x;
                if (m == c.u || m == c.v || !first_in_window(c, 1, j)) continue;
                if (redo & kVGs) v_node<true, GlobalSink, MODE == 1>(c, P, gr, t.grp, t.row, m, sk, next, kVGs);
              }
            } else {
              parts = redo;
            }
          }
        }
        if (!parts) ja = jb = 0;
      }
#if TM_TMA_TASKS
      const int a2 = ja & ~1;
      const bool staged = !cand && jb > ja && jb - a2 <= kStageEntries;
      if (staged) {
        __syncwarp();
        if (lane == 0) bulk_load(sbuf, c.g.np[1] + a2, (uint32_t)(((jb - a2) * 8 + 15) & ~15), sbar);
        mbar_wait(sbar, sphase);
        sphase ^= 1;
      }
#endif
      for (int k = ja + lane; k < jb; k += 32) {
        int m;
        if (cand) {
          m = cand[k];
          if (m == c.u || m == c.v || !exists_hub(c, 1, c.v, vs, ve, m)) continue;
        } else {
#if TM_TMA_TASKS
          const int2 sl = staged ? sbuf[k - a2] : slot_np(c, 1, k);
#else
          const int2 sl = slot_np(c, 1, k);
#endif
          m = sl.x;
          if (m == c.u || m == c.v || !first_of(c, sl)) continue;
        }
        v_node<true, GlobalSink, MODE == 1>(c, P, gr, t.grp, t.row, m, sk, next, parts);
      }
    }
    }  // MODE != 2
    if constexpr (MODE != 1) {
    if (!item_task) {  // a chain node's window (or its useful nodes)
      CycAcc acc;
#pragma unroll
      for (int k = 0; k < kMaxCyc; ++k) acc.e[k] = 0;
      const int L = t.level & 7;
      const int path[kMaxChain] = {t.path[0], t.path[1], t.path[2], t.path[3], t.path[4]};
      int ja = t.a, jb = t.b;
      const int *cand = nullptr;
      if (t.level & kPullFlag) {
        const Win w{t.a, t.b};
        if (pull_candidates(c, gr.cyc, gr.cyc.maxd, L + 1, w, use, ja, jb)) {
          cand = use;
        } else {
          bool ok = false;
          if (lane == 0 && !(next.bloom && t.b - t.a <= kInPlace))
            ok = emit(next, t.row, t.grp, L, path[0], path[1], path[2], path[3], path[4], t.a, t.b);
          // split into chain tasks for the next round, or (filters built) walk the window here
          if (__shfl_sync(0xffffffffu, ok, 0)) ja = jb = 0;
        }
      }
      for (int k = ja + lane; k < jb; k += 32)  // one entry per lane per step
        cycles_resume(c, gr.cyc, t.row, t.grp, L, path, k, k + 1, cand, acc, next);
#pragma unroll
      for (int k = 0; k < kMaxCyc; ++k) {
        const long long sum = warp_sum(acc.e[k]);
        if (lane == 0 && k < gr.cyc.n && sum)
          atomicAdd(reinterpret_cast<unsigned long long *>(orow + gr.cyc.col[k]), (unsigned long long)sum);
      }
    }
    }  // MODE != 1
  }
}

// deferred chain descents (push_chain), one record per thread: the trigger's
// context is rebuilt (u's in-window closes every chain), chains a2.. below
// a1 are enumerated with the task-kernel semantics (wide nodes: pull
// candidates or chain tasks for the rounds that follow), counts are added
// to the trigger's row
template <bool ONE = false>
__global__ void __launch_bounds__(256) k_mine_chains(const __grid_constant__ DevGraph g,
                                                     const __grid_constant__ DevPlans P, int64_t lo,
                                                     long long *__restrict__ out, ChainQ cq, Queue qu) {
  const unsigned long long n = min(*cq.count, cq.cap);
  for (unsigned long long i = (unsigned long long)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (unsigned long long)gridDim.x * blockDim.x) {
    const ChainRec rc = cq.rec[i];
    const DevGroup &gr = P.gr[ONE ? 0 : rc.grp];
    const int e = (int)(lo + rc.row);
    const uint32_t r = __ldg(g.e_rank + e);
    uint32_t wlo;
    int slab;
    if (gr.lo_slab) {
      const int2 ls = __ldg(gr.lo_slab + rc.row);
      wlo = (uint32_t)ls.x;
      slab = ls.y;
    } else {
      wlo = __ldg(gr.lo_tab + r);
      slab = slab_of(gr, r);
    }
    Ctx c{gr.view, __ldg(g.e_src + e), __ldg(g.e_dst + e), wlo, r, {}, {}, {}, {}, (int64_t)slab * gr.stride};
    c.wui = Win{rc.ua, rc.ub};
    CycAcc acc;
#pragma unroll
    for (int k = 0; k < kMaxCyc; ++k) acc.e[k] = 0;
    int path[kMaxChain] = {rc.a1, -1, -1, -1, -1};
    chain_level<1, true>(c, gr.cyc, rc.row, rc.grp, path, rc.wa, rc.wb, nullptr, acc, qu);
    long long *orow = out + (int64_t)rc.row * P.n;
#pragma unroll
    for (int k = 0; k < kMaxCyc; ++k)
      if (k < gr.cyc.n && acc.e[k])
        atomicAdd(reinterpret_cast<unsigned long long *>(orow + gr.cyc.col[k]), (unsigned long long)acc.e[k]);
  }
}

// rows whose slices went to domain tasks: whole-count columns from scratch
__global__ void k_mine_finalize(const __grid_constant__ DevPlans P, long long *__restrict__ out,
                                const int32_t *__restrict__ split_rows,
                                const int32_t *__restrict__ split_n, const int32_t *__restrict__ scratch,
                                int32_t split_cap, const unsigned int *__restrict__ gate) {
  if (gate && *(volatile const unsigned int *)gate == 0) return;
  const int n = min(*split_n, split_cap);
  for (int s = blockIdx.x * blockDim.x + threadIdx.x; s < n; s += gridDim.x * blockDim.x) {
    const int row = split_rows[2 * s], gi = split_rows[2 * s + 1];
    const long long a = scratch[3 * s], d = scratch[3 * s + 1], c3 = scratch[3 * s + 2];
    const DevGroup &gr = P.gr[gi];
    long long *orow = out + (int64_t)row * P.n;
    for (int i = 0; i < gr.ncols; ++i) {
      const int ci = gr.cols[i];
      const DevPlan &p = P.p[ci];
      if (p.family == TM_STACK)
        orow[ci] = (a > 0 && d > 0 && a >= p.min_size && d >= p.min_size) ? a * d : 0;
      else if (p.family == TM_CYCLE && p.cycle_len == 3)
        orow[ci] = c3 >= p.min_size ? c3 : 0;
    }
  }
}

// per trigger row: (lo_tab[rank], slab of rank) — one coalesced 8-byte read
// in the trigger kernel instead of two loads that wait for e_rank
__global__ void k_lo_slab(const uint32_t *__restrict__ e_rank, int64_t lo, int64_t rows,
                          const uint32_t *__restrict__ lo_tab, const uint16_t *__restrict__ slab_of,
                          int2 *__restrict__ out) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= rows) return;
  const uint32_t r = __ldg(e_rank + lo + i);
  out[i] = make_int2((int)__ldg(lo_tab + r), slab_of ? (int)__ldg(slab_of + r) : 0);
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

// own-window table of CSR direction dir: slot p of owner x (edge e = eid[p])
// is inside x's window at e's own time, so that window's lower bound is
// searched in [a, p] only and its upper bound galloped forward from p.
// Consecutive slots share their search paths (one run, nearby targets), so
// the bisections of a hub run are L1 broadcasts instead of the dependent
// DRAM chains the trigger would otherwise walk.  Written by edge id: the
// trigger kernels read it coalesced.
__global__ void k_own_windows(const __grid_constant__ DevGraph g, const uint32_t *__restrict__ lo_tab,
                              int dir, int64_t lo, int64_t hi, int2 *__restrict__ tab) {
  const int64_t p = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (p >= g.n_edges) return;
  const int e = __ldg(g.eid[dir] + p);
  if (e < lo || e >= hi) return;
  const int x = __ldg(g.owner[dir] + p);  // coalesced (was a gather through the edge table)
  const int a = __ldg(g.ptr[dir] + x), b = __ldg(g.ptr[dir] + x + 1);
  const uint32_t *rk = g.rnk[dir];
  const uint32_t r = __ldg(rk + p);
  const int lb = lb_u32(rk, a, (int)p, __ldg(lo_tab + r));
  tab[e - lo] = make_int2(lb, ub_gallop(rk, (int)p + 1, b, r));
}

// the same tables in a slab view: slot p's copy in its own slab sits at
// sptr[s][x] + (p - start[s][x]); the window is searched inside that short
// slab run (tm_slab.cu)
__global__ void k_own_windows_slab(const __grid_constant__ DevGraph g, const uint32_t *__restrict__ lo_tab,
                                   int dir, int64_t lo, int64_t hi, const uint16_t *__restrict__ slab_of,
                                   int64_t stride, const int32_t *__restrict__ start,
                                   const int32_t *__restrict__ sptr, const uint32_t *__restrict__ srnk,
                                   int2 *__restrict__ tab) {
  const int64_t p = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (p >= g.n_edges) return;
  const int e = __ldg(g.eid[dir] + p);
  if (e < lo || e >= hi) return;
  const int x = __ldg(g.owner[dir] + p);
  const uint32_t r = __ldg(g.rnk[dir] + p);
  const int64_t cell = (int64_t)__ldg(slab_of + r) * stride + x;
  const int a = __ldg(sptr + cell), b = __ldg(sptr + cell + 1);
  const int q = a + (int)(p - __ldg(start + cell));
  const int lb = lb_u32(srnk, a, q, __ldg(lo_tab + r));
  tab[e - lo] = make_int2(lb, ub_gallop(srnk, q + 1, b, r));
}

}  // namespace
}  // namespace tmb

using namespace tmb;

#ifndef TM_LOSLAB
#define TM_LOSLAB 1
#endif

// TM_SPLIT_TASKS=1: item / chain task kernels with deferral at any size (tests)
static bool split_tasks_forced() {
  static bool on = [] {
    const char *e = getenv("TM_SPLIT_TASKS");
    return e && e[0] == '1';
  }();
  return on;
}

// TM_DEFER=0: the trigger kernel enumerates chain descents inline (A/B)
static bool defer_chains_enabled() {
  static bool on = [] {
    const char *e = getenv("TM_DEFER");
    return !(e && e[0] == '0');
  }();
  return on;
}

// TM_ORDER=1 processes full-range calls in out-CSR (source) order; measured
// neutral (HI-Small -3%, HI-Medium +2%), so edge-id order stays the default
static bool source_order() {
  static bool on = [] {
    const char *e = getenv("TM_ORDER");
    return e && e[0] == '1';
  }();
  return on;
}

// TM_OWN=0 turns the own-window tables off (A/B)
static bool own_windows_enabled() {
  static bool on = [] {
    const char *e = getenv("TM_OWN");
    return !(e && e[0] == '0');
  }();
  return on;
}

// TM_OWN=2 also builds own-window tables in slab views (A/B)
static bool own_in_slabs() {
  static bool on = [] {
    const char *e = getenv("TM_OWN");
    return e && e[0] == '2';
  }();
  return on;
}

static int mine_impl(tm_graph *g, const tm_plan_desc *plans, int n_plans, int64_t lo, int64_t hi,
                     int64_t *out, int out_on_device, void *stream, bool allow_defer);

extern "C" int tm_mine(tm_graph *g, const tm_plan_desc *plans, int n_plans, int64_t lo, int64_t hi,
                       int64_t *out, int out_on_device, void *stream) {
  return mine_impl(g, plans, n_plans, lo, hi, out, out_on_device, stream, true);
}

static int mine_impl(tm_graph *g, const tm_plan_desc *plans, int n_plans, int64_t lo, int64_t hi,
                     int64_t *out, int out_on_device, void *stream, bool allow_defer) {
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
  g->last.light_ms = g->last.heavy_ms = g->last.total_ms = g->last.prep_ms = -1.f;
  if (rows == 0 || n_plans == 0) return TM_OK;
  TM_CUDA(cudaSetDevice(g->device));
  cudaStream_t s = stream ? static_cast<cudaStream_t>(stream) : g->stream;
  TM_CUDA(g->begin(s));  // the shared scratch below may still be in use by the previous call
  const int64_t launches0 = tm_kernel_launch_count();

  // delta groups (one window set + one lower-bound table per distinct delta)
  DevPlans dp{};
  dp.n = n_plans;
  int64_t deltas[kMaxGroups];
  for (int i = 0; i < n_plans; ++i) {
    // same delta -> same group, unless its cycle enumeration is full
    const bool cyc = plans[i].family == TM_CYCLE && plans[i].cycle_len >= 3;
    int k = 0;
    while (k < dp.ngroups && (deltas[k] != plans[i].delta || (cyc && dp.gr[k].cyc.n == kMaxCyc))) ++k;
    if (k == dp.ngroups) {
      if (dp.ngroups == kMaxGroups)
        return fail(TM_E_UNSUPPORTED_PLAN, "more than " + std::to_string(kMaxGroups) +
                                               " column groups (distinct deltas, or > " +
                                               std::to_string(kMaxCyc) +
                                               " cycle columns per delta) in one tm_mine call");
      deltas[dp.ngroups++] = plans[i].delta;
    }
    const tm_plan_desc &p = plans[i];
    dp.p[i] = DevPlan{p.family, p.endpoint, p.direction, p.exclude_trigger, p.cycle_len, p.min_size, k};
    DevGroup &gr = dp.gr[k];
    gr.cols[gr.ncols++] = (int8_t)i;
    {
      const int packed = i | p.endpoint << 10 | p.direction << 11 | (p.exclude_trigger ? 1 : 0) << 12;
      if (p.family == TM_FAN || p.family == TM_DEGREE || (p.family == TM_CYCLE && p.cycle_len == 2)) {
        gr.lane_d[gr.n_lane] = packed | (p.family == TM_CYCLE ? kLaneCyc2 : 0);
        gr.lane_k[gr.n_lane++] = p.min_size;
      } else if (p.family == TM_STACK || (p.family == TM_CYCLE && p.cycle_len == 3)) {
        gr.end_d[gr.n_end] = packed | (p.family == TM_STACK ? kLaneStack : 0);
        gr.end_k[gr.n_end++] = p.min_size;
      }
    }
    switch (p.family) {
      case TM_FAN:
      case TM_DEGREE: gr.need |= 1 << (2 * p.endpoint + p.direction); break;
      case TM_CYCLE:
        gr.need |= p.cycle_len == 2 ? 8 : (1 | 8);
        if (p.cycle_len >= 3) {
          CycGroup &cg = gr.cyc;
          const int d = p.cycle_len - 3;
          cg.depth[cg.n] = (int8_t)d;
          cg.k[cg.n] = p.min_size;
          cg.col[cg.n] = (int8_t)i;
          cg.n++;
          cg.mask |= 1 << d;
          cg.maxd = std::max(cg.maxd, d);
          if (d == 0) gr.udom = 1; else gr.vdom = 1;
        }
        break;
      case TM_SG: gr.need |= 1 | 4; gr.udom = 1; gr.sg_col[gr.n_sg++] = (int8_t)i; break;
      case TM_GS: gr.need |= 8 | 2; gr.vdom = 1; gr.gs_col[gr.n_gs++] = (int8_t)i; break;
      case TM_STACK: gr.need |= 1 | 8; gr.udom = gr.vdom = 1; gr.has_stack = 1; break;
      default: break;
    }
  }
  const int64_t R = g->n_ranks;
  int rc;
  if (g->prof) TM_CUDA(cudaEventRecord(g->ev[3], s));
  if ((rc = g->lo_tabs.ensure_pooled(sizeof(uint32_t) * (size_t)(R > 0 ? R : 1) * dp.ngroups, s, g->stream))) return rc;
  // own-window tables pay off when a group needs them for many triggers
  const int64_t E = g->n_edges;
  const bool own_on = own_windows_enabled() && rows * 64 >= E;
  int n_own = 0;
  if (own_on)
    for (int k = 0; k < dp.ngroups; ++k) n_own += ((dp.gr[k].need >> 1) & 1) + ((dp.gr[k].need >> 2) & 1);
  if (n_own && (rc = g->own_tabs.ensure_pooled(sizeof(int2) * (size_t)rows * n_own, s, g->stream))) return rc;
#if TM_LOSLAB
  if ((rc = g->lo_slab.ensure_pooled(sizeof(int2) * (size_t)rows * dp.ngroups, s, g->stream))) return rc;
#endif
  const DevGraph dg = g->dev();
  int rounds = 0;
  int own_i = 0;
  const PreparedViews &pv = g->prep;
  const bool prepared = pv.valid && lo >= pv.lo && hi <= pv.hi;
  for (int k = 0; k < dp.ngroups; ++k) {
    int pi = -1;  // the prepared tables of this delta (tm_mine_prepare), if any
    for (int i = 0; prepared && i < pv.n; ++i)
      if (pv.delta[i] == deltas[k]) pi = i;
    if (pi >= 0) {
      dp.gr[k].lo_tab = pv.lo_tabs.as<uint32_t>() + (size_t)pi * R;
      dp.gr[k].view = pv.view[pi];
      dp.gr[k].slab_of = pv.slab_of[pi];
      dp.gr[k].stride = pv.stride[pi];
    } else {
      dp.gr[k].lo_tab = g->lo_tabs.as<uint32_t>() + (size_t)k * R;
      k_lo_table<<<grid_for(R, 256), 256, 0, s>>>(g->uniq_time.as<int64_t>(), R, deltas[k],
                                                  g->lo_tabs.as<uint32_t>() + (size_t)k * R);
      TM_LAUNCHED("k_lo_table");
    }
    // the group's view of the graph: time slabs when the call covers a good
    // share of the edges (the view costs O(E + n_slabs N) to build)
    if (pi >= 0) {
      // prepared
    } else if (rows * 16 >= E) {
      if ((rc = build_slab_view(g, g->slabs[k], deltas[k], dp.gr[k].lo_tab, s, lo, hi, false, &dp.gr[k].view,
                                &dp.gr[k].slab_of, &dp.gr[k].stride)))
        return rc;
    } else {
      dp.gr[k].view = dg;
      dp.gr[k].slab_of = nullptr;
      dp.gr[k].stride = 0;
    }
    // own-window tables: global view only — in a slab view the windows are
    // short bisections of L2-resident runs, cheaper than the table passes
    // (HI-Large: 131 vs 145 ms per step, TM_OWN A/B)
    const bool own_here = own_on && (!dp.gr[k].slab_of || own_in_slabs());
    for (int dir = 0; dir < 2 && own_here; ++dir) {
      if (!((dp.gr[k].need >> (dir ? 1 : 2)) & 1)) continue;
      int2 *tab = g->own_tabs.as<int2>() + (size_t)rows * own_i++;
      if (dp.gr[k].slab_of) {
        const DevGraph &v = dp.gr[k].view;
        const SlabIndex &si = pi >= 0 ? pv.slabs[pi] : g->slabs[k];
        k_own_windows_slab<<<grid_for(E, 256), 256, 0, s>>>(
            dg, dp.gr[k].lo_tab, dir, lo, hi, dp.gr[k].slab_of, dp.gr[k].stride,
            si.start[dir].as<int32_t>() - (int64_t)si.s0 * dp.gr[k].stride, v.ptr[dir], v.rnk[dir], tab);
        TM_LAUNCHED("k_own_windows_slab");
      } else {
        k_own_windows<<<grid_for(E, 256), 256, 0, s>>>(dg, dp.gr[k].lo_tab, dir, lo, hi, tab);
        TM_LAUNCHED("k_own_windows");
      }
      dp.gr[k].own[dir] = tab;
    }
#if TM_LOSLAB
    {
      int2 *ls = g->lo_slab.as<int2>() + (size_t)rows * k;
      k_lo_slab<<<grid_for(rows, 256), 256, 0, s>>>(g->e_rank.as<uint32_t>(), lo, rows, dp.gr[k].lo_tab,
                                                     dp.gr[k].slab_of, ls);
      TM_LAUNCHED("k_lo_slab");
      dp.gr[k].lo_slab = ls;
    }
#endif
    // Hand-off width for chain nodes: with short windows (mean windowed
    // degree <= 2) backward pruning in the task kernel wins for any node
    // wider than kDeepSplit; with long windows nearly every node is that
    // wide and the per-task overhead dominates, so only hubs (> 64) leave.
    {
      const double mean_w = (double)g->n_edges / (double)std::max<int64_t>(g->n_nodes, 1) *
                            (double)deltas[k] / (double)std::max<int64_t>(g->t_span, 1);
      dp.gr[k].cyc.deep_split = mean_w <= 2.0 ? kDeepSplit : 64;
    }
    // task rounds: domain tasks, then one per chain level below a1
    if (dp.gr[k].udom || dp.gr[k].vdom)
      rounds = std::max(rounds, 3 + std::max(0, dp.gr[k].cyc.maxd - 1));  // + 2: declined pull tasks
  }

  long long *d_out;
  if (out_on_device) {
    d_out = reinterpret_cast<long long *>(out);
  } else {
    if ((rc = g->out_scratch.ensure_pooled(sizeof(long long) * (size_t)rows * n_plans, s, g->stream))) return rc;
    d_out = g->out_scratch.as<long long>();
  }
#ifdef TM_TASK_CAP  // tiny-cap test builds: queue-full / split-slot fallbacks
  const int64_t task_cap = TM_TASK_CAP;
#else
  const int64_t task_cap = std::min<int64_t>(std::max<int64_t>(1 << 18, rows / 8), 1 << 24);
#endif
#ifdef TM_SPLIT_CAP
  const int64_t split_cap = TM_SPLIT_CAP;
#else
  const int64_t split_cap = std::min<int64_t>(std::max<int64_t>(1 << 16, rows / 16), 1 << 22);
#endif
  if ((rc = g->heavy_n.ensure_pooled(sizeof(unsigned long long) * 6, s, g->stream)) ||
      (rc = g->heavy_q.ensure_pooled(sizeof(int32_t) * 2 * (size_t)split_cap, s, g->stream)) ||
      (rc = g->split_scratch.ensure_pooled(sizeof(int32_t) * 3 * (size_t)split_cap, s, g->stream)) ||
      (rc = g->split_win.ensure_pooled(sizeof(int4) * 2 * (size_t)split_cap, s, g->stream)) ||
      (rc = g->tasks.ensure_pooled(sizeof(Task) * (size_t)task_cap * 2, s, g->stream)))
    return rc;
  // [0] split rows (int32 in the low word), [1] [2] task queues A / B
  unsigned long long *cnt64 = g->heavy_n.as<unsigned long long>();
  int32_t *cnt = reinterpret_cast<int32_t *>(cnt64);
  // [4] (low word): overflow of the deferred chain descents, for the whole call
  unsigned int *overflow = reinterpret_cast<unsigned int *>(cnt64 + 4);
  TM_CUDA(cudaMemsetAsync(cnt64, 0, sizeof(unsigned long long) * 6, s));
  Queue qa{g->tasks.as<Task>(), cnt64 + 1, (int32_t)task_cap, nullptr, ChainQ{}};
  Queue qb{g->tasks.as<Task>() + task_cap, cnt64 + 2, (int32_t)task_cap, nullptr, ChainQ{}};
  // [3] deferred chain descents of the trigger kernel (k_mine_chains)
  // Deferral pays for short windows, where a1's window is a few entries and
  // records are fewer than triggers; with long windows (mean windowed degree
  // > 2, the deep_split switch above) nearly every V item would become a
  // record and the queue would overflow into the rescue pass, so the
  // trigger kernel enumerates inline there.
  bool any_chains = false, long_windows = false;
  for (int k = 0; k < dp.ngroups; ++k) {
    any_chains |= dp.gr[k].cyc.maxd >= 2;
    long_windows |= dp.gr[k].cyc.maxd >= 2 && dp.gr[k].cyc.deep_split != kDeepSplit;
  }
  ChainQ cq{};
  if (any_chains && !long_windows && allow_defer && defer_chains_enabled()) {
#ifdef TM_CHAIN_CAP  // tiny-cap test builds: the overflow -> inline rescue path
    const int64_t chain_cap = TM_CHAIN_CAP;
#else
    const int64_t chain_cap = std::max<int64_t>(1 << 20, rows);
#endif
    if ((rc = g->chain_q.ensure_pooled(sizeof(ChainRec) * (size_t)chain_cap, s, g->stream))) return rc;
    cq = ChainQ{g->chain_q.as<ChainRec>(), cnt64 + 3, (unsigned long long)chain_cap, overflow};
  }

  for (int i = 0; i < n_plans; ++i) {
    const int f = plans[i].family;
    const bool staged = f == TM_SG || f == TM_GS || (f == TM_CYCLE && plans[i].cycle_len >= 4);
    dp.slot[i] = (int8_t)(staged ? dp.n_stage : -1);
    if (staged) dp.slot_col[dp.n_stage++] = (int8_t)i;
  }
  const size_t smem = sizeof(long long) * kThreads * std::max(dp.n_stage, 1);
  // one delta group (the common case): kernel instances with P.gr[0] fixed
  const bool one_group = TM_ONE_GROUP && dp.ngroups == 1;
  if (smem > 48 * 1024)
    for (const void *kf : {(const void *)k_mine_warp<true, false>, (const void *)k_mine_warp<true, true>,
                           (const void *)k_mine_warp<false, false>})
      TM_CUDA(cudaFuncSetAttribute(kf, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  // TM_CARVEOUT=pct: preferred shared-memory share of the L1/shared array
  // for the mining kernels (A/B: the walkers' loads are L1-cached)
  if (const char *co = getenv("TM_CARVEOUT")) {
    const int pct = atoi(co);
    TM_CUDA(cudaFuncSetAttribute(k_mine_warp<true, false>, cudaFuncAttributePreferredSharedMemoryCarveout, pct));
    TM_CUDA(cudaFuncSetAttribute(k_mine_warp<true, true>, cudaFuncAttributePreferredSharedMemoryCarveout, pct));
    TM_CUDA(cudaFuncSetAttribute(k_mine_warp<false, false>, cudaFuncAttributePreferredSharedMemoryCarveout, pct));
    for (const void *kf : {(const void *)k_mine_tasks<0>, (const void *)k_mine_tasks<1>, (const void *)k_mine_tasks<2>,
                           (const void *)k_mine_tasks<1, true>, (const void *)k_mine_tasks<2, true>})
      TM_CUDA(cudaFuncSetAttribute(kf, cudaFuncAttributePreferredSharedMemoryCarveout, pct));
  }
  // Host output: mine the range in pieces and copy each finished piece back
  // on a copy stream while the next piece is mined — the D2H of the int64
  // block (8*C bytes per trigger over PCIe) is the largest end-to-end cost.
  // Only for page-locked output: a D2H into pageable memory blocks the host
  // thread, which would serialize the pieces instead of overlapping them.
  bool pinned = false;
  if (!out_on_device) {
    cudaPointerAttributes pa{};
    pinned = cudaPointerGetAttributes(&pa, out) == cudaSuccess && pa.type == cudaMemoryTypeHost;
    cudaGetLastError();
  }
  const int pieces = (pinned && rows >= (1 << 20)) ? kHostPieces : 1;
  if (pieces > 1 && !g->copy_stream) {
    TM_CUDA(cudaStreamCreateWithFlags(&g->copy_stream, cudaStreamNonBlocking));
    for (int i = 0; i < kHostPieces; ++i)
      TM_CUDA(cudaEventCreateWithFlags(&g->piece_ev[i], cudaEventDisableTiming));
  }
  const int task_grid = 148 * (2048 / kTaskThreads);
  if ((rc = g->bloom_lists.ensure_pooled(sizeof(int32_t) * 2 * kBloomList * (size_t)task_grid * (kTaskThreads / 32),
                                         s, g->stream)))
    return rc;
  if ((rc = g->split_counts.ensure_pooled(sizeof(int32_t) * kHostPieces, s, g->stream))) return rc;
  int32_t *piece_split = g->split_counts.as<int32_t>();
  g->prof_pending = g->prof;
  if (g->prof) TM_CUDA(cudaEventRecord(g->ev[0], s));
  const int64_t per = (rows + pieces - 1) / pieces;
  // one pass over piece pc: the trigger kernel (deferring chain descents when
  // cq is set), the deferred descents, the task rounds, the split-row
  // finalize.  gate != null: a rescue pass that runs only if the deferred
  // pass overflowed (*gate != 0), recomputing every row inline.
  auto run_piece = [&](int pc, bool defer, const unsigned int *gate) -> int {
    const int64_t r0 = std::min<int64_t>(rows, pc * per), r1 = std::min<int64_t>(rows, r0 + per);
    long long *po = d_out + r0 * n_plans;
    Queue a = qa, b = qb;
    DevPlans dpp = dp;  // own-window tables are indexed relative to the piece
    for (int k = 0; k < dpp.ngroups; ++k) {
      for (int d = 0; d < 2; ++d)
        if (dpp.gr[k].own[d]) dpp.gr[k].own[d] += r0;
      if (dpp.gr[k].lo_slab) dpp.gr[k].lo_slab += r0;
    }
    TM_CUDA(cudaMemsetAsync(cnt64, 0, sizeof(unsigned long long) * 4, s));
    // full-range device-output calls: triggers in time order when the edge
    // ids are not (slab views are then read slab by slab), or out-CSR order
    // (TM_ORDER=1 A/B); rows are always written by edge id
    const bool full = pieces == 1 && lo == 0 && hi == g->n_edges;
    bool any_slabs = false;
    for (int k = 0; k < dp.ngroups; ++k) any_slabs |= dp.gr[k].slab_of != nullptr;
    const int32_t *order = !full ? nullptr
                           : source_order() ? g->eid[1].as<int32_t>()
                           : (any_slabs && !g->ids_time_ordered) ? g->time_order.as<int32_t>()
                                                                 : nullptr;
    if (defer) {
      Queue aw = a;
      aw.chains = cq;
      auto warp_kernel = one_group ? k_mine_warp<true, true> : k_mine_warp<true, false>;
      warp_kernel<<<grid_for(r1 - r0, kThreads), kThreads, smem, s>>>(
          dg, dpp, lo + r0, r1 - r0, po, aw, g->heavy_q.as<int32_t>(), cnt, g->split_scratch.as<int32_t>(),
          g->split_win.as<int4>(), (int32_t)split_cap, order, nullptr);
      TM_LAUNCHED("k_mine_warp");
      (one_group ? k_mine_chains<true> : k_mine_chains<false>)<<<148 * 8, 256, 0, s>>>(dg, dpp, lo + r0, po, cq, a);
      TM_LAUNCHED("k_mine_chains");
    } else {
      // the gated rescue pass: a resident-size grid strides over the rows
      const unsigned grid = gate ? std::min<unsigned>(grid_for(r1 - r0, kThreads), 148 * 16)
                                 : grid_for(r1 - r0, kThreads);
      k_mine_warp<false, false><<<grid, kThreads, smem, s>>>(
          dg, dpp, lo + r0, r1 - r0, po, a, g->heavy_q.as<int32_t>(), cnt, g->split_scratch.as<int32_t>(),
          g->split_win.as<int4>(), (int32_t)split_cap, order, gate);
      TM_LAUNCHED("k_mine_warp");
    }
    if (g->prof && pc == pieces - 1 && !gate) TM_CUDA(cudaEventRecord(g->ev[1], s));
    // big calls: item tasks defer too (a spill-free item-task kernel; HI-Large
    // task rounds 9.6 -> 8.4 ms); small ones keep one launch per round (the
    // two extra launches per round cost more there: HI-Small 0.85 -> 0.99 ms)
    const bool split_tasks = defer && (r1 - r0 >= (int64_t)1 << 24 || split_tasks_forced());
    for (int r = 0; r < rounds; ++r) {
      TM_CUDA(cudaMemsetAsync(b.count, 0, sizeof(unsigned long long), s));
      if (split_tasks) {
        // item tasks defer their chain descents to records; chain tasks and
        // the records (which may emit chain tasks for the next round) follow
        TM_CUDA(cudaMemsetAsync(cq.count, 0, sizeof(unsigned long long), s));
        Queue bd = b;
        bd.chains = cq;
        (one_group ? k_mine_tasks<1, true> : k_mine_tasks<1, false>)<<<task_grid, kTaskThreads, 0, s>>>(
            dg, dpp, lo + r0, po, g->split_scratch.as<int32_t>(), a,
                                                           bd, g->bloom_lists.as<int32_t>(),
                                                           g->split_win.as<int4>(), nullptr);
        TM_LAUNCHED("k_mine_tasks");
        (one_group ? k_mine_tasks<2, true> : k_mine_tasks<2, false>)<<<task_grid, kTaskThreads, 0, s>>>(
            dg, dpp, lo + r0, po, g->split_scratch.as<int32_t>(), a,
                                                           b, g->bloom_lists.as<int32_t>(),
                                                           g->split_win.as<int4>(), nullptr);
        TM_LAUNCHED("k_mine_tasks");
        (one_group ? k_mine_chains<true> : k_mine_chains<false>)<<<148 * 8, 256, 0, s>>>(dg, dpp, lo + r0, po, cq, b);
        TM_LAUNCHED("k_mine_chains");
      } else {
        k_mine_tasks<0><<<task_grid, kTaskThreads, 0, s>>>(dg, dpp, lo + r0, po, g->split_scratch.as<int32_t>(), a,
                                                           b, g->bloom_lists.as<int32_t>(),
                                                           g->split_win.as<int4>(), gate);
        TM_LAUNCHED("k_mine_tasks");
      }
      std::swap(a, b);
    }
    if (rounds > 0) {
      k_mine_finalize<<<148, 256, 0, s>>>(dp, po, g->heavy_q.as<int32_t>(), cnt, g->split_scratch.as<int32_t>(),
                                          (int32_t)split_cap, gate);
      TM_LAUNCHED("k_mine_finalize");
    }
    if (!gate) TM_CUDA(cudaMemcpyAsync(piece_split + pc, cnt, sizeof(int32_t), cudaMemcpyDeviceToDevice, s));
    return TM_OK;
  };
  for (int pc = 0; pc < pieces; ++pc) {
    const int64_t r0 = std::min<int64_t>(rows, pc * per), r1 = std::min<int64_t>(rows, r0 + per);
    if ((rc = run_piece(pc, cq.rec != nullptr, nullptr))) return rc;
    // device output: a deferred pass that overflowed is redone inline on the
    // device (gated on the overflow word, no host round trip)
    if (cq.rec && out_on_device && (rc = run_piece(pc, false, overflow))) return rc;
    if (pieces > 1) {
      TM_CUDA(cudaEventRecord(g->piece_ev[pc], s));
      TM_CUDA(cudaStreamWaitEvent(g->copy_stream, g->piece_ev[pc], 0));
      TM_CUDA(cudaMemcpyAsync(out + r0 * n_plans, d_out + r0 * n_plans,
                              sizeof(long long) * (size_t)(r1 - r0) * n_plans, cudaMemcpyDeviceToHost,
                              g->copy_stream));
    }
  }
  if (g->prof) TM_CUDA(cudaEventRecord(g->ev[2], s));
  if (!out_on_device) {
    if (pieces == 1)
      TM_CUDA(cudaMemcpyAsync(out, d_out, sizeof(long long) * (size_t)rows * n_plans,
                              cudaMemcpyDeviceToHost, s));
    int32_t ns[kHostPieces] = {};
    TM_CUDA(cudaMemcpyAsync(ns, piece_split, sizeof(int32_t) * pieces, cudaMemcpyDeviceToHost, s));
    unsigned int ov = 0;
    if (cq.rec) TM_CUDA(cudaMemcpyAsync(&ov, overflow, sizeof(ov), cudaMemcpyDeviceToHost, s));
    if (pieces > 1) TM_CUDA(cudaStreamSynchronize(g->copy_stream));
    TM_CUDA(cudaStreamSynchronize(s));
    if (ov) {  // a deferred descent found no room: the whole call again, inline
      TM_CUDA(g->end(s));
      return mine_impl(g, plans, n_plans, lo, hi, out, out_on_device, stream, false);
    }
    g->last.heavy_triggers = 0;
    for (int i = 0; i < pieces; ++i) g->last.heavy_triggers += ns[i];
  } else {
    g->last.heavy_triggers = -1;  // not read back on the async path
  }
  TM_CUDA(g->end(s));
  g->last.kernel_launches = tm_kernel_launch_count() - launches0;
  return TM_OK;
}

// Window-start tables and time-slab views of the plans' deltas, built for
// triggers [lo, hi) and kept on the graph: tm_mine calls on sub-ranges of
// [lo, hi) reuse them (the pieces of a multi-GPU step: each rank prepares its
// own trigger range once per step, and only the slabs those triggers read).
extern "C" int tm_mine_prepare(tm_graph *g, const tm_plan_desc *plans, int n_plans, int64_t lo, int64_t hi,
                               void *stream) {
  if (!g) return fail(TM_E_BAD_ARG, "graph is NULL");
  if (n_plans < 0 || n_plans > kMaxPlans || (n_plans > 0 && !plans))
    return fail(TM_E_BAD_ARG, "bad plans");
  if (lo < 0 || hi < lo || hi > g->n_edges) return fail(TM_E_BAD_ARG, "bad trigger range");
  TM_CUDA(cudaSetDevice(g->device));
  cudaStream_t s = stream ? static_cast<cudaStream_t>(stream) : g->stream;
  TM_CUDA(g->begin(s));
  PreparedViews &pv = g->prep;
  pv.valid = false;
  pv.n = 0;
  for (int i = 0; i < n_plans; ++i) {
    if (plans[i].delta < 0) return fail(TM_E_BAD_ARG, "negative delta");
    bool seen = false;
    for (int k = 0; k < pv.n; ++k) seen |= pv.delta[k] == plans[i].delta;
    if (seen) continue;
    if (pv.n == kMaxGroups) return fail(TM_E_UNSUPPORTED_PLAN, "more than 8 distinct deltas");
    pv.delta[pv.n++] = plans[i].delta;
  }
  const int64_t R = g->n_ranks;
  int rc;
  if ((rc = pv.lo_tabs.ensure_pooled(sizeof(uint32_t) * (size_t)(R > 0 ? R : 1) * std::max(pv.n, 1), s,
                                     g->stream)))
    return rc;
  for (int k = 0; k < pv.n; ++k) {
    uint32_t *lt = pv.lo_tabs.as<uint32_t>() + (size_t)k * R;
    if (R > 0) {
      k_lo_table<<<grid_for(R, 256), 256, 0, s>>>(g->uniq_time.as<int64_t>(), R, pv.delta[k], lt);
      TM_LAUNCHED("k_lo_table");
    }
    if ((rc = build_slab_view(g, pv.slabs[k], pv.delta[k], lt, s, lo, hi, true, &pv.view[k], &pv.slab_of[k],
                              &pv.stride[k])))
      return rc;
  }
  pv.lo = lo;
  pv.hi = hi;
  pv.valid = true;
  TM_CUDA(g->end(s));
  return TM_OK;
}

// Drop the prepared tables (their memory stays with the graph for re-use).
extern "C" int tm_mine_release(tm_graph *g) {
  if (!g) return fail(TM_E_BAD_ARG, "graph is NULL");
  g->prep.valid = false;
  g->prep.n = 0;
  return TM_OK;
}

// diagnostic: work counters of the mining kernels (-DTM_COUNTERS=1 builds;
// tools/work_profile.py).  Not part of the public header.
extern "C" int tm_debug_counters(int reset, int64_t *out, int n) {
#if TM_COUNTERS
  unsigned long long h[kCtrN] = {};
  TM_CUDA(cudaMemcpyFromSymbol(h, dev::tm_ctr, sizeof(h)));
  for (int i = 0; i < n && i < kCtrN; ++i) out[i] = (int64_t)h[i];
  if (reset) {
    unsigned long long z[kCtrN] = {};
    TM_CUDA(cudaMemcpyToSymbol(dev::tm_ctr, z, sizeof(z)));
  }
  return kCtrN;
#else
  (void)reset; (void)out; (void)n;
  return 0;
#endif
}

extern "C" int tm_last_mine_stats(tm_graph *g, tm_mine_stats *stats) {
  if (!g || !stats) return fail(TM_E_BAD_ARG, "NULL argument");
  if (g->prof_pending) {
    TM_CUDA(cudaSetDevice(g->device));
    TM_CUDA(cudaEventSynchronize(g->ev[2]));
    TM_CUDA(cudaEventElapsedTime(&g->last.light_ms, g->ev[0], g->ev[1]));
    TM_CUDA(cudaEventElapsedTime(&g->last.heavy_ms, g->ev[1], g->ev[2]));
    TM_CUDA(cudaEventElapsedTime(&g->last.total_ms, g->ev[3], g->ev[2]));
    TM_CUDA(cudaEventElapsedTime(&g->last.prep_ms, g->ev[3], g->ev[0]));
    g->prof_pending = false;
  }
  *stats = g->last;
  return TM_OK;
}

extern "C" int tm_set_profiling(tm_graph *g, int on) {
  if (!g) return fail(TM_E_BAD_ARG, "NULL graph");
  TM_CUDA(cudaSetDevice(g->device));
  for (int i = 0; i < 4; ++i)
    if (!g->ev[i]) TM_CUDA(cudaEventCreate(&g->ev[i]));
  g->prof = on != 0;
  return TM_OK;
}
