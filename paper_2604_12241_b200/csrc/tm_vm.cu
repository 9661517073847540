// tm_vm.cu — GENERIC stage programs on the GPU.
//
// The reference runs every plan without a kernel hint through its generic
// interpreter: run_plan_on_trigger (engine.py:516-562) walks the loop tree
// of cells, execute_cell (:325-430) evaluates one cell — gate predicates,
// constant node predicates, operand maps (scalar / set / windowed
// adjacency, _adjacency_map :284-317), the cell op (for_all / intersect /
// union / differentiate), candidate node predicates and existential order
// constraints (_order_satisfiable :220-262) — and _EmissionState
// (:433-513) counts per binding and materializes instances.
//
// Device design: one thread interprets one trigger.  A cell's result (the
// reference's {node: {symbol: [(t, eid)]}}) is a segment of 16-byte
// entries (node, eid, rank, symbol) sorted by node, in a per-thread arena
// used as a stack: a loop scope's allocations are popped when its member
// advances, exactly mirroring the slot overwrite / bound-edge restore
// discipline of the reference.  Symbol -1 marks a node with no edge lists
// (scalar operands, a bound `X.self`).  A trigger whose arena overflows is
// queued and re-run with a larger arena (fewer threads), so no trigger is
// ever truncated.  Counting writes one value per trigger at the end; the
// instance-producing modes write tm_collect_instances records, and members
// attribution is derived from those records (last-member rule,
// engine.py:636-640), so every retry is side-effect free.
#include "tm_device.cuh"

namespace tmb {
namespace {

using namespace dev;

struct Ent {
  int32_t node, eid;
  uint32_t rank;
  int32_t sym;  // -1: node marker
};

struct Seg {
  int off, len;
};

struct VmAttrs {
  const double *amount;
  const int32_t *currency;
  const int32_t *cur_rank;
  const int64_t *uniq_time;
};

constexpr int kFrames = TM_VM_MAX_CELLS + 1;
constexpr int kVars = TM_VM_MAX_CELLS + 2;
constexpr int kOrderSyms = 4;

struct Frame {
  int cell;     // driver cell, -1 = trigger level
  Seg res;      // the driver's result
  int m0, m1;   // current member group [m0, m1) inside res
  int next;     // next cell index to consider as a child
  int mark;     // arena top for this member's scope
  uint32_t syms;  // symbols present in the member's edge lists
};

// record sink: MODE 0 counts only, 1 sizes records, 2 writes them
template <int MODE>
struct Sink {
  int32_t *buf;
  long long n;
  __device__ __forceinline__ void put(int32_t x) {
    if (MODE == 2) buf[n] = x;
    ++n;
  }
};

struct Vm {
  const tm_vm_program *P;
  const DevGraph *g;
  VmAttrs at;
  int u, v, e;
  uint32_t r;
  uint32_t blo, bhi;  // backward window (rank space)
  uint32_t flo, fhi;  // forward window; empty when flo > fhi
  Ent *A;
  int cap, top;
  bool overflow;
  Seg slot[TM_VM_MAX_CELLS];
  int scalar[kVars];
  Frame fr[kFrames];
  int nf;
  long long count;
  int plan_index;
};

__device__ __forceinline__ bool push(Vm &m, const Ent &x) {
  if (m.top >= m.cap) {
    m.overflow = true;
    return false;
  }
  m.A[m.top++] = x;
  return true;
}

__device__ __forceinline__ bool cmp_holds(int op, double a, double b) {
  switch (op) {
    case TM_VM_EQ: return a == b;
    case TM_VM_NE: return a != b;
    case TM_VM_LE: return a <= b;
    case TM_VM_LT: return a < b;
    case TM_VM_GE: return a >= b;
    default: return a > b;
  }
}
__device__ __forceinline__ bool cmp_holds_i(int op, long long a, long long b) {
  switch (op) {
    case TM_VM_EQ: return a == b;
    case TM_VM_NE: return a != b;
    case TM_VM_LE: return a <= b;
    case TM_VM_LT: return a < b;
    case TM_VM_GE: return a >= b;
    default: return a > b;
  }
}

// value of an edge-predicate term for entry (eid, rank) (engine.py:202-217):
// edge ids and timestamps are Python ints, amounts and DSL numbers floats
// (dsl.py:222).  Python compares an int with a float exactly, so integer
// terms stay int64 and mixed pairs go through cmp_mixed.
struct Num {
  bool is_int;
  long long i;
  double d;
};
__device__ __forceinline__ Num term_num(const Vm &m, int k, int ref, double num, int eid, uint32_t rank) {
  switch (k) {
    case TM_VM_T_NUMBER: return Num{false, 0, num};
    case TM_VM_T_EID: return Num{true, (long long)(ref ? eid : m.e), 0.0};
    case TM_VM_T_TIME: return Num{true, (long long)__ldg(m.at.uniq_time + rank), 0.0};
    case TM_VM_T_AMOUNT: return Num{false, 0, __ldg(m.at.amount + (ref ? eid : m.e))};
    default: return Num{false, 0, 0.0};
  }
}

// sign of (a - d) for int64 a and double d, exactly (-2: unordered, NaN)
__device__ __forceinline__ int cmp_int_double(long long a, double d) {
  if (d != d) return -2;
  if (d >= 9223372036854775808.0) return -1;   // 2^63 > every int64
  if (d < -9223372036854775808.0) return 1;
  const double f = floor(d);                   // |f| <= 2^63, exactly an int64 unless f == 2^63
  const long long fi = (long long)f;
  if (a < fi) return -1;
  if (a > fi) return 1;
  return d > f ? -1 : 0;                       // a == floor(d): below d iff d has a fraction
}

__device__ __forceinline__ bool sign_holds(int op, int s) {
  if (s == -2) return op == TM_VM_NE;          // NaN: only != holds
  switch (op) {
    case TM_VM_EQ: return s == 0;
    case TM_VM_NE: return s != 0;
    case TM_VM_LE: return s <= 0;
    case TM_VM_LT: return s < 0;
    case TM_VM_GE: return s >= 0;
    default: return s > 0;
  }
}

__device__ __forceinline__ bool cmp_num(int op, const Num &a, const Num &b) {
  if (a.is_int && b.is_int) return cmp_holds_i(op, a.i, b.i);
  if (!a.is_int && !b.is_int) return cmp_holds(op, a.d, b.d);
  if (a.is_int) return sign_holds(op, cmp_int_double(a.i, b.d));
  const int s = cmp_int_double(b.i, a.d);      // sign of (b - a)
  return sign_holds(op, s == -2 ? -2 : -s);
}

// does the skip predicate hold for entry (eid, rank)?  (_edge_pred_keeps negated)
__device__ bool pred_holds(const Vm &m, const tm_vm_pred &p, int eid, uint32_t rank) {
  if (p.lk == TM_VM_T_CONST) return p.lnum != 0.0;
  if (p.lk == TM_VM_T_CURRENCY || p.rk == TM_VM_T_CURRENCY) {
    if (p.table >= 0) {
      const bool lcur = p.lk == TM_VM_T_CURRENCY;
      const int ref = lcur ? p.lref : p.rref;
      const int c = __ldg(m.at.currency + (ref ? eid : m.e));
      return m.P->table[p.table + c] != 0;
    }
    const int a = __ldg(m.at.cur_rank + __ldg(m.at.currency + (p.lref ? eid : m.e)));
    const int b = __ldg(m.at.cur_rank + __ldg(m.at.currency + (p.rref ? eid : m.e)));
    return cmp_holds_i(p.cmp, a, b);
  }
  if (p.lk == TM_VM_T_EID && p.rk == TM_VM_T_EID)
    return cmp_holds_i(p.cmp, p.lref ? eid : m.e, p.rref ? eid : m.e);
  return cmp_num(p.cmp, term_num(m, p.lk, p.lref, p.lnum, eid, rank),
                 term_num(m, p.rk, p.rref, p.rnum, eid, rank));
}

// the bound edge list of symbol s: innermost frame whose member carries s
// (bound_edges save/restore, engine.py:547-557); s = 0 is the trigger
struct BoundList {
  int a, b;  // entry range in the arena (filter by sym), a < 0: the trigger itself
  bool any;
};
__device__ __forceinline__ BoundList bound_list(const Vm &m, int s) {
  if (s < 0) return BoundList{0, 0, false};
  if (s == 0) return BoundList{-1, -1, true};
  for (int f = m.nf - 1; f >= 1; --f)
    if (m.fr[f].syms & (1u << s)) return BoundList{m.fr[f].m0, m.fr[f].m1, true};
  return BoundList{0, 0, false};
}

// group [a, b) of node n inside a node-sorted segment (binary search)
__device__ __forceinline__ Seg find_group(const Vm &m, Seg s, int n) {
  int a = s.off, b = s.off + s.len;
  while (a < b) {
    const int mid = (a + b) >> 1;
    if (m.A[mid].node < n) a = mid + 1; else b = mid;
  }
  int c = a;
  while (c < s.off + s.len && m.A[c].node == n) ++c;
  return Seg{a, c - a};
}

// stable sort of [off, off + n) by node, scratch = the n entries above
__device__ bool sort_by_node(Vm &m, int off, int n) {
  if (n <= 1) return true;
  if (n <= 24) {
    for (int i = off + 1; i < off + n; ++i) {
      const Ent x = m.A[i];
      int j = i - 1;
      while (j >= off && m.A[j].node > x.node) {
        m.A[j + 1] = m.A[j];
        --j;
      }
      m.A[j + 1] = x;
    }
    return true;
  }
  if (off + 2 * n > m.cap) {
    m.overflow = true;
    return false;
  }
  Ent *src = m.A + off, *dst = m.A + off + n;
  for (int w = 1; w < n; w <<= 1) {
    for (int lo = 0; lo < n; lo += 2 * w) {
      const int mid = min(lo + w, n), hi = min(lo + 2 * w, n);
      int i = lo, j = mid, k = lo;
      while (i < mid && j < hi) dst[k++] = (src[j].node < src[i].node) ? src[j++] : src[i++];
      while (i < mid) dst[k++] = src[i++];
      while (j < hi) dst[k++] = src[j++];
    }
    Ent *t = src;
    src = dst;
    dst = t;
  }
  if (src != m.A + off)
    for (int i = 0; i < n; ++i) m.A[off + i] = src[i];
  return true;
}

// windowed adjacency of x (engine.py:284-317): self-loops skipped, per-entry
// skip predicates of the operand's symbol applied; node-sorted segment
__device__ bool adjacency(Vm &m, const tm_vm_cell &C, const tm_vm_operand &op, uint32_t lo, uint32_t hi,
                          Seg &out, long long &survivors) {
  const int x = m.scalar[op.var];
  const int d = op.dir;
  out = Seg{m.top, 0};
  if (lo > hi) return true;
  const int a = __ldg(m.g->ptr[d] + x), b = __ldg(m.g->ptr[d] + x + 1);
  const int ja = lb_u32(m.g->rnk[d], a, b, lo);
  const int jb = ub_u32(m.g->rnk[d], ja, b, hi);
  for (int j = ja; j < jb; ++j) {
    const int n = __ldg(m.g->nbr[d] + j);
    if (n == x) continue;
    const int eid = __ldg(m.g->eid[d] + j);
    const uint32_t rk = __ldg(m.g->rnk[d] + j);
    bool keep = true;
    for (int q = 0; q < C.n_edge && keep; ++q)
      if (C.edge[q].sym == op.sym && pred_holds(m, C.edge[q], eid, rk)) keep = false;
    if (!keep) continue;
    ++survivors;
    if (!push(m, Ent{n, eid, rk, op.sym})) return false;
  }
  out.len = m.top - out.off;
  return sort_by_node(m, out.off, out.len);
}

// candidate group: up to TM_VM_MAX_OPS entry ranges holding node n
struct Group {
  int n;
  int k;
  Seg part[TM_VM_MAX_OPS];
};

// order constraints (engine.py:220-262): one timestamp per referenced
// symbol — from the candidate's lists, else the bound edges — such that
// every constraint holds.  Values are staged above the arena top.
__device__ bool order_ok(Vm &m, const tm_vm_cell &C, const Group &gp) {
  int syms[kOrderSyms], ns = 0;
  for (int q = 0; q < C.n_order; ++q)
    for (int side = 1; side <= 2; ++side) {
      const int s = C.order[q][side];
      if (s < 0) continue;
      bool have = false;
      for (int i = 0; i < ns; ++i) have |= syms[i] == s;
      if (!have) {
        if (ns == kOrderSyms) return false;  // rejected by the host lowering
        syms[ns++] = s;
      }
    }
  int base = m.top, beg[kOrderSyms], end[kOrderSyms];
  for (int i = 0; i < ns; ++i) {
    const int s = syms[i];
    beg[i] = m.top;
    bool from_cand = false;
    for (int k = 0; k < gp.k; ++k)
      for (int j = gp.part[k].off; j < gp.part[k].off + gp.part[k].len; ++j)
        if (m.A[j].sym == s) {
          from_cand = true;
          if (!push(m, m.A[j])) { m.top = base; return false; }
        }
    if (!from_cand) {
      const BoundList bl = bound_list(m, s);
      if (bl.any) {
        if (bl.a < 0) {
          if (!push(m, Ent{0, m.e, m.r, 0})) { m.top = base; return false; }
        } else {
          for (int j = bl.a; j < bl.b; ++j)
            if (m.A[j].sym == s && !push(m, m.A[j])) { m.top = base; return false; }
        }
      }
    }
    end[i] = m.top;
    if (end[i] == beg[i]) {
      m.top = base;
      return false;
    }
  }
  // backtracking over one value per symbol
  int idx[kOrderSyms];
  uint32_t val[kOrderSyms];
  int lvl = 0;
  idx[0] = beg[0];
  bool ok = false;
  while (lvl >= 0) {
    if (lvl == ns) { ok = true; break; }
    if (idx[lvl] >= end[lvl]) {
      --lvl;
      if (lvl >= 0) ++idx[lvl];
      continue;
    }
    val[lvl] = m.A[idx[lvl]].rank;
    bool cons = true;
    for (int q = 0; q < C.n_order && cons; ++q) {
      long long side[2];
      bool known = true;
      for (int t = 0; t < 2; ++t) {
        const int s = C.order[q][1 + t];
        if (s < 0) { side[t] = m.r; continue; }
        int i = 0;
        while (syms[i] != s) ++i;
        if (i > lvl) known = false; else side[t] = val[i];
      }
      if (known && !cmp_holds_i(C.order[q][0], side[0], side[1])) cons = false;
    }
    if (cons) {
      ++lvl;
      if (lvl < ns) idx[lvl] = beg[lvl];
    } else {
      ++idx[lvl];
    }
  }
  m.top = base;
  return ok;
}

__device__ __forceinline__ bool node_pred_holds(const Vm &m, const int (&np)[3], int cand_var, int cand) {
  const int a = np[1] == cand_var ? cand : m.scalar[np[1]];
  const int b = np[2] == cand_var ? cand : m.scalar[np[2]];
  return np[0] == TM_VM_EQ ? a == b : a != b;
}

// execute_cell (engine.py:325-430): the cell's result segment + iterations
__device__ bool exec_cell(Vm &m, int ci, Seg &res, long long &iters) {
  const tm_vm_cell &C = m.P->cells[ci];
  const uint32_t lo = C.forward ? m.flo : m.blo, hi = C.forward ? m.fhi : m.bhi;
  const int base = m.top;
  res = Seg{base, 0};
  iters = 0;
  // gate predicates: some bound edge of the tested symbol must survive
  for (int q = 0; q < C.n_gate; ++q) {
    const tm_vm_pred &p = C.gate[q];
    const BoundList bl = bound_list(m, p.sym);
    bool kept = false;
    if (bl.any) {
      if (bl.a < 0) kept = !pred_holds(m, p, m.e, m.r);
      else
        for (int j = bl.a; j < bl.b && !kept; ++j)
          if (m.A[j].sym == p.sym) kept = !pred_holds(m, p, m.A[j].eid, m.A[j].rank);
    }
    if (!kept) return true;
  }
  const int cand_var = 2 + ci;
  for (int q = 0; q < C.n_node; ++q)
    if (C.node[q][1] != cand_var && C.node[q][2] != cand_var && node_pred_holds(m, C.node[q], -1, 0))
      return true;
  // operand maps
  Seg ops[TM_VM_MAX_OPS];
  long long survivors = 0;
  for (int k = 0; k < C.n_ops; ++k) {
    const tm_vm_operand &op = C.ops[k];
    if (op.kind == TM_VM_SCALAR) {
      ops[k] = Seg{m.top, 1};
      if (!push(m, Ent{m.scalar[op.var], -1, 0, -1})) return false;
    } else if (op.kind == TM_VM_SET) {
      const Seg stored = m.slot[op.slot];
      const int bound = m.scalar[op.var];
      if (bound >= 0) {
        const Seg gq = find_group(m, stored, bound);
        if (gq.len > 0) {
          ops[k] = gq;
        } else {
          ops[k] = Seg{m.top, 1};
          if (!push(m, Ent{bound, -1, 0, -1})) return false;
        }
      } else {
        ops[k] = stored;
      }
    } else {
      if (!adjacency(m, C, op, lo, hi, ops[k], survivors)) return false;
    }
  }
  (void)survivors;
  // candidates in node order, filtered, copied to the result
  const int out0 = m.top;
  Group gp;
  auto emit_group = [&](const Group &g) -> bool {
    for (int q = 0; q < C.n_node; ++q)
      if ((C.node[q][1] == cand_var || C.node[q][2] == cand_var) && node_pred_holds(m, C.node[q], cand_var, g.n))
        return true;
    if (C.n_order > 0 && !order_ok(m, C, g)) return !m.overflow;
    for (int k = 0; k < g.k; ++k)
      for (int j = g.part[k].off; j < g.part[k].off + g.part[k].len; ++j) {
        const Ent x = m.A[j];
        if (!push(m, x)) return false;
        if (x.sym >= 0) ++iters;
      }
    return true;
  };
  if (C.op == TM_VM_FOR_ALL || C.op == TM_VM_DIFFERENTIATE) {
    const Seg s = ops[0];
    for (int j = s.off; j < s.off + s.len;) {
      int k = j;
      while (k < s.off + s.len && m.A[k].node == m.A[j].node) ++k;
      gp.n = m.A[j].node;
      gp.k = 1;
      gp.part[0] = Seg{j, k - j};
      if (!emit_group(gp)) return false;
      j = k;
    }
  } else if (C.op == TM_VM_INTERSECT) {
    const Seg s = ops[0];
    for (int j = s.off; j < s.off + s.len;) {
      int k = j;
      while (k < s.off + s.len && m.A[k].node == m.A[j].node) ++k;
      gp.n = m.A[j].node;
      gp.k = C.n_ops;
      gp.part[0] = Seg{j, k - j};
      bool all = true;
      for (int o = 1; o < C.n_ops && all; ++o) {
        gp.part[o] = find_group(m, ops[o], gp.n);
        all = gp.part[o].len > 0;
      }
      if (all && !emit_group(gp)) return false;
      j = k;
    }
  } else {  // union: k-way merge of the node-sorted operands
    int pos[TM_VM_MAX_OPS];
    for (int o = 0; o < C.n_ops; ++o) pos[o] = ops[o].off;
    while (true) {
      int n = INT_MAX;
      for (int o = 0; o < C.n_ops; ++o)
        if (pos[o] < ops[o].off + ops[o].len) n = min(n, m.A[pos[o]].node);
      if (n == INT_MAX) break;
      gp.n = n;
      gp.k = C.n_ops;
      for (int o = 0; o < C.n_ops; ++o) {
        int k = pos[o];
        while (k < ops[o].off + ops[o].len && m.A[k].node == n) ++k;
        gp.part[o] = Seg{pos[o], k - pos[o]};
        pos[o] = k;
      }
      if (!emit_group(gp)) return false;
    }
  }
  // compact: the result replaces this cell's operand scratch
  const int len = m.top - out0;
  for (int i = 0; i < len; ++i) m.A[base + i] = m.A[out0 + i];
  m.top = base + len;
  res = Seg{base, len};
  return true;
}

__device__ __forceinline__ int n_groups(const Vm &m, Seg s) {
  int n = 0;
  for (int j = s.off; j < s.off + s.len; ++j) n += (j == s.off || m.A[j].node != m.A[j - 1].node);
  return n;
}

// instance members common to every unit of a binding (_base_members,
// engine.py:447-453): trigger + every bound edge list (innermost wins per
// symbol) + trigger endpoints + bound loop variables
template <int MODE>
__device__ void base_edges(const Vm &m, Sink<MODE> &sk, int &ne) {
  sk.put(m.e);
  ++ne;
  uint32_t inner = 0;
  for (int f = m.nf - 1; f >= 1; --f) {
    for (int j = m.fr[f].m0; j < m.fr[f].m1; ++j) {
      const int s = m.A[j].sym;
      if (s >= 0 && !(inner & (1u << s))) {
        sk.put(m.A[j].eid);
        ++ne;
      }
    }
    inner |= m.fr[f].syms;
  }
}
template <int MODE>
__device__ void base_nodes(const Vm &m, Sink<MODE> &sk, int &nn) {
  sk.put(m.u);
  sk.put(m.v);
  nn += 2;
  for (int f = 1; f < m.nf; ++f) {
    sk.put(m.A[m.fr[f].m0].node);
    ++nn;
  }
}

template <int MODE>
__device__ __forceinline__ long long open_rec(Sink<MODE> &sk, int plan, int e) {
  const long long at = sk.n;
  sk.put(plan);
  sk.put(e);
  sk.put(0);
  sk.put(0);
  return at;
}
template <int MODE>
__device__ __forceinline__ void close_rec(Sink<MODE> &sk, long long at, int ne, int nn) {
  if (MODE == 2) {
    sk.buf[at + 2] = ne;
    sk.buf[at + 3] = nn;
  }
}

// _EmissionState.on_cell (engine.py:455-499)
template <int MODE>
__device__ void on_cell(Vm &m, int ci, Seg res, long long iters, Sink<MODE> &sk) {
  const tm_vm_program &P = *m.P;
  if (P.mode == TM_VM_PAIR_PRODUCT || ci != P.target[0]) return;
  const int K = P.min_size;
  const int groups = n_groups(m, res);
  if (P.mode == TM_VM_SET_CARDINALITY || P.mode == TM_VM_INSTANCE_LIST) {
    if (groups < K) return;
    m.count += groups;
    if (MODE == 0) return;
    for (int j = res.off; j < res.off + res.len;) {
      int k = j;
      while (k < res.off + res.len && m.A[k].node == m.A[j].node) ++k;
      const long long at = open_rec(sk, m.plan_index, m.e);
      int ne = 0, nn = 0;
      base_edges(m, sk, ne);
      for (int q = j; q < k; ++q)
        if (m.A[q].sym >= 0) { sk.put(m.A[q].eid); ++ne; }
      base_nodes(m, sk, nn);
      sk.put(m.A[j].node);
      ++nn;
      close_rec(sk, at, ne, nn);
      j = k;
    }
  } else if (P.mode == TM_VM_EDGE_COUNT) {
    if (iters < K) return;
    m.count += iters;
    if (MODE == 0) return;
    for (int q = res.off; q < res.off + res.len; ++q) {
      if (m.A[q].sym < 0) continue;
      const long long at = open_rec(sk, m.plan_index, m.e);
      int ne = 0, nn = 0;
      base_edges(m, sk, ne);
      sk.put(m.A[q].eid);
      ++ne;
      base_nodes(m, sk, nn);
      sk.put(m.A[q].node);
      ++nn;
      close_rec(sk, at, ne, nn);
    }
  } else {  // SOURCE_COUNT
    if (groups < K) return;
    m.count += 1;
    if (MODE == 0) return;
    const long long at = open_rec(sk, m.plan_index, m.e);
    int ne = 0, nn = 0;
    base_edges(m, sk, ne);
    for (int q = res.off; q < res.off + res.len; ++q)
      if (m.A[q].sym >= 0) { sk.put(m.A[q].eid); ++ne; }
    base_nodes(m, sk, nn);
    for (int j = res.off; j < res.off + res.len; ++j)
      if (j == res.off || m.A[j].node != m.A[j - 1].node) { sk.put(m.A[j].node); ++nn; }
    close_rec(sk, at, ne, nn);
  }
}

// _EmissionState.finish_pair_product (engine.py:501-513)
template <int MODE>
__device__ void finish_pair(Vm &m, Sink<MODE> &sk) {
  const tm_vm_program &P = *m.P;
  if (P.mode != TM_VM_PAIR_PRODUCT) return;
  const Seg a = m.slot[P.target[0]], c = m.slot[P.target[1]];
  const long long na = n_groups(m, a), nc = n_groups(m, c);
  if (na < P.min_size || nc < P.min_size) return;
  m.count += na * nc;
  if (MODE == 0) return;
  for (int i = a.off; i < a.off + a.len;) {
    int i2 = i;
    while (i2 < a.off + a.len && m.A[i2].node == m.A[i].node) ++i2;
    for (int j = c.off; j < c.off + c.len;) {
      int j2 = j;
      while (j2 < c.off + c.len && m.A[j2].node == m.A[j].node) ++j2;
      const long long at = open_rec(sk, m.plan_index, m.e);
      int ne = 1, nn = 4;
      sk.put(m.e);
      for (int q = i; q < i2; ++q)
        if (m.A[q].sym >= 0) { sk.put(m.A[q].eid); ++ne; }
      for (int q = j; q < j2; ++q)
        if (m.A[q].sym >= 0) { sk.put(m.A[q].eid); ++ne; }
      sk.put(m.u);
      sk.put(m.v);
      sk.put(m.A[i].node);
      sk.put(m.A[j].node);
      close_rec(sk, at, ne, nn);
      j = j2;
    }
    i = i2;
  }
}

__device__ __forceinline__ void bind_member(Vm &m, Frame &f) {
  int k = f.m0;
  while (k < f.res.off + f.res.len && m.A[k].node == m.A[f.m0].node) ++k;
  f.m1 = k;
  uint32_t s = 0;
  for (int j = f.m0; j < f.m1; ++j)
    if (m.A[j].sym >= 0) s |= 1u << m.A[j].sym;
  f.syms = s;
  m.scalar[2 + f.cell] = m.A[f.m0].node;
  f.next = 0;
  f.mark = m.top;
}

// run_plan_on_trigger (engine.py:516-562) as an explicit-stack loop
template <int MODE>
__device__ bool run_trigger(Vm &m, Sink<MODE> &sk) {
  const tm_vm_program &P = *m.P;
  m.nf = 1;
  m.fr[0] = Frame{-1, Seg{0, 0}, 0, 0, 0, m.top, 0};
  while (m.nf > 0) {
    Frame &f = m.fr[m.nf - 1];
    int ci = f.next;
    while (ci < P.n_cells && P.cells[ci].parent != f.cell) ++ci;
    if (ci < P.n_cells) {
      f.next = ci + 1;
      Seg res;
      long long iters;
      if (!exec_cell(m, ci, res, iters)) return false;
      m.slot[ci] = res;
      on_cell(m, ci, res, iters, sk);
      bool has_children = false;
      for (int c = ci + 1; c < P.n_cells; ++c) has_children |= P.cells[c].parent == ci;
      if (has_children && res.len > 0) {
        Frame &nf = m.fr[m.nf++];
        nf.cell = ci;
        nf.res = res;
        nf.m0 = res.off;
        bind_member(m, nf);
      }
      continue;
    }
    // this member's children are done: next member, or leave the loop
    if (m.nf == 1) break;
    m.top = f.mark;
    if (f.m1 < f.res.off + f.res.len) {
      f.m0 = f.m1;
      bind_member(m, f);
    } else {
      m.scalar[2 + f.cell] = -1;
      --m.nf;
    }
  }
  m.nf = 1;
  finish_pair(m, sk);
  return true;
}

__device__ __forceinline__ uint32_t rank_ub(const int64_t *uniq, int64_t R, long long x) {
  int64_t a = 0, b = R;
  while (a < b) {
    const int64_t mid = (a + b) >> 1;
    if (__ldg(uniq + mid) <= x) a = mid + 1; else b = mid;
  }
  return (uint32_t)a;  // first rank with time > x
}
__device__ __forceinline__ uint32_t rank_lb(const int64_t *uniq, int64_t R, long long x) {
  int64_t a = 0, b = R;
  while (a < b) {
    const int64_t mid = (a + b) >> 1;
    if (__ldg(uniq + mid) < x) a = mid + 1; else b = mid;
  }
  return (uint32_t)a;
}

// one trigger; false = arena overflow (nothing observable was written)
template <int MODE>
__device__ bool vm_trigger(const tm_vm_program *P, const DevGraph &g, const VmAttrs &at, int64_t R, int e,
                           Ent *arena, int cap, Sink<MODE> &sk, long long &count, int plan_index) {
  Vm m;
  m.P = P;
  m.g = &g;
  m.at = at;
  m.e = e;
  m.u = __ldg(g.e_src + e);
  m.v = __ldg(g.e_dst + e);
  m.r = __ldg(g.e_rank + e);
  const long long t = __ldg(at.uniq_time + m.r), d = P->delta;
  m.bhi = m.r;
  m.blo = rank_lb(at.uniq_time, R, t >= LLONG_MIN + d ? t - d : LLONG_MIN);
  m.flo = m.r;
  m.fhi = rank_ub(at.uniq_time, R, t <= LLONG_MAX - d ? t + d : LLONG_MAX) - 1;
  m.A = arena;
  m.cap = cap;
  m.top = 0;
  m.overflow = false;
  m.count = 0;
  m.plan_index = plan_index;
  for (int i = 0; i < kVars; ++i) m.scalar[i] = -1;
  m.scalar[0] = m.u;
  m.scalar[1] = m.v;
  for (int i = 0; i < TM_VM_MAX_CELLS; ++i) m.slot[i] = Seg{0, 0};
  if (!run_trigger(m, sk) || m.overflow) return false;
  count = m.count;
  return true;
}

// MODE 0: counts into out[i];  1: record words into size[i];  2: records at size[i]
template <int MODE>
__global__ void __launch_bounds__(128) k_vm(const tm_vm_program *__restrict__ P, const __grid_constant__ DevGraph g,
                                            VmAttrs at, int64_t R, int64_t lo, int64_t n_rows,
                                            const int32_t *__restrict__ list, Ent *__restrict__ arena, int cap,
                                            long long *__restrict__ out, unsigned long long *__restrict__ size,
                                            int32_t *__restrict__ buf, int32_t *__restrict__ ovf,
                                            int32_t *__restrict__ n_ovf, int plan_index) {
  const int64_t tid = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const int64_t nthreads = (int64_t)gridDim.x * blockDim.x;
  Ent *A = arena + tid * (int64_t)cap;
  for (int64_t i0 = tid; i0 < n_rows; i0 += nthreads) {
    const int64_t i = list ? list[i0] : i0;  // row
    const int e = (int)(lo + i);
    Sink<MODE> sk{MODE == 2 ? buf + size[i] : nullptr, 0};
    long long count = 0;
    if (!vm_trigger<MODE>(P, g, at, R, e, A, cap, sk, count, plan_index)) {
      ovf[atomicAdd(n_ovf, 1)] = (int32_t)i;
      continue;
    }
    if (MODE == 0) out[i] = count;
    if (MODE == 1) size[i] = (unsigned long long)sk.n;
  }
}

// members from records: a trigger's instance counts when the trigger is its
// temporally last member ((time, eid) order, engine.py:636-640); then every
// distinct member edge gains 1
__global__ void k_vm_members(const __grid_constant__ DevGraph g, int64_t lo, int64_t n_rows,
                             const unsigned long long *__restrict__ size, int32_t *__restrict__ buf,
                             long long *__restrict__ out) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n_rows) return;
  const int e = (int)(lo + i);
  const uint32_t re = __ldg(g.e_rank + e);
  long long p = (long long)size[i];
  const long long end = (long long)size[i + 1];
  while (p < end) {
    const int ne = buf[p + 2], nn = buf[p + 3];
    int32_t *ed = buf + p + 4;
    bool last = true;
    for (int k = 0; k < ne && last; ++k) {
      const int f = ed[k];
      const uint32_t rf = __ldg(g.e_rank + f);
      if (rf > re || (rf == re && f > e)) last = false;
    }
    if (last) {
      for (int a = 1; a < ne; ++a) {  // dedup: insertion sort in place
        const int x = ed[a];
        int b = a - 1;
        while (b >= 0 && ed[b] > x) {
          ed[b + 1] = ed[b];
          --b;
        }
        ed[b + 1] = x;
      }
      for (int k = 0; k < ne; ++k)
        if (k == 0 || ed[k] != ed[k - 1]) atomicAdd(reinterpret_cast<unsigned long long *>(out + ed[k]), 1ull);
    }
    p += 4 + ne + nn;
  }
}

// arena tiers: (entries per thread, threads); a trigger overflowing the
// last tier is an error
struct Tier {
  int cap;
  int threads;
};
constexpr Tier kTiers[] = {{512, 148 * 512}, {8192, 148 * 32}, {1 << 17, 148 * 2}, {1 << 22, 8}, {1 << 25, 1}};
constexpr int kNumTiers = sizeof(kTiers) / sizeof(kTiers[0]);

int check_program(const tm_graph *g, const tm_vm_program *p) {
  if (!p) return fail(TM_E_BAD_ARG, "program is NULL");
  if (p->n_cells < 1 || p->n_cells > TM_VM_MAX_CELLS) return fail(TM_E_BAD_ARG, "bad cell count");
  if (p->min_size < 1) return fail(TM_E_BAD_ARG, "min_size < 1");
  if (p->delta < 0) return fail(TM_E_BAD_ARG, "negative delta");
  if (p->mode < TM_VM_SET_CARDINALITY || p->mode > TM_VM_INSTANCE_LIST) return fail(TM_E_BAD_ARG, "bad mode");
  const int nt = p->mode == TM_VM_PAIR_PRODUCT ? 2 : 1;
  for (int i = 0; i < nt; ++i)
    if (p->target[i] < 0 || p->target[i] >= p->n_cells) return fail(TM_E_BAD_ARG, "bad emission target");
  if (p->uses_attrs && !g->attr_amount.p) return fail(TM_E_STATE, "attribute predicates need tm_graph_set_attrs");
  for (int c = 0; c < p->n_cells; ++c) {
    const tm_vm_cell &C = p->cells[c];
    if (C.parent < -1 || C.parent >= c) return fail(TM_E_BAD_ARG, "cell parent must precede the cell");
    if (C.n_ops < 1 || C.n_ops > TM_VM_MAX_OPS || C.n_node > TM_VM_MAX_PREDS || C.n_edge > TM_VM_MAX_PREDS ||
        C.n_gate > TM_VM_MAX_PREDS || C.n_order > TM_VM_MAX_PREDS || C.n_node < 0 || C.n_edge < 0 ||
        C.n_gate < 0 || C.n_order < 0)
      return fail(TM_E_BAD_ARG, "cell " + std::to_string(c) + ": bad counts");
    for (int k = 0; k < C.n_ops; ++k) {
      const tm_vm_operand &o = C.ops[k];
      if (o.var < 0 || o.var >= 2 + c) return fail(TM_E_BAD_ARG, "operand variable out of scope");
      if ((o.kind == TM_VM_SET || o.kind == TM_VM_MEMBER_ADJ) && (o.slot < 0 || o.slot >= c))
        return fail(TM_E_BAD_ARG, "operand reads a later slot");
      if ((o.kind == TM_VM_ADJ || o.kind == TM_VM_MEMBER_ADJ) &&
          (o.dir < 0 || o.dir > 1 || o.sym < 1 || o.sym >= TM_VM_MAX_SYMS))
        return fail(TM_E_BAD_ARG, "bad adjacency operand");
    }
    for (int q = 0; q < C.n_order; ++q)
      for (int s = 1; s <= 2; ++s)
        if (C.order[q][s] < -1 || C.order[q][s] >= TM_VM_MAX_SYMS) return fail(TM_E_BAD_ARG, "bad order symbol");
  }
  return TM_OK;
}

VmAttrs attrs_of(const tm_graph *g) {
  return VmAttrs{g->attr_amount.as<double>(), g->attr_currency.as<int32_t>(), g->attr_cur_rank.as<int32_t>(),
                 g->uniq_time.as<int64_t>()};
}

// run MODE over rows [0, rows) with overflow tiers; size / out / buf as k_vm
template <int MODE>
int vm_pass(tm_graph *g, const tm_vm_program *dprog, int64_t lo, int64_t rows, long long *out,
            unsigned long long *size, int32_t *buf, int plan_index) {
  cudaStream_t s = g->stream;
  int rc;
  if ((rc = g->vm_ovf.ensure(sizeof(int32_t) * 2 * (size_t)(rows + 1))) || (rc = g->vm_novf.ensure(8)))
    return rc;
  int32_t *ovf[2] = {g->vm_ovf.as<int32_t>(), g->vm_ovf.as<int32_t>() + rows + 1};
  int32_t *novf = g->vm_novf.as<int32_t>();
  const int32_t *list = nullptr;
  int64_t n = rows;
  for (int t = 0; t < kNumTiers && n > 0; ++t) {
    const Tier tr = kTiers[t];
    const int64_t threads = std::min<int64_t>(tr.threads, ((n + 127) / 128) * 128);
    if ((rc = g->vm_arena.ensure(sizeof(Ent) * (size_t)tr.cap * (size_t)threads))) return rc;
    int32_t *dst = ovf[t & 1];
    TM_CUDA(cudaMemsetAsync(novf + (t & 1), 0, sizeof(int32_t), s));
    k_vm<MODE><<<grid_for(threads, 128), 128, 0, s>>>(dprog, g->dev(), attrs_of(g), g->n_ranks, lo, n, list,
                                                      g->vm_arena.as<Ent>(), tr.cap, out, size, buf, dst,
                                                      novf + (t & 1), plan_index);
    TM_LAUNCHED("k_vm");
    int32_t h = 0;
    TM_CUDA(cudaMemcpyAsync(&h, novf + (t & 1), sizeof(int32_t), cudaMemcpyDeviceToHost, s));
    TM_CUDA(cudaStreamSynchronize(s));
    n = h;
    list = dst;
  }
  if (n > 0) return fail(TM_E_OVERFLOW, "a trigger's stage program exceeds the largest VM arena");
  return TM_OK;
}

int upload_program(tm_graph *g, const tm_vm_program *prog, const tm_vm_program **dprog) {
  int rc;
  if ((rc = g->vm_prog.ensure(sizeof(tm_vm_program)))) return rc;
  TM_CUDA(cudaMemcpyAsync(g->vm_prog.p, prog, sizeof(tm_vm_program), cudaMemcpyHostToDevice, g->stream));
  *dprog = g->vm_prog.as<tm_vm_program>();
  return TM_OK;
}

// records of [lo, hi) into g->inst_buf, per-row offsets in `size` (rows + 1)
int vm_records(tm_graph *g, const tm_vm_program *prog, int32_t plan_index, int64_t lo, int64_t hi,
               DevBuf &size, int64_t *words) {
  const tm_vm_program *dp;
  int rc;
  if ((rc = check_program(g, prog)) || (rc = upload_program(g, prog, &dp))) return rc;
  const int64_t rows = hi - lo;
  cudaStream_t s = g->stream;
  if ((rc = size.ensure(sizeof(unsigned long long) * (size_t)(rows + 1)))) return rc;
  unsigned long long *sz = size.as<unsigned long long>();
  if ((rc = vm_pass<1>(g, dp, lo, rows, nullptr, sz, nullptr, plan_index))) return rc;
  TM_CUDA(cudaMemsetAsync(sz + rows, 0, sizeof(unsigned long long), s));
  if ((rc = scan_u64_exclusive(sz, rows + 1, s))) return rc;
  unsigned long long total = 0;
  TM_CUDA(cudaMemcpyAsync(&total, sz + rows, 8, cudaMemcpyDeviceToHost, s));
  TM_CUDA(cudaStreamSynchronize(s));
  if (total > (1ull << 33)) return fail(TM_E_OVERFLOW, "instance records exceed 32 GiB");
  if ((rc = g->inst_buf.ensure(sizeof(int32_t) * (size_t)(total ? total : 1)))) return rc;
  if ((rc = vm_pass<2>(g, dp, lo, rows, nullptr, sz, g->inst_buf.as<int32_t>(), plan_index))) return rc;
  g->inst_words = (int64_t)total;
  *words = (int64_t)total;
  return TM_OK;
}

}  // namespace
}  // namespace tmb

using namespace tmb;

extern "C" int tm_graph_set_attrs(tm_graph *g, const double *amount, const int32_t *currency, int32_t n_vocab,
                                  const int32_t *cur_rank) {
  if (!g || n_vocab < 0 || (g->n_edges > 0 && (!amount || !currency)) || (n_vocab > 0 && !cur_rank))
    return fail(TM_E_BAD_ARG, "bad attribute arrays");
  for (int64_t i = 0; i < g->n_edges; ++i)
    if (currency[i] < 0 || currency[i] >= n_vocab) return fail(TM_E_BAD_ARG, "currency id out of range");
  if (n_vocab > TM_VM_TABLE) return fail(TM_E_UNSUPPORTED_PLAN, "currency vocabulary too large");
  TM_CUDA(cudaSetDevice(g->device));
  const size_t E = (size_t)(g->n_edges > 0 ? g->n_edges : 1);
  int rc;
  if ((rc = g->attr_amount.ensure(8 * E)) || (rc = g->attr_currency.ensure(4 * E)) ||
      (rc = g->attr_cur_rank.ensure(4 * (size_t)(n_vocab > 0 ? n_vocab : 1))))
    return rc;
  if (g->n_edges > 0) {
    TM_CUDA(cudaMemcpy(g->attr_amount.p, amount, 8 * (size_t)g->n_edges, cudaMemcpyHostToDevice));
    TM_CUDA(cudaMemcpy(g->attr_currency.p, currency, 4 * (size_t)g->n_edges, cudaMemcpyHostToDevice));
  }
  if (n_vocab > 0) TM_CUDA(cudaMemcpy(g->attr_cur_rank.p, cur_rank, 4 * (size_t)n_vocab, cudaMemcpyHostToDevice));
  g->n_vocab = n_vocab;
  return TM_OK;
}

extern "C" int tm_vm_mine(tm_graph *g, const tm_vm_program *prog, int64_t lo, int64_t hi, int64_t *out) {
  if (!g) return fail(TM_E_BAD_ARG, "graph is NULL");
  if (lo < 0 || hi < lo || hi > g->n_edges) return fail(TM_E_BAD_ARG, "bad trigger range");
  if (hi > lo && !out) return fail(TM_E_BAD_ARG, "out is NULL");
  const tm_vm_program *dp;
  int rc;
  if ((rc = check_program(g, prog))) return rc;
  const int64_t rows = hi - lo;
  if (rows == 0) return TM_OK;
  TM_CUDA(cudaSetDevice(g->device));
  if ((rc = upload_program(g, prog, &dp))) return rc;
  DevBuf dout;
  if ((rc = dout.ensure(8 * (size_t)rows))) return rc;
  if ((rc = vm_pass<0>(g, dp, lo, rows, dout.as<long long>(), nullptr, nullptr, 0))) return rc;
  TM_CUDA(cudaMemcpyAsync(out, dout.p, 8 * (size_t)rows, cudaMemcpyDeviceToHost, g->stream));
  TM_CUDA(cudaStreamSynchronize(g->stream));
  return TM_OK;
}

extern "C" int tm_vm_collect(tm_graph *g, const tm_vm_program *prog, int32_t plan_index, int64_t lo, int64_t hi,
                             int64_t *out_words) {
  if (!g || !out_words) return fail(TM_E_BAD_ARG, "NULL argument");
  *out_words = 0;
  g->inst_words = 0;
  if (lo < 0 || hi < lo || hi > g->n_edges) return fail(TM_E_BAD_ARG, "bad trigger range");
  int rc;
  if ((rc = check_program(g, prog))) return rc;
  if (hi == lo) return TM_OK;
  TM_CUDA(cudaSetDevice(g->device));
  DevBuf size;
  return vm_records(g, prog, plan_index, lo, hi, size, out_words);
}

extern "C" int tm_vm_members(tm_graph *g, const tm_vm_program *prog, int64_t lo, int64_t hi, int64_t *out) {
  if (!g) return fail(TM_E_BAD_ARG, "graph is NULL");
  if (lo < 0 || hi < lo || hi > g->n_edges) return fail(TM_E_BAD_ARG, "bad trigger range");
  const int64_t E = g->n_edges;
  if (E > 0 && !out) return fail(TM_E_BAD_ARG, "out is NULL");
  int rc;
  if ((rc = check_program(g, prog))) return rc;
  if (E == 0) return TM_OK;
  TM_CUDA(cudaSetDevice(g->device));
  DevBuf acc, size;
  if ((rc = acc.ensure(8 * (size_t)E))) return rc;
  TM_CUDA(cudaMemsetAsync(acc.p, 0, 8 * (size_t)E, g->stream));
  constexpr int64_t kChunk = 1 << 16;  // bounds the record buffer
  for (int64_t a = lo; a < hi; a += kChunk) {
    const int64_t b = std::min(hi, a + kChunk);
    int64_t words = 0;
    if ((rc = vm_records(g, prog, 0, a, b, size, &words))) return rc;
    k_vm_members<<<grid_for(b - a, 128), 128, 0, g->stream>>>(g->dev(), a, b - a, size.as<unsigned long long>(),
                                                              g->inst_buf.as<int32_t>(), acc.as<long long>());
    TM_LAUNCHED("k_vm_members");
  }
  TM_CUDA(cudaMemcpyAsync(out, acc.p, 8 * (size_t)E, cudaMemcpyDeviceToHost, g->stream));
  TM_CUDA(cudaStreamSynchronize(g->stream));
  return TM_OK;
}
