"""Lowering of GENERIC execution plans onto the device stage VM (csrc/tm_vm.cu).

A plan whose compiled cells do not match one of the GPU families (see
plan.recognize) — union / differentiate stages, order constraints, forward
windows, attribute predicates, any loop nest — is the reference's generic
interpreter's job (engine.py:325-562).  `lower_program` turns such a plan
into a tm_vm_program (include/tempmine_b200.h): variables and edge symbols
numbered, skip predicates classified exactly as _PreparedCell does
(engine.py:139-162: node / per-entry edge / gate), and every predicate
pre-typed the way Python would evaluate it in _edge_pred_keeps
(engine.py:192-217): numeric terms compare as numbers, currency against a
string literal through a per-vocabulary truth table, None / mixed-type
equality folded to a constant.  Plans the VM cannot express raise
UnsupportedPlanError — never a CPU fallback.
"""

from __future__ import annotations

import ctypes
from dataclasses import dataclass

from . import _lib
from ._lib import TM_E_UNSUPPORTED_PLAN, UnsupportedPlanError

_OPS = {"for_all": 0, "intersect": 1, "union": 2, "differentiate": 3}
_KINDS = {"scalar": 0, "set": 1, "adj": 2, "member_adj": 3}
_MODES = {"set_cardinality": 0, "source_count": 1, "pair_product": 2, "edge_count": 3, "instance_list": 4}
_CMP = {"==": 0, "!=": 1, "<=": 2, "<": 3, ">=": 4, ">": 5}
T_NUMBER, T_EID, T_TIME, T_AMOUNT, T_CURRENCY, T_CONST = 0, 1, 2, 3, 4, 5
_NUMERIC = (T_NUMBER, T_EID, T_TIME, T_AMOUNT)


def _py_compare(a, b, op: str) -> bool:
    """engine.py:_compare"""
    if op == "==":
        return a == b
    if op == "!=":
        return a != b
    if op == "<=":
        return a <= b
    if op == "<":
        return a < b
    if op == ">=":
        return a >= b
    return a > b


@dataclass
class VmProgram:
    """A lowered GENERIC plan: the ctypes program plus host-side facts."""

    name: str
    prog: _lib.TmVmProgram
    members: bool
    uses_attrs: bool


class _Unsupported(Exception):
    pass


def _sym_id(name: str) -> int:
    if not (isinstance(name, str) and name.startswith("e") and name[1:].isdigit()):
        raise _Unsupported(f"edge symbol {name!r}")
    k = int(name[1:])
    if k >= _lib.VM_MAX_SYMS:
        raise _Unsupported(f"more than {_lib.VM_MAX_SYMS - 1} edge symbols")
    return k


def _edge_term(t):
    """(kind, ref, num, string) of a term as _edge_pred_keeps values it;
    kind None = Python None."""
    if t.kind == "edge":
        return (T_EID, 0 if t.name == "e0" else 1, 0.0, None)
    if t.kind == "etime":
        return (None, 0, 0.0, None) if t.name == "e0" else (T_TIME, 1, 0.0, None)
    if t.kind == "eattr":
        ref = 0 if t.name == "e0" else 1
        if t.attr == "amount":
            return (T_AMOUNT, ref, 0.0, None)
        return (T_CURRENCY, ref, 0.0, None)
    if t.kind == "number":
        return (T_NUMBER, 0, float(t.value), None)
    if t.kind == "string":
        return ("str", 0, 0.0, str(t.value))
    return (None, 0, 0.0, None)  # node / trigger_time / window_end -> None


def _lower_pred(pred, sym: int, vocab, table: list) -> _lib.TmVmPred:
    p = _lib.TmVmPred()
    p.cmp = _CMP[pred.op]
    p.sym = sym
    p.table = -1
    lk, lref, lnum, lstr = _edge_term(pred.lhs)
    rk, rref, rnum, rstr = _edge_term(pred.rhs)
    ordering = pred.op not in ("==", "!=")

    def const(v: bool):
        p.lk = T_CONST
        p.lnum = 1.0 if v else 0.0
        return p

    if lk is None or rk is None:  # None == x only for x None
        if ordering:
            raise _Unsupported(f"ordering comparison with None in {pred!r}")
        both = lk is None and rk is None
        return const(both if pred.op == "==" else not both)
    lstrlike = lk in ("str", T_CURRENCY)
    rstrlike = rk in ("str", T_CURRENCY)
    if lstrlike != rstrlike:
        if ordering:
            raise _Unsupported(f"ordering comparison between a string and a number in {pred!r}")
        return const(pred.op == "!=")
    if lstrlike:  # both string-valued
        if lk == "str" and rk == "str":
            return const(_py_compare(lstr, rstr, pred.op))
        if lk == T_CURRENCY and rk == T_CURRENCY:
            p.lk, p.lref, p.rk, p.rref = T_CURRENCY, lref, T_CURRENCY, rref
            return p
        if vocab is None:
            raise _Unsupported("currency predicate without a currency vocabulary")
        off = len(table)
        if off + len(vocab) > _lib.VM_TABLE:
            raise _Unsupported("currency truth tables exceed the program table")
        for word in vocab:
            table.append(1 if (_py_compare(word, rstr, pred.op) if lk == T_CURRENCY
                               else _py_compare(lstr, word, pred.op)) else 0)
        p.table = off
        p.lk, p.lref = (T_CURRENCY, lref) if lk == T_CURRENCY else (T_NUMBER, 0)
        p.rk, p.rref = (T_CURRENCY, rref) if rk == T_CURRENCY else (T_NUMBER, 0)
        return p
    p.lk, p.lref, p.lnum = lk, lref, lnum
    p.rk, p.rref, p.rnum = rk, rref, rnum
    return p


def _uses_attr(pred) -> bool:
    return any(t.kind == "eattr" for t in (pred.lhs, pred.rhs))


def lower_program(plan, vocab=None) -> VmProgram:
    """ExecutionPlan (reference or ours) -> VmProgram; UnsupportedPlanError
    when the VM limits (8 cells, 4 operands, 8 predicates of each kind, 15
    edge symbols, 4 symbols per order group) or types rule it out."""
    name = getattr(plan, "name", "?")
    try:
        return _lower(plan, vocab)
    except _Unsupported as exc:
        raise UnsupportedPlanError(TM_E_UNSUPPORTED_PLAN, f"plan {name}: {exc}") from None


def _lower(plan, vocab) -> VmProgram:
    attribution = getattr(plan, "attribution", "trigger")
    if attribution not in ("trigger", "members"):
        raise _Unsupported(f"unknown attribution {attribution!r}")
    cells = plan.cells
    if not 1 <= len(cells) <= _lib.VM_MAX_CELLS:
        raise _Unsupported(f"{len(cells)} cells (VM limit {_lib.VM_MAX_CELLS})")
    if int(plan.delta) < 0:
        raise ValueError(f"plan {plan.name}: delta must be non-negative")
    if int(plan.emission.min_size) < 1:
        raise ValueError(f"plan {plan.name}: min_size must be >= 1")
    prog = _lib.TmVmProgram()
    prog.n_cells = len(cells)
    prog.mode = _MODES[plan.emission.mode]
    prog.min_size = int(plan.emission.min_size)
    targets = tuple(plan.emission.target_slots)
    prog.target[0] = targets[0]
    prog.target[1] = targets[1] if len(targets) > 1 else -1
    prog.delta = int(plan.delta)
    var = {"N0": 0, "N1": 1}
    table: list[int] = []
    uses_attrs = False
    for i, cell in enumerate(cells):
        c = prog.cells[i]
        c.op = _OPS[cell.op]
        c.parent = int(cell.parent)
        c.forward = 1 if cell.window_lo == "t" else 0
        if len(cell.src) > _lib.VM_MAX_OPS:
            raise _Unsupported(f"cell {i}: {len(cell.src)} operands (VM limit {_lib.VM_MAX_OPS})")
        c.n_ops = len(cell.src)
        own = set()
        for k, d in enumerate(cell.src):
            o = c.ops[k]
            o.kind = _KINDS[d.kind]
            if d.base not in var:
                raise _Unsupported(f"cell {i}: operand base {d.base!r} is not bound")
            o.var = var[d.base]
            o.slot = int(d.slot)
            o.dir = 0 if d.direction == "in" else 1
            o.sym = _sym_id(d.symbol) if d.symbol else -1
            if d.symbol:
                own.add(d.symbol)
        var_here = dict(var)
        var_here[cell.dst_var] = 2 + i
        n_node = n_edge = n_gate = 0
        for pred in cell.skip_preds:
            kinds = {pred.lhs.kind, pred.rhs.kind}
            if kinds == {"node"}:  # engine.py:147-150
                if n_node == _lib.VM_MAX_PREDS:
                    raise _Unsupported(f"cell {i}: too many node predicates")
                for t in (pred.lhs, pred.rhs):
                    if t.name not in var_here:
                        raise _Unsupported(f"cell {i}: node {t.name!r} is not bound")
                c.node[n_node][0] = _CMP[pred.op] if pred.op in ("==", "!=") else -1
                if c.node[n_node][0] < 0:
                    raise _Unsupported(f"cell {i}: node comparison {pred.op}")
                c.node[n_node][1] = var_here[pred.lhs.name]
                c.node[n_node][2] = var_here[pred.rhs.name]
                n_node += 1
                continue
            uses_attrs |= _uses_attr(pred)
            sym = None
            for t in (pred.lhs, pred.rhs):  # engine.py:152-156 (last own symbol wins)
                if t.kind in ("edge", "etime", "eattr") and t.name in own:
                    sym = t.name
            if sym is not None:
                if n_edge == _lib.VM_MAX_PREDS:
                    raise _Unsupported(f"cell {i}: too many edge predicates")
                c.edge[n_edge] = _lower_pred(pred, _sym_id(sym), vocab, table)
                n_edge += 1
            else:  # gate (engine.py:341-352): target = last edge-like term
                target = None
                for t in (pred.lhs, pred.rhs):
                    if t.kind in ("edge", "etime", "eattr"):
                        target = t.name
                if n_gate == _lib.VM_MAX_PREDS:
                    raise _Unsupported(f"cell {i}: too many gate predicates")
                c.gate[n_gate] = _lower_pred(pred, _sym_id(target) if target else -1, vocab, table)
                n_gate += 1
        c.n_node, c.n_edge, c.n_gate = n_node, n_edge, n_gate
        if len(cell.order_preds) > _lib.VM_MAX_PREDS:
            raise _Unsupported(f"cell {i}: too many order constraints")
        osyms = set()
        for q, pred in enumerate(cell.order_preds):
            c.order[q][0] = _CMP[pred.op]
            for side, t in ((1, pred.lhs), (2, pred.rhs)):
                if t.kind == "trigger_time":
                    c.order[q][side] = -1
                elif t.kind == "etime":
                    c.order[q][side] = _sym_id(t.name)
                    osyms.add(t.name)
                else:
                    raise _Unsupported(f"cell {i}: order term {t.kind}")
        if len(osyms) > 4:
            raise _Unsupported(f"cell {i}: order constraints over more than 4 symbols")
        c.n_order = len(cell.order_preds)
        var[cell.dst_var] = 2 + i
    for k, b in enumerate(table):
        prog.table[k] = b
    prog.uses_attrs = 1 if uses_attrs else 0
    return VmProgram(getattr(plan, "name", "?"), prog, attribution == "members", uses_attrs)


# ---------------------------------------------------------------------------
# calls


def _prepare(dgraph, vp: VmProgram) -> None:
    if vp.uses_attrs:
        dgraph.ensure_attrs()


def vm_mine(dgraph, vp: VmProgram, lo: int = 0, hi: int | None = None):
    """Trigger-attribution counts of rows [lo, hi) (engine.py:607-646)."""
    import numpy as np
    hi = dgraph.edge_count if hi is None else hi
    out = np.zeros(hi - lo, dtype=np.int64)
    if hi <= lo:
        return out
    with dgraph.lock:
        _prepare(dgraph, vp)
        _lib.check(_lib.load().tm_vm_mine(dgraph.handle, ctypes.byref(vp.prog), lo, hi, _lib.ptr(out)),
                   "tm_vm_mine")
    return out


def vm_members(dgraph, vp: VmProgram, lo: int = 0, hi: int | None = None):
    """Members attribution (engine.py:629-640): the full n_edges column."""
    import numpy as np
    hi = dgraph.edge_count if hi is None else hi
    out = np.zeros(dgraph.edge_count, dtype=np.int64)
    if dgraph.edge_count == 0:
        return out
    with dgraph.lock:
        _prepare(dgraph, vp)
        _lib.check(_lib.load().tm_vm_members(dgraph.handle, ctypes.byref(vp.prog), lo, hi, _lib.ptr(out)),
                   "tm_vm_members")
    return out


def vm_instance_stream(dgraph, vp: VmProgram, plan_index: int, lo: int, hi: int):
    """Raw instance records of rows [lo, hi) (tm_collect_instances format)."""
    import numpy as np
    if hi <= lo:
        return np.zeros(0, dtype=np.int32)
    lib = _lib.load()
    words = ctypes.c_int64()
    with dgraph.lock:  # collect + fetch share the graph's record buffer: one unit
        _prepare(dgraph, vp)
        _lib.check(lib.tm_vm_collect(dgraph.handle, ctypes.byref(vp.prog), plan_index, lo, hi,
                                     ctypes.byref(words)), "tm_vm_collect")
        buf = np.empty(words.value, dtype=np.int32)
        _lib.check(lib.tm_fetch_instances(dgraph.handle, _lib.ptr(buf), words.value), "tm_fetch_instances")
    return buf
