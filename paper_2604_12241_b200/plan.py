"""Execution plans and their lowering onto the GPU families.

Two kinds of plan objects reach `mine`:

* the reference's own `tempmine.plan.ExecutionPlan` (compile_pattern,
  plan.py:134-187) — the drop-in case: a user keeps the reference's DSL
  front-end and swaps `mine`;
* this module's structurally identical dataclasses, built by
  `builtin_plan(name, ...)` for the 11 builtins (patterns/*.pat) and the
  extended families cycle_5..8 / gs_count, so the
  engine is usable without the reference installed.

`lower_plan` maps either to a `PlanDesc` (the C-ABI tm_plan_desc).  A hinted
plan is dispatched exactly as `_kernel_fn` does (engine.py:569-589: FAN /
DEGREE read cells[0].src[0].base/.direction, CYCLE_n its length, emission
min_size).  A GENERIC plan — custom DSL, `force_generic=True`, or one of the
extended families, which the reference only runs on its interpreter — is
matched structurally on its compiled cells with the analyst-chosen names
erased (the reference does the same on the DSL, plan.py:194-229).  Anything
else raises UnsupportedPlanError: there is no CPU fallback.
"""

from __future__ import annotations

from dataclasses import dataclass, field

from ._lib import (TM_CYCLE, TM_DEGREE, TM_FAN, TM_GS, TM_SG, TM_STACK, TM_E_UNSUPPORTED_PLAN,
                   UnsupportedPlanError)

GENERIC = "GENERIC"
FAN = "FAN"
DEGREE = "DEGREE"
CYCLE_2 = "CYCLE_2"
CYCLE_3 = "CYCLE_3"
CYCLE_4 = "CYCLE_4"
SCATTER_GATHER = "SCATTER_GATHER"
STACK = "STACK"

# plan.py:28-33 — CSV column contract, builtin order
BUILTIN_COLUMNS = (
    "fan_in", "fan_out",
    "deg_in_src", "deg_out_src", "deg_in_dst", "deg_out_dst",
    "cycle_2", "cycle_3", "cycle_4",
    "sg_count", "stack_count",
)
# north-star families the reference only runs on its generic interpreter
EXTENDED_COLUMNS = ("cycle_5", "cycle_6", "cycle_7", "cycle_8", "gs_count")
# the headline "full pattern set" (BASELINE.json config 1): C = 14
FULL_PATTERN_SET = BUILTIN_COLUMNS + ("cycle_5", "cycle_6", "gs_count")

BUILTIN_DELTA = 604800  # every shipped .pat file (patterns/*.pat)

# ---------------------------------------------------------------------------
# plan dataclasses (field-for-field the reference's, plan.py:40-91, dsl.py:80-118)


@dataclass(frozen=True)
class Term:
    kind: str
    name: str = ""
    attr: str = ""
    value: float | str = 0


@dataclass(frozen=True)
class ConstraintExpr:
    kind: str
    lhs: Term
    op: str
    rhs: Term


@dataclass(frozen=True)
class OperandDesc:
    kind: str
    base: str
    slot: int
    direction: str = ""
    symbol: str | None = None


@dataclass(frozen=True)
class LoopCell:
    op: str
    src: tuple
    dst_slot: int
    dst_var: str
    parent: int
    skip_preds: tuple
    order_preds: tuple
    window_lo: str = "t-delta"
    window_hi: str = "t"


@dataclass(frozen=True)
class CompiledEmission:
    mode: str
    min_size: int
    target_slots: tuple
    target_vars: tuple


@dataclass(frozen=True)
class ExecutionPlan:
    name: str
    delta: int
    cells: tuple
    slot_count: int
    emission: CompiledEmission
    kernel_hint: str
    attribution: str = "trigger"


@dataclass(frozen=True)
class PlanDesc:
    """One tm_plan_desc (include/tempmine_b200.h)."""

    family: int
    endpoint: int = 0
    direction: int = 0
    exclude_trigger: int = 0
    cycle_len: int = 0
    min_size: int = 1
    delta: int = 0
    members: bool = False  # attribution "members" -> tm_mine_members (not a C field)


# ---------------------------------------------------------------------------
# builders


def _node(name: str) -> Term:
    return Term("node", name)


def _skip(a: str, b: str) -> ConstraintExpr:
    return ConstraintExpr("skip_if", _node(a), "==", _node(b))


class _Builder:
    def __init__(self):
        self.cells: list[LoopCell] = []
        self.var_slot: dict[str, int] = {}
        self.sym = 0

    def operand(self, base: str, accessor: str) -> OperandDesc:
        trig = base in ("N0", "N1")
        if accessor == "self":
            return OperandDesc("scalar", base, -1) if trig else OperandDesc("set", base, self.var_slot[base])
        self.sym += 1
        direction = "in" if accessor == "in_neigh" else "out"
        if trig:
            return OperandDesc("adj", base, -1, direction, f"e{self.sym}")
        return OperandDesc("member_adj", base, self.var_slot[base], direction, f"e{self.sym}")

    def stage(self, op: str, srcs, dst_var: str, skips=(), edge_skips=()):
        slot = len(self.cells)
        ops = tuple(self.operand(b, a) for b, a in srcs)
        parent = -1
        for o in ops:
            if o.kind == "member_adj":
                parent = o.slot
        preds = tuple(_skip(a, b) for a, b in skips)
        preds += tuple(ConstraintExpr("skip_if", Term("edge", ops[0].symbol), "==", Term("edge", "e0"))
                       for _ in edge_skips)
        self.cells.append(LoopCell(op, ops, slot, dst_var, parent, preds, ()))
        self.var_slot[dst_var] = slot

    def plan(self, name, delta, mode, targets, min_size, hint) -> ExecutionPlan:
        slots = tuple(self.var_slot[t] for t in targets)
        return ExecutionPlan(name, int(delta), tuple(self.cells), len(self.cells),
                             CompiledEmission(mode, int(min_size), slots, tuple(targets)), hint)


_DEGREE_SHAPES = {  # name -> (endpoint var, accessor)
    "deg_in_src": ("N0", "in_neigh"), "deg_out_src": ("N0", "out_neigh"),
    "deg_in_dst": ("N1", "in_neigh"), "deg_out_dst": ("N1", "out_neigh"),
}
_FAN_SHAPES = {"fan_in": ("N1", "in_neigh"), "fan_out": ("N0", "out_neigh")}


def _cycle_k(b: _Builder, k: int) -> None:
    chain = k - 3
    for i in range(1, chain + 1):
        skips = [("N0", "N1")] if i == 1 else []
        skips.append((f"A{i}", "N0"))
        if i >= 2:
            skips.append((f"A{i}", "N1"))
        skips += [(f"A{i}", f"A{j}") for j in range(1, i - 1)]
        b.stage("for_all", [("N1" if i == 1 else f"A{i-1}", "out_neigh")], f"A{i}", skips)
    b.stage("intersect", [(f"A{chain}", "out_neigh"), ("N0", "in_neigh")], "C",
            [("C", "N1")] + [("C", f"A{j}") for j in range(1, chain)])


def builtin_plan(name: str, delta: int | None = None, min_size: int | None = None,
                 column: str | None = None, hinted: bool = True) -> ExecutionPlan:
    """Compiled plan of a builtin (patterns/*.pat) or extended family.

    delta defaults to the shipped 604800 ticks; min_size to the pattern's
    emission default (sg_count / gs_count: 2, else 1).  `column` renames the
    output column; `hinted=False` mimics compile_pattern(force_generic=True).
    """
    delta = BUILTIN_DELTA if delta is None else int(delta)
    b = _Builder()
    if name in _FAN_SHAPES:
        base, acc = _FAN_SHAPES[name]
        b.stage("for_all", [(base, acc)], "F", edge_skips=[True])
        mode, targets, k0, hint = "edge_count", ("F",), 1, FAN
    elif name in _DEGREE_SHAPES:
        base, acc = _DEGREE_SHAPES[name]
        b.stage("for_all", [(base, acc)], "D")
        mode, targets, k0, hint = "edge_count", ("D",), 1, DEGREE
    elif name == "cycle_2":
        b.stage("intersect", [("N1", "out_neigh"), ("N0", "self")], "C")
        mode, targets, k0, hint = "set_cardinality", ("C",), 1, CYCLE_2
    elif name == "cycle_3":
        b.stage("intersect", [("N1", "out_neigh"), ("N0", "in_neigh")], "C", [("N0", "N1")])
        mode, targets, k0, hint = "set_cardinality", ("C",), 1, CYCLE_3
    elif name in ("cycle_4", "cycle_5", "cycle_6", "cycle_7", "cycle_8"):
        k = int(name.split("_")[1])
        if k == 4:
            b.stage("for_all", [("N1", "out_neigh")], "M", [("N0", "N1"), ("M", "N0")])
            b.stage("intersect", [("M", "out_neigh"), ("N0", "in_neigh")], "C", [("C", "N1")])
        else:
            _cycle_k(b, k)
        mode, targets, k0 = "set_cardinality", ("C",), 1
        hint = CYCLE_4 if k == 4 else GENERIC
    elif name == "sg_count":
        b.stage("for_all", [("N0", "in_neigh")], "S", [("S", "N1")])
        b.stage("intersect", [("S", "out_neigh"), ("N1", "in_neigh")], "M")
        mode, targets, k0, hint = "source_count", ("M",), 2, SCATTER_GATHER
    elif name == "gs_count":
        b.stage("for_all", [("N1", "out_neigh")], "D", [("D", "N0")])
        b.stage("intersect", [("D", "in_neigh"), ("N0", "out_neigh")], "M")
        mode, targets, k0, hint = "source_count", ("M",), 2, GENERIC
    elif name == "stack_count":
        b.stage("for_all", [("N0", "in_neigh")], "A", [("A", "N1")])
        b.stage("for_all", [("N1", "out_neigh")], "C", [("C", "N0")])
        mode, targets, k0, hint = "pair_product", ("A", "C"), 1, STACK
    else:
        raise KeyError(f"no builtin or extended pattern {name!r}")
    k = k0 if min_size is None else int(min_size)
    return b.plan(column or name, delta, mode, targets, k, hint if hinted else GENERIC)


def plan_from_dict(d: dict) -> ExecutionPlan:
    """Rebuild a compiled plan from dataclasses.asdict() of a reference (or
    our) ExecutionPlan — how compiled custom patterns travel as fixtures."""
    t = lambda x: Term(x["kind"], x["name"], x["attr"], x["value"])  # noqa: E731
    c = lambda x: ConstraintExpr(x["kind"], t(x["lhs"]), x["op"], t(x["rhs"]))  # noqa: E731
    cells = tuple(LoopCell(cl["op"], tuple(OperandDesc(**o) for o in cl["src"]), cl["dst_slot"],
                           cl["dst_var"], cl["parent"], tuple(c(p) for p in cl["skip_preds"]),
                           tuple(c(p) for p in cl["order_preds"]), cl["window_lo"], cl["window_hi"])
                  for cl in d["cells"])
    em = d["emission"]
    return ExecutionPlan(d["name"], d["delta"], cells, d["slot_count"],
                         CompiledEmission(em["mode"], em["min_size"], tuple(em["target_slots"]),
                                          tuple(em["target_vars"])), d["kernel_hint"],
                         d.get("attribution", "trigger"))


def load_builtin(name: str, delta: int | None = None, min_size: int | None = None) -> ExecutionPlan:
    if name not in BUILTIN_COLUMNS:
        raise KeyError(f"no builtin pattern {name!r}")
    return builtin_plan(name, delta, min_size)


def full_pattern_set(delta: int = 86400, names=FULL_PATTERN_SET) -> list[ExecutionPlan]:
    return [builtin_plan(n, delta) for n in names]


# ---------------------------------------------------------------------------
# structural canonical form (names erased)


def _canon_term(t, var_slot: dict, own_syms: dict, own_var: str):
    kind = t.kind
    if kind == "node":
        if t.name in ("N0", "N1"):
            return ("node", t.name)
        if t.name == own_var:
            return ("node", "$cand")
        return ("node", f"$s{var_slot.get(t.name, -99)}")
    if kind in ("edge", "etime", "eattr"):
        if t.name == "e0":
            return (kind, "e0", t.attr)
        return (kind, own_syms.get(t.name, "$foreign"), t.attr)
    return (kind, str(t.value))


def canonical_shape(plan) -> tuple:
    """Structure of a compiled plan with variable / edge-symbol names erased."""
    var_slot = {c.dst_var: i for i, c in enumerate(plan.cells)}
    shape = []
    for i, cell in enumerate(plan.cells):
        ops = []
        own_syms = {}
        for j, d in enumerate(cell.src):
            base = d.base if d.base in ("N0", "N1") else f"$s{d.slot}"
            ops.append((d.kind, base, d.direction or ""))
            if d.symbol:
                own_syms[d.symbol] = f"$op{base}{d.direction}"
        if cell.op in ("intersect", "union"):
            ops = sorted(ops)
        preds = []
        for p in cell.skip_preds:
            lhs = _canon_term(p.lhs, var_slot, own_syms, cell.dst_var)
            rhs = _canon_term(p.rhs, var_slot, own_syms, cell.dst_var)
            if p.op in ("==", "!=") and rhs < lhs:
                lhs, rhs = rhs, lhs
            preds.append((lhs, p.op, rhs))
        order = tuple(sorted(str(p) for p in cell.order_preds))
        shape.append((cell.op, tuple(ops), tuple(sorted(preds)), order, cell.parent,
                      cell.window_lo, cell.window_hi))
    em = plan.emission
    return (tuple(shape), em.mode, tuple(em.target_slots))


def _family_of(name: str, delta: int, k: int) -> PlanDesc:
    if name in _FAN_SHAPES or name in _DEGREE_SHAPES:
        base, acc = (_FAN_SHAPES.get(name) or _DEGREE_SHAPES[name])
        return PlanDesc(TM_FAN if name in _FAN_SHAPES else TM_DEGREE, 0 if base == "N0" else 1,
                        0 if acc == "in_neigh" else 1, 1 if name in _FAN_SHAPES else 0, 0, k, delta)
    if name.startswith("cycle_"):
        return PlanDesc(TM_CYCLE, cycle_len=int(name.split("_")[1]), min_size=k, delta=delta)
    if name == "sg_count":
        return PlanDesc(TM_SG, min_size=k, delta=delta)
    if name == "gs_count":
        return PlanDesc(TM_GS, min_size=k, delta=delta)
    if name == "stack_count":
        return PlanDesc(TM_STACK, min_size=k, delta=delta)
    raise KeyError(name)


_SHAPES: dict | None = None


def _shape_table() -> dict:
    global _SHAPES
    if _SHAPES is None:
        _SHAPES = {canonical_shape(builtin_plan(n)): n for n in BUILTIN_COLUMNS + EXTENDED_COLUMNS}
    return _SHAPES


def recognize(plan) -> str | None:
    """Family name of a structurally recognized plan, else None."""
    return _shape_table().get(canonical_shape(plan))


def lower_plan(plan) -> PlanDesc:
    """ExecutionPlan (reference or ours) -> PlanDesc; raises UnsupportedPlanError."""
    import dataclasses
    name = getattr(plan, "name", "?")
    attribution = getattr(plan, "attribution", "trigger")
    if attribution not in ("trigger", "members"):
        raise UnsupportedPlanError(TM_E_UNSUPPORTED_PLAN, f"plan {name}: unknown attribution {attribution!r}")
    desc = _lower_trigger(plan, name)
    return dataclasses.replace(desc, members=True) if attribution == "members" else desc


def _lower_trigger(plan, name) -> PlanDesc:
    delta = int(plan.delta)
    if delta < 0:
        raise ValueError(f"plan {name}: delta must be non-negative")
    k = int(plan.emission.min_size)
    if k < 1:
        raise ValueError(f"plan {name}: min_size must be >= 1")
    hint = getattr(plan, "kernel_hint", GENERIC)
    # hinted dispatch, exactly as _kernel_fn (engine.py:569-589)
    if hint in (FAN, DEGREE):
        d = plan.cells[0].src[0]
        return PlanDesc(TM_FAN if hint == FAN else TM_DEGREE, 0 if d.base == "N0" else 1,
                        0 if d.direction == "in" else 1, 1 if hint == FAN else 0, 0, k, delta)
    if hint in (CYCLE_2, CYCLE_3, CYCLE_4):
        return PlanDesc(TM_CYCLE, cycle_len={CYCLE_2: 2, CYCLE_3: 3, CYCLE_4: 4}[hint], min_size=k,
                        delta=delta)
    if hint == SCATTER_GATHER:
        return PlanDesc(TM_SG, min_size=k, delta=delta)
    if hint == STACK:
        return PlanDesc(TM_STACK, min_size=k, delta=delta)
    if hint != GENERIC:
        raise UnsupportedPlanError(TM_E_UNSUPPORTED_PLAN, f"plan {name}: unknown kernel hint {hint}")
    fam = recognize(plan)
    if fam is None:
        raise UnsupportedPlanError(
            TM_E_UNSUPPORTED_PLAN,
            f"plan {name}: GENERIC plan does not match a GPU family (fan/degree, cycle_2..8, "
            "sg, gs, stack); arbitrary DSL stage programs are not on the GPU path")
    return _family_of(fam, delta, k)
