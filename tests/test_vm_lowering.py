"""Host half of the GENERIC stage VM: lowering compiled plans (the
reference's own compile_pattern output, tests/golden/vm.npz) into
tm_vm_program structs.  No GPU needed."""

from __future__ import annotations

import ctypes
import json

import numpy as np
import pytest

from conftest import load_npz
from paper_2604_12241_b200 import _lib
from paper_2604_12241_b200 import plan as P
from paper_2604_12241_b200.vm import lower_program


def _plans():
    z = load_npz("vm.npz")
    return [P.plan_from_dict(d) for d in json.loads(str(z["plans"]))]


def test_every_fixture_program_lowers():
    vocab = ("USD", "EUR", "GBP", "CHF")
    for p in _plans():
        vp = lower_program(p, vocab)
        assert vp.prog.n_cells == len(p.cells)
        assert vp.prog.min_size == p.emission.min_size
        for i, cell in enumerate(p.cells):
            assert vp.prog.cells[i].parent == cell.parent
            assert vp.prog.cells[i].n_ops == len(cell.src)


def test_predicate_classification_and_typing():
    byname = {p.name: p for p in _plans()}
    vocab = ("USD", "EUR", "GBP", "CHF")
    g = lower_program(byname["gate_cur"], vocab).prog
    c = g.cells[0]
    # e0.amount > 700 gates the stage; e1.currency != "USD" filters entries
    assert (c.n_gate, c.n_edge, c.n_node) == (1, 1, 0)
    assert c.gate[0].sym == 0 and c.gate[0].lk == 3 and c.gate[0].rk == 0 and c.gate[0].rnum == 700.0
    t = c.edge[0].table
    assert t >= 0 and [g.table[t + i] for i in range(4)] == [0, 1, 1, 1]
    a = lower_program(byname["gate_anc"], vocab).prog
    assert a.cells[1].n_gate == 1 and a.cells[1].gate[0].sym == 1  # ancestor symbol e1
    o = lower_program(byname["ord_cycle3"], vocab).prog.cells[1]
    assert o.n_order == 3 and [o.order[2][k] for k in range(3)] == [2, 3, -1]  # e3.t <= t
    f = lower_program(byname["fwd_fan"], vocab).prog
    assert f.cells[0].forward == 1 and f.mode == 3 and f.min_size == 2
    n = lower_program(byname["nest_self"], vocab).prog
    assert [n.cells[i].parent for i in range(4)] == [-1, 0, 1, 1]
    kinds = {(n.cells[2].ops[k].kind, n.cells[2].ops[k].var) for k in range(2)}
    assert kinds == {(1, 2), (3, 3)}  # A.self (A bound) and B.out_neigh (member adjacency)


def test_currency_predicate_needs_vocabulary():
    byname = {p.name: p for p in _plans()}
    with pytest.raises(_lib.UnsupportedPlanError):
        lower_program(byname["gate_cur"], None)


def test_struct_layout_matches_header():
    assert ctypes.sizeof(_lib.TmVmPred) == 48
    assert ctypes.sizeof(_lib.TmVmCell) == 1072
    assert ctypes.sizeof(_lib.TmVmProgram) == 9632


def test_limits_raise_unsupported():
    import dataclasses
    p = _plans()[0]
    big = dataclasses.replace(p, cells=p.cells * 9, slot_count=len(p.cells) * 9)
    with pytest.raises(_lib.UnsupportedPlanError):
        lower_program(big)
