"""Synthetic IBM-AML-shaped transaction graphs (vectorized, array output).

Same generative model and the same PCG64 draw sequence as the reference
generator (synth.py:73-163): power-law source weights k^-alpha over a seeded
permutation `hub_order`, uniform destinations redrawn until dst != src,
uniform integer timestamps, then planted sg / cycle / stack instances
appended after the background.  The reference builds one Python record per
edge; this module returns numpy arrays, so HI-Medium / HI-Large shapes
 can be generated on the GPU box.  For cfg1 the arrays are
bit-identical to synth.generate (pinned by tests/golden/cfg1.npz hashes).
"""

from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np

PLANT_KINDS = ("sg_count", "cycle_2", "cycle_3", "cycle_4", "stack_count")


@dataclass(frozen=True)
class PlantSpec:
    kind: str
    count: int
    fanout: tuple = (3, 8)
    span: int = 3600


@dataclass(frozen=True)
class SynthConfig:
    node_count: int
    background_edge_count: int
    time_horizon: int
    seed: int = 7
    plants: tuple = ()
    label_planted: bool = True
    powerlaw_exponent: float = 2.1


@dataclass
class SynthGraph:
    src: np.ndarray
    dst: np.ndarray
    time: np.ndarray
    amount: np.ndarray
    label: np.ndarray  # int8, -1 unlabeled
    node_count: int
    truth_triggers: np.ndarray
    config: SynthConfig = field(repr=False)

    @property
    def edge_count(self) -> int:
        return len(self.src)


def _plants_for(scale: int) -> tuple:
    return (PlantSpec("sg_count", 2 * scale), PlantSpec("cycle_2", scale), PlantSpec("cycle_3", scale),
            PlantSpec("cycle_4", scale), PlantSpec("stack_count", scale))


# SURVEY.md §8d table; † horizons / alpha are the survey's stated assumptions
CONFIGS = {
    "cfg1": SynthConfig(10_000, 100_000, 16 * 86400, seed=7,
                        plants=(PlantSpec("sg_count", 100), PlantSpec("cycle_2", 50),
                                PlantSpec("cycle_3", 50), PlantSpec("cycle_4", 50),
                                PlantSpec("stack_count", 50))),
    "hi-small": SynthConfig(515_088, 5_078_345, 10 * 86400, seed=2604, plants=_plants_for(500),
                            powerlaw_exponent=1.0),
    "hi-medium": SynthConfig(2_077_023, 31_898_238, 16 * 86400, seed=2604, plants=_plants_for(3000),
                             powerlaw_exponent=1.0),
    "hi-large": SynthConfig(2_116_168, 179_702_229, 97 * 86400, seed=2604, plants=_plants_for(17500),
                            powerlaw_exponent=1.0),
}


def generate(config: SynthConfig) -> SynthGraph:
    """Background + planted edges; deterministic under config.seed."""
    if config.node_count <= 1:
        raise ValueError("node_count must be at least 2")
    rng = np.random.Generator(np.random.PCG64(config.seed))
    n = config.node_count
    weights = np.arange(1, n + 1, dtype=np.float64) ** (-config.powerlaw_exponent)
    weights /= weights.sum()
    hub_order = rng.permutation(n)
    m = config.background_edge_count
    src = hub_order[rng.choice(n, size=m, p=weights)]
    del weights
    dst = rng.integers(0, n, size=m)
    clash = src == dst
    while clash.any():
        dst[clash] = rng.integers(0, n, size=int(clash.sum()))
        clash = src == dst
    times = rng.integers(0, config.time_horizon, size=m)
    amounts = np.round(rng.uniform(10.0, 10000.0, size=m), 2)

    ps, pd, pt, triggers = [], [], [], []
    eid = m
    for plant in config.plants:
        lo, hi = plant.fanout
        for _ in range(plant.count):
            span = plant.span
            t0 = int(rng.integers(0, config.time_horizon - span))
            es, ed, et = [], [], []
            if plant.kind == "sg_count":
                f = int(rng.integers(lo, hi + 1))
                nodes = rng.choice(n, size=f + 2, replace=False)
                s, d = int(nodes[0]), int(nodes[1])
                mids = nodes[2:].tolist()
                for i, mid in enumerate(mids):
                    es.append(s); ed.append(mid); et.append(t0 + i)
                for i, mid in enumerate(mids):
                    es.append(mid); ed.append(d); et.append(t0 + span // 2 + i)
            elif plant.kind.startswith("cycle_"):
                length = int(plant.kind.split("_")[1])
                nodes = rng.choice(n, size=length, replace=False).tolist()
                step = max(1, span // length)
                for i in range(length):
                    es.append(nodes[i]); ed.append(nodes[(i + 1) % length]); et.append(t0 + i * step)
            elif plant.kind == "stack_count":
                f_in = int(rng.integers(lo, hi + 1))
                f_out = int(rng.integers(lo, hi + 1))
                nodes = rng.choice(n, size=f_in + f_out + 2, replace=False).tolist()
                u, v = nodes[0], nodes[1]
                for i, a in enumerate(nodes[2:2 + f_in]):
                    es.append(a); ed.append(u); et.append(t0 + i)
                for j, c in enumerate(nodes[2 + f_in:]):
                    es.append(v); ed.append(c); et.append(t0 + span // 2 + j)
                es.append(u); ed.append(v); et.append(t0 + span)
            else:
                raise ValueError(f"unknown plant kind {plant.kind}")
            ids = list(range(eid, eid + len(es)))
            # trigger = temporally last member, (timestamp, edge id) order
            triggers.append(max(ids, key=lambda e, et=et, base=eid: (et[e - base], e)))
            eid += len(es)
            ps += es; pd += ed; pt += et
    n_plant = len(ps)
    all_src = np.concatenate([src, np.asarray(ps, dtype=np.int64)])
    all_dst = np.concatenate([dst, np.asarray(pd, dtype=np.int64)])
    all_time = np.concatenate([times, np.asarray(pt, dtype=np.int64)])
    plant_ids = np.arange(m, m + n_plant)
    plant_amount = amounts[plant_ids % max(m, 1)] if m else np.round(10 + (plant_ids % 9990) * 1.0, 2)
    all_amount = np.concatenate([amounts, plant_amount])
    if config.label_planted:
        label = np.concatenate([np.zeros(m, dtype=np.int8), np.ones(n_plant, dtype=np.int8)])
    else:
        label = np.full(m + n_plant, -1, dtype=np.int8)
    return SynthGraph(all_src.astype(np.int64), all_dst.astype(np.int64), all_time.astype(np.int64),
                      all_amount, label, n, np.asarray(triggers, dtype=np.int64), config)


def stable_time_order(t: np.ndarray) -> np.ndarray:
    """np.argsort(t, kind="stable"), fast for large logs: when (t - min) * E + id
    fits int64 the (time, id) keys are distinct, so an unstable sort of them
    gives the same permutation (numpy's stable int64 argsort is a merge sort:
    75 s at HI-Large; this is ~10 s)."""
    E = len(t)
    if E == 0:
        return np.zeros(0, dtype=np.int64)
    t0, t1 = int(t.min()), int(t.max())
    if (t1 - t0 + 1) * E >= 2**62:
        return np.argsort(t, kind="stable")
    key = (t - t0).astype(np.int64)
    key *= E
    key += np.arange(E, dtype=np.int64)
    key.sort()
    key %= E
    return key


def time_ordered(g: SynthGraph) -> SynthGraph:
    """Re-number edge ids in (time, old id) order — a time-ordered transaction
    log.  Counts per edge are unchanged up to the renumbering."""
    order = stable_time_order(g.time)
    inv = np.empty_like(order)
    inv[order] = np.arange(len(order))
    return SynthGraph(g.src[order], g.dst[order], g.time[order], g.amount[order], g.label[order],
                      g.node_count, inv[g.truth_triggers] if len(g.truth_triggers) else g.truth_triggers,
                      g.config)
