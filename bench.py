#!/usr/bin/env python
"""Benchmark: transactions mined/s, full pattern set (C = 14), on B200.

One step = one pass of the mining stage over every trigger edge of the
workload graph (all 14 feature columns for all E edges), graph resident in
HBM, output int64 (E, 14) in HBM; for N > 1 each rank takes a contiguous
edge range (prepared once per step: its time slabs only), mined in pieces
whose NCCL all-gathers overlap the next piece's mining.  `value` = E / max-over-ranks
step time.  Default workload: the north-star HI-Large shape
(BASELINE.json:north_star, ~180 M transactions) on 1 B200.

After the timed steps the GPU output is checked against the CPU oracle
(oracle/tm_oracle.c, pinned to the reference's own outputs) on >= 1024
random 1000-trigger blocks of the same graph — the reference's _mine_range
seam (engine.py:607-646); the oracle's time on those blocks is the
cpu_baseline.  Any mismatch: the JSON line still prints, exit status 1.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config hi-large]
    python bench.py --impl reference ...   # CPU oracle port on the host cores

Prints ONE JSON line (rank 0).  See DESIGN.md §6.
"""

from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
import tempfile
import threading
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

METRIC = "transactions mined/sec, full pattern set, 1/2/4/8 B200; % HBM roofline"
UNIT = "edges/s"
DELTA = 86400
FALLBACK_HBM = 6650.0  # /opt/skills/guides/B200_PROFILING.md fallback, GB/s
# per-family breakdown (report per-family fractions)
FAMILIES = {
    "streaming": ["fan_in", "fan_out", "deg_in_src", "deg_out_src", "deg_in_dst", "deg_out_dst", "cycle_2"],
    "cycles_3_6": ["cycle_3", "cycle_4", "cycle_5", "cycle_6"],
    "sg": ["sg_count"],
    "gs": ["gs_count"],
    "stack": ["stack_count"],
}


def log(*a):
    print(*a, file=sys.stderr, flush=True)


def args_parse():
    p = argparse.ArgumentParser()
    p.add_argument("--gpus", type=int, default=1)
    p.add_argument("--steps", type=int, default=10)
    p.add_argument("--warmup", type=int, default=3)
    p.add_argument("--config", default="hi-large", choices=["cfg1", "hi-small", "hi-medium", "hi-large"])
    p.add_argument("--impl", default="ours", choices=["ours", "reference"])
    p.add_argument("--cpu-seconds", type=float, default=12.0, help="CPU baseline sample budget (s)")
    p.add_argument("--parity-blocks", type=int, default=1024, help="sampled 1000-trigger blocks checked")
    p.add_argument("--no-parity", action="store_true", help="skip the oracle check (and cpu_baseline)")
    p.add_argument("--no-e2e", action="store_true")
    p.add_argument("--e2e-steps", type=int, default=10)
    p.add_argument("--no-families", action="store_true")
    p.add_argument("--pieces", type=int, default=4, help="N > 1: pipelined all-gather pieces")
    p.add_argument("--wide", action="store_true", help="N > 1: int64 transport (default int32 + flags)")
    return p.parse_args()


def generate(name: str):
    from paper_2604_12241_b200 import synth
    cfg = synth.CONFIGS[name]
    t0 = time.perf_counter()
    g = synth.time_ordered(synth.generate(cfg))
    log(f"[bench] generated {name}: {g.edge_count} edges, {g.node_count} nodes in "
        f"{time.perf_counter() - t0:.1f}s")
    return cfg, g


class Workload:
    """Edge arrays of the synthetic graph (what every rank's replica is built from)."""

    def __init__(self, cfg, src, dst, time_, node_count):
        self.cfg, self.src, self.dst, self.time, self.node_count = cfg, src, dst, time_, node_count
        self.edge_count = len(src)


def workload(name: str, rank: int = 0, world: int = 1, dist=None) -> Workload:
    """Generate once: with N > 1 rank 0 generates and the other ranks map its
    arrays (no per-rank 180 M-edge regeneration)."""
    from paper_2604_12241_b200 import synth
    if world == 1:
        cfg, g = generate(name)
        return Workload(cfg, g.src, g.dst, g.time, g.node_count)
    tag = f"tmb_{name}_{os.environ.get('MASTER_PORT', '0')}"
    base = Path(tempfile.gettempdir())
    if rank == 0:
        cfg, g = generate(name)
        for k in ("src", "dst", "time"):
            np.save(base / f"{tag}_{k}.npy", getattr(g, k))
    dist.barrier()
    arr = {k: np.load(base / f"{tag}_{k}.npy", mmap_mode="r") for k in ("src", "dst", "time")}
    cfg = synth.CONFIGS[name]
    n = int(max(arr["src"].max(), arr["dst"].max())) + 1
    w = Workload(cfg, np.ascontiguousarray(arr["src"]), np.ascontiguousarray(arr["dst"]),
                 np.ascontiguousarray(arr["time"]), max(n, cfg.node_count))
    dist.barrier()
    if rank == 0:
        for k in ("src", "dst", "time"):
            (base / f"{tag}_{k}.npy").unlink(missing_ok=True)
    return w


def workload_config(name, w: Workload, n_cols):
    cfg = w.cfg
    return {"workload": name, "n_nodes": int(w.node_count), "n_edges": int(w.edge_count),
            "columns": n_cols, "delta": DELTA, "powerlaw_alpha": cfg.powerlaw_exponent,
            "horizon_ticks": cfg.time_horizon, "seed": cfg.seed, "edge_order": "time-ordered",
            "pattern_set": "fan_in/out, deg x4, cycle_2..6, sg_count, gs_count, stack_count",
            "l2": "flushed (256 MiB device write) before every timed step"}


def peaks():
    p = ROOT / "MEASURED_PEAKS.json"
    if p.exists():
        d = json.loads(p.read_text())
        return float(d["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)"
    return FALLBACK_HBM, "fallback (B200_PROFILING.md)"


def bytes_per_edge(n_cols: int, n_nodes: int, n_edges: int) -> float:
    """SURVEY §8d compulsory bytes per trigger: 16 (src, dst, t) + 24 (one
    out + one in CSR entry) + 8 C (features) + 8 (N + 1) / E (indptr)."""
    return 16 + 24 + 8 * n_cols + 8 * (n_nodes + 1) / max(n_edges, 1)


def cpu_model() -> str:
    try:
        for line in Path("/proc/cpuinfo").read_text().splitlines():
            if line.startswith("model name"):
                return line.split(":", 1)[1].strip()
    except OSError:
        pass
    return "unknown"


class ClockSampler:
    """SM clock + clock-event reasons sampled DURING the timed region.

    NVML (nvidia_ml_py) polled every ~2 ms from a thread — the timed region
    of a short run is tens of milliseconds, too short for nvidia-smi's
    100 ms loop; nvidia-smi is the fallback."""

    REASONS = {"sw_power_cap": 0x4, "hw_slowdown": 0x8, "sw_thermal_slowdown": 0x20,
               "hw_thermal_slowdown": 0x40, "hw_power_brake_slowdown": 0x80}

    def __init__(self, device: int):
        self.rows = []
        self.stop_flag = False
        self.nvml = None
        try:
            import pynvml
            pynvml.nvmlInit()
            self.nvml = pynvml
            self.h = pynvml.nvmlDeviceGetHandleByIndex(device)
            self.max_mhz = pynvml.nvmlDeviceGetMaxClockInfo(self.h, pynvml.NVML_CLOCK_SM)
        except Exception:
            self.nvml = None
        self.t = threading.Thread(target=self._poll, daemon=True)
        self.t.start()

    def _poll(self):
        while not self.stop_flag:
            if self.nvml is not None:
                try:
                    sm = self.nvml.nvmlDeviceGetClockInfo(self.h, self.nvml.NVML_CLOCK_SM)
                    rs = self.nvml.nvmlDeviceGetCurrentClocksEventReasons(self.h)
                    self.rows.append((sm, rs))
                except Exception:
                    pass
                time.sleep(0.002)
            else:
                try:
                    out = subprocess.run(["nvidia-smi", "--query-gpu=clocks.sm,clocks.max.sm",
                                          "--format=csv,noheader,nounits"], capture_output=True,
                                         text=True, timeout=5).stdout.split(",")
                    self.max_mhz = float(out[1])
                    self.rows.append((float(out[0]), 0))
                except Exception:
                    return

    def stop(self):
        self.stop_flag = True
        self.t.join(timeout=5)
        if not self.rows:
            return None
        sm = [r[0] for r in self.rows]
        reasons = sorted({k for _, rs in self.rows for k, bit in self.REASONS.items() if rs & bit})
        return {"sm_mhz": float(np.median(sm)), "sm_max_mhz": float(self.max_mhz), "reasons": reasons,
                "samples": len(self.rows), "source": "nvml" if self.nvml is not None else "nvidia-smi"}


# ---------------------------------------------------------------------------
# the CPU oracle (oracle/tm_oracle.c): parity checker, cpu_baseline and the
# reference arm — never on the measured GPU path


_ORACLE = {}


def oracle_graph(w: Workload):
    from oracle.oracle import OracleGraph
    t0 = time.perf_counter()
    if id(w) not in _ORACLE:
        _ORACLE[id(w)] = OracleGraph(w.src, w.dst, w.time, node_count=w.node_count)
    return _ORACLE[id(w)], time.perf_counter() - t0


def sample_blocks(n_edges: int, n_blocks: int, seed: int, size: int = 1000) -> list[tuple[int, int]]:
    rng = np.random.default_rng(seed)
    out = []
    for _ in range(n_blocks):
        lo = int(rng.integers(0, max(1, n_edges - size)))
        out.append((lo, min(lo + size, n_edges)))
    return out


def oracle_blocks(w: Workload, names, blocks, threads: int):
    """Oracle rows of each block, and the seconds spent mining them."""
    from oracle.oracle import column
    og, _ = oracle_graph(w)
    cols = [column(n, DELTA) for n in names]
    res, spent = [], 0.0
    for lo, hi in blocks:
        t = time.perf_counter()
        res.append(og.mine(cols, lo, hi, threads=threads))
        spent += time.perf_counter() - t
    return res, spent


def run_reference(a):
    """--impl reference: the reference's CPU algorithm (the pinned C port, on
    all host threads) on the same workload; rank 0 only."""
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return 0
    import paper_2604_12241_b200 as tmb
    w = workload(a.config)
    names = list(tmb.FULL_PATTERN_SET)
    og, build_s = oracle_graph(w)
    threads = os.cpu_count() or 1
    per_step = max(2.0, min(6.0, 90.0 / max(1, a.steps + a.warmup)))
    vals = []
    for step in range(a.warmup + a.steps):
        blocks, rows, spent, k = [], 0, 0.0, 0
        while spent < per_step:
            bl = sample_blocks(w.edge_count, 16, seed=1000 * step + k)
            k += 1
            _, s = oracle_blocks(w, names, bl, threads)
            spent += s
            rows += sum(h - l for l, h in bl)
            blocks += bl
        if step >= a.warmup:
            vals.append((rows / spent, rows, spent, len(blocks)))
    value = float(np.mean([v for v, *_ in vals]))
    ms = float(np.mean([s / r * w.edge_count * 1e3 for _, r, s, _ in vals]))
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": a.gpus,
        "steps": a.steps, "warmup": a.warmup, "ms_per_step": ms, "higher_is_better": True,
        "scaling": "strong", "vs_baseline": None, "dtype": "int64",
        "data": "synthetic (reference synth model)",
        "config": workload_config(a.config, w, len(names)),
        "cpu_baseline": {"value": value, "unit": UNIT, "cores": threads, "kind": "port",
                         "cpu": cpu_model(),
                         "sample": f"per step: random contiguous 1000-trigger blocks of the {a.config} "
                                   f"graph, all 14 columns, ~{per_step:.0f}s of CPU work on {threads} threads "
                                   f"(oracle/tm_oracle.c, the reference's algorithm restated in C and pinned "
                                   f"to its outputs); ms_per_step extrapolated to all {w.edge_count} triggers; "
                                   f"CPU graph build {build_s:.1f}s untimed"},
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)
    return 0


# ---------------------------------------------------------------------------


def timed_mine(tmb, g, descs, lo, hi, out, stream, flush, steps, warmup, sampler_dev=None):
    """CUDA-event times (ms) of `steps` full mining calls after `warmup`, L2
    flushed before each; returns (step_ms, warp_kernel_ms, launches, clocks)."""
    import torch
    from paper_2604_12241_b200 import _lib
    step_ms, light_ms, prep_ms, heavy_ms = [], [], [], []
    launches = 0
    sampler = None
    for step in range(warmup + steps):
        timed = step >= warmup
        if timed and step == warmup:
            torch.cuda.synchronize()
            if sampler_dev is not None:
                sampler = ClockSampler(sampler_dev)
        flush.zero_()
        ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        c0 = _lib.kernel_launch_count()
        ev0.record(stream)
        tmb.mine_rows_device(g, descs, lo, hi, out.data_ptr(), stream.cuda_stream)
        ev1.record(stream)
        ev1.synchronize()
        st = tmb.last_stats(g)
        if timed:
            launches += _lib.kernel_launch_count() - c0
            step_ms.append(ev0.elapsed_time(ev1))
            light_ms.append(st.light_ms)
            prep_ms.append(st.prep_ms)
            heavy_ms.append(st.heavy_ms)
    clocks = sampler.stop() if sampler else None
    timed_mine.parts = {"prep_ms": float(np.mean(prep_ms)), "task_kernels_ms": float(np.mean(heavy_ms))}
    return step_ms, light_ms, launches, clocks


timed_mine.parts = None


def main():
    a = args_parse()
    if a.impl == "reference":
        return run_reference(a)

    import torch
    import torch.distributed as dist

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world > 1:
        torch.cuda.set_device(local)
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    else:
        torch.cuda.set_device(0)
    dev = torch.cuda.current_device()

    import paper_2604_12241_b200 as tmb
    from paper_2604_12241_b200 import _lib

    w = workload(a.config, rank, world, dist if world > 1 else None)
    plans = tmb.full_pattern_set(DELTA)
    plans, descs = tmb.lower_all(plans)
    names = [p.name for p in plans]
    C = len(descs)
    E = w.edge_count
    pieces = a.pieces if world > 1 else 1
    narrow = world > 1 and not a.wide

    # page-locked edge arrays (as a loader would hand them over): the build
    # below and the e2e steps read them
    pin = lambda x: torch.from_numpy(np.ascontiguousarray(x, dtype=np.int64)).pin_memory().numpy()
    hs, hd, ht = pin(w.src), pin(w.dst), pin(w.time)
    t0 = time.perf_counter()
    g = tmb.DeviceGraph(hs, hd, ht, node_count=w.node_count, device=dev)
    torch.cuda.synchronize()
    build_s = time.perf_counter() - t0
    info = g.info()
    log(f"[bench] rank {rank}: graph built in {build_s:.2f}s, {info.device_bytes / 2**30:.2f} GiB, "
        f"max out/in degree {info.max_out_degree}/{info.max_in_degree}")

    # a non-default stream: its handle is non-NULL, so the library launches on
    # it (NULL would select the graph's own stream) and the events below see
    # exactly the mining kernels' stream
    stream = torch.cuda.Stream()
    torch.cuda.set_stream(stream)
    flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
    _lib.check(_lib.load().tm_set_profiling(g.handle, 1), "tm_set_profiling")

    if world == 1:
        out = torch.empty((E, C), dtype=torch.int64, device="cuda")
        step_ms, light_ms, launches, clocks = timed_mine(tmb, g, descs, 0, E, out, stream, flush, a.steps,
                                                         a.warmup, sampler_dev=dev)
        total_ms = compute_ms = float(np.sum(step_ms))
        full_out = out
    else:
        from paper_2604_12241_b200.distributed import mine_pipelined
        step_ms, light_ms, mine_ms = [], [], []
        launches = 0
        sampler = None
        full_out = None
        for step in range(a.warmup + a.steps):
            timed = step >= a.warmup
            if timed and step == a.warmup:
                dist.barrier()
                torch.cuda.synchronize()
                sampler = ClockSampler(dev)
            flush.zero_()
            ev0, ev1, evm = (torch.cuda.Event(enable_timing=True) for _ in range(3))
            c0 = _lib.kernel_launch_count()
            ev0.record(stream)
            # one step: prepare this rank's window tables / slab views (its
            # contiguous trigger range), mine its pieces, gather each piece
            # while the next is mined, reorder into the final rows
            full_out = mine_pipelined(
                E, C, rank, world,
                lambda lo, hi, o: tmb.mine_rows_device(g, descs, lo, hi, o.data_ptr(), stream.cuda_stream),
                pieces=pieces, device="cuda", narrow=narrow,
                prepare=lambda lo, hi: tmb.prepare_views(g, descs, lo, hi, stream.cuda_stream),
                on_mined=lambda: evm.record(stream))
            tmb.release_views(g)
            ev1.record(stream)
            ev1.synchronize()
            st = tmb.last_stats(g)
            if timed:
                launches += _lib.kernel_launch_count() - c0
                step_ms.append(ev0.elapsed_time(ev1))
                mine_ms.append(ev0.elapsed_time(evm))
                light_ms.append(st.light_ms)
        torch.cuda.synchronize()
        clocks = sampler.stop()
        t = torch.tensor([float(np.sum(step_ms)), float(np.sum(mine_ms))], dtype=torch.float64, device="cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        total_ms, compute_ms = float(t[0].item()), float(t[1].item())
    ms_per_step = total_ms / a.steps
    value = E / (ms_per_step / 1e3)

    # roofline (compulsory-bytes model): the whole mining step
    # is the unit — every kernel of the step (window tables, k_mine_warp, task
    # rounds) is charged, none is credited with another's bytes
    peak, peak_src = peaks()
    b_edge = bytes_per_edge(C, w.node_count, E)
    lm = float(np.mean(light_ms))
    step_alone_ms = compute_ms / a.steps  # mining only (N > 1: gathers excluded)
    achieved = E / world * b_edge / (step_alone_ms / 1e3) / 1e9 if world > 1 else E * b_edge / (ms_per_step / 1e3) / 1e9
    traffic = None
    tfile = ROOT / "profiles" / "ncu_traffic.json"
    if tfile.exists():
        ent = json.loads(tfile.read_text()).get(a.config, {})
        if ent.get("step_dram_bytes"):
            traffic = ent["step_dram_bytes"]
    roofline = {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s", "frac": achieved / peak,
                "traffic": traffic, "kernel": "mining step (k_own_windows + k_mine_warp + task rounds)",
                "step_ms": step_alone_ms, "warp_kernel_ms": lm,
                "prep_ms": (timed_mine.parts or {}).get("prep_ms"),
                "task_kernels_ms": (timed_mine.parts or {}).get("task_kernels_ms"),
                "prep": "per call: rank-window tables + the time-slab view of the dual CSR (tm_slab.cu)",
                "warp_kernel_share": lm / step_alone_ms if step_alone_ms > 0 else None,
                "bytes_per_edge": b_edge, "peak_source": peak_src,
                "traffic_source": "profiles/ncu_traffic.json: dram__bytes_read.sum + dram__bytes_write.sum "
                                  "summed over the step's kernels (ncu --set full, one step)",
                "model": "compulsory bytes per trigger = 16 (src,dst,t) + 24 (one out + one in CSR "
                         "entry) + 8*C (features) + 8(N+1)/E (indptr), SURVEY.md §8d; E x B / step time"}

    # per-family fractions, 1 GPU: each family mined alone
    families = None
    if world == 1 and not a.no_families:
        families = {}
        for fam, cols in FAMILIES.items():
            fdescs = [d for d, n in zip(descs, names) if n in cols]
            fout = torch.empty((E, len(fdescs)), dtype=torch.int64, device="cuda")
            fms, flm, _, _ = timed_mine(tmb, g, fdescs, 0, E, fout, stream, flush, max(3, a.steps // 2), 2)
            del fout
            fb = bytes_per_edge(len(fdescs), w.node_count, E)
            fstep = float(np.mean(fms))
            families[fam] = {"columns": cols, "ms_per_step": fstep, "edges_per_s": E / (fstep / 1e3),
                             "warp_kernel_ms": float(np.mean(flm)), "bytes_per_edge": fb,
                             "frac": E * fb / (fstep / 1e3) / 1e9 / peak}
            log(f"[bench] family {fam}: {fstep:.2f} ms, frac {families[fam]['frac']:.3f}")
        torch.cuda.synchronize()

    # parity on sampled blocks + the CPU baseline on the same blocks (rank 0)
    parity = cpu = None
    if rank == 0 and not a.no_parity:
        threads = os.cpu_count() or 1
        og, build_cpu = oracle_graph(w)
        blocks = sample_blocks(E, a.parity_blocks, seed=2604)
        want, spent = oracle_blocks(w, names, blocks, threads)
        # keep sampling for the CPU baseline until its budget is spent
        extra = 0
        while world == 1 and spent < a.cpu_seconds:
            more = sample_blocks(E, 64, seed=9000 + extra)
            extra += 1
            rws, s = oracle_blocks(w, names, more, threads)
            blocks += more
            want += rws
            spent += s
        # only the sampled rows come back to the host
        idx = torch.from_numpy(np.concatenate([np.arange(lo, hi) for lo, hi in blocks])).to(full_out.device)
        got = full_out.index_select(0, idx).cpu().numpy()
        bad_rows = 0
        bad_cols = set()
        at = 0
        for (lo, hi), wv in zip(blocks, want):
            diff = got[at:at + hi - lo] != wv
            at += hi - lo
            if diff.any():
                bad_rows += int(diff.any(axis=1).sum())
                bad_cols.update(names[j] for j in np.nonzero(diff.any(axis=0))[0])
        rows = sum(h - l for l, h in blocks)
        parity = {"blocks": len(blocks), "rows": rows, "mismatches": bad_rows, "bad_columns": sorted(bad_cols),
                  "checker": "oracle/tm_oracle.c (CPU restatement pinned to the reference's outputs, "
                             "tests/test_oracle_golden.py) on random 1000-trigger blocks, all columns, "
                             "bit-exact int64"}
        if world == 1:
            cpu = {"value": rows / spent, "unit": UNIT, "cores": threads, "kind": "port", "cpu": cpu_model(),
                   "sample": f"{len(blocks)} random contiguous 1000-trigger blocks ({rows} triggers) of the "
                             f"same graph, all {C} columns, {spent:.1f}s on {threads} threads; "
                             f"oracle/tm_oracle.c (CPU graph build {build_cpu:.1f}s untimed)"}
        log(f"[bench] parity: {bad_rows} mismatching rows of {rows} ({len(blocks)} blocks)")

    # end to end through the drop-in API: pinned host edge arrays -> mine()
    # (H2D + GPU CSR build + mining + D2H into the pinned FeatureMatrix)
    e2e = None
    if not a.no_e2e:
        from types import SimpleNamespace

        from paper_2604_12241_b200 import hostmem
        from paper_2604_12241_b200.distributed import mine_distributed
        lab = np.full(E, -1, dtype=np.int8)
        e2e_ms = []
        for step in range(2 + a.e2e_steps):  # two untimed warm-up calls (pool, pinned pages)
            if world > 1:
                dist.barrier()
            # a fresh graph object every step: mine() uploads and builds it
            host_graph = SimpleNamespace(edge_src=hs, edge_dst=hd, edge_time=ht, node_count=w.node_count,
                                         edge_label=lab)
            t = time.perf_counter()
            if world == 1:
                fm = tmb.mine(host_graph, plans)
            else:
                fm = mine_distributed(host_graph, plans, pieces=pieces, narrow=narrow)
            dt = (time.perf_counter() - t) * 1e3
            fm.device_graph.free()
            del fm, host_graph
            if step >= 2:
                e2e_ms.append(dt)
        em, med = float(np.mean(e2e_ms)), float(np.median(e2e_ms))
        if world > 1:
            t = torch.tensor([em, med], dtype=torch.float64, device="cuda")
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            em, med = float(t[0].item()), float(t[1].item())
        e2e = {"value": E / (em / 1e3), "unit": UNIT, "h2d_bytes_per_step": 24 * E * world,
               "d2h_bytes_per_step": 8 * E * C * world, "ms_per_step": em, "median_ms": med,
               "median_value": E / (med / 1e3), "max_over_median": float(np.max(e2e_ms)) / med,
               "step_ms": [round(x, 3) for x in e2e_ms],
               "pinned_pool": dict(hostmem.stats),
               "api": "paper_2604_12241_b200.mine(graph, plans)" if world == 1 else
                      "paper_2604_12241_b200.distributed.mine_distributed(graph, plans)",
               "includes": "H2D of src/dst/time (pinned), GPU CSR build, mining, D2H of the int64 "
                           "feature block into the FeatureMatrix (pinned host pool)"}

    if rank == 0:
        line = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": a.steps,
            "warmup": a.warmup, "ms_per_step": ms_per_step, "higher_is_better": True,
            "scaling": "strong", "vs_baseline": None, "dtype": "int64",
            "data": "synthetic (reference synth model: power-law sources, uniform dst/time, planted "
                    "instances; edge ids time-ordered)",
            "config": dict(workload_config(a.config, w, C),
                           parallelism=(f"contiguous edge range per rank (its slabs prepared once per step), "
                                        f"{pieces} pieces, NCCL all-gather "
                                        f"({'int32 + overflow flags' if narrow else 'int64'}) per piece "
                                        f"overlapped with mining" if world > 1 else "1 GPU"),
                           graph_build_s=build_s, graph_build="H2D of pinned src/dst/time + GPU CSR, pair "
                           "indexes, ranks (tm_graph_build)", graph_device_gib=info.device_bytes / 2**30),
            "roofline": roofline, "families": families, "parity": parity, "cpu_baseline": cpu, "e2e": e2e,
            "gpu_launches": int(launches), "clocks": clocks,
            # scaling with and without the feature all-gather
            "compute_only": {"value": E / (compute_ms / a.steps / 1e3), "unit": UNIT,
                             "ms_per_step": compute_ms / a.steps,
                             "note": "mining only (max over ranks), all-gather excluded"},
        }
        print(json.dumps(line), flush=True)
    g.free()
    if world > 1:
        dist.destroy_process_group()
    if parity is not None and parity["mismatches"]:
        return 1
    return 0


if __name__ == "__main__":
    sys.exit(main())
