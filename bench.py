#!/usr/bin/env python
"""Benchmark: transactions mined/s, full pattern set (C = 14), on B200.

One step = one pass of the mining stage over every trigger edge of the
workload graph (all 14 feature columns for all E edges), graph resident in
HBM, output int64 (E, 14) in HBM; for N > 1 the edge range is split into N
equal chunks (one per rank) and the columns are assembled on every GPU by one
NCCL all-gather.  `value` = E / max-over-ranks step time.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config hi-small]
    python bench.py --impl reference ...   # CPU oracle port on the host cores

Prints ONE JSON line (rank 0).  See DESIGN.md §Measurement.
"""

from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
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


def log(*a):
    print(*a, file=sys.stderr, flush=True)


def args_parse():
    p = argparse.ArgumentParser()
    p.add_argument("--gpus", type=int, default=1)
    p.add_argument("--steps", type=int, default=10)
    p.add_argument("--warmup", type=int, default=3)
    p.add_argument("--config", default="hi-small", choices=["cfg1", "hi-small", "hi-medium", "hi-large"])
    p.add_argument("--impl", default="ours", choices=["ours", "reference"])
    p.add_argument("--cpu-seconds", type=float, default=12.0, help="CPU baseline sample budget")
    p.add_argument("--no-cpu-baseline", action="store_true")
    p.add_argument("--no-e2e", action="store_true")
    p.add_argument("--pieces", type=int, default=4, help="N > 1: pipelined all-gather pieces")
    return p.parse_args()


def workload(name: str):
    from paper_2604_12241_b200 import synth
    cfg = synth.CONFIGS[name]
    t0 = time.perf_counter()
    g = synth.time_ordered(synth.generate(cfg))
    log(f"[bench] generated {name}: {g.edge_count} edges, {g.node_count} nodes in "
        f"{time.perf_counter() - t0:.1f}s")
    return cfg, g


def workload_config(name, cfg, g, n_cols):
    return {"workload": name, "n_nodes": int(g.node_count), "n_edges": int(g.edge_count),
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
# CPU baseline / reference arm: the oracle port (oracle/tm_oracle.c), which
# restates the reference's per-trigger algorithm, on all host threads


_ORACLE = {}


def cpu_sample(g, names, budget_s: float, seed: int = 0):
    """Time the oracle on random contiguous 1000-trigger blocks until the
    budget is spent.  Returns (edges_per_s, rows, seconds, blocks, build_s);
    the CPU graph build is done once and not timed."""
    from oracle.oracle import OracleGraph, column
    t0 = time.perf_counter()
    if id(g) not in _ORACLE:
        _ORACLE[id(g)] = OracleGraph(g.src, g.dst, g.time, node_count=g.node_count)
    og = _ORACLE[id(g)]
    build_s = time.perf_counter() - t0
    cols = [column(n, DELTA) for n in names]
    rng = np.random.default_rng(seed)
    rows = blocks = 0
    spent = 0.0
    threads = os.cpu_count() or 1
    while spent < budget_s and blocks < 4096:
        lo = int(rng.integers(0, max(1, g.edge_count - 1000)))
        hi = min(lo + 1000, g.edge_count)
        t = time.perf_counter()
        og.mine(cols, lo, hi, threads=threads)
        spent += time.perf_counter() - t
        rows += hi - lo
        blocks += 1
    return rows / spent, rows, spent, blocks, build_s


def run_reference(a):
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return 0
    import paper_2604_12241_b200 as tmb
    cfg, g = workload(a.config)
    names = list(tmb.FULL_PATTERN_SET)
    per_step = max(2.0, min(10.0, 150.0 / max(1, a.steps + a.warmup)))
    vals = []
    for step in range(a.warmup + a.steps):
        v, rows, spent, blocks, build_s = cpu_sample(g, names, per_step, seed=step)
        if step >= a.warmup:
            vals.append((v, rows, spent, blocks))
    value = float(np.mean([v for v, *_ in vals]))
    ms = float(np.mean([s / r * g.edge_count * 1e3 for _, r, s, _ in vals]))
    cores = os.cpu_count() or 1
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": a.gpus,
        "steps": a.steps, "warmup": a.warmup, "ms_per_step": ms, "higher_is_better": True,
        "scaling": "strong", "vs_baseline": None, "dtype": "int64",
        "data": "synthetic (reference synth model)",
        "config": workload_config(a.config, cfg, g, len(names)),
        "cpu_baseline": {"value": value, "unit": UNIT, "cores": cores, "kind": "port",
                         "sample": f"per step: random contiguous 1000-trigger blocks of the {a.config} "
                                   f"graph, all 14 columns, ~{per_step:.0f}s of CPU work; "
                                   f"ms_per_step extrapolated to all {g.edge_count} triggers"},
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)
    return 0


# ---------------------------------------------------------------------------


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

    cfg, g0 = workload(a.config)
    plans = tmb.full_pattern_set(DELTA)
    plans, descs = tmb.lower_all(plans)
    C = len(descs)
    E = g0.edge_count
    chunk = (E + world - 1) // world
    lo, hi = min(rank * chunk, E), min((rank + 1) * chunk, E)
    # N > 1: interleaved pieces, each piece's all-gather overlaps the next
    # piece's mining (distributed.piece_bounds)
    from paper_2604_12241_b200.distributed import piece_bounds
    pieces = a.pieces if world > 1 else 1
    P, sub, pbounds = piece_bounds(E, world, pieces)
    rows_local = sum(h - l for l, h in pbounds[rank]) if world > 1 else hi - lo

    t0 = time.perf_counter()
    g = tmb.DeviceGraph(g0.src, g0.dst, g0.time, node_count=g0.node_count, device=dev)
    torch.cuda.synchronize()
    build_s = time.perf_counter() - t0
    info = g.info()
    log(f"[bench] rank {rank}: graph built in {build_s:.2f}s, {info.device_bytes / 2**30:.2f} GiB, "
        f"max out/in degree {info.max_out_degree}/{info.max_in_degree}, rows [{lo},{hi})")

    # a non-default stream: its handle is non-NULL, so the library launches on
    # it (NULL would select the graph's own stream) and the events below see
    # exactly the mining kernels' stream
    stream = torch.cuda.Stream()
    torch.cuda.set_stream(stream)
    out_local = torch.empty((chunk, C), dtype=torch.int64, device="cuda")
    out_pieces = torch.zeros((pieces, sub, C), dtype=torch.int64, device="cuda") if world > 1 else None
    out_full = torch.empty((pieces * P, C), dtype=torch.int64, device="cuda") if world > 1 else None
    flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
    _lib.check(_lib.load().tm_set_profiling(g.handle, 1), "tm_set_profiling")

    step_ms, light_ms, heavy_ms, heavy_n, mine_ms = [], [], [], [], []
    launches = 0
    clocks = None
    for step in range(a.warmup + a.steps):
        timed = step >= a.warmup
        if timed and step == a.warmup:
            if world > 1:
                dist.barrier()
            torch.cuda.synchronize()
            sampler = ClockSampler(dev)
        flush.zero_()
        ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        evm = torch.cuda.Event(enable_timing=True)
        c0 = _lib.kernel_launch_count()
        ev0.record(stream)
        if world == 1:
            tmb.mine_rows_device(g, descs, lo, hi, out_local.data_ptr(), stream.cuda_stream)
            evm.record(stream)
        else:
            works = []
            for p in range(pieces):
                plo, phi = pbounds[rank][p]
                if phi > plo:
                    tmb.mine_rows_device(g, descs, plo, phi, out_pieces[p].data_ptr(), stream.cuda_stream)
                # NCCL waits for this stream, then gathers while the next piece is mined
                works.append(dist.all_gather_into_tensor(out_full[p * P:(p + 1) * P], out_pieces[p],
                                                         async_op=True))
            evm.record(stream)  # all pieces mined (gathers may still run)
            for w in works:
                w.wait()
        ev1.record(stream)
        ev1.synchronize()
        st = tmb.last_stats(g)
        if timed:
            launches += _lib.kernel_launch_count() - c0
            step_ms.append(ev0.elapsed_time(ev1))
            mine_ms.append(ev0.elapsed_time(evm))
            light_ms.append(st.light_ms)
            heavy_ms.append(st.heavy_ms)
    torch.cuda.synchronize()
    clocks = sampler.stop()
    total_ms = float(np.sum(step_ms))
    compute_ms = float(np.sum(mine_ms))
    if world > 1:
        t = torch.tensor([total_ms, compute_ms], dtype=torch.float64, device="cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        total_ms, compute_ms = float(t[0].item()), float(t[1].item())
    ms_per_step = total_ms / a.steps
    value = E / (ms_per_step / 1e3)

    # roofline of the dominant kernel (compulsory-bytes model)
    peak, peak_src = peaks()
    b_edge = 16 + 24 + 8 * C + 8 * (g0.node_count + 1) / E
    rows = rows_local
    lm, hm = float(np.mean(light_ms)), float(np.mean(heavy_ms))
    dom_name, dom_ms = ("k_mine_warp", lm) if lm >= hm else ("k_mine_tasks+finalize", hm)
    achieved = rows * b_edge / (dom_ms / 1e3) / 1e9
    traffic = None
    tfile = ROOT / "profiles" / "ncu_traffic.json"
    if tfile.exists():
        tj = json.loads(tfile.read_text())
        ent = tj.get(a.config, {}).get(dom_name)
        if ent:
            traffic = ent.get("dram_bytes")
    roofline = {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s",
                "frac": achieved / peak, "traffic": traffic, "kernel": dom_name,
                "kernel_ms": dom_ms, "warp_kernel_ms": lm, "task_kernels_ms": hm,
                "bytes_per_edge": b_edge, "peak_source": peak_src,
                "step_frac": E * b_edge / (ms_per_step / 1e3) / 1e9 / peak,
                "model": "compulsory bytes per trigger = 16 (src,dst,t) + 24 (one out + one in CSR "
                         "entry) + 8*C (features) + 8(N+1)/E (indptr), SURVEY.md §8d"}

    # end-to-end through the public API: pinned host arrays -> build -> mine -> host
    e2e = None
    if not a.no_e2e:
        pin = lambda x: torch.from_numpy(np.ascontiguousarray(x, dtype=np.int64)).pin_memory().numpy()
        hs, hd, ht = pin(g0.src), pin(g0.dst), pin(g0.time)
        hout = torch.empty((hi - lo, C), dtype=torch.int64).pin_memory().numpy()
        e2e_ms = []
        n_e2e = max(1, min(a.steps, 5))
        for step in range(2 + n_e2e):  # two untimed warm-up builds (pool, pinned pages)
            if world > 1:
                dist.barrier()
            t = time.perf_counter()
            ge = tmb.DeviceGraph(hs, hd, ht, node_count=g0.node_count, device=dev)
            tmb.mine_rows(ge, descs, lo, hi, out=hout)
            dt = (time.perf_counter() - t) * 1e3
            ge.free()
            if step >= 2:
                e2e_ms.append(dt)
        em = float(np.mean(e2e_ms))
        if world > 1:
            t = torch.tensor([em], dtype=torch.float64, device="cuda")
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            em = float(t.item())
        e2e = {"value": E / (em / 1e3), "unit": UNIT, "h2d_bytes_per_step": 24 * E * world,
               "d2h_bytes_per_step": 8 * E * C, "ms_per_step": em,
               "step_ms": [round(x, 3) for x in e2e_ms], "median_ms": float(np.median(e2e_ms)),
               "includes": "H2D of src/dst/time (pinned), GPU CSR build, mining, D2H of the int64 "
                           "feature block (pinned)"}
    cpu = None
    if rank == 0 and world == 1 and not a.no_cpu_baseline:
        try:
            names = [p.name for p in plans]
            v, r, s, blocks, build_cpu = cpu_sample(g0, names, a.cpu_seconds)
            cpu = {"value": v, "unit": UNIT, "cores": os.cpu_count() or 1, "kind": "port",
                   "sample": f"{blocks} random contiguous 1000-trigger blocks ({r} triggers) of the "
                             f"same graph, all {C} columns, {s:.1f}s; oracle/tm_oracle.c on "
                             f"{os.cpu_count()} threads (CPU graph build {build_cpu:.1f}s untimed)"}
        except Exception as exc:  # reported, never substituted for the GPU number
            cpu = {"value": None, "unit": UNIT, "cores": os.cpu_count() or 1, "kind": "port",
                   "sample": f"failed: {exc}"}

    if rank == 0:
        line = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": a.steps,
            "warmup": a.warmup, "ms_per_step": ms_per_step, "higher_is_better": True,
            "scaling": "strong", "vs_baseline": None, "dtype": "int64",
            "data": "synthetic (reference synth model: power-law sources, uniform dst/time, planted "
                    "instances; edge ids time-ordered)",
            "config": dict(workload_config(a.config, cfg, g0, C),
                           parallelism=(f"edge ranges x{world}, {pieces} interleaved pieces, NCCL all-gather "
                                        f"per piece overlapped with mining" if world > 1 else "1 GPU"),
                           graph_build_s=build_s, graph_device_gib=info.device_bytes / 2**30),
            "roofline": roofline, "cpu_baseline": cpu, "e2e": e2e,
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
    return 0


if __name__ == "__main__":
    sys.exit(main())
