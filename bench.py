#!/usr/bin/env python
"""Benchmark of the fused ragged paged attention (the Pensieve hot path) on B200.

A "step" is one attention pass over every layer of the model for one ragged batch
(n_layer launches of pb_attn_run, each layer with its own KV pools), inputs resident in HBM.
Default workload: BASELINE config 4 (Llama-2-70B GQA-8, 64 conversations, mixed prefill +
decode, 80 layers) — the config the north star scales across GPUs by KV head.  With N ranks
the kv heads are sharded (8/N per rank, the same spans and block tables everywhere, no
collective on the attention path): total work is fixed, so scaling is "strong".

  python bench.py [--gpus N] [--steps K] [--warmup W] [--config C] [--layers L]
  python bench.py --impl reference ...   # the reference CPU implementation (oracle/_ref)

Prints one JSON line (rank 0).  Timing: CUDA events on the launching stream, barrier +
synchronize on both sides, max over ranks.  Per-step inputs (n_layer x pool bytes) are far
larger than the 126 MB L2, so no explicit flush is needed.
"""
from __future__ import annotations

import argparse
import json
import math
import os
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

MODEL_LAYERS = {1: 1, 2: 40, 3: 40, 4: 80}
UNITS = {1: "GB/s", 2: "GB/s", 3: "GB/s", 4: "TFLOP/s"}
FALLBACK_PEAKS = {"hbm_gbs": 6650.0, "bf16_tflops": 1590.0, "bf16_tflops_sustained": 1400.0}


def load_peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        d = json.load(open(p))
        return d, "measured (MEASURED_PEAKS.json)"
    return FALLBACK_PEAKS, "fallback (B200_PROFILING.md)"


def dist_env():
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return rank, world, local


class ClockSampler:
    """nvidia-smi clocks + throttle reasons during the timed region (B200_PROFILING.md)."""

    FIELDS = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.hw_slowdown,"
              "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
              "clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int):
        self.index = index
        self.proc = None
        self.lines = []

    def start(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.FIELDS}", "--format=csv,noheader,nounits",
                 "-lms", "100"], stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except (FileNotFoundError, OSError):
            self.proc = None

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def stop(self):
        if not self.proc:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except subprocess.TimeoutExpired:
            self.proc.kill()
        sm, mx, reasons = [], [], set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in self.lines:
            parts = [x.strip() for x in ln.split(",")]
            if len(parts) < 7:
                continue
            try:
                sm.append(float(parts[0]))
                mx.append(float(parts[1]))
            except ValueError:
                continue
            for n, v in zip(names, parts[3:7]):
                if v.lower().startswith("active"):
                    reasons.add(n)
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": sorted(reasons), "samples": len(sm)}


def select_cpu_sample(w, threads: int, budget_s: float):
    """Bounded, deterministic sample of spans for the CPU reference (~budget_s of work at
    ~0.1 GFLOP/s per thread, measured for this code in this container)."""
    from paper_2312_05516_b200.workloads import SplitMix64
    order = list(range(len(w.spans)))
    rng = SplitMix64(99)
    for i in range(len(order), 1, -1):
        j = rng.next() % i
        order[i - 1], order[j] = order[j], order[i - 1]
    budget = budget_s * 0.1e9 * max(1, threads)
    chosen, acc = [], 0.0
    for i in order:
        fl, _ = w.flops_bytes([i])
        if acc + fl <= budget:
            chosen.append(i)
            acc += fl
    if not chosen:
        chosen = [min(order, key=lambda i: w.flops_bytes([i])[0])]
    return sorted(chosen)


def run_reference_cpu(w, threads: int, budget_s: float, reps: int = 1):
    """The reference's own paged_multi_token_attention (oracle/_ref), per sub-request on
    `threads` host threads, over a bounded span sample.  Returns (seconds, flops, bytes, ids)."""
    import numpy as np

    from oracle.oracle import Reference

    ids = select_cpu_sample(w, threads, budget_s)
    shape, batch, q, keys, values = w.compact_host_inputs(ids)
    ref = Reference()
    store = ref.store(shape.chunk_size, shape.n_kv_head, shape.head_size, shape.n_slots, keys, values)
    try:
        best = None
        for _ in range(reps):
            t0 = time.perf_counter()
            st, _ = ref.attention_mt(store, shape, batch, q, threads)
            dt = time.perf_counter() - t0
            assert st == 0, st
            best = dt if best is None else min(best, dt)
    finally:
        ref.destroy_store(store)
    fl, by = w.flops_bytes(ids)
    return best, fl, by, ids


def metric_value(unit, flops, bytes_, seconds):
    return (flops / seconds / 1e12) if unit == "TFLOP/s" else (bytes_ / seconds / 1e9)


def bench_reference(args):
    rank, world, _ = dist_env()
    if rank != 0:
        return 0
    from paper_2312_05516_b200.workloads import config
    w = config(args.config)
    unit = UNITS[args.config]
    threads = os.cpu_count() or 1
    vals = []
    ids = None
    for s in range(args.warmup + args.steps):
        sec, fl, by, ids = run_reference_cpu(w, threads, args.cpu_budget)
        if s >= args.warmup:
            vals.append(metric_value(unit, fl, by, sec))
    v = statistics.median(vals)
    line = {
        "impl": "reference", "metric": f"ragged paged-attn {unit} (reference CPU kvsim::paged_multi_token_attention)",
        "value": v, "unit": unit, "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
        "higher_is_better": True, "dtype": "f32 (bf16-rounded inputs, double accumulation)",
        "data": "synthetic (SplitMix64, workloads.config)",
        "config": {"workload": w.name, "sample_spans": len(ids)},
        "cpu_baseline": {"value": v, "unit": unit, "cores": threads, "kind": "reference",
                         "sample": f"{len(ids)} of {len(w.spans)} spans (one layer), per-span std::thread split"},
        "e2e": {"value": v, "unit": unit, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)
    return 0


def bench_ours(args):
    import torch
    import torch.distributed as dist

    from paper_2312_05516_b200 import abi
    from paper_2312_05516_b200.abi import PB_BF16, AttentionPlan
    from paper_2312_05516_b200.workloads import config

    rank, world, local = dist_env()
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if world > 1:
        dist.init_process_group("nccl", device_id=dev)
    w = config(args.config)
    n_layer = args.layers or MODEL_LAYERS[args.config]
    unit = UNITS[args.config]
    if w.n_kv_head % world:
        raise SystemExit(f"n_kv_head {w.n_kv_head} not divisible by {world} ranks")
    nkv = w.n_kv_head // world
    # every rank gets rank 0's span/block-table descriptors (the same migration plan,
    # PAPER.md:741-744) and its own kv-head shard; no collective touches the attention
    from paper_2312_05516_b200.sharding import broadcast_batch, shard_shape
    shape = shard_shape(w.shape(), rank, world)
    batch = broadcast_batch(w.batch() if rank == 0 else None) if world > 1 else w.batch()
    dt = torch.bfloat16 if w.dtype == PB_BF16 else torch.float32
    eb = 2 if w.dtype == PB_BF16 else 4
    row = nkv * w.head_size
    pool_elems = w.n_slots * w.chunk * row
    q_elems = w.total_tokens * shape.n_head * w.head_size
    # pools for every layer; rank r holds kv heads [r*nkv, (r+1)*nkv) (synthetic draws offset by rank)
    pools_k, pools_v = [], []
    for l in range(n_layer):
        k = torch.empty(pool_elems, dtype=dt, device=dev)
        v = torch.empty(pool_elems, dtype=dt, device=dev)
        abi.fill_unit(k.data_ptr(), w.dtype, pool_elems, w.seed + 7919 * rank, 2 * l * pool_elems)
        abi.fill_unit(v.data_ptr(), w.dtype, pool_elems, w.seed + 7919 * rank, (2 * l + 1) * pool_elems)
        pools_k.append(k)
        pools_v.append(v)
    q = torch.empty(q_elems, dtype=dt, device=dev)
    abi.fill_unit(q.data_ptr(), w.dtype, q_elems, w.seed + 104729, 0)
    out = torch.empty_like(q)
    stream = torch.cuda.current_stream()
    sh = stream.cuda_stream
    plan = AttentionPlan(shape, batch)
    plan.upload(sh)
    ws = torch.zeros(max(1, plan.workspace_bytes()), dtype=torch.uint8, device=dev)
    stats = plan.stats()

    def step():
        for l in range(n_layer):
            plan.run(q.data_ptr(), pools_k[l].data_ptr(), pools_v[l].data_ptr(), out.data_ptr(),
                     ws.data_ptr(), sh)

    def barrier():
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()

    for _ in range(max(3, args.warmup)):
        step()
    barrier()
    # ---- timed region: K steps, per-layer events for the dominant kernel's duration ----
    clocks = ClockSampler(local)
    clocks.start()
    n_ev = args.steps * n_layer
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(n_ev + 1)]
    launches0 = abi.launch_count()
    barrier()
    ev[0].record(stream)
    i = 0
    for _ in range(args.steps):
        for l in range(n_layer):
            plan.run(q.data_ptr(), pools_k[l].data_ptr(), pools_v[l].data_ptr(), out.data_ptr(),
                     ws.data_ptr(), sh)
            i += 1
            ev[i].record(stream)
    barrier()
    launches = abi.launch_count() - launches0
    total_ms = ev[0].elapsed_time(ev[n_ev])
    per_launch = [ev[j].elapsed_time(ev[j + 1]) for j in range(n_ev)]
    clk = clocks.stop()
    t = torch.tensor([total_ms], device=dev, dtype=torch.float64)
    if world > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    ms_per_step = float(t.item()) / args.steps

    # ---- e2e through the C-ABI with host buffers: plan build+upload, per-layer H2D q and
    # D2H out from pinned memory, every step ----
    q_host = torch.empty(q_elems, dtype=dt, pin_memory=True)
    q_host.copy_(q.cpu())
    out_host = torch.empty(q_elems, dtype=dt, pin_memory=True)
    e2e_steps = max(2, min(args.steps, 10))
    barrier()
    e0 = torch.cuda.Event(enable_timing=True)
    e1 = torch.cuda.Event(enable_timing=True)
    t0 = time.perf_counter()
    e0.record(stream)
    for _ in range(e2e_steps):
        p2 = AttentionPlan(shape, batch)
        p2.upload(sh)
        for l in range(n_layer):
            q.copy_(q_host, non_blocking=True)
            p2.run(q.data_ptr(), pools_k[l].data_ptr(), pools_v[l].data_ptr(), out.data_ptr(), ws.data_ptr(), sh)
            out_host.copy_(out, non_blocking=True)
        stream.synchronize()
    e1.record(stream)
    barrier()
    wall = time.perf_counter() - t0
    te = torch.tensor([wall], device=dev, dtype=torch.float64)
    if world > 1:
        dist.all_reduce(te, op=dist.ReduceOp.MAX)
    e2e_s = float(te.item()) / e2e_steps
    desc_bytes = 32 * batch.n_spans + 4 * int(batch.bt_off[-1]) + 40 * (stats["prefill_tiles"] + stats["decode_units"] + stats["simt_tiles"])

    if rank != 0:
        if world > 1:
            dist.destroy_process_group()
        return 0

    # whole-job work: every rank computes its kv-head shard of every layer
    fl_layer, by_layer = w.flops_bytes()
    value = metric_value(unit, fl_layer * n_layer, by_layer * n_layer, ms_per_step / 1e3)
    e2e_value = metric_value(unit, fl_layer * n_layer, by_layer * n_layer, e2e_s)
    peaks, peak_src = load_peaks()
    # dominant kernel: one layer's attention launch on rank 0 (its shard)
    avg_launch_s = statistics.mean(per_launch) / 1e3
    if unit == "TFLOP/s":
        achieved = stats["flops"] / avg_launch_s / 1e12
        peak = peaks.get("bf16_tflops_sustained", peaks["bf16_tflops"])
        roof = {"bound": "tensor", "achieved": achieved, "peak": peak, "unit": "TFLOP/s"}
    else:
        achieved = stats["bytes"] / avg_launch_s / 1e9
        peak = peaks["hbm_gbs"]
        roof = {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s"}
    roof["frac"] = achieved / peak
    roof["traffic"] = load_traffic(w.name)
    roof["peak_source"] = peak_src
    roof["per_launch_us"] = avg_launch_s * 1e6
    roof["hbm_gbs"] = stats["bytes"] / avg_launch_s / 1e9
    roof["tflops"] = stats["flops"] / avg_launch_s / 1e12

    cpu = None
    if not args.no_cpu_baseline:
        threads = os.cpu_count() or 1
        sec, fl, by, ids = run_reference_cpu(w, threads, args.cpu_budget)
        cpu = {"value": metric_value(unit, fl, by, sec), "unit": unit, "cores": threads, "kind": "reference",
               "sample": f"{len(ids)} of {len(w.spans)} spans, one layer, all {shape.n_head * world} heads; "
                         f"{sec:.2f} s wall on {threads} threads"}
    line = {
        "metric": f"ragged paged-attn {unit} (fused prefill+decode, {n_layer} layers/step)",
        "value": value, "unit": unit, "n_gpus": world, "steps": args.steps, "warmup": max(3, args.warmup),
        "ms_per_step": ms_per_step, "higher_is_better": True, "scaling": "strong",
        "vs_baseline": None, "dtype": "bf16" if w.dtype == PB_BF16 else "f32",
        "data": "synthetic (SplitMix64 fill on device; random-init KV pools per layer)",
        "config": {"workload": w.name, "n_layer": n_layer, "spans": len(w.spans), "tokens": w.total_tokens,
                   "n_head": w.n_head, "n_kv_head": w.n_kv_head, "head_size": w.head_size, "page_tokens": w.chunk,
                   "parallelism": f"kv-head shard x{world}",
                   "l2": "inputs larger than L2 (per step: n_layer pools)",
                   "plan": {k: stats[k] for k in ("prefill_tiles", "decode_units", "split_spans", "simt_tiles")}},
        "roofline": roof,
        "cpu_baseline": cpu,
        "e2e": {"value": e2e_value, "unit": unit,
                "h2d_bytes_per_step": n_layer * q_elems * eb + desc_bytes,
                "d2h_bytes_per_step": n_layer * q_elems * eb},
        "gpu_launches": int(launches),
        "clocks": clk,
    }
    print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()
    return 0


def load_traffic(name):
    p = os.path.join(ROOT, "profiles", "traffic.json")
    if os.path.exists(p):
        return json.load(open(p)).get(name)
    return None


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--config", type=int, default=4, choices=[1, 2, 3, 4])
    ap.add_argument("--layers", type=int, default=0)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--cpu-budget", type=float, default=12.0, help="seconds of CPU reference work")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    args = ap.parse_args()
    if args.impl == "reference":
        return bench_reference(args)
    return bench_ours(args)


if __name__ == "__main__":
    sys.exit(main())
