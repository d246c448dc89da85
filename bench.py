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
larger than the 126 MB L2, so no explicit flush is needed.  At one GPU the default line also
carries `configs`: the HBM-bound configs 2 and 3 and the swap config 5 (driven over the
reference's own ShareGPT trace), each with its roofline fraction and clock record.

Both arms print the same `metric`, `unit` and `config` for a config, so the driver can divide
them; the reference arm loads only oracle/_ref/libkvsim_ref.so (the workload generators it
shares with this arm are host-only and never load the product library).
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
# one metric name per config, printed identically by both arms (BASELINE.json metric:
# "ragged paged-attn TFLOP/s & HBM GB/s vs roofline; KV swap GB/s; x CPU ref")
METRICS = {1: "ragged paged-attn HBM GB/s", 2: "ragged paged-attn HBM GB/s", 3: "ragged paged-attn HBM GB/s",
           4: "ragged paged-attn TFLOP/s"}


def bench_config(w, n_layer, world):
    """The `config` object of a config's line (identical in both arms)."""
    return {"workload": w.name, "n_layer": n_layer, "spans": len(w.spans), "tokens": w.total_tokens,
            "n_head": w.n_head, "n_kv_head": w.n_kv_head, "head_size": w.head_size, "page_tokens": w.chunk,
            "parallelism": f"kv-head shard x{world}", "l2": "inputs larger than L2 (per step: n_layer pools)"}


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
        self.lines = []  # (arrival time, line)
        self.t_begin = None

    def start(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.FIELDS}", "--format=csv,noheader,nounits",
                 "-lms", "10"], stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except (FileNotFoundError, OSError):
            self.proc = None

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append((time.time(), line.strip()))

    def wait_ready(self, timeout_s: float = 3.0):
        """Block until nvidia-smi delivers its first sample (it starts slowly)."""
        t_end = time.time() + timeout_s
        while self.proc and not self.lines and time.time() < t_end:
            time.sleep(0.01)

    def begin(self):
        """Mark the start of the timed region (start() runs earlier: nvidia-smi needs a few
        hundred ms before its first sample, longer than some timed regions)."""
        self.t_begin = time.time()

    def stop(self):
        if not self.proc:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        t_end = time.time()
        time.sleep(0.03)  # the last in-window sample reaches the reader
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except subprocess.TimeoutExpired:
            self.proc.kill()
        sm, mx, reasons = [], [], set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        t0 = self.t_begin if self.t_begin is not None else 0.0
        window = [ln for t, ln in self.lines if t0 <= t <= t_end + 0.02]
        for ln in window:
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
    """The reference's own CPU implementation (oracle/_ref: kvsim::paged_multi_token_attention
    compiled from /root/reference sources), on all host threads, on this config's workload.
    A step is one bounded sample of the workload's spans (about --cpu-budget seconds)."""
    rank, world, _ = dist_env()
    if rank != 0:
        return 0
    from paper_2312_05516_b200.workloads import config
    w = config(args.config)
    unit = UNITS[args.config]
    n_layer = args.layers or MODEL_LAYERS[args.config]
    threads = os.cpu_count() or 1
    vals, secs = [], []
    ids = None
    for s in range(args.warmup + args.steps):
        sec, fl, by, ids = run_reference_cpu(w, threads, args.cpu_budget)
        if s >= args.warmup:
            vals.append(metric_value(unit, fl, by, sec))
            secs.append(sec)
    v = statistics.median(vals)
    sample = f"{len(ids)} of {len(w.spans)} spans (one layer, all heads), per-span std::thread split"
    line = {
        "impl": "reference", "metric": METRICS[args.config],
        "value": v, "unit": unit, "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": statistics.median(secs) * 1e3, "higher_is_better": True, "scaling": "strong",
        "vs_baseline": None, "dtype": "f32 (bf16-rounded inputs, double accumulation)",
        "data": "synthetic (SplitMix64, workloads.config)",
        "config": bench_config(w, n_layer, 1),
        "cpu_baseline": {"value": v, "unit": unit, "cores": threads, "kind": "reference", "sample": sample},
        "e2e": {"value": v, "unit": unit, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
        "gpu_launches": 0,
    }
    print(json.dumps(line), flush=True)
    return 0


def measure_attention(args, cfg, n_layer, steps, warmup, rank, world, dev, with_e2e):
    """One config's attention step on this rank's kv-head shard: device-timed value, per-launch
    roofline of the dominant kernel (one layer's fused launch), and (with_e2e) the same metric
    through the C-ABI with host q/out buffers.  Returns a dict (rank 0 reports it)."""
    import torch
    import torch.distributed as dist

    from paper_2312_05516_b200 import abi
    from paper_2312_05516_b200.abi import PB_BF16, AttentionPlan
    from paper_2312_05516_b200.sharding import broadcast_batch, shard_shape
    from paper_2312_05516_b200.workloads import config

    w = config(cfg)
    unit = UNITS[cfg]
    if w.n_kv_head % world:
        raise SystemExit(f"n_kv_head {w.n_kv_head} not divisible by {world} ranks")
    nkv = w.n_kv_head // world
    # every rank gets rank 0's span/block-table descriptors (the same migration plan,
    # PAPER.md:741-744) and its own kv-head shard; no collective touches the attention
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

    # the layer loop is one CUDA graph launch per step (pb_attn_run_layers: captured during
    # the warm-up, replayed while the pointers stay the same)
    qs = [q.data_ptr()] * n_layer
    outs = [out.data_ptr()] * n_layer
    kps = [x.data_ptr() for x in pools_k]
    vps = [x.data_ptr() for x in pools_v]

    def step():
        plan.run_layers(qs, kps, vps, outs, ws.data_ptr(), sh)

    def barrier():
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()

    clocks = ClockSampler(dev.index)
    clocks.start()
    clocks.wait_ready()
    for _ in range(warmup):
        step()
    barrier()
    # ---- timed region: K steps, an event pair around each step's graph launch; the dominant
    # kernel's average launch duration is the step time over its n_layer launches (the one
    # kernel per layer, back to back inside the graph, so inter-launch gaps count against it) ----
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(steps + 1)]
    launches0 = abi.launch_count()
    barrier()
    clocks.begin()
    ev[0].record(stream)
    for i in range(steps):
        step()
        ev[i + 1].record(stream)
    barrier()
    launches = abi.launch_count() - launches0
    total_ms = ev[0].elapsed_time(ev[steps])
    per_launch = [ev[j].elapsed_time(ev[j + 1]) / n_layer for j in range(steps)]
    clk = clocks.stop()
    t = torch.tensor([total_ms], device=dev, dtype=torch.float64)
    if world > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    ms_per_step = float(t.item()) / steps
    fl_layer, by_layer = w.flops_bytes()
    res = {"w": w, "unit": unit, "n_layer": n_layer, "ms_per_step": ms_per_step, "clocks": clk,
           "gpu_launches": int(launches), "stats": stats,
           # whole-job work: every rank computes its kv-head shard of every layer
           "value": metric_value(unit, fl_layer * n_layer, by_layer * n_layer, ms_per_step / 1e3)}
    peaks, peak_src = load_peaks()
    avg_launch_s = statistics.mean(per_launch) / 1e3
    if unit == "TFLOP/s":
        achieved = stats["flops"] / avg_launch_s / 1e12
        peak = peaks.get("bf16_tflops_sustained", peaks["bf16_tflops"])
        roof = {"bound": "tensor", "achieved": achieved, "peak": peak, "unit": "TFLOP/s",
                "peak_kind": "bf16 sustained (kernel timed inside a long step)"}
    else:
        achieved = stats["bytes"] / avg_launch_s / 1e9
        peak = peaks["hbm_gbs"]
        roof = {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s", "peak_kind": "HBM copy"}
    roof["frac"] = achieved / peak
    roof["traffic"] = load_traffic(w.name)
    roof["peak_source"] = peak_src
    roof["per_launch_us"] = avg_launch_s * 1e6
    roof["hbm_gbs"] = stats["bytes"] / avg_launch_s / 1e9
    roof["tflops"] = stats["flops"] / avg_launch_s / 1e12
    res["roofline"] = roof

    if with_e2e:
        # ---- e2e through the C-ABI with host buffers, every step: plan build + upload, then
        # pb_attn_run_layers_host (per-layer H2D of q and D2H of out from pinned memory,
        # overlapped with the neighbouring layers' attention on two copy streams) ----
        q_host = torch.empty(q_elems, dtype=dt, pin_memory=True)
        q_host.copy_(q.cpu())
        out_host = torch.empty(q_elems, dtype=dt, pin_memory=True)
        e2e_steps = max(2, min(steps, 10))
        stage = torch.empty(max(1, plan.stage_bytes()), dtype=torch.uint8, device=dev)
        kp = [x.data_ptr() for x in pools_k]
        vp = [x.data_ptr() for x in pools_v]
        barrier()
        t0 = time.perf_counter()
        for _ in range(e2e_steps):
            p2 = AttentionPlan(shape, batch)
            p2.upload(sh)
            p2.run_layers_host([q_host.data_ptr()] * n_layer, [out_host.data_ptr()] * n_layer, kp, vp,
                               stage.data_ptr(), ws.data_ptr(), sh)
            stream.synchronize()
        barrier()
        wall = time.perf_counter() - t0
        te = torch.tensor([wall], device=dev, dtype=torch.float64)
        if world > 1:
            dist.all_reduce(te, op=dist.ReduceOp.MAX)
        e2e_s = float(te.item()) / e2e_steps
        desc_bytes = 32 * batch.n_spans + 4 * int(batch.bt_off[-1]) + 40 * (
            stats["prefill_tiles"] + stats["decode_units"] + stats["simt_tiles"])
        io_bytes = n_layer * q_elems * eb
        # pinned-copy peaks of this box (the e2e line is bound by these: every layer's q and
        # out cross the host link)
        h2d_peak, d2h_peak = pinned_copy_peaks(torch, dev, 1 << 28)
        res["e2e"] = {"value": metric_value(unit, fl_layer * n_layer, by_layer * n_layer, e2e_s), "unit": unit,
                      "h2d_bytes_per_step": io_bytes + desc_bytes, "d2h_bytes_per_step": io_bytes,
                      "ms_per_step": e2e_s * 1e3,
                      "link": {"h2d_gbs": (io_bytes + desc_bytes) / e2e_s / 1e9, "d2h_gbs": io_bytes / e2e_s / 1e9,
                               "pinned_h2d_peak_gbs": h2d_peak, "pinned_d2h_peak_gbs": d2h_peak,
                               "h2d_frac": (io_bytes + desc_bytes) / e2e_s / 1e9 / h2d_peak,
                               "d2h_frac": io_bytes / e2e_s / 1e9 / d2h_peak}}
        del q_host, out_host, stage
    del pools_k, pools_v, q, out, ws, plan
    torch.cuda.empty_cache()
    return res


def pinned_copy_peaks(torch, dev, nbytes):
    """cudaMemcpyAsync pinned H2D and D2H GB/s on this box (best of 3, CUDA events)."""
    big = torch.empty(nbytes, dtype=torch.uint8, device=dev)
    hbuf = torch.empty(nbytes, dtype=torch.uint8, pin_memory=True)
    big.copy_(hbuf, non_blocking=True)
    torch.cuda.synchronize()
    best = [0.0, 0.0]
    for _ in range(3):
        e = [torch.cuda.Event(enable_timing=True) for _ in range(4)]
        e[0].record(); big.copy_(hbuf, non_blocking=True); e[1].record()
        e[2].record(); hbuf.copy_(big, non_blocking=True); e[3].record()
        torch.cuda.synchronize()
        best[0] = max(best[0], nbytes / (e[0].elapsed_time(e[1]) / 1e3) / 1e9)
        best[1] = max(best[1], nbytes / (e[2].elapsed_time(e[3]) / 1e3) / 1e9)
    del big, hbuf
    return best[0], best[1]


def duplex_microbench(torch, dev, nbytes=1 << 28, reps=3):
    """Isolated PCIe/C2C duplex measurement (the paper reports an 18-20% per-direction drop
    when H2D and D2H overlap; the reference models 0.20,
    proj/include/kvsim/swap_engine.hpp:15): H2D alone, D2H alone, then both at once on two
    streams, each timed with CUDA events on its own stream."""
    dev_a = torch.empty(nbytes, dtype=torch.uint8, device=dev)
    dev_b = torch.empty(nbytes, dtype=torch.uint8, device=dev)
    h_a = torch.empty(nbytes, dtype=torch.uint8, pin_memory=True)
    h_b = torch.empty(nbytes, dtype=torch.uint8, pin_memory=True)
    s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()

    def timed(h2d, d2h):
        torch.cuda.synchronize()
        e = [torch.cuda.Event(enable_timing=True) for _ in range(4)]
        if h2d:
            e[0].record(s1)
            with torch.cuda.stream(s1):
                dev_a.copy_(h_a, non_blocking=True)
            e[1].record(s1)
        if d2h:
            e[2].record(s2)
            with torch.cuda.stream(s2):
                h_b.copy_(dev_b, non_blocking=True)
            e[3].record(s2)
        torch.cuda.synchronize()
        g = lambda a, b: nbytes / (e[a].elapsed_time(e[b]) / 1e3) / 1e9  # noqa: E731
        return (g(0, 1) if h2d else None), (g(2, 3) if d2h else None)

    timed(True, True)
    h_alone = max(timed(True, False)[0] for _ in range(reps))
    d_alone = max(timed(False, True)[1] for _ in range(reps))
    both = [timed(True, True) for _ in range(reps)]
    h_both = max(b[0] for b in both)
    d_both = max(b[1] for b in both)
    del dev_a, dev_b, h_a, h_b
    return {"bytes_each": nbytes, "h2d_alone_gbs": h_alone, "d2h_alone_gbs": d_alone,
            "h2d_concurrent_gbs": h_both, "d2h_concurrent_gbs": d_both,
            "h2d_drop": 1 - h_both / h_alone, "d2h_drop": 1 - d_both / d_alone,
            "paper_drop": "0.18-0.20 per direction (PAPER.md:760-762)", "reference_model": 0.20}


def bench_ours(args):
    import torch
    import torch.distributed as dist

    rank, world, local = dist_env()
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if world > 1:
        dist.init_process_group("nccl", device_id=dev)
    n_layer = args.layers or MODEL_LAYERS[args.config]
    warmup = max(3, args.warmup)
    r = measure_attention(args, args.config, n_layer, args.steps, warmup, rank, world, dev, with_e2e=True)
    # the other BASELINE configs at one GPU, each a sub-result with its own roofline and clocks
    # (configs 2 and 3 have 40 and 10 kv heads: not the multi-GPU workload)
    subs = {}
    if world == 1 and args.config == 4 and not args.no_subconfigs:
        for c in (2, 3):
            m = measure_attention(args, c, MODEL_LAYERS[c], args.steps, warmup, rank, world, dev, with_e2e=False)
            subs[f"cfg{c}"] = {"metric": METRICS[c], "value": m["value"], "unit": m["unit"],
                               "ms_per_step": m["ms_per_step"], "n_layer": m["n_layer"], "workload": m["w"].name,
                               "roofline": m["roofline"], "clocks": m["clocks"], "gpu_launches": m["gpu_launches"]}
        subs["cfg5"] = config5_result(args, warmup)
    if rank != 0:
        if world > 1:
            dist.destroy_process_group()
        return 0
    w = r["w"]
    unit = r["unit"]
    cpu = None
    if not args.no_cpu_baseline:
        threads = os.cpu_count() or 1
        sec, fl, by, ids = run_reference_cpu(w, threads, args.cpu_budget)
        cpu = {"value": metric_value(unit, fl, by, sec), "unit": unit, "cores": threads, "kind": "reference",
               "sample": f"{len(ids)} of {len(w.spans)} spans, one layer, all {w.n_head} heads; "
                         f"{sec:.2f} s wall on {threads} threads"}
    cfgd = bench_config(w, n_layer, world)
    line = {
        "metric": METRICS[args.config],
        "value": r["value"], "unit": unit, "n_gpus": world, "steps": args.steps, "warmup": warmup,
        "ms_per_step": r["ms_per_step"], "higher_is_better": True, "scaling": "strong",
        "vs_baseline": None, "dtype": "bf16" if w.dtype == 1 else "f32",
        "data": "synthetic (SplitMix64 fill on device; random-init KV pools per layer)",
        "config": cfgd,
        "roofline": r["roofline"],
        "plan": {k: r["stats"][k] for k in ("prefill_tiles", "decode_units", "split_spans", "simt_tiles")},
        "cpu_baseline": cpu,
        "e2e": r["e2e"],
        "gpu_launches": r["gpu_launches"],
        "clocks": r["clocks"],
    }
    if subs:
        line["configs"] = subs
    print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()
    return 0


def plan_sharegpt_steps(n_steps: int, dev_frac: float = 0.3, host_factor: float = 0.05, think: float = 1.0):
    """Config 5: drive the step planner (pb_sched_*) over the reference's own
    ShareGPT-like trace (proj/data/traces/synthetic_sharegpt_200.trace, committed as
    tests/golden/sharegpt_200_trace.json) with the device tier at ~30% of the working set and
    a host tier small enough to overflow, so leading chunks get dropped and come back as
    dropped-prefix recompute spans while other conversations swap in and out.  Returns the
    window of n_steps consecutive planned steps that carries the most swap-ins, swap-outs and
    recompute spans (the whole run is planned; the window is the densest stretch of it)."""
    from paper_2312_05516_b200.abi import KvCache
    from paper_2312_05516_b200.planner import Scheduler, default_params
    from paper_2312_05516_b200.workloads import reference_trace

    trace = reference_trace()
    ws = sum((sum(p + o for p, o in turns) + 15) // 16 for _, turns in trace)
    dev_slots = max(64, int(dev_frac * ws))
    host_slots = max(1, int(host_factor * dev_slots))
    cache = KvCache(16, dev_slots, host_slots)
    sched = Scheduler(cache, params=default_params(token_budget=4096))
    pending = [(0.02 * c, c, 0) for c, _ in trace]
    turns = dict(trace)
    req, req_conv, now, steps, history = 0, {}, 0.0, 0, []
    while (pending or sched.queue_size or sched.running_size) and steps < 20000:
        steps += 1
        now += 0.05
        for item in sorted(p for p in pending if p[0] <= now):
            pending.remove(item)
            t, c, k = item
            pr, ou = turns[c][k]
            sched.enqueue(req, c, t, pr, ou, k)
            req_conv[req] = (c, k)
            req += 1
        plans = sched.step(now)
        history.extend(plans)
        for i in range(len(plans)):
            for r in sched.complete(i, now + 0.01):
                c, k = req_conv[r]
                if k + 1 < len(turns[c]):
                    pending.append((now + think, c, k + 1))  # think time
    score = [(len(p.in_moves) > 0) + (len(p.out_moves) > 0) + (p.recompute_tokens > 0) for p in history]
    n = min(n_steps, len(history))
    best = max(range(len(history) - n + 1), key=lambda i: sum(score[i:i + n]))
    return history[best:best + n], dev_slots, host_slots, {"trace_conversations": len(trace),
                                                           "planned_steps": len(history), "window_start": best}


def config5_result(args, warmup):
    """Config 5: CPU-tier swap-in/out (pb_swap_step, layer-pipelined) + the ragged attention of
    the same planned steps, Llama-2-13B shape, one GPU.  Returns the result dict."""
    import torch

    from paper_2312_05516_b200 import abi
    from paper_2312_05516_b200.abi import PB_BF16, AttentionPlan, AttnShape, KvTier

    n_layer = 40 if args.config != 5 else (args.layers or 40)
    n_head, n_kv, d, chunk = 40, 10, 128, 16
    c5_steps = max(args.steps, 12)  # at least 12 timed steps (>= 10 of them carry swaps)
    steps, dev_slots, host_slots, plan_info = plan_sharegpt_steps(warmup + c5_steps)
    dev = torch.device("cuda", torch.cuda.current_device())
    page_elems = chunk * n_kv * d
    page_bytes = page_elems * 2
    k = torch.empty((n_layer, dev_slots, page_elems), dtype=torch.bfloat16, device=dev)
    v = torch.empty_like(k)
    abi.fill_unit(k.data_ptr(), PB_BF16, k.numel(), 5, 0)
    abi.fill_unit(v.data_ptr(), PB_BF16, v.numel(), 5, k.numel())
    max_tok = max(p.total_tokens for p in steps)
    q = torch.empty(max_tok * n_head * d, dtype=torch.bfloat16, device=dev)
    abi.fill_unit(q.data_ptr(), PB_BF16, q.numel(), 6, 0)
    out = torch.empty_like(q)
    max_chunks = max(max(len(p.in_moves), len(p.out_moves)) for p in steps) + 1
    tier = KvTier(n_layer, host_slots, page_bytes, max_chunks)
    shape = AttnShape(n_head, n_kv, d, chunk, dev_slots, PB_BF16, math.sqrt(d))
    cs, xs = torch.cuda.Stream(), torch.cuda.Stream()
    plans = [AttentionPlan(shape, p.batch()) for p in steps]
    wss = max(pl.workspace_bytes() for pl in plans)
    wsb = torch.zeros(max(1, wss), dtype=torch.uint8, device=dev)
    layer_stride = dev_slots * page_bytes

    def run(i, ev=None):
        p, pl = steps[i], plans[i]
        if ev:
            ev[0].record(xs)
        tier.step(k.data_ptr(), v.data_ptr(), layer_stride, p.out_moves, p.in_moves, cs.cuda_stream, xs.cuda_stream)
        if ev:
            ev[1].record(xs)
        pl.upload(cs.cuda_stream)
        for l in range(n_layer):
            tier.wait_layer(l, cs.cuda_stream)
            pl.run(q.data_ptr(), k.data_ptr() + l * layer_stride, v.data_ptr() + l * layer_stride, out.data_ptr(),
                   wsb.data_ptr(), cs.cuda_stream)

    clocks = ClockSampler(dev.index)
    clocks.start()
    clocks.wait_ready()
    for i in range(warmup):
        run(i)
    torch.cuda.synchronize()
    t0 = torch.cuda.Event(enable_timing=True)
    t1 = torch.cuda.Event(enable_timing=True)
    swap_ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(c5_steps)]
    launches0 = abi.launch_count()
    torch.cuda.synchronize()
    clocks.begin()
    t0.record(cs)
    for s in range(c5_steps):
        run(warmup + s, swap_ev[s])
    # the step's work includes its swap-out D2H (on the tier's own stream)
    tier.sync()
    xs.wait_stream(cs)
    cs.wait_stream(xs)
    t1.record(cs)
    torch.cuda.synchronize()
    launches = abi.launch_count() - launches0
    clk = clocks.stop()
    total_ms = t0.elapsed_time(t1)
    swap_ms = sum(a.elapsed_time(b) for a, b in swap_ev)

    # the two halves alone, same steps: attention without swaps, swaps without attention
    def timed_loop(fn):
        torch.cuda.synchronize()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(cs)
        for s in range(c5_steps):
            fn(warmup + s)
        tier.sync()
        xs.wait_stream(cs)
        cs.wait_stream(xs)
        b.record(cs)
        torch.cuda.synchronize()
        return a.elapsed_time(b) / c5_steps

    def attn_only(i):
        pl = plans[i]
        pl.upload(cs.cuda_stream)
        for l in range(n_layer):
            pl.run(q.data_ptr(), k.data_ptr() + l * layer_stride, v.data_ptr() + l * layer_stride, out.data_ptr(),
                   wsb.data_ptr(), cs.cuda_stream)

    def swap_only(i):
        p = steps[i]
        tier.step(k.data_ptr(), v.data_ptr(), layer_stride, p.out_moves, p.in_moves, cs.cuda_stream, xs.cuda_stream)
        tier.wait_layer(n_layer - 1, cs.cuda_stream)

    attn_only_ms = timed_loop(attn_only)
    swap_only_ms = timed_loop(swap_only)

    # untimed audit pass: device-stamped swap-in completions vs attention starts per layer,
    # checked by the LayerDependencyAuditor restatement (pb_evlog_audit)
    log = abi.EventLog(1 << 16)
    tier.set_event_log(log)

    def audited(i):
        p, pl = steps[i], plans[i]
        tier.step(k.data_ptr(), v.data_ptr(), layer_stride, p.out_moves, p.in_moves, cs.cuda_stream, xs.cuda_stream)
        pl.upload(cs.cuda_stream)
        for l in range(n_layer):
            tier.wait_layer(l, cs.cuda_stream)
            log.mark(abi.PB_EV_ATTN_START, l, -1, cs.cuda_stream)
            pl.run(q.data_ptr(), k.data_ptr() + l * layer_stride, v.data_ptr() + l * layer_stride, out.data_ptr(),
                   wsb.data_ptr(), cs.cuda_stream)
        log.mark(abi.PB_EV_STEP_END, -1, -1, cs.cuda_stream)

    for s_ in range(c5_steps):
        audited(warmup + s_)
    tier.sync()
    torch.cuda.synchronize()
    events = log.read()
    tier.set_event_log(None)
    violations, audited_steps = abi.audit_events(events, per_step=True)
    timed = steps[warmup:warmup + c5_steps]
    attn_bytes = sum(pl.stats()["bytes"] for pl in plans[warmup:warmup + c5_steps]) * n_layer
    attn_flops = sum(pl.stats()["flops"] for pl in plans[warmup:warmup + c5_steps]) * n_layer
    n_in = sum(len(p.in_moves) for p in timed)
    n_out = sum(len(p.out_moves) for p in timed)
    in_bytes, out_bytes = n_in * tier.chunk_bytes, n_out * tier.chunk_bytes
    del k, v, q, out, wsb, plans, tier
    torch.cuda.empty_cache()
    h2d_peak, d2h_peak = pinned_copy_peaks(torch, dev, 1 << 30)
    duplex = duplex_microbench(torch, dev)
    peaks, peak_src = load_peaks()
    value = attn_bytes / (total_ms / 1e3) / 1e9
    swap_s = swap_only_ms * c5_steps / 1e3
    return {
        "metric": "ragged paged-attn HBM GB/s with layer-pipelined KV swap", "value": value, "unit": "GB/s",
        "ms_per_step": total_ms / c5_steps, "steps": c5_steps, "warmup": warmup, "n_layer": n_layer,
        "workload": "cfg5-sharegpt-llama2-13b",
        "trace": "proj/data/traces/synthetic_sharegpt_200.trace (tests/golden/sharegpt_200_trace.json)",
        "plan": dict(plan_info, device_slots=dev_slots, host_slots=host_slots, chunk_bytes=page_bytes * 2 * n_layer,
                     spans_per_step=sum(len(p.spans) for p in timed) / len(timed),
                     recompute_tokens=sum(p.recompute_tokens for p in timed),
                     steps_with_swap_in=sum(1 for p in timed if p.in_moves),
                     steps_with_swap_out=sum(1 for p in timed if p.out_moves),
                     steps_with_swaps=sum(1 for p in timed if p.in_moves or p.out_moves),
                     steps_with_recompute=sum(1 for p in timed if p.recompute_tokens)),
        "roofline": {"bound": "hbm", "achieved": value, "peak": peaks["hbm_gbs"], "unit": "GB/s",
                     "frac": value / peaks["hbm_gbs"], "traffic": None, "peak_source": peak_src,
                     "tflops": attn_flops / (total_ms / 1e3) / 1e12,
                     "attention_only_gbs": attn_bytes / (attn_only_ms * c5_steps / 1e3) / 1e9,
                     "attention_only_frac": attn_bytes / (attn_only_ms * c5_steps / 1e3) / 1e9 / peaks["hbm_gbs"]},
        "pipeline_audit": {"violations": violations, "steps": audited_steps,
                           "swap_in_layer_events": int((events["kind"] == abi.PB_EV_SWAP_IN_LAYER).sum()),
                           "attn_start_events": int((events["kind"] == abi.PB_EV_ATTN_START).sum())},
        "parts_ms_per_step": {"attention_only": attn_only_ms, "swap_only": swap_only_ms,
                              "both": total_ms / c5_steps},
        "swap": {"chunks_in": n_in, "chunks_out": n_out, "bytes_in": in_bytes, "bytes_out": out_bytes,
                 "swap_only_gbs": (in_bytes + out_bytes) / swap_s / 1e9 if swap_s > 0 else None,
                 "h2d_gbs_swap_only": in_bytes / swap_s / 1e9 if swap_s > 0 else None,
                 "d2h_gbs_swap_only": out_bytes / swap_s / 1e9 if swap_s > 0 else None,
                 "h2d_frac_of_pinned_peak": in_bytes / swap_s / 1e9 / h2d_peak if swap_s > 0 else None,
                 "d2h_frac_of_pinned_peak": out_bytes / swap_s / 1e9 / d2h_peak if swap_s > 0 else None,
                 # the busier direction sets the swap time: its share of the swap-only time
                 "link_busy_frac": max(in_bytes / h2d_peak, out_bytes / d2h_peak) / 1e9 / swap_s
                 if swap_s > 0 else None,
                 "swap_events_ms": swap_ms,
                 "pinned_h2d_peak_gbs": h2d_peak, "pinned_d2h_peak_gbs": d2h_peak},
        "duplex": duplex,
        "clocks": clk, "gpu_launches": int(launches),
    }


def bench_config5(args):
    import torch
    torch.cuda.set_device(0)
    warmup = max(3, args.warmup)
    r = config5_result(args, warmup)
    line = {"metric": r.pop("metric"), "value": r.pop("value"), "unit": r.pop("unit"), "n_gpus": 1,
            "steps": r.pop("steps"), "warmup": r.pop("warmup"), "ms_per_step": r.pop("ms_per_step"),
            "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "bf16",
            "data": "reference ShareGPT trace planned by pb_sched; synthetic KV values",
            "config": {"workload": r.pop("workload"), "n_layer": r.pop("n_layer")}}
    line.update(r)
    print(json.dumps(line), flush=True)
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
    ap.add_argument("--config", type=int, default=4, choices=[1, 2, 3, 4, 5])
    ap.add_argument("--layers", type=int, default=0)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--cpu-budget", type=float, default=12.0, help="seconds of CPU reference work")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-subconfigs", action="store_true", help="headline config only (no cfg2/3/5 sub-results)")
    args = ap.parse_args()
    if args.config == 5:
        if args.impl == "reference":
            print(json.dumps({"impl": "reference", "unavailable": "config 5 has no CPU reference: the "
                              "reference swap engine moves no bytes (SPEC.md:458)"}))
            return 0
        return bench_config5(args)
    if args.impl == "reference":
        return bench_reference(args)
    return bench_ours(args)


if __name__ == "__main__":
    sys.exit(main())
