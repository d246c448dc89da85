"""Synthetic workloads of BASELINE.json's configs, bit-reproducible.

Every value is ``float(2*u01 - 1)`` drawn from SplitMix64 (reference
/root/reference/proj/src/workload.cpp:30-40), exactly like the reference fixtures
(proj/tests/acceptance.cpp:98, proj/tests/test_attention.cpp:19).  Draw order for one
instance:

  1. layout draws (per conversation: past context, then query length),
  2. Fisher-Yates shuffle of the physical slot pool with ``next() % i``
     (proj/tests/acceptance.cpp:143-146), slots then handed out in conversation order,
  3. layer-0 K pool, layer-0 V pool, q, then K/V pools of layers 1, 2, ... .

SplitMix64 is counter based (draw j of ``SplitMix64{seed}`` is ``mix(seed + (j+1)*golden)``),
so pools are filled on the GPU by ``pb_fill_splitmix_unit`` with the right first-draw index
and equal the sequential CPU stream bit for bit (``unit_draws`` below is the numpy form).
For bf16 configs the stored values are those floats rounded to bf16 (round-to-nearest-even);
the CPU oracle is fed the same bf16-rounded values widened back to fp32.
"""
from __future__ import annotations

import math
from dataclasses import dataclass, field
from typing import List, Optional, Sequence, Tuple

import numpy as np

from .descriptors import PB_BF16, PB_F32, AttnShape, Batch

GOLDEN = 0x9E3779B97F4A7C15
MASK64 = (1 << 64) - 1


class SplitMix64:
    """Sequential SplitMix64 (workload.cpp:30-40) that also counts its draws."""

    def __init__(self, seed: int):
        self.seed = seed & MASK64
        self.state = self.seed
        self.draws = 0

    def next(self) -> int:
        self.state = (self.state + GOLDEN) & MASK64
        z = self.state
        z = ((z ^ (z >> 30)) * 0xBF58476D1CE4E5B9) & MASK64
        z = ((z ^ (z >> 27)) * 0x94D049BB133111EB) & MASK64
        self.draws += 1
        return z ^ (z >> 31)

    def u01(self) -> float:
        return (self.next() >> 11) * (1.0 / 9007199254740992.0)

    def skip(self, n: int) -> None:
        """Advance past n draws (consumed elsewhere, e.g. by a GPU fill)."""
        self.state = (self.state + n * GOLDEN) & MASK64
        self.draws += n


def unit_draws(seed: int, first: int, n: int) -> np.ndarray:
    """float32(2*u01-1) for draws first..first+n-1 of SplitMix64{seed}, vectorised."""
    with np.errstate(over="ignore"):
        idx = np.arange(first + 1, first + 1 + n, dtype=np.uint64)
        z = np.uint64(seed) + idx * np.uint64(GOLDEN)
        z = (z ^ (z >> np.uint64(30))) * np.uint64(0xBF58476D1CE4E5B9)
        z = (z ^ (z >> np.uint64(27))) * np.uint64(0x94D049BB133111EB)
        z = z ^ (z >> np.uint64(31))
    u = (z >> np.uint64(11)).astype(np.float64) * (1.0 / 9007199254740992.0)
    return (2.0 * u - 1.0).astype(np.float32)


def round_bf16(x: np.ndarray) -> np.ndarray:
    """Round fp32 -> bf16 (RNE) and widen back to fp32 (finite inputs)."""
    u = np.ascontiguousarray(x, dtype=np.float32).view(np.uint32).astype(np.uint64)
    r = ((u + 0x7FFF + ((u >> 16) & 1)) >> 16) << 16
    return r.astype(np.uint32).view(np.float32)


def to_bf16_bits(x: np.ndarray) -> np.ndarray:
    u = np.ascontiguousarray(x, dtype=np.float32).view(np.uint32).astype(np.uint64)
    return (((u + 0x7FFF + ((u >> 16) & 1)) >> 16)).astype(np.uint16)


@dataclass
class Workload:
    name: str
    n_head: int
    n_kv_head: int
    head_size: int
    chunk: int
    dtype: int
    seed: int
    # spans: (conversation index, causal_offset, query_len)
    spans: List[Tuple[int, int, int]]
    conv_tables: List[np.ndarray]
    n_slots: int
    pool_first_draw: int  # draw index of the first layer-0 K element
    n_layer: int = 1
    scale: float = 0.0
    notes: str = ""

    def __post_init__(self):
        if not self.scale:
            self.scale = math.sqrt(self.head_size)

    # ---- sizes -------------------------------------------------------------------
    @property
    def row_elems(self) -> int:
        return self.n_kv_head * self.head_size

    @property
    def pool_elems(self) -> int:
        return self.n_slots * self.chunk * self.row_elems

    @property
    def total_tokens(self) -> int:
        return sum(q for _, _, q in self.spans)

    @property
    def q_elems(self) -> int:
        return self.total_tokens * self.n_head * self.head_size

    def k_first_draw(self, layer: int = 0) -> int:
        if layer == 0:
            return self.pool_first_draw
        return self.pool_first_draw + 2 * self.pool_elems + self.q_elems + 2 * (layer - 1) * self.pool_elems

    def v_first_draw(self, layer: int = 0) -> int:
        return self.k_first_draw(layer) + self.pool_elems

    def q_first_draw(self) -> int:
        return self.pool_first_draw + 2 * self.pool_elems

    # ---- descriptors ---------------------------------------------------------------
    def shape(self, n_kv_head: Optional[int] = None, dtype: Optional[int] = None) -> AttnShape:
        nkv = self.n_kv_head if n_kv_head is None else n_kv_head
        nh = self.n_head * nkv // self.n_kv_head
        return AttnShape(nh, nkv, self.head_size, self.chunk, self.n_slots,
                         self.dtype if dtype is None else dtype, self.scale)

    def batch(self, span_ids: Optional[Sequence[int]] = None) -> Batch:
        ids = range(len(self.spans)) if span_ids is None else span_ids
        ql, co, tables = [], [], []
        for i in ids:
            conv, off, q = self.spans[i]
            ql.append(q)
            co.append(off)
            ctx = off + q
            tables.append(self.conv_tables[conv][: (ctx + self.chunk - 1) // self.chunk])
        return Batch(ql, co, tables)

    def span_token_offsets(self) -> np.ndarray:
        q = np.array([s[2] for s in self.spans], dtype=np.int64)
        off = np.zeros(len(q) + 1, dtype=np.int64)
        off[1:] = np.cumsum(q)
        return off

    # ---- host copies (checkers / CPU baseline) ---------------------------------------
    def host_q(self) -> np.ndarray:
        q = unit_draws(self.seed, self.q_first_draw(), self.q_elems)
        return round_bf16(q) if self.dtype == PB_BF16 else q

    def host_pool(self, which: str, layer: int = 0) -> np.ndarray:
        first = self.k_first_draw(layer) if which == "k" else self.v_first_draw(layer)
        x = unit_draws(self.seed, first, self.pool_elems)
        return round_bf16(x) if self.dtype == PB_BF16 else x

    def host_pages(self, which: str, slots: Sequence[int], layer: int = 0) -> np.ndarray:
        """Only the listed pages (cheap for sampled parity at full config sizes)."""
        first = self.k_first_draw(layer) if which == "k" else self.v_first_draw(layer)
        page = self.chunk * self.row_elems
        out = np.empty((len(slots), page), dtype=np.float32)
        for j, s in enumerate(slots):
            out[j] = unit_draws(self.seed, first + int(s) * page, page)
        return round_bf16(out) if self.dtype == PB_BF16 else out

    def compact_host_inputs(self, span_ids: Sequence[int], layer: int = 0):
        """(shape, batch, q, keys, values) on the host for the chosen spans only: just the pages
        they touch, slots renumbered densely (slot relocation is bit-exact for the reference,
        proj/tests/test_attention.cpp:407-432).  Feeds the CPU checkers / CPU baseline."""
        full = self.batch(span_ids)
        slots = sorted(set(int(s) for i in range(full.n_spans) for s in full.table(i)))
        remap = {s: j for j, s in enumerate(slots)}
        tables = [[remap[int(s)] for s in full.table(i)] for i in range(full.n_spans)]
        batch = Batch(full.query_len, full.causal_offset, tables)
        shape = self.shape()
        shape.n_slots = len(slots)
        keys = self.host_pages("k", slots, layer).reshape(-1)
        values = self.host_pages("v", slots, layer).reshape(-1)
        tok = self.span_token_offsets()
        row = self.n_head * self.head_size
        q = np.concatenate([unit_draws(self.seed, self.q_first_draw() + int(tok[i]) * row,
                                       int(tok[i + 1] - tok[i]) * row) for i in span_ids])
        if self.dtype == PB_BF16:
            q = round_bf16(q)
        return shape, batch, q, keys, values

    def flops_bytes(self, span_ids: Optional[Sequence[int]] = None) -> Tuple[float, float]:
        """flops over unmasked score pairs; bytes = K+V once per kv head + Q + O
        + block table."""
        eb = 4 if self.dtype == PB_F32 else 2
        fl = by = 0.0
        ids = range(len(self.spans)) if span_ids is None else span_ids
        d = self.head_size
        for i in ids:
            _, off, q = self.spans[i]
            if q == 0:
                continue
            fl += 4.0 * self.n_head * d * (q * off + q * (q + 1) / 2)
            ctx = off + q
            by += 2.0 * ctx * self.n_kv_head * d * eb + 2.0 * q * self.n_head * d * eb + 4.0 * (
                (ctx + self.chunk - 1) // self.chunk)
        return fl, by


def _build(name: str, n_head: int, n_kv: int, d: int, chunk: int, dtype: int, seed: int,
           convs: List[List[Tuple[int, int]]], rng: SplitMix64, n_layer: int = 1,
           notes: str = "") -> Workload:
    """convs[c] = list of (causal_offset, query_len) spans of conversation c."""
    pages = []
    for spans in convs:
        ctx = max(off + q for off, q in spans)
        pages.append((ctx + chunk - 1) // chunk)
    n_slots = sum(pages)
    pool = list(range(n_slots))
    for i in range(len(pool), 1, -1):  # acceptance.cpp:143-146
        j = rng.next() % i
        pool[i - 1], pool[j] = pool[j], pool[i - 1]
    tables, k = [], 0
    for p in pages:
        tables.append(np.array(pool[k:k + p], dtype=np.int32))
        k += p
    flat = [(c, off, q) for c, spans in enumerate(convs) for off, q in spans]
    w = Workload(name, n_head, n_kv, d, chunk, dtype, rng.seed, flat, tables, n_slots,
                 rng.draws, n_layer, notes=notes)
    rng.skip(2 * w.pool_elems + w.q_elems)  # layer-0 K, V and q
    return w


def config(cfg: int, n_layer: int = 1) -> Workload:
    """BASELINE.json configs 1-4."""
    if cfg == 1:
        rng = SplitMix64(1)
        convs = [[(0, 40)], [(96, 1)], [(0, 32), (112, 17)], [(63, 1)]]
        return _build("cfg1-tiny", 8, 8, 64, 16, PB_F32, 1, convs, rng, n_layer,
                      "tiny synthetic, fp32 validation mode, dropped-prefix pair in conv 2")
    if cfg == 2:
        rng = SplitMix64(2)
        convs = []
        for i in range(64):
            past = rng.next() % 2049
            q = 1 + rng.next() % 512 if i % 4 == 0 else 1
            convs.append([(past, q)])
        return _build("cfg2-opt13b", 40, 40, 128, 16, PB_BF16, 2, convs, rng, n_layer,
                      "OPT-13B attention shape, 64 conversations mixed prefill/decode")
    if cfg == 3:
        rng = SplitMix64(3)
        convs = [[(1 + rng.next() % 4096, 1)] for _ in range(256)]
        return _build("cfg3-llama2-13b", 40, 10, 128, 16, PB_BF16, 3, convs, rng, n_layer,
                      "Llama-2-13B GQA-4, 256 decode spans")
    if cfg == 4:
        rng = SplitMix64(4)
        convs = []
        for i in range(64):
            if i % 4 == 0:
                past = rng.next() % 2049
                q = 1 + rng.next() % 1024
            else:
                past = 1 + rng.next() % 4096
                q = 1
            convs.append([(past, q)])
        return _build("cfg4-llama2-70b", 64, 8, 128, 16, PB_BF16, 4, convs, rng, n_layer,
                      "Llama-2-70B GQA-8 mixed prefill+decode, shardable by kv head")
    raise ValueError(f"unknown config {cfg}")


def random_instance(rng: SplitMix64, n_head: int, n_kv: int, d: int, chunk: int, dtype: int,
                    n_spans: int, max_ctx: int, all_decode: bool = False,
                    max_q: Optional[int] = None) -> Workload:
    """acceptance.cpp make_instance-style random ragged batch (one span per conversation)."""
    convs = []
    for s in range(n_spans):
        ctx = 1 + rng.next() % max_ctx
        if all_decode:
            q = 1
        else:
            q = 1 + rng.next() % (ctx if max_q is None else min(ctx, max_q))
        convs.append([(ctx - q, q)])
    return _build("random", n_head, n_kv, d, chunk, dtype, rng.seed, convs, rng)


# --------------------------------------------------------------------------- config 5
def sharegpt_trace(n_conv: int, seed: int = 5, mean_turns: float = 5.5, mean_prompt: float = 37.77,
                   sigma_prompt: float = 0.6, mean_output: float = 204.58, sigma_output: float = 0.5,
                   max_prompt: int = 512, max_output: int = 2048, max_context: int = 16384):
    """Synthetic ShareGPT-like multi-turn trace: geometric turn counts, lognormal prompt and
    output lengths with the ShareGPT statistics the paper reports (the
    reference's synthetic generator uses the same distribution family and parameters).
    Returns [(conv_id, [(prompt, output), ...])]."""
    rng = SplitMix64(seed)

    def normal():
        u1 = max(rng.u01(), 1e-300)
        u2 = rng.u01()
        return math.sqrt(-2.0 * math.log(u1)) * math.cos(2.0 * math.pi * u2)

    def lognormal(mean, sigma):
        mu = math.log(mean) - 0.5 * sigma * sigma
        return math.exp(mu + sigma * normal())

    p_stop = 1.0 / mean_turns
    out = []
    for c in range(n_conv):
        turns, total = [], 0
        while True:
            pr = max(1, min(max_prompt, int(round(lognormal(mean_prompt, sigma_prompt)))))
            ou = max(1, min(max_output, int(round(lognormal(mean_output, sigma_output)))))
            if total + pr + ou > max_context:
                break
            turns.append((pr, ou))
            total += pr + ou
            if rng.u01() < p_stop:
                break
        if turns:
            out.append((c, turns))
    return out


def reference_trace(path: Optional[str] = None):
    """The reference's own ShareGPT-like trace (proj/data/traces/synthetic_sharegpt_200.trace),
    as committed in tests/golden/sharegpt_200_trace.json by tests/golden/make_trace_fixture.py.
    Returns [(conv_id, [(prompt, output), ...])] like sharegpt_trace."""
    import json
    import os
    if path is None:
        path = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests", "golden",
                            "sharegpt_200_trace.json")
    with open(path) as f:
        convs = json.load(f)["conversations"]
    return [(int(c), [(int(p), int(o)) for p, o in turns]) for c, turns in convs]
