"""CPU-side checks of the C-ABI library: it loads, exports every symbol the header
declares, and its host-side validation (check_batch, proj/src/attention.cpp:23-48) and plan
accounting behave like the reference — no GPU needed for any of these."""
import math
import os
import re
import subprocess

import numpy as np
import pytest

import paper_2312_05516_b200 as pb
from paper_2312_05516_b200 import abi
from paper_2312_05516_b200.abi import PB_BF16, PB_F32, AttnShape, AttentionPlan, Batch
from paper_2312_05516_b200.workloads import SplitMix64, config, random_instance

ROOT = os.path.abspath(os.path.join(os.path.dirname(__file__), ".."))


def header_symbols():
    text = open(os.path.join(ROOT, "include", "pensieve_b200.h")).read()
    return sorted(set(re.findall(r"\b(pb_[a-z0-9_]+)\s*\(", text)))


def test_library_exports_every_header_symbol():
    out = subprocess.run(["nm", "-D", "--defined-only", pb.so_path()], capture_output=True,
                         text=True, check=True).stdout
    exported = set(re.findall(r" T (pb_[a-z0-9_]+)", out))
    missing = [s for s in header_symbols() if s not in exported]
    assert not missing, missing
    assert set(abi.exported_symbols()) <= exported


def test_library_is_sm100a():
    out = subprocess.run(["cuobjdump", "--list-elf", pb.so_path()], capture_output=True, text=True).stdout
    assert "sm_100a" in out


def _shape(**kw):
    d = dict(n_head=2, n_kv_head=1, head_size=8, chunk_size=16, n_slots=4, dtype=PB_F32, scale=math.sqrt(8))
    d.update(kw)
    return AttnShape(**d)


@pytest.mark.parametrize("mutate,err", [
    (lambda s, b: (_shape(n_head=0), b), abi.DimensionMismatch),
    (lambda s, b: (_shape(n_head=3, n_kv_head=2), b), abi.DimensionMismatch),
    (lambda s, b: (_shape(scale=0.0), b), abi.DimensionMismatch),
    (lambda s, b: (s, Batch([3], [0], [[0]], query_start=[1])), abi.DimensionMismatch),
    (lambda s, b: (s, Batch([3], [0], [[0]], context_len=[4])), abi.DimensionMismatch),
    (lambda s, b: (s, Batch([3], [-1], [[0]], context_len=[2])), abi.DimensionMismatch),
    (lambda s, b: (s, Batch([3], [0], [[]])), abi.DimensionMismatch),
    (lambda s, b: (s, Batch([3], [20], [[0]])), abi.DimensionMismatch),
    (lambda s, b: (s, Batch([3], [0], [[4]])), abi.Error),
    (lambda s, b: (s, Batch([3], [0], [[-1]])), abi.Error),
])
def test_plan_validation_matches_reference_errors(mutate, err, oracle):
    s0, b0 = _shape(), Batch([3], [0], [[0]])
    s, b = mutate(s0, b0)
    with pytest.raises(err):
        AttentionPlan(s, b)
    # the oracle (restating check_batch) reports the same class
    q = np.zeros(max(1, b.total_tokens) * max(1, s.n_head) * max(1, s.head_size), np.float32)
    q = q[: b.total_tokens * max(0, s.n_head) * max(0, s.head_size)]
    kv = np.zeros(max(1, s.n_slots * s.chunk_size * max(1, s.n_kv_head) * max(1, s.head_size)), np.float32)
    st, _ = oracle.attention(s, b, q, kv, kv)
    assert st == err.code


def test_single_token_plan_rejects_long_spans():
    with pytest.raises(abi.DimensionMismatch):
        AttentionPlan(_shape(), Batch([2], [0], [[0]]), flags=abi.PB_PLAN_SINGLE_TOKEN)
    AttentionPlan(_shape(), Batch([1, 1], [0, 5], [[0], [1]]), flags=abi.PB_PLAN_SINGLE_TOKEN)


def test_one_shot_api_checks_numerics_on_host():
    s = _shape()
    b = Batch([1], [0], [[0]])
    q = np.zeros(16, np.float32)
    q[3] = np.nan
    kv = np.zeros(4 * 16 * 8, np.float32)
    with pytest.raises(abi.NumericError):
        abi.paged_multi_token_attention(s, b, q, kv, kv)
    q[3] = 0
    k = kv.copy()
    k[0] = np.inf  # k_row[0] of the attended position
    with pytest.raises(abi.NumericError):
        abi.paged_multi_token_attention(s, b, q, k, kv)


@pytest.mark.parametrize("cfg", [1, 2, 3, 4])
def test_plan_accounting_matches_survey(cfg):
    w = config(cfg)
    plan = AttentionPlan(w.shape(), w.batch())
    st = plan.stats()
    fl, by = w.flops_bytes()
    assert st["flops"] == pytest.approx(fl, rel=1e-12)
    assert st["bytes"] == pytest.approx(by, rel=1e-12)
    assert st["total_tokens"] == w.total_tokens
    # SURVEY §8(d) table
    expect = {1: (0.01e9, 1.6e6, 91, 5), 2: (127.6e9, 1.757e9, None, 64),
              3: (11.07e9, 2.773e9, 256, 256), 4: (432.3e9, 0.735e9, None, 64)}[cfg]
    assert fl == pytest.approx(expect[0], rel=0.02 if cfg > 1 else 1.0)
    assert by == pytest.approx(expect[1], rel=0.02 if cfg > 1 else 1.0)
    if expect[2]:
        assert w.total_tokens == expect[2]
    assert len(w.spans) == expect[3]


def test_work_list_covers_every_row():
    """Each (span, kv head, query token) appears in exactly one work item; decode splits
    tile [0, context)."""
    rng = SplitMix64(9)
    w = random_instance(rng, 8, 2, 128, 16, PB_BF16, 12, 3000)
    plan = AttentionPlan(w.shape(), w.batch())
    st = plan.stats()
    assert st["rows"] == w.total_tokens * w.n_head
    for force in (abi.PB_PLAN_FORCE_SIMT, abi.PB_PLAN_NO_SPLIT):
        st2 = AttentionPlan(w.shape(), w.batch(), flags=force).stats()
        assert st2["rows"] == w.total_tokens * w.n_head


def test_run_layers_checks_arguments_before_any_device_call():
    """pb_attn_run_layers rejects a plan that was never uploaded and mismatched per-layer
    lists before touching the device (its run_impl checks, in the same order)."""
    w = config(2)
    plan = AttentionPlan(w.shape(), w.batch())
    with pytest.raises(abi.Error):
        plan.run_layers([1, 1], [1, 1], [1, 1], [1, 1], 1, None)
    with pytest.raises(abi.DimensionMismatch):
        plan.run_layers([1, 1], [1], [1, 1], [1, 1], 1, None)
