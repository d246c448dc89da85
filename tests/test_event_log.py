"""Pipeline event log and its LayerDependencyAuditor restatement (pb_evlog_audit):
the reference's own known-answer cases (proj/tests/test_event_log.cpp:74-109), a
differential check against the reference auditor on random event streams (CPU), and on the
GPU the real swap-in -> attention ordering of the layer-pipelined swap engine."""
import numpy as np
import pytest

from paper_2312_05516_b200 import abi
from paper_2312_05516_b200.abi import (EVENT_DTYPE, PB_EV_ATTN_START, PB_EV_STEP_END, PB_EV_SWAP_IN_LAYER,
                                       PB_EV_SWAP_OUT, audit_events)
from paper_2312_05516_b200.workloads import SplitMix64


def _ev(rows):
    """rows of (t_seconds, kind, layer) -> EVENT_DTYPE records in ns"""
    out = np.zeros(len(rows), dtype=EVENT_DTYPE)
    for i, (t, kind, layer) in enumerate(rows):
        out[i] = (int(round(t * 1e9)), kind, layer, -1)
    return out


def test_reference_kat_clean_pipelined_step():
    # proj/tests/test_event_log.cpp:74-91 ({t, kind, req, layer})
    ev = _ev([(0.001, PB_EV_SWAP_IN_LAYER, 0), (0.001, PB_EV_ATTN_START, 0), (0.002, PB_EV_SWAP_IN_LAYER, 1),
              (0.0025, PB_EV_ATTN_START, 1), (0.004, PB_EV_STEP_END, -1), (0.005, PB_EV_ATTN_START, 0),
              (0.006, PB_EV_STEP_END, -1)])
    assert audit_events(ev) == (0, 2)


def test_reference_kat_attention_before_swap_in():
    # proj/tests/test_event_log.cpp:93-109
    ev = _ev([(0.002, PB_EV_SWAP_IN_LAYER, 0), (0.0015, PB_EV_ATTN_START, 0), (0.004, PB_EV_STEP_END, -1)])
    assert audit_events(ev)[0] == 1
    multi = _ev([(0.001, PB_EV_SWAP_IN_LAYER, 0), (0.003, PB_EV_SWAP_IN_LAYER, 0), (0.002, PB_EV_ATTN_START, 0),
                 (0.004, PB_EV_STEP_END, -1)])
    assert audit_events(multi)[0] == 1
    assert audit_events(_ev([(0.001, PB_EV_SWAP_IN_LAYER, -1)]))[0] == 1  # swap-in without a layer


def test_audit_matches_reference_auditor(reference):
    rng = SplitMix64(2024)
    kinds = [PB_EV_SWAP_IN_LAYER, PB_EV_SWAP_OUT, PB_EV_ATTN_START, PB_EV_STEP_END]
    for trial in range(200):
        n = 1 + rng.next() % 60
        rows = []
        for _ in range(n):
            k = kinds[rng.next() % 4]
            layer = int(rng.next() % 6) - 1
            t = 10 * (rng.next() % 1000)  # ns, multiples of 10 (away from the 1 ns tolerance)
            rows.append((t, k, layer))
        ev = np.zeros(n, dtype=EVENT_DTYPE)
        for i, (t, k, layer) in enumerate(rows):
            ev[i] = (t, k, layer, -1)
        want = reference.audit_layer_deps([r[1] for r in rows], [r[2] for r in rows], [r[0] / 1e9 for r in rows])
        assert audit_events(ev) == want, (trial, rows)


@pytest.mark.gpu
def test_swap_pipeline_audit_on_gpu(cuda):
    """Layer-pipelined swap-in + attention with the tier's per-layer events: every layer's
    attention is stamped after its pages landed (0 violations).  Skipping the wait for the
    last layer is caught by the same audit."""
    torch = cuda
    n_layer, page_bytes, slots = 12, 4 * 16 * 128 * 2, 64
    k = torch.zeros((n_layer, slots, page_bytes // 2), dtype=torch.bfloat16, device="cuda")
    v = torch.zeros_like(k)
    tier = abi.KvTier(n_layer, 32, page_bytes, 32)
    log = abi.EventLog(4096)
    tier.set_event_log(log)
    cs, xs = torch.cuda.Stream(), torch.cuda.Stream()
    layer_stride = slots * page_bytes
    moves_in = [(i, i, 2 * i) for i in range(24)]  # (chunk, host src, device dst)
    for step in range(3):
        tier.step(k.data_ptr(), v.data_ptr(), layer_stride, [], moves_in, cs.cuda_stream, xs.cuda_stream)
        for l in range(n_layer):
            tier.wait_layer(l, cs.cuda_stream)
            log.mark(PB_EV_ATTN_START, l, -1, cs.cuda_stream)
        log.mark(PB_EV_STEP_END, -1, -1, cs.cuda_stream)
    torch.cuda.synchronize()
    ev = log.read()
    assert (ev["kind"] == PB_EV_SWAP_IN_LAYER).sum() == 3 * n_layer
    assert audit_events(ev) == (0, 3)
    assert audit_events(ev, per_step=True) == (0, 3)
    # an attention of the last layer stamped before the step's swap-in was even issued: the
    # per-step audit flags it (the streaming form sees a layer that is not "ready" yet)
    log.reset()
    log.mark(PB_EV_ATTN_START, n_layer - 1, -1, cs.cuda_stream)
    tier.step(k.data_ptr(), v.data_ptr(), layer_stride, [], moves_in, cs.cuda_stream, xs.cuda_stream)
    for l in range(n_layer - 1):
        tier.wait_layer(l, cs.cuda_stream)
        log.mark(PB_EV_ATTN_START, l, -1, cs.cuda_stream)
    tier.wait_layer(n_layer - 1, cs.cuda_stream)
    log.mark(PB_EV_STEP_END, -1, -1, cs.cuda_stream)
    torch.cuda.synchronize()
    bad = log.read()
    assert audit_events(bad, per_step=True) == (1, 1)
    assert audit_events(bad) == (0, 1)


def test_per_step_audit_cases():
    ev = _ev([(0.002, PB_EV_ATTN_START, 0), (0.003, PB_EV_SWAP_IN_LAYER, 0), (0.004, PB_EV_STEP_END, -1),
              (0.005, PB_EV_SWAP_IN_LAYER, 0), (0.006, PB_EV_ATTN_START, 0), (0.007, PB_EV_STEP_END, -1)])
    assert audit_events(ev, per_step=True) == (1, 2)
    assert audit_events(ev) == (0, 2)
