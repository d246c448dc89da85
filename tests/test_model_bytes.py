"""ModelConfig byte arithmetic and the KV-head shard geometry through the
C-ABI: pb_model_* restates /root/reference/proj/src/model_config.cpp:13-68 and is pinned
against the reference-written golden file (tests/golden/model_bytes.json, make_golden.py) and,
when it is built, the reference library itself; pb_shard_shape follows :25-26 / :36-40."""
import json
import os

import pytest

from paper_2312_05516_b200 import abi
from paper_2312_05516_b200.abi import (AttnShape, ConfigError, DimensionMismatch, ModelConfig, PB_BF16,
                                       chunk_bytes, kv_token_bytes, model_preset, model_validate, shard_shape)

HERE = os.path.dirname(os.path.abspath(__file__))
PRESETS = ("opt-13b", "opt-66b", "llama2-13b", "llama2-70b")


def _golden():
    with open(os.path.join(HERE, "golden", "model_bytes.json")) as f:
        return json.load(f)["kv_token_bytes_chunk_bytes"]


def test_presets_match_the_reference_golden_file():
    gold = _golden()
    assert len(gold) == 12
    for key, (tok, ch) in gold.items():
        preset, chunk = key.split("/")
        m = model_preset(preset)
        assert kv_token_bytes(m) == tok, key
        assert chunk_bytes(m, int(chunk)) == ch, key


def test_known_answers_from_survey():
    # OPT-13B 819,200 B/token; Llama-2-70B chunk 32 at 4 partitions 2,621,440 B
    assert kv_token_bytes(model_preset("opt-13b")) == 819200
    assert chunk_bytes(model_preset("llama2-70b"), 32) == 2621440


def test_against_the_reference_library(reference):
    for preset in PRESETS:
        for n_kv in (0, 1, 8):
            m = model_preset(preset)
            if n_kv:
                m.n_kv_head = n_kv
            for chunk in (1, 7, 16, 32, 64):
                st, tok, ch = reference.model_bytes(preset, chunk, n_kv)
                assert st == 0
                assert (kv_token_bytes(m), chunk_bytes(m, chunk)) == (tok, ch), (preset, n_kv, chunk)


def test_validation_order_and_errors():
    good = model_preset("llama2-70b")
    model_validate(good)
    bad = [dict(n_layer=-1), dict(n_head=0), dict(hidden=1), dict(n_kv_head=3, n_head=64, hidden=8192),
           dict(bytes_per_scalar=0), dict(n_partitions=0), dict(n_partitions=3)]
    for b in bad:
        m = model_preset("llama2-70b")
        for k, v in b.items():
            setattr(m, k, v)
        with pytest.raises(ConfigError):
            model_validate(m)
    with pytest.raises(ConfigError):
        chunk_bytes(good, 0)
    with pytest.raises(ConfigError):
        model_preset("gpt-5")


def test_shard_shape_matches_per_worker_chunk_bytes():
    """A rank's shard holds chunk_bytes(n_partitions = world) per chunk: page bytes of the
    shard shape times 2 (K, V) times n_layer."""
    m = model_preset("llama2-70b")
    full = AttnShape(m.n_head, m.n_kv_head, m.head_size, 16, 1024, PB_BF16, m.head_size ** 0.5)
    for world in (1, 2, 4, 8):
        for rank in range(world):
            s, h0, k0 = shard_shape(full, rank, world)
            assert (s.n_head, s.n_kv_head) == (64 // world, 8 // world)
            assert (h0, k0) == (rank * 64 // world, rank * 8 // world)
            assert (s.head_size, s.chunk_size, s.n_slots, s.dtype) == (128, 16, 1024, PB_BF16)
        mw = model_preset("llama2-70b")
        mw.n_partitions = world
        page_bytes = 16 * s.n_kv_head * s.head_size * mw.bytes_per_scalar
        assert 2 * mw.n_layer * page_bytes == chunk_bytes(mw, 16)
    with pytest.raises(DimensionMismatch):
        shard_shape(full, 0, 3)
    with pytest.raises(ConfigError):
        shard_shape(full, 4, 4)


def test_exported():
    for n in ("pb_model_validate", "pb_model_kv_token_bytes", "pb_model_chunk_bytes", "pb_model_preset",
              "pb_shard_shape", "pb_tier_set_policy"):
        assert n in abi.exported_symbols()


def test_reference_model_config_unit_tests_pass_on_pb_model():
    """The reference's OWN ModelConfig unit tests (proj/tests/test_model_config.cpp, 7 cases,
    compiled unchanged) with ModelConfig::validate / kv_token_bytes / chunk_bytes / preset
    resolved to this library's pb_model_* at link time (oracle/ref_tests_b200_model.cpp,
    oracle/Makefile).  Host code only."""
    import os
    import subprocess

    exe = os.path.join(os.path.dirname(os.path.abspath(__file__)), "..", "oracle", "_ref",
                       "kvsim_model_config_tests_b200")
    if not os.path.exists(exe) or not os.path.isdir("/root/reference/proj/data"):
        pytest.skip("needs the reference build and its data directory (this container only)")
    r = subprocess.run([exe], capture_output=True, text=True, timeout=120)
    assert r.returncode == 0, r.stdout + r.stderr
    assert "test cases: 7 | 7 passed | 0 failed" in r.stdout, r.stdout
