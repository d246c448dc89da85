"""The drop-in check from the reference's side: a kvsim C++ program (reference headers and
sources, unmodified) calls the B200 library through include/pensieve_b200_kvsim.hpp where it
would call kvsim::paged_multi_token_attention / single_token_attention (oracle/dropin_test.cpp,
built by oracle/Makefile)."""
import os
import subprocess

import pytest

ROOT = os.path.abspath(os.path.join(os.path.dirname(__file__), ".."))
EXE = os.path.join(ROOT, "oracle", "_ref", "kvsim_dropin_test")


def _run(*args):
    if not os.path.exists(EXE):
        pytest.skip("oracle/_ref/kvsim_dropin_test not built (needs /root/reference at build time)")
    r = subprocess.run([EXE, *args], capture_output=True, text=True, timeout=600)
    print(r.stdout)
    return r


def test_dropin_error_behaviour_matches_kvsim():
    r = _run("--no-gpu")
    assert r.returncode == 0, r.stdout + r.stderr
    assert r.stdout.count("[PASS]") >= 5


@pytest.mark.gpu
def test_dropin_values_match_kvsim(cuda):
    r = _run()
    assert r.returncode == 0, r.stdout + r.stderr
    assert "FAIL" not in r.stdout


REF_TESTS = os.path.join(ROOT, "oracle", "_ref", "kvsim_attention_tests_b200")


@pytest.mark.gpu
def test_reference_attention_unit_tests_pass_on_the_b200_path(cuda):
    """The reference's OWN unit tests (proj/tests/test_attention.cpp, 13 test cases, compiled
    unchanged against a doctest stand-in) with kvsim::paged_multi_token_attention and
    kvsim::single_token_attention resolved to the B200 library (oracle/ref_tests_b200.cpp,
    link-time substitution in oracle/Makefile).  Includes its bit-identity checks (one position
    returns that V row exactly, causal masking leaves token 0 bit-identical, GQA with duplicated
    kv heads == MHA, permuted slots bit-identical) and its 1e-5 dense-oracle comparison."""
    if not os.path.exists(REF_TESTS):
        pytest.skip("oracle/_ref/kvsim_attention_tests_b200 not built (needs /root/reference at build time)")
    r = subprocess.run([REF_TESTS], capture_output=True, text=True, timeout=900)
    print(r.stdout, r.stderr)
    assert r.returncode == 0, r.stdout + r.stderr
    assert "| 0 failed" in r.stdout and "test cases: 13 | 13 passed" in r.stdout, r.stdout
