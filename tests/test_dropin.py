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
