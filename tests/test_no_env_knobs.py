"""The production library has no runtime knobs: no `PB_*` environment variable changes what it
computes (round-1 builds read PB_ONLY / PB_TILE_HALF / PB_SWAP_IN ... and PB_ONLY=1 silently
skipped every decode unit).  Profiling variants are separate builds (scripts/build_variants.sh).

CPU: the default library carries no `PB_*` strings and no product source calls getenv.
GPU: a fused prefill+decode batch run in a child process with every former knob set gives
bit-identical outputs to a clean child process."""
import glob
import json
import os
import re
import subprocess
import sys

import numpy as np
import pytest

import paper_2312_05516_b200 as pb

ROOT = os.path.abspath(os.path.join(os.path.dirname(__file__), ".."))
FORMER_KNOBS = {
    "PB_ONLY": "1", "PB_ABLATE": "1", "PB_TILE_HALF": "1", "PB_DEC_UNITS": "3", "PB_FUSE_DECODE_ONLY": "0",
    "PB_TILE_ORDER": "1", "PB_DEC_CTA_SCALE": "4", "PB_DECODE": "simt", "PB_SWAP_IN": "zc",
    "PB_SWAP_DUPLEX": "0", "PB_SWAP_LB": "1", "PB_SWAP_BATCH": "0", "PB_PLAN_FLAGS": "7",
}


def test_library_has_no_env_knob_strings():
    out = subprocess.run(["strings", pb.so_path()], capture_output=True, text=True, check=True).stdout
    knobs = sorted({ln for ln in out.splitlines() if re.match(r"^PB_[A-Z_]+$", ln)})
    assert knobs == [], knobs


def test_product_sources_do_not_read_the_environment():
    srcs = glob.glob(os.path.join(ROOT, "paper_2312_05516_b200", "csrc", "*.[ch]*"))
    assert srcs
    hits = [os.path.basename(s) for s in srcs if re.search(r"\bgetenv\s*\(|secure_getenv", open(s).read())]
    assert hits == [], hits


_CHILD = r"""
import sys, json, hashlib
sys.path.insert(0, sys.argv[1]); sys.path.insert(0, sys.argv[1] + '/tests')
import numpy as np
import gpu_helpers as gh
from paper_2312_05516_b200.workloads import PB_BF16, SplitMix64, _build
convs = [[(0, 200)], [(700, 1)], [(0, 64), (300, 45)], [(1500, 1)], [(90, 1)], [(0, 513)], [(2047, 1)]]
w = _build('knobs', 32, 8, 128, 16, PB_BF16, 99, convs, SplitMix64(99))
q, k, v = gh.device_inputs(w)
out, plan = gh.run_plan(w, q, k, v)
st = plan.stats()
print(json.dumps({'sha': hashlib.sha256(out.tobytes()).hexdigest(), 'tiles': st['prefill_tiles'],
                  'units': st['decode_units'], 'finite': bool(np.isfinite(out).all())}))
"""


def _child(env_extra):
    env = {k: v for k, v in os.environ.items() if not k.startswith("PB_")}
    env.update(env_extra)
    r = subprocess.run([sys.executable, "-c", _CHILD, ROOT], capture_output=True, text=True, env=env, timeout=600)
    assert r.returncode == 0, r.stderr[-2000:]
    return json.loads(r.stdout.strip().splitlines()[-1])


@pytest.mark.gpu
def test_former_env_knobs_change_nothing():
    clean = _child({})
    assert clean["finite"] and clean["tiles"] > 0 and clean["units"] > 0, clean
    knobbed = _child(FORMER_KNOBS)
    assert knobbed == clean
