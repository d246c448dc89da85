"""bench.py's reference arm on CPU (the driver computes the headline ratio from the two arms'
lines): it prints the same metric string and config object as our arm would for the same
config, carries ms_per_step / e2e / cpu_baseline, and never maps the product library (it runs
the reference's own kvsim::paged_multi_token_attention from oracle/_ref)."""
import json
import os
import subprocess
import sys

import pytest

ROOT = os.path.abspath(os.path.join(os.path.dirname(__file__), ".."))

_CHILD = r"""
import sys, json, io, contextlib
sys.path.insert(0, sys.argv[1])
sys.argv = ['bench.py', '--impl', 'reference', '--steps', '1', '--warmup', '1', '--cpu-budget', '1']
import bench
buf = io.StringIO()
with contextlib.redirect_stdout(buf):
    rc = bench.main()
line = json.loads(buf.getvalue().strip().splitlines()[-1])
maps = open('/proc/self/maps').read()
print(json.dumps({'rc': rc, 'line': line,
                  'product_mapped': 'libpensieve_b200.so' in maps,
                  'ref_mapped': 'libkvsim_ref.so' in maps}))
"""


@pytest.mark.skipif(not os.path.exists(os.path.join(ROOT, "oracle", "_ref", "libkvsim_ref.so")),
                    reason="oracle/_ref not built")
def test_reference_arm_line_matches_our_arm_contract():
    r = subprocess.run([sys.executable, "-c", _CHILD, ROOT], capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stderr[-2000:]
    res = json.loads(r.stdout.strip().splitlines()[-1])
    line = res["line"]
    sys.path.insert(0, ROOT)
    import bench
    from paper_2312_05516_b200.workloads import config

    assert res["rc"] in (0, None)
    assert line["impl"] == "reference"
    assert line["metric"] == bench.METRICS[4] and line["unit"] == bench.UNITS[4]
    assert line["config"] == bench.bench_config(config(4), bench.MODEL_LAYERS[4], 1)
    assert line["value"] > 0 and line["ms_per_step"] > 0 and line["higher_is_better"] is True
    assert line["e2e"]["value"] == line["value"] and line["e2e"]["h2d_bytes_per_step"] == 0
    assert line["cpu_baseline"]["kind"] == "reference" and line["cpu_baseline"]["cores"] >= 1
    assert line["gpu_launches"] == 0
    assert res["ref_mapped"] and not res["product_mapped"]
