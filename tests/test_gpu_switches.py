"""Scheduling switches must not change results: the attention work order
(LPT vs kv-group-major), the dead-warp softmax skip, the scan placement and
the attention's CTAs per SM only reorder or skip exactly-zero work, so every
output must be bit-identical across them (each run in its own process: the
switches are read once per process)."""
import json
import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _run(env_extra):
    env = dict(os.environ)
    env.update(env_extra)
    r = subprocess.run([sys.executable, "tests/switch_worker.py"], cwd=ROOT, env=env, capture_output=True,
                       text=True, timeout=600)
    assert r.returncode == 0, r.stderr[-3000:]
    return json.loads(r.stdout.strip().splitlines()[-1])


@pytest.mark.gpu
def test_switches_bit_identical():
    base = _run({})
    for extra in ({"SA_ATTN_SKIP": "0"}, {"SA_ATTN_ORDER": "1"}, {"SA_ATTN_ORDER": "0"}, {"SA_ATTN_CTAS": "1"},
                  {"SA_SCAN_AT": "0"}):
        got = _run(extra)
        assert got == base, (extra, {k for k in base if got[k] != base[k]})
