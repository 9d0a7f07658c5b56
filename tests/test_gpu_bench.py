"""bench.py contract checks on one GPU (the driver's own invocation shapes)."""
import json
import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu
REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _run(args, env=None, timeout=600):
    e = dict(os.environ)
    e.pop("WORLD_SIZE", None)
    e.update(env or {})
    r = subprocess.run([sys.executable, "bench.py"] + args, cwd=REPO, capture_output=True, text=True,
                       timeout=timeout, env=e)
    assert r.returncode == 0, r.stderr[-3000:]
    lines = [ln for ln in r.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1, r.stdout[-2000:]
    return json.loads(lines[0]), r.stderr


def test_bench_self_launches_ranks():
    """`bench.py --gpus 2` without torchrun spawns two ranks itself (here both
    on the one GPU over gloo) and reports n_gpus = 2."""
    line, err = _run(["--gpus", "2", "--ctx", "4096", "--steps", "2", "--warmup", "3", "--no-e2e", "--ttft-layers", "2", "--ttft-ctx", "2048",
                      "--no-cpu-baseline", "--no-128k", "--no-est"], env={"SA_DIST_BACKEND": "gloo"})
    assert line["n_gpus"] == 2 and line["config"]["n_gpus"] == 2
    assert "rank 1/2" in err and "rank 0/2" in err
    assert line["value"] > 0


def test_bench_world_size_mismatch_fails():
    e = dict(os.environ, WORLD_SIZE="1", RANK="0", LOCAL_RANK="0")
    r = subprocess.run([sys.executable, "bench.py", "--gpus", "2", "--ctx", "1024", "--steps", "1"], cwd=REPO,
                       capture_output=True, text=True, timeout=300, env=e)
    assert r.returncode != 0 and "must match" in (r.stderr + r.stdout)


def test_bench_line_fields_small():
    """One small run: the step includes the finiteness scan and the cache fill,
    the line carries the roofline / e2e / clocks keys and the same config keys
    as the reference arm."""
    line, _ = _run(["--ctx", "4096", "--steps", "3", "--warmup", "3", "--no-cpu-baseline", "--no-128k", "--ttft-layers", "3", "--ttft-ctx", "4096"])
    for key in ("roofline", "e2e", "e2e_numpy_f32", "clocks", "gpu_launches", "estimator_roofline"):
        assert line.get(key) is not None, key
    ref, _ = _run(["--impl", "reference", "--ctx", "1024", "--steps", "2", "--warmup", "1"])
    assert set(ref["config"]) == set(line["config"])
    assert ref["cpu_baseline"]["kind"] in ("reference", "port")
