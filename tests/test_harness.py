"""Harness, SATN I/O and CLI parity (reference pkg/tests/test_bench.py,
test_tensorio.py): CPU tests cover the report/threshold/config/file logic,
the GPU tests run sweeps and the CLI subcommands on the device path."""

import struct

import numpy as np
import pytest

from paper_2412_06198_b200.harness import (
    BenchConfigError,
    BenchRecord,
    MethodThreshold,
    ThresholdReport,
    attention_io_bytes,
    emit_report,
    estimate_attention_memory,
    find_threshold,
    fixed_pattern_for,
    parse_config,
    parse_report_csv,
    run_sweep,
    synth_qkv,
)
from paper_2412_06198_b200.cli import main as cli_main
from paper_2412_06198_b200.patterns import BlockSparse, Triangular, VerticalSlash
from paper_2412_06198_b200.runtime import ModelConfig
from paper_2412_06198_b200.tensorio import TensorFormatError, read_tensor, write_tensor


def small_cfg(max_context=256, heads=2, d_head=8):
    return ModelConfig(n_heads=heads, d_model=heads * d_head, d_head=d_head, max_context=max_context)


def rec(ctx, method, latency, seed=0):
    return BenchRecord(ctx=ctx, method=method, pattern="-", latency_s=latency, flops=1, mem_bytes=1,
                       frob_err=None, seed=seed)


# ---- memory model, fixed patterns, inputs (test_bench.py:40-100) ----

def test_memory_model():
    cfg = small_cfg(max_context=4096)
    assert estimate_attention_memory("dense", 0, cfg) == attention_io_bytes(0, cfg)
    assert estimate_attention_memory("dense", 64, cfg) == 64 * 64 * 4 + attention_io_bytes(64, cfg)
    for m in ("triangular", "vertical-slash", "block-sparse"):
        assert estimate_attention_memory(m, 1024, cfg) < estimate_attention_memory("dense", 1024, cfg)
    d1, d2 = (estimate_attention_memory("dense", c, cfg) - attention_io_bytes(c, cfg) for c in (512, 1024))
    assert d2 == 4 * d1


def test_fixed_patterns_and_half_even():
    assert fixed_pattern_for("triangular", 1000) == Triangular(100, 0)
    assert fixed_pattern_for("vertical-slash", 1000) == VerticalSlash(50, 50)
    assert fixed_pattern_for("block-sparse", 1000) == BlockSparse(64, 2)
    assert fixed_pattern_for("vertical-slash", 5) == VerticalSlash(1, 1)  # round(0.25) = 0 -> clamp 1
    assert fixed_pattern_for("triangular", 131072) == Triangular(13107, 0)
    with pytest.raises(BenchConfigError):
        fixed_pattern_for("dense", 8)


def test_synth_qkv_deterministic():
    a = synth_qkv(3, 16, 2, 4)
    b = synth_qkv(3, 16, 2, 4)
    for x, y in zip(a, b):
        np.testing.assert_array_equal(x, y)
        assert x.shape == (1, 2, 16, 4) and x.dtype == np.float32 and np.abs(x).max() <= 1.0
    rng = np.random.default_rng([3, 16])
    np.testing.assert_array_equal(a[0][0], rng.uniform(-1, 1, (2, 16, 4)).astype(np.float32))


def test_sweep_validation_before_timing():
    cfg = small_cfg(max_context=64)
    for bad in ([], [0], [64, 32], [128]):
        with pytest.raises(BenchConfigError):
            run_sweep(bad, ["dense"], cfg)
    with pytest.raises(BenchConfigError):
        run_sweep([32], ["bogus"], cfg)
    with pytest.raises(BenchConfigError):
        run_sweep([32], ["dense"], cfg, repeats=0)


# ---- thresholds (test_bench.py:164-202) ----

def test_threshold_cases():
    r = [rec(c, "dense", 10.0 * c) for c in (1, 2, 4, 8)] + [rec(c, "vertical-slash", 1.0 * c) for c in (1, 2, 4, 8)]
    assert find_threshold(r).methods[0].crossover_ctx == 1
    r = [rec(c, "dense", 1.0) for c in (1, 2, 4, 8)] + [rec(c, "vertical-slash", 2.0) for c in (1, 2, 4, 8)]
    assert find_threshold(r).methods[0].crossover_ctx is None
    ctxs = [1024, 2048, 4096, 8192, 16384]
    dense = {1024: 0.1, 2048: 0.4, 4096: 1.6, 8192: 6.4, 16384: 25.6}
    sparse = {1024: 0.5, 2048: 0.9, 4096: 1.7, 8192: 3.3, 16384: 6.5}
    th = find_threshold([rec(c, "dense", dense[c]) for c in ctxs] + [rec(c, "block-sparse", sparse[c]) for c in ctxs])
    assert th.methods[0].crossover_ctx == 8192 and th.methods[0].gradient < th.dense_gradient
    with pytest.raises(BenchConfigError):
        find_threshold([rec(1, "dense", 1.0)])
    with pytest.raises(BenchConfigError, match="no shared ctx"):
        find_threshold([rec(1, "dense", 1.0), rec(2, "vertical-slash", 1.0)])


# ---- reports (test_bench.py:203-255) ----

def test_reports(tmp_path):
    p = tmp_path / "r.csv"
    emit_report([rec(1, "dense", 1.0)], None, "csv", p)
    assert p.read_text().splitlines()[0] == "ctx,method,pattern,latency_s,flops,mem_bytes,frob_err,seed"
    r = BenchRecord(ctx=8, method="dense", pattern="-", latency_s=None, flops=10, mem_bytes=20, frob_err=None, seed=0)
    emit_report([r], None, "csv", p)
    assert p.read_text().splitlines()[1] == "8,dense,-,-,10,20,-,0"
    recs = [rec(32, "dense", 0.125), BenchRecord(64, "auto", "auto(block-sparse=2)", 1e-3, 123, 456, 0.5, 7)]
    emit_report(recs, None, "csv", p)
    assert parse_report_csv(p) == recs
    th = ThresholdReport(dense_gradient=2e-5, methods=(MethodThreshold("vertical-slash", 8192, 1e-5),))
    text = emit_report([rec(1, "dense", 1.0)], th, "markdown")
    assert "Effectiveness threshold" in text and "8192" in text
    assert "Effectiveness threshold" not in emit_report([rec(1, "dense", 1.0)], None, "markdown")
    with pytest.raises(BenchConfigError):
        emit_report([], None, "csv")
    with pytest.raises(BenchConfigError):
        emit_report([rec(1, "dense", 1.0)], None, "xml")
    bad = tmp_path / "bad.csv"
    bad.write_text("a,b,c\n1,2,3\n")
    with pytest.raises(BenchConfigError):
        parse_report_csv(bad)


def test_parse_config(tmp_path):
    p = tmp_path / "cfg.txt"
    p.write_text("# comment\nctx = 32,64\nseed=7\n\nmethods=dense\n")
    assert parse_config(p) == {"ctx": "32,64", "seed": "7", "methods": "dense"}
    p.write_text("just-words\n")
    with pytest.raises(BenchConfigError, match="key=value"):
        parse_config(p)


# ---- SATN files (test_tensorio.py) ----

def test_satn_round_trip_and_errors(tmp_path):
    a = np.random.default_rng(0).standard_normal((3, 5, 2)).astype(np.float32)
    p = tmp_path / "t.satn"
    write_tensor(p, a)
    np.testing.assert_array_equal(read_tensor(p), a)
    write_tensor(p, np.arange(6, dtype=np.float64).reshape(2, 3))
    b = read_tensor(p)
    assert b.dtype == np.float32 and b.shape == (2, 3)
    raw = p.read_bytes()
    for data, msg in ((b"JUNKJUNK", "not a SATN"), (b"SATN" + struct.pack("<HH", 2, 1) + struct.pack("<Q", 1) + b"\0" * 4,
                                                      "unsupported format version"),
                      (raw[:-4], "payload size mismatch"), (b"SATN\x01", "truncated header"),
                      (raw[:12], "truncated dims"),
                      (b"SATN" + struct.pack("<HH", 1, 2) + struct.pack("<2Q", 1 << 30, 1 << 30), "implausible")):
        p.write_bytes(data)
        with pytest.raises(TensorFormatError, match=msg) as ei:
            read_tensor(p)
        assert isinstance(ei.value.offset, int)


# ---- CLI error paths (test_bench.py:336-355) ----

def test_cli_error_lines(tmp_path, capsys):
    rc = cli_main(["attn", "--q", "missing.satn", "--k", "missing.satn", "--v", "missing.satn",
                   "--out", str(tmp_path / "y.satn")])
    assert rc == 1
    err = capsys.readouterr().err
    assert err.startswith("error: ") and len(err.strip().splitlines()) == 1
    bad = tmp_path / "bad.satn"
    bad.write_bytes(b"JUNKJUNK")
    rc = cli_main(["attn", "--q", str(bad), "--k", str(bad), "--v", str(bad), "--out", str(tmp_path / "y.satn")])
    assert rc == 1 and "not a SATN tensor file" in capsys.readouterr().err


# ---- on the B200: sweeps and subcommands (test_bench.py:115-160, 204-210, 271-335) ----

@pytest.mark.gpu
def test_sweep_csv_round_trip_and_labels(tmp_path):
    cfg = small_cfg(max_context=256)
    records = run_sweep([32, 64], ["dense", "triangular"], cfg, repeats=1, seed=5)
    p = tmp_path / "report.csv"
    emit_report(records, None, "csv", p)
    assert parse_report_csv(p) == records
    assert all(r.latency_s is not None and r.latency_s > 0 for r in records)
    assert records[0].frob_err == 0.0 and records[1].frob_err is not None
    cap = run_sweep([64, 128], ["dense", "vertical-slash"], cfg, repeats=1, dense_cap_mb=0.05)
    assert [r.latency_s is None for r in cap if r.method == "dense"] == [False, True]
    auto = run_sweep([64], ["auto"], small_cfg(max_context=64, heads=2, d_head=16), repeats=1,
                     families=("vertical-slash",))
    assert auto[0].pattern == "auto(vertical-slash=2)"
    host = run_sweep([64], ["triangular"], cfg, repeats=1, inputs="host")
    dev = run_sweep([64], ["triangular"], cfg, repeats=1, inputs="device")
    assert host[0].latency_s > 0 and (host[0].pattern, host[0].flops, host[0].frob_err) == (
        dev[0].pattern, dev[0].flops, dev[0].frob_err)


@pytest.mark.gpu
def test_cli_bench_attn_select(tmp_path, capsys):
    out = tmp_path / "r.csv"
    rc = cli_main(["bench", "--ctx", "32,64", "--methods", "dense,vertical-slash", "--heads", "2", "--d-head", "8",
                   "--repeats", "1", "--seed", "1", "--out", str(out), "--quiet"])
    assert rc == 0 and len(parse_report_csv(out)) == 4
    cfgfile = tmp_path / "cfg.txt"
    cfgfile.write_text("ctx=32\nmethods=dense\nheads=2\nd_head=8\nrepeats=1\nepsilon=0.1\nfamilies=vertical-slash\n")
    rc = cli_main(["bench", "--config", str(cfgfile), "--ctx", "16", "--out", str(out), "--quiet"])
    assert rc == 0 and [r.ctx for r in parse_report_csv(out)] == [16]
    rng = np.random.default_rng(12)
    for name in ("q", "k", "v"):
        write_tensor(tmp_path / f"{name}.satn", rng.uniform(-1, 1, (2, 32, 8)).astype(np.float32))
    y = tmp_path / "y.satn"
    args = ["--q", str(tmp_path / "q.satn"), "--k", str(tmp_path / "k.satn"), "--v", str(tmp_path / "v.satn")]
    assert cli_main(["attn", *args, "--out", str(y), "--method", "dense"]) == 0
    assert read_tensor(y).shape == (2, 32, 8)
    assert cli_main(["attn", *args, "--out", str(y), "--method", "auto", "--cal-window", "16"]) == 0
    capsys.readouterr()
    assert cli_main(["select", *args, "--cal-window", "16"]) == 0
    lines = capsys.readouterr().out.strip().splitlines()
    assert len(lines) >= 2 and lines[-1].startswith("head 1:")
