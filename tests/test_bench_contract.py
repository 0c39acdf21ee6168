"""bench.py contract checks that need no GPU: the reference arm prints one
JSON line with the driver's keys (impl, metric, value, unit, cpu_baseline,
e2e), timing the compiled reference (oracle/_ref) on host cores."""
import json
import os
import subprocess
import sys

import pytest

import oracle as O

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.mark.skipif(not O.ref_available(), reason="oracle/_ref not built")
def test_reference_arm_json_line():
    out = subprocess.run([sys.executable, "bench.py", "--impl", "reference", "--steps", "2",
                          "--warmup", "1", "--d", "200000"], capture_output=True, text=True,
                         cwd=ROOT, timeout=300)
    assert out.returncode == 0, out.stderr
    lines = [l for l in out.stdout.splitlines() if l.startswith("{")]
    assert len(lines) == 1
    j = json.loads(lines[0])
    assert j["impl"] == "reference"
    for k in ("metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step",
              "higher_is_better", "config", "cpu_baseline", "e2e"):
        assert k in j, k
    assert j["value"] > 0 and j["cpu_baseline"]["kind"] == "reference"
    assert j["e2e"]["h2d_bytes_per_step"] == 0 and j["e2e"]["value"] == j["value"]
    # the reference's own code on every host thread (coordinate shards)
    assert j["cpu_baseline"]["cores"] == len(os.sched_getaffinity(0))


@pytest.mark.skipif(not O.ref_available(), reason="oracle/_ref not built")
def test_sharded_reference_timing():
    """ref_time_rounds_sharded: d split into coordinate shards, one reference
    run (simulator rules) per shard, concurrently; a sharded threaded
    transport is refused (it is timed unsharded, tools/cpu_reference.py)."""
    h = O.HyperParams(alpha0=0.1, anneal_at=(), mu=0.9, weight_decay=1e-4, beta_ea=0.1)
    for proto in (O.ALLREDUCE, O.PULL, O.ELASTIC):
        assert O.ref_time_rounds(proto, 2, 100_003, 3, False, h, "pool", shards=4) > 0
    with pytest.raises(RuntimeError, match="simulator rules"):
        O.ref_time_rounds(O.ALLREDUCE, 2, 100_003, 3, True, h, "pool", shards=4)


@pytest.mark.gpu
def test_bench_json_line_on_gpu():
    """One N = 1 bench line carries every key of the driver contract and the
    round-1 additions (roofline with traffic, e2e with copy bytes, clocks,
    gpu_launches) with sane values."""
    out = subprocess.run([sys.executable, "bench.py", "--steps", "5", "--warmup", "3",
                          "--no-extras", "--no-cpu"], capture_output=True, text=True,
                         cwd=ROOT, timeout=600)
    assert out.returncode == 0, out.stderr[-3000:]
    lines = [l for l in out.stdout.splitlines() if l.startswith("{")]
    assert len(lines) == 1
    j = json.loads(lines[0])
    for k in ("metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step",
              "higher_is_better", "scaling", "vs_baseline", "dtype", "data", "config",
              "roofline", "e2e", "clocks", "gpu_launches"):
        assert k in j, k
    assert j["n_gpus"] == 1 and j["steps"] == 5 and j["warmup"] == 3
    assert j["value"] > 1e10 and j["higher_is_better"] is True
    assert "workload" in j["config"]
    r = j["roofline"]
    for k in ("bound", "achieved", "peak", "unit", "frac", "traffic"):
        assert k in r, k
    assert r["bound"] == "hbm" and 0.3 < r["frac"] <= 1.05
    e = j["e2e"]
    assert e["value"] > 0 and e["h2d_bytes_per_step"] == 4 * 25_000_000
    assert e["d2h_bytes_per_step"] > 0
    assert j["gpu_launches"] >= 5
    assert j["clocks"]["sm_mhz"] is not None


@pytest.mark.skipif(not O.ref_available(), reason="oracle/_ref not built")
def test_cpu_reference_sweep_tool():
    """tools/cpu_reference.py --sweep (profiles/r2_cpu_reference_sweep.md) at a
    tiny size: one JSON line per (protocol, p, path), every figure positive
    or an explicit error record."""
    out = subprocess.run([sys.executable, "tools/cpu_reference.py", "--sweep", "--sizes", "4096",
                          "--max-seconds", "60"], capture_output=True, text=True, cwd=ROOT,
                         timeout=300)
    assert out.returncode == 0, out.stderr
    rows = [json.loads(l) for l in out.stdout.splitlines() if l.startswith("{")]
    assert "host" in rows[0]
    runs = [r for r in rows[1:] if "param_updates_per_s" in r]
    assert len(runs) + sum("error" in r for r in rows[1:]) == 3 * 3 * 3
    assert all(r["param_updates_per_s"] > 0 for r in runs)
    assert {r["path"] for r in runs} >= {"simulator rules, all threads (coordinate shards)",
                                          "simulator rules (1 thread)"}
