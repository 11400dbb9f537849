"""bench.py host-side contract (CPU): the config object both arms print, the
host-gap summary, the clock sampler without NVML, and the reference arm's
JSON line (the oracle on a bounded C1 sample, run as the driver runs it)."""
import json
import os
import subprocess
import sys
import types

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import bench  # noqa: E402
import synth  # noqa: E402


def _args(**kw):
    d = dict(batch=0, force_gather=False, no_pipeline=False, steps=20, warmup=5)
    d.update(kw)
    return types.SimpleNamespace(**d)


def test_workload_config_c3_one_gpu():
    c = bench.workload_config(synth.CONFIGS[3], _args(), 1)
    assert c["frames_per_step_per_gpu"] == 64
    assert c["pipelined_calls"] is True and c["sharded_path"] is False
    assert c["resident_batches_per_gpu"] == 25            # warmup + steps < 157 batches
    assert "configs[2]" in c["workload"] and c["parallelism"] == "frames sharded by batch, dp1"
    assert c["l2"].startswith("inputs larger than L2: 398 MB")


def test_workload_config_c5_eight_gpus_shards_streams():
    c = bench.workload_config(synth.CONFIGS[5], _args(), 8)
    assert c["frames_per_step_per_gpu"] == 32                # 256 streams / 8 ranks, all per call
    assert c["sharded_path"] is True
    assert c["parallelism"] == "camera streams sharded (s mod 8), dp8"
    assert "256 streams" in c["workload"]


def test_host_gaps_summary():
    g = bench.host_gaps([0.0, 0.0001, 0.0003, 0.0023])
    assert g["median_us"] == pytest.approx(200.0)
    assert g["max_us"] == pytest.approx(2000.0)
    assert g["over_1ms"] == 1 and g["sum_over_1ms_ms"] == pytest.approx(2.0)
    assert g["first_us"] == [100.0, 200.0, 2000.0]
    assert bench.host_gaps([1.0]) is None


def test_clock_sampler_without_nvml_reports_it():
    s = bench.ClockSampler(0)
    if s.ok:
        pytest.skip("NVML is available here")
    s.start()
    s.active = True
    s.sample_now()
    s.stop()
    assert s.summary()["reasons"] == ["nvml unavailable"]


def test_reference_arm_json_line():
    env = dict(os.environ, CUDA_VISIBLE_DEVICES="")
    r = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--impl", "reference",
                        "--config", "1", "--steps", "2", "--warmup", "1"],
                       capture_output=True, text=True, timeout=300, env=env, cwd=ROOT)
    assert r.returncode == 0, r.stderr[-2000:]
    lines = [l for l in r.stdout.splitlines() if l.startswith("{")]
    assert len(lines) == 1
    d = json.loads(lines[0])
    assert d["impl"] == "reference" and d["unit"] == "frames/s" and d["value"] > 0
    assert d["metric"] == bench.METRIC and d["higher_is_better"] is True
    assert d["steps"] == 2 and d["warmup"] == 1 and d["n_gpus"] == 1
    assert d["config"] == bench.workload_config(synth.CONFIGS[1], _args(steps=2, warmup=1), 1)
    cb = d["cpu_baseline"]
    assert cb["kind"] == "oracle" and cb["value"] == d["value"] and cb["cores"] >= 1 and cb["sample"]
    assert d["e2e"] == {"value": d["value"], "unit": "frames/s", "h2d_bytes_per_step": 0,
                        "d2h_bytes_per_step": 0}
