"""bench.py keeps the driver's JSON contract: one JSON line with the required
keys, on CPU for the reference arm (the oracle) and on a GPU for our arm."""
import json
import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
BASE_KEYS = {"metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step",
             "higher_is_better", "scaling", "vs_baseline", "dtype", "data", "config", "e2e",
             "cpu_baseline"}


def _run(args, timeout=600):
    r = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py")] + args,
                       capture_output=True, text=True, timeout=timeout, cwd=ROOT)
    assert r.returncode == 0, r.stderr[-2000:]
    lines = [ln for ln in r.stdout.splitlines() if ln.strip().startswith("{")]
    assert len(lines) == 1, r.stdout
    return json.loads(lines[0])


def test_reference_arm_contract():
    d = _run(["--impl", "reference", "--config", "tiny", "--steps", "3", "--warmup", "3"])
    assert BASE_KEYS <= set(d)
    assert d["impl"] == "reference" and d["value"] > 0
    assert d["cpu_baseline"]["kind"] == "oracle" and d["cpu_baseline"]["cores"] >= 1
    assert d["e2e"]["h2d_bytes_per_step"] == 0 and d["e2e"]["d2h_bytes_per_step"] == 0
    assert "workload" in d["config"]


def test_capacity_override_reaches_the_run():
    """--capacity (the SURVEY §8d C sweep) replaces the config's C on both arms."""
    d = _run(["--impl", "reference", "--config", "tiny", "--steps", "2", "--warmup", "3",
              "--capacity", "64"])
    assert d["config"]["capacity_blocks_per_gpu"] == 64 and d["value"] > 0


@pytest.mark.gpu
def test_our_arm_contract():
    d = _run(["--config", "tiny", "--steps", "4", "--warmup", "3", "--cpu-sample-s", "1"])
    assert BASE_KEYS | {"roofline", "clocks", "gpu_launches", "link_roofline"} <= set(d)
    assert d["value"] > 0 and d["gpu_launches"] > 0 and d["n_gpus"] == 1
    r = d["roofline"]
    assert r["bound"] == "hbm" and r["peak"] > 0 and 0 < r["frac"] == pytest.approx(
        r["achieved"] / r["peak"])
    assert d["e2e"]["value"] > 0 and d["e2e"]["h2d_bytes_per_step"] > 0
    assert {"sm_mhz", "sm_max_mhz", "reasons"} <= set(d["clocks"])
    assert d["cpu_baseline"]["kind"] == "oracle"
    # e2e covers the device-timed steps themselves (same rows), through the public API
    assert d["e2e"]["device_value_same_steps"] == pytest.approx(d["value"], rel=1e-3)
    det = d["detail"]
    assert det["step_ms"]["p50"] > 0 and det["step_ms"]["p99"] >= det["step_ms"]["p50"]
    assert {"evict_per_step", "readmissions_per_step", "cold_restart_ratio"} <= set(det["churn"])
    assert 0 <= r["fresh_row_share"] <= 1
    assert 0 < det["locality"]["mean_K_over_Kloc"] <= 1
    assert 0 <= det["locality"]["jaccard_consecutive_K"] <= 1


def test_gpus_n_self_launches_ranks():
    """`bench.py --gpus 2` outside torchrun launches 2 ranks itself (127.0.0.1
    rendezvous); rank 0 alone prints the line (reference arm: CPU only)."""
    d = _run(["--impl", "reference", "--gpus", "2", "--config", "tiny", "--steps", "2",
              "--warmup", "3"])
    assert d["impl"] == "reference" and d["value"] > 0


@pytest.mark.gpu
def test_our_arm_two_ranks_on_one_gpu():
    """TGS_BENCH_BACKEND=gloo bench.py --gpus 2: two libtidegs ranks share the
    GPU, the library issues C1 / C2 through torch_comm; one n_gpus = 2 line."""
    env = dict(os.environ, TGS_BENCH_BACKEND="gloo")
    r = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--gpus", "2", "--config",
                        "tiny", "--steps", "4", "--warmup", "3", "--no-cpu-baseline"],
                       capture_output=True, text=True, timeout=600, cwd=ROOT, env=env)
    assert r.returncode == 0, r.stderr[-2000:]
    lines = [ln for ln in r.stdout.splitlines() if ln.strip().startswith("{")]
    assert len(lines) == 1, r.stdout
    d = json.loads(lines[0])
    assert d["n_gpus"] == 2 and d["value"] > 0 and d["config"]["world_size"] == 2
