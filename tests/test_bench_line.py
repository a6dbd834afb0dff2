"""bench.py's JSON lines against the driver's contract: the reference arm (the float64 oracle on the
host cores; runs without a GPU) and, on a GPU box, one short run of the product arm on the small
configuration.  Checks the keys, their internal consistency (value = frames / time, roofline.frac =
achieved / peak, e2e byte counts from the workload's shapes) and that kernels were launched."""
import json
import os
import subprocess
import sys

import pytest

from synth import CONFIGS

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
BASE = json.load(open(os.path.join(ROOT, "BASELINE.json")))


def _bench(*args, env=None, timeout=900):
    r = subprocess.run([sys.executable, "bench.py", *args], cwd=ROOT, capture_output=True, text=True,
                       timeout=timeout, env=dict(os.environ, **(env or {})))
    assert r.returncode == 0, r.stderr[-4000:]
    lines = [ln for ln in r.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1, r.stdout[-2000:]
    return json.loads(lines[0])


def test_reference_arm_line():
    d = _bench("--impl", "reference", "--config", "tiny", "--steps", "2", "--warmup", "1")
    cfg = CONFIGS["tiny"]
    assert d["impl"] == "reference" and d["metric"] == BASE["metric"] and d["unit"] == "frames/s"
    assert d["higher_is_better"] is True and d["steps"] == 2 and d["warmup"] == 1 and d["n_gpus"] == 1
    assert d["config"]["workload"] == "tiny" and d["dtype"] == "f64"
    assert d["value"] > 0 and abs(d["ms_per_step"] - 1e3 * cfg.S / d["value"]) <= 1e-6 * d["ms_per_step"]
    cb = d["cpu_baseline"]
    assert cb["kind"] == "oracle" and cb["cores"] >= 1 and cb["value"] == d["value"] and cb["sample"]
    assert d["e2e"] == {"value": d["value"], "unit": d["unit"], "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}


def test_reference_arm_other_ranks_do_no_work():
    r = subprocess.run([sys.executable, "bench.py", "--impl", "reference", "--config", "tiny", "--gpus", "2"],
                       cwd=ROOT, capture_output=True, text=True, timeout=300,
                       env=dict(os.environ, RANK="1", LOCAL_RANK="1", WORLD_SIZE="2"))
    assert r.returncode == 0 and r.stdout.strip() == ""


@pytest.mark.gpu
def test_product_arm_line_small_config():
    d = _bench("--config", "tiny", "--steps", "8", "--warmup", "3")
    cfg = CONFIGS["tiny"]
    assert "impl" not in d or d["impl"] != "reference"
    assert d["metric"] == BASE["metric"] and d["unit"] == "frames/s" and d["higher_is_better"] is True
    assert d["n_gpus"] == 1 and d["steps"] == 8 and d["warmup"] >= 3 and d["data"].startswith("synthetic")
    assert d["config"]["workload"] == "tiny" and "l2" in d["config"]
    assert abs(d["value"] - cfg.S / (d["ms_per_step"] * 1e-3)) <= 1e-6 * d["value"]
    rf = d["roofline"]
    assert rf["bound"] == "hbm" and rf["unit"] == "GB/s" and rf["kernel"] == "project_kernel"
    assert abs(rf["frac"] - rf["achieved"] / rf["peak"]) < 1e-12 and 0 < rf["frac"] < 1.2
    fb = cfg.Q * cfg.Q * (2 if cfg.dtype == "u16" else 4)
    assert d["e2e"]["value"] > 0 and d["e2e"]["h2d_bytes_per_step"] == cfg.S * fb
    assert d["e2e"]["d2h_bytes_per_step"] >= cfg.S * 8
    assert d["gpu_launches"] > 0
    assert {"sm_mhz", "sm_max_mhz", "reasons"} <= set(d["clocks"])
    cb = d["cpu_baseline"]
    assert cb["kind"] == "oracle" and cb["value"] > 0 and cb["cores"] >= 1
    assert d["latency"]["ingest_batch_us"]["n"] >= 1 and d["latency"]["readout_us"]["n"] >= 1
