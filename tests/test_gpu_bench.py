"""GPU: bench.py keeps its JSON-line contract (both arms), on a short run."""
import json
import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _run(args, timeout=600):
    out = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), *args], cwd=ROOT, capture_output=True,
                         text=True, timeout=timeout)
    assert out.returncode == 0, out.stderr[-2000:]
    lines = [ln for ln in out.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1, out.stdout[-2000:]
    return json.loads(lines[0])


def test_bench_line_contract():
    d = _run(["--steps", "3", "--warmup", "3", "--no-cpu-baseline", "--e2e-steps", "1"])
    for k in ("metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better", "scaling",
              "vs_baseline", "dtype", "data", "config", "roofline", "e2e", "gpu_launches", "clocks"):
        assert k in d, k
    assert d["value"] > 0 and d["n_gpus"] == 1 and d["steps"] == 3 and d["warmup"] == 3
    assert d["higher_is_better"] is True and d["scaling"] == "weak" and d["vs_baseline"] is None
    assert "workload" in d["config"]
    rf = d["roofline"]
    for k in ("bound", "achieved", "peak", "unit", "frac", "traffic"):
        assert k in rf, k
    assert rf["bound"] == "hbm" and 0 < rf["frac"] < 1.2 and abs(rf["achieved"] / rf["peak"] - rf["frac"]) < 1e-9
    e = d["e2e"]
    assert e["value"] > 0 and e["h2d_bytes_per_step"] > 0 and e["d2h_bytes_per_step"] > 0
    assert e["value"] < d["value"]  # host copies cannot be free
    assert d["gpu_launches"] >= 6 * 3
    assert {"sm_mhz", "sm_max_mhz", "reasons"} <= set(d["clocks"])
    cf = d["configs"]
    assert set(cf) == {"c1_c128", "c2_c128", "c3_c128", "c4_c128", "c5_c64"}, cf
    for k, rec in cf.items():
        assert "error" not in rec, (k, rec)
        assert rec["ms_per_step"] > 0 and rec["solves_per_s"] > 0 and rec["bound"] in ("latency", "hbm", "fp64")
    assert 0 < cf["c4_c128"]["spread_fp_frac"] < 1.2


def test_bench_single_config_flag():
    d = _run(["--config", "c3", "--steps", "3", "--warmup", "3"])
    assert d["record"]["cfg"] == 3 and d["value"] > 0 and d["config"]["rhs_per_gpu"] == 256


def test_bench_reference_arm_contract():
    d = _run(["--impl", "reference", "--steps", "1", "--warmup", "3"])
    ours = _run(["--steps", "3", "--warmup", "3", "--no-cpu-baseline", "--no-e2e", "--no-configs"])
    assert d["config"] == ours["config"]  # same workload description in both arms
    assert d["impl"] == "reference" and d["value"] > 0 and d["unit"] == "solves/s"
    assert d["cpu_baseline"]["kind"] == "oracle" and d["cpu_baseline"]["cores"] >= 1
    assert d["e2e"]["h2d_bytes_per_step"] == 0 and d["e2e"]["d2h_bytes_per_step"] == 0
