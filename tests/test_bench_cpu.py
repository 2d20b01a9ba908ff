"""Host logic of bench.py (no GPU): the algorithmic work counts behind the roofline objects and
the reference-arm JSON contract."""
import json
import os
import subprocess
import sys
import types

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import bench  # noqa: E402


def test_fused_bytes_dense_and_csr():
    # dense C-SVC: X 4d + |x|^2 4 + G r/w 8 + status 1 per row (4d + 13)
    assert bench.fused_bytes_per_iter("c4", 500000, 54, 1) == 500000 * (4 * 54 + 13)
    # eps-SVR: both dual copies per row (4d + 22)
    assert bench.fused_bytes_per_iter("c2", 50000, 100, 2) == 50000 * (4 * 100 + 22)
    # CSR: 8 B per nonzero (value + index) + indptr 8 + norm 4 + G/status 9 per row
    assert bench.fused_bytes_per_iter("c5", 10, 400, 1, nnz=400) == 8 * 400 + 10 * 21


def test_batched_roofline_counts():
    info = types.SimpleNamespace(n_problem=10, pass_ms=57.0 * 100 / 1e3, passes=100)
    r = bench.batched_roofline(info, 60000, 784, {"bf16_tflops": 1695.0, "hbm_gbs": 6464.9},
                               "measured")
    flops = 2.0 * 60000 * 784 * 160
    assert r["bound"] == "tensor" and r["unit"] == "TFLOP/s"
    assert r["algorithmic_flops_per_launch"] == flops
    assert abs(r["us_per_launch"] - 57.0) < 1e-9
    assert abs(r["achieved"] - flops / 57e-6 / 1e12) < 1e-6
    assert abs(r["peak"] - 1695.0 / 3) < 1e-9
    assert abs(r["frac"] - r["achieved"] / r["peak"]) < 1e-12


@pytest.mark.timeout(600)
def test_reference_arm_json_contract():
    """bench.py --impl reference prints one JSON line with the contract's keys (the oracle arm,
    rank 0, a bounded sample)."""
    out = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--impl", "reference",
                          "--config", "c1", "--steps", "1", "--warmup", "0", "--cpu-seconds", "0.5"],
                         capture_output=True, text=True, timeout=600, cwd=ROOT)
    assert out.returncode == 0, out.stderr[-2000:]
    line = json.loads(out.stdout.strip().splitlines()[-1])
    for k in ("impl", "metric", "value", "unit", "n_gpus", "steps", "warmup", "higher_is_better",
              "config", "cpu_baseline", "e2e"):
        assert k in line, k
    assert line["impl"] == "reference" and line["higher_is_better"] is False
    assert line["e2e"]["h2d_bytes_per_step"] == 0 and line["cpu_baseline"]["kind"] == "oracle"
    assert line["value"] > 0
