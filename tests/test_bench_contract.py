"""bench.py contract checks that run on CPU: the reference arm (the reference's CPU
path, oracle port) prints one JSON line with the keys the driver reads; the MUFU
roofline helper's arithmetic."""

import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def test_reference_arm_json_line():
    r = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--impl", "reference", "--steps", "1",
                        "--warmup", "1"], capture_output=True, text=True, timeout=600, cwd=ROOT)
    assert r.returncode == 0, r.stderr[-2000:]
    line = json.loads(r.stdout.strip().splitlines()[-1])
    for k in ("metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better",
              "scaling", "vs_baseline", "dtype", "data", "config", "impl", "cpu_baseline", "e2e"):
        assert k in line, k
    assert line["impl"] == "reference" and line["value"] > 0 and line["unit"] == "images/s"
    cb = line["cpu_baseline"]
    assert cb["kind"] == "port" and cb["cores"] >= 1 and cb["value"] == line["value"] and cb["sample"]
    assert line["e2e"] == {"value": line["value"], "unit": line["unit"], "h2d_bytes_per_step": 0,
                           "d2h_bytes_per_step": 0}
    assert "workload" in line["config"]


def test_xu_roofline_helper():
    import bench

    r = bench.xu_roofline(256, 197, 384, 16, 0.1536, {"sm_mhz": 1965.0})
    assert r["ops_per_launch"] == 20 * 256 * 197 * 384
    assert abs(r["peak"] - 16 * 148 * 1965e6 / 1e9) < 1e-6
    assert abs(r["frac"] - r["achieved"] / r["peak"]) < 1e-12 and 0.3 < r["frac"] < 0.8


def test_gpus_flag_self_launches_ranks():
    """``bench.py --gpus 2`` outside torchrun starts 2 ranks itself; under the
    reference arm rank 0 alone prints the JSON line with n_gpus = 2."""
    r = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--impl", "reference", "--gpus", "2",
                        "--steps", "1", "--warmup", "1"], capture_output=True, text=True, timeout=900, cwd=ROOT)
    assert r.returncode == 0, r.stderr[-2000:]
    lines = [ln for ln in r.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1
    assert json.loads(lines[0])["n_gpus"] == 2


def test_world_size_mismatch_is_an_error():
    env = dict(os.environ, WORLD_SIZE="1", RANK="0", LOCAL_RANK="0")
    r = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--impl", "reference", "--gpus", "2"],
                       capture_output=True, text=True, timeout=300, cwd=ROOT, env=env)
    assert r.returncode == 2


def test_cpu_op_baseline_leg():
    """The op-level CPU leg (the reference's fused-op composition and the
    engine alone, lanes/s and GB/s) runs on the host and reports both config rows."""
    import bench

    r = bench.cpu_op_baseline(reps=1)
    assert r["kind"] == "port" and r["cores"] >= 1
    for name in ("cfg1", "cfg2"):
        row = r["rows"][name]
        for k in ("fused_op_ms", "fused_op_ms_scaled", "fused_lanes_per_s", "fused_gbs", "engine_lbm_ms",
                  "engine_fwd_ms", "engine_lbm_over_fwd", "sample"):
            assert k in row, (name, k)
        assert row["fused_op_ms"] > 0 and row["engine_lbm_ms"] > 0
        assert row["fused_op_ms_scaled"] >= row["fused_op_ms"]
