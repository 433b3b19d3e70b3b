"""bench.py contract pieces that run without a GPU: the reference arm's JSON line (the reference's own CPU
implementation on the host cores), the roofline selection and the launcher command."""
import json
import subprocess
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))


def test_reference_arm_prints_one_json_line():
    out = subprocess.run([sys.executable, str(ROOT / "bench.py"), "--impl", "reference", "--steps", "2", "--warmup", "1",
                          "--cpu-rows", "200000"], capture_output=True, text=True, cwd=ROOT)
    assert out.returncode == 0, out.stderr[-2000:]
    lines = [l for l in out.stdout.splitlines() if l.startswith("{")]
    assert len(lines) == 1
    d = json.loads(lines[0])
    assert d["impl"] == "reference" and d["unit"] == "GB/s" and d["higher_is_better"] is True
    assert d["value"] > 0 and d["steps"] == 2 and d["dtype"] == "f64"
    assert d["cpu_baseline"]["kind"] in ("reference", "port") and d["cpu_baseline"]["cores"] >= 1
    assert d["e2e"] == {"value": d["value"], "unit": "GB/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}
    assert d["config"]["m"] == 200000 and d["config"]["same_config"] is False


def test_reference_arm_ranks_other_than_zero_stay_silent():
    import os
    env = dict(os.environ, RANK="1", WORLD_SIZE="2", LOCAL_RANK="1")
    out = subprocess.run([sys.executable, str(ROOT / "bench.py"), "--impl", "reference", "--steps", "1", "--warmup", "0",
                          "--cpu-rows", "1000"], capture_output=True, text=True, cwd=ROOT, env=env)
    assert out.returncode == 0 and out.stdout.strip() == ""


def test_roofline_bound_follows_the_column_count():
    import bench
    m = 1 << 27
    assert bench.roofline_bound("tsqr", m, 8, 6540.0)[0] == "hbm"
    assert bench.roofline_bound("tsqr", m, 12, 6540.0)[0] == "hbm"
    assert bench.roofline_bound("tsqr", m, 22, 6540.0)[0] == "hbm"
    assert bench.roofline_bound("tsqr", m, 23, 6540.0)[0] == "fp64"   # 2mn^2 at 36.9 TFLOP/s outlasts 8mn at the copy rate
    assert bench.roofline_bound("gram", m, 32, 6540.0)[0] == "hbm"
    assert bench.roofline_bound("gram", m, 64, 6540.0)[0] == "fp64"
    bound, t, flops = bench.roofline_bound("tsqr", m, 32, 6540.0)
    assert abs(t - 2.0 * m * 32 * 32 / 36.9e12) < 1e-12 and flops == 2.0 * m * 32 * 32


def test_reference_rows_fit_the_host(monkeypatch):
    import bench
    assert bench.reference_rows(1 << 27, 8, 12345) == 12345
    rows = bench.reference_rows(1 << 40, 8, 0)  # never more than the host can hold
    assert rows < (1 << 40) and rows >= 1024
