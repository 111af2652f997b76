"""bench.py's reference arm on the host cores (no GPU): one JSON line with the
keys the driver reads, the same workload string and config keys as the GPU arm,
and a CPU baseline that says what was timed."""
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_reference_arm_line():
    r = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--impl", "reference", "--steps", "1",
                        "--warmup", "0"], capture_output=True, text=True, timeout=600, cwd=ROOT)
    assert r.returncode == 0, r.stderr[-2000:]
    line = json.loads(r.stdout.strip().splitlines()[-1])
    assert line["impl"] == "reference"
    for key in ("metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better",
                "scaling", "vs_baseline", "dtype", "data", "config", "cpu_baseline", "e2e"):
        assert key in line, key
    assert line["unit"] == "grid_points/s" and line["higher_is_better"] is True and line["dtype"] == "f64"
    assert line["steps"] == 1 and line["value"] > 0
    cfg = line["config"]
    assert cfg["workload"].startswith("c1:") and cfg["points_per_step"] == 5 * 1023 * 1023
    cb = line["cpu_baseline"]
    assert cb["kind"] in ("port", "reference") and cb["cores"] >= 1 and cb["value"] == line["value"]
    assert line["e2e"]["h2d_bytes_per_step"] == 0 and line["e2e"]["d2h_bytes_per_step"] == 0
    # the GPU arm prints the same config keys (the driver compares the two dicts)
    sys.path.insert(0, ROOT)
    import bench
    assert set(bench.bench_config(1)) == set(cfg)
