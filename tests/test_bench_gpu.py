"""bench.py contract on the B200: the default arm prints one JSON line with the
driver's keys, the roofline and pair rates, and launches only this repo's
kernels inside the timed region."""
import json
import subprocess
import sys
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parents[1]


@pytest.mark.gpu
def test_bench_json_line_contract():
    out = subprocess.run([sys.executable, str(ROOT / "bench.py"), "--steps", "3", "--warmup", "3",
                          "--no-cpu-baseline"],
                         capture_output=True, text=True, timeout=600, cwd=str(ROOT))
    assert out.returncode == 0, out.stderr[-2000:]
    lines = [ln for ln in out.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1
    d = json.loads(lines[0])
    for key in ("metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step",
                "higher_is_better", "scaling", "vs_baseline", "dtype", "data", "config",
                "roofline", "e2e", "gpu_launches", "clocks"):
        assert key in d, key
    assert d["n_gpus"] == 1 and d["steps"] == 3 and d["warmup"] >= 3 and d["value"] > 0
    # prepare + forward + backward per step, all from libgridmaker_b200.so
    assert d["gpu_launches"] == 3 * 3
    r = d["roofline"]
    assert r["bound"] == "hbm" and r["unit"] == "GB/s" and 0 < r["frac"] < 2
    assert abs(r["frac"] - r["achieved"] / r["peak"]) < 1e-9
    assert 0 < r["pairs_cutoff_per_grid"] < r["pairs_box_per_grid"]
    assert r["fwd_cutoff_pairs_per_s"] > 0 and r["bwd_cutoff_pairs_per_s"] > 0
    e = d["e2e"]
    assert e["value"] > 0 and e["h2d_bytes_per_step"] > 0 and e["d2h_bytes_per_step"] > 0


@pytest.mark.gpu
def test_bench_latency_config_graph_leg():
    """C1 (one ligand per call): the line carries the CUDA-graph replay rate
    beside the eager headline, and the replay is the faster of the two."""
    out = subprocess.run([sys.executable, str(ROOT / "bench.py"), "--config", "c1", "--steps", "20",
                          "--warmup", "3", "--no-cpu-baseline"],
                         capture_output=True, text=True, timeout=600, cwd=str(ROOT))
    assert out.returncode == 0, out.stderr[-2000:]
    d = json.loads([ln for ln in out.stdout.splitlines() if ln.startswith("{")][-1])
    g = d["graph"]
    assert g["unit"] == "grids/s" and g["value"] > d["value"] > 0
