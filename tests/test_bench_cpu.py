"""bench.py contract on CPU: the reference arm (the C oracle on the host
cores) prints one JSON line with the driver's keys."""
import json
import subprocess
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]


def test_reference_arm_json_line():
    out = subprocess.run([sys.executable, str(ROOT / "bench.py"), "--impl", "reference",
                          "--steps", "1", "--warmup", "1"],
                         capture_output=True, text=True, timeout=600, cwd=str(ROOT))
    assert out.returncode == 0, out.stderr[-2000:]
    lines = [ln for ln in out.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1
    d = json.loads(lines[0])
    for key in ("impl", "metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step",
                "higher_is_better", "scaling", "dtype", "data", "config", "cpu_baseline", "e2e"):
        assert key in d, key
    assert d["impl"] == "reference" and d["value"] > 0
    assert d["cpu_baseline"]["kind"] == "port" and d["cpu_baseline"]["cores"] >= 1
    assert d["e2e"]["h2d_bytes_per_step"] == 0 and d["e2e"]["value"] == d["value"]


def test_pair_counts_match_survey_figures():
    """bench.pair_counts (the roofline's compute side) against SURVEY 8(d)'s
    measured (atom, voxel) pairs per grid (C2: 733,027 box / 383,482 in the
    cutoff; C4 per nonzero weight: 2,601,905 / 1,364,529), within 2% (other
    synthetic draws, untransformed frame)."""
    sys.path.insert(0, str(ROOT))
    import bench
    from paper_1912_04822_b200 import GridMaker

    for name, box_ref, cut_ref in (("c2", 733027, 383482), ("c4", 2601905, 1364529)):
        cfg = bench.CONFIGS[name]
        exs, _ = bench.make_batch(cfg, 0, 1, n=8)
        gm = GridMaker(resolution=cfg["resolution"], dimension=cfg["dimension"],
                       binary=cfg["binary"])
        box, cut = bench.pair_counts(gm, exs)
        assert abs(box / box_ref - 1) < 0.02, (name, box)
        assert abs(cut / cut_ref - 1) < 0.02, (name, cut)
        assert cut < box
