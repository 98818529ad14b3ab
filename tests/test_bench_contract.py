"""bench.py's JSON contract on the CPU: the reference arm's line (the oracle
timed on host threads over a bounded sample) and the roofline records."""
import json
import subprocess
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))


def test_reference_arm_line():
    out = subprocess.run([sys.executable, str(ROOT / "bench.py"), "--impl", "reference", "--config", "C1", "--steps",
                          "1", "--warmup", "0", "--cpu-seconds", "0.5"], capture_output=True, text=True, timeout=300,
                         cwd=ROOT)
    assert out.returncode == 0, out.stderr
    line = json.loads(out.stdout.strip().splitlines()[-1])
    for key in ("metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better", "scaling",
                "vs_baseline", "dtype", "data", "config", "cpu_baseline", "e2e"):
        assert key in line, key
    assert line["impl"] == "reference" and line["higher_is_better"] is False and line["value"] > 0
    assert line["cpu_baseline"]["kind"] == "port" and line["cpu_baseline"]["cores"] >= 1
    assert line["e2e"]["h2d_bytes_per_step"] == 0 and line["e2e"]["value"] == line["value"]


def test_rooflines_records():
    import bench

    prof = {"epoch": {"count": 2, "ms": 30.0, "bytes": 2 * 6.55e9, "flops": 2 * 6.55e11},
            "gram_p1": {"count": 4, "ms": 2.0, "bytes": 4 * 3.28e9, "flops": 4 * 1.6e9},
            "qr": {"count": 0, "ms": 0.0, "bytes": 0.0, "flops": 0.0}}
    r = bench.rooflines(prof)
    assert set(r) == {"epoch", "gram_p1"}
    assert r["epoch"]["bound"] == "tensor" and r["epoch"]["unit"] == "TFLOP/s"
    assert abs(r["epoch"]["achieved"] - 6.55e11 / 15e-3 / 1e12) < 1e-9
    assert r["gram_p1"]["bound"] == "hbm" and abs(r["gram_p1"]["frac"] - r["gram_p1"]["achieved"] / r["gram_p1"]["peak"]) < 1e-12
    assert "note" in r["gram_p1"]
