"""bench.py keeps the driver's contract (one JSON line with the required keys).

The CPU test runs the reference arm on a small configuration; the GPU tests
run our arm on C2 (and the multi-rank path at one rank), with few steps.
"""
from __future__ import annotations

import json
import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
REQUIRED = {"metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better", "scaling",
            "vs_baseline", "dtype", "data", "config", "e2e"}


def _run(*args, timeout=600):
    r = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), *args], capture_output=True, text=True,
                       timeout=timeout, cwd=ROOT)
    assert r.returncode == 0, r.stdout + r.stderr
    lines = [ln for ln in r.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1, r.stdout
    return json.loads(lines[0])


def test_reference_arm_contract():
    if not os.path.exists(os.path.join(ROOT, "oracle", "_ref", "libndg_ref.so")):
        pytest.skip("oracle/_ref not built")
    line = _run("--impl", "reference", "--config", "c2", "--steps", "1", "--warmup", "1")
    assert REQUIRED <= set(line)
    assert line["impl"] == "reference" and line["value"] > 0
    assert line["cpu_baseline"]["kind"] == "reference" and line["cpu_baseline"]["cores"] >= 1
    assert line["e2e"]["h2d_bytes_per_step"] == 0


@pytest.mark.gpu
def test_bench_contract_on_gpu():
    line = _run("--config", "c2", "--steps", "3", "--warmup", "3", "--no-cpu-baseline")
    assert REQUIRED <= set(line) | {"roofline", "clocks", "gpu_launches"}
    assert line["value"] > 0 and line["e2e"]["value"] > 0 and line["gpu_launches"] > 0
    assert 0 < line["roofline"]["frac"] < 1.5 and line["roofline"]["bound"] == "hbm"
    assert line["exact_mode"]["value"] > 0
    assert line["n_gpus"] == 1 and line["scaling"] == "weak"


@pytest.mark.gpu
def test_bench_csv_row_in_the_reference_schema(tmp_path):
    from paper_2510_05254_b200 import report as rp
    path = tmp_path / "bench.csv"
    line = _run("--config", "c2", "--steps", "3", "--warmup", "3", "--no-cpu-baseline", "--no-exact-arm",
                "--csv", str(path))
    lines = path.read_text().splitlines()
    assert lines[0] == "# ndg-bench report" and lines[2] == ",".join(rp.COLUMNS)
    row = dict(zip(rp.COLUMNS, lines[3].split(",")))
    assert row["experiment"] == "timing" and row["steps"] == "3" and row["rk"] == "rk4"
    assert abs(float(row["wall_seconds"]) * 1e3 / 3 - line["ms_per_step"]) < 1e-9 * line["ms_per_step"]


@pytest.mark.gpu
def test_bench_multi_rank_path_at_one_rank():
    line = _run("--config", "c2", "--steps", "3", "--warmup", "3", "--no-cpu-baseline", "--no-exact-arm",
                "--force-exchange")
    assert line["value"] > 0
    assert "NCCL" in line["config"]["parallelism"]
