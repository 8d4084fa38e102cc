"""bench.py's roofline inputs come from committed files (CPU): the pipe peaks
(profiles/r02_peaks.json, measured by scripts/probe.py) and the ncu DRAM
traffic of the generation kernel (profiles/r0*_k_run_traffic.json), so every
`frac` in a bench line recomputes from committed numbers."""

from __future__ import annotations

import json
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))

import bench  # noqa: E402


def test_peaks_come_from_committed_probe_output():
    peaks = bench.load_peaks()
    probe = json.loads((ROOT / "profiles" / "r02_peaks.json").read_text())
    assert peaks["popc_per_s"] == probe["popc_per_s"] and 4e12 < peaks["popc_per_s"] < 5e12
    assert peaks["int8_tc_dense_ops_per_s"] > 4e15
    assert peaks["mma_64x64x32_per_s_per_sm"] > 1e7
    assert peaks["hbm_gbs"] > 6000


def test_traffic_parses_nested_ncu_metrics():
    for name in ("r01_k_run_traffic.json", "r02_k_run_traffic.json"):
        path = ROOT / "profiles" / name
        if not path.exists():
            continue
        d = json.loads(path.read_text())["metrics"]
        unit_r, val_r = d["dram__bytes_read.sum"]
        unit_w, val_w = d["dram__bytes_write.sum"]
        want = float(val_r) * bench._NCU_SCALE[unit_r] + float(val_w) * bench._NCU_SCALE[unit_w]
        got = bench.ncu_traffic(path)
        assert got is not None and abs(got - want) < 1.0 and got > 1e5, name


def test_algorithmic_bytes_of_the_bench_generation():
    # 4N fitness read + 2N parents read + 4N records + 4N fitness written
    assert bench.algorithmic_bytes_per_generation(20, 10_000) == 5_440_000
