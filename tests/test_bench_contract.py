"""bench.py's constants and derived figures (CPU): the algorithmic bytes per
correlation of SURVEY 8(d), the workload shapes of BASELINE configs[1..4] and
the paper's perf-ratio arithmetic (proj/src/harness.cpp:15-25)."""
import math
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import bench  # noqa: E402


def test_algorithmic_bytes_per_correlation():
    # 8(N/2+1)/B + 4n + (4W + 8W + 8(N/2+1))/C, N = 870,912, n = 65,741
    assert bench.B_CODE_HALF == 3_483_656
    assert bench.B_REPLICA == 262_964
    assert abs(bench.bytes_per_corr(9, 64) - 854_469) < 1.0


def test_search_workload_shape():
    assert bench.W == 800_000 and bench.ADV == 720_000 and bench.FS == 8.0e6
    assert bench.N_WIN == 11            # 1 s of stream at advance 720,000
    assert len(bench.BINS) == 9 and bench.BINS[0] == -400e3 and bench.BINS[-1] == 400e3
    for wl in ("search", "roster", "streams"):
        cfg = bench.workload_config(1, wl)
        assert cfg["windows"] == 11 and cfg["bins"] == 9 and cfg["window_len"] == 800_000
    assert bench.workload_config(8, "roster")["codes_per_gpu"] * 8 >= 1024


def test_paper_perf_ratio_arithmetic():
    # perf_ratio = (time per pattern) / window duration; tags at a 50 % share = floor(0.5 / ratio)
    corr_per_s = 445_000.0
    ratio = (1.0 / corr_per_s) / (bench.W / bench.FS)
    assert abs(ratio - 2.247e-5) < 1e-8
    assert int(math.floor(0.5 / ratio)) == 22_250


def test_roofline_formula():
    # bound fp32, frac = achieved / peak, attainable = min(HBM roof, FP32 roof)
    r = bench.roofline(6336, 13.0, 150.0, 6556.2, bench.bytes_per_corr(9, 64))
    assert r["bound"] == "fp32" and r["unit"] == "TFLOP/s"
    assert abs(r["achieved"] - 6336 * 47.6e6 / 13e-3 / 1e12) < 1e-9
    assert abs(r["frac"] - r["achieved"] / 150.0) < 1e-12
    fp32_roof = 150e12 / 47.6e6
    hbm_roof = 6556.2e9 / bench.bytes_per_corr(9, 64)
    assert abs(r["attainable_corr_per_s"] - min(fp32_roof, hbm_roof)) < 1e-6
    assert abs(r["frac_of_attainable"] - (6336 / 13e-3) / min(fp32_roof, hbm_roof)) < 1e-12
    assert abs(r["hbm"]["frac"] - bench.bytes_per_corr(9, 64) * 6336 / 13e-3 / 6556.2e9) < 1e-12
