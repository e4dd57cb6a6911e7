"""bench.py's roofline denominator rule (choose_peak): sustained peak when the in-kernel SM
clock shows the power-limited regime, burst otherwise or when no clock was measured."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402

PEAKS = {"bf16_tflops": 1633.4, "bf16_tflops_sustained": 1374.5, "sm_max_mhz": 1965.0,
         "clocks_under_load": {"sm_mhz_median": 1320.0}}


def test_power_limited_clock_takes_sustained():
    peak, sus, why = bench.choose_peak(PEAKS, 1229)
    assert sus and peak == 1374.5 and "1229 MHz" in why


def test_boundary_is_inclusive_at_ten_percent():
    assert bench.choose_peak(PEAKS, 1452)[1]
    assert not bench.choose_peak(PEAKS, 1453)[1]


def test_full_clock_or_unmeasured_takes_burst():
    assert bench.choose_peak(PEAKS, 1965)[:2] == (1633.4, False)
    assert bench.choose_peak(PEAKS, None)[:2] == (1633.4, False)
    fallback = {"hbm_gbs": 6650.0, "bf16_tflops": 1590.0, "bf16_tflops_sustained": 1400.0}
    assert bench.choose_peak(fallback, 1200)[:2] == (1590.0, False)  # no clock record: burst
