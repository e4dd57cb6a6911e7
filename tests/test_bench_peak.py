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


class _FakeCtx:
    """Writes a synthetic trace: launches 0..5 alternate ag, rs; clock events carry cycles."""

    def __init__(self, mhz_by_launch):
        self.mhz = mhz_by_launch

    def trace_enable(self, cap):
        pass

    def trace_dump(self, path):
        import json
        ev = []
        for launch, mhz in enumerate(self.mhz):
            for k in range(5):
                dur = 10.0 + k  # us
                ev.append({"name": f"clock {int(mhz * dur)}", "cat": "clock", "ph": "X", "ts": 0, "dur": dur,
                           "pid": 0, "tid": 8, "args": {"launch": launch}})
                ev.append({"name": "mma 0", "cat": "mma", "ph": "X", "ts": 0, "dur": dur, "pid": 0, "tid": 3,
                           "args": {"launch": launch}})
        json.dump({"traceEvents": ev}, open(path, "w"))
        return len(ev)


def test_kernel_clocks_reads_ag_and_rs_launches_after_the_first_step():
    # launches: ag 1900 (first step, skipped), rs 1900 (skipped), ag 1200, rs 1300, ag 1210, rs 1290
    ctx = _FakeCtx([1900, 1900, 1200, 1300, 1210, 1290])
    calls = []
    out = bench.kernel_clocks(ctx, lambda: calls.append(1), steps=3)
    assert len(calls) == 3
    assert abs(out["ag_gemm"] - 1205) <= 5 and abs(out["gemm_rs"] - 1295) <= 5


def test_nvlink_roofline_matches_survey_table():
    """SURVEY §8(d) table, TP=8 rows: AG 58.7 MB / RS 117.4 MB of wire per rank; at 900 GB/s the
    RS is link-bound (130.5 us) and the AG tensor-bound."""
    r = bench.nvlink_roofline(8, 8192, 1792, False, 0.1, 0.14, 1626.5, 120.26e9)
    assert r["ag_gemm"]["wire_bytes_per_rank"] == 7 * 8192 * 4096 * 2 // 8 == 58720256
    assert r["gemm_rs"]["wire_bytes_per_rank"] == 7 * 8192 * 4096 * 4 // 8
    assert r["ag_gemm"]["bound"] == "tensor" and abs(r["ag_gemm"]["t_gemm_ms"] - 0.0739) < 1e-3
    assert r["gemm_rs"]["bound"] == "nvlink" and abs(r["gemm_rs"]["t_link_ms"] - 0.1305) < 1e-3
    loop = bench.nvlink_roofline(8, 8192, 1792, True, 0.77, 0.83, 1374.5, 962.07e9)
    assert not loop["exercised"] and "frac" not in loop["gemm_rs"]
