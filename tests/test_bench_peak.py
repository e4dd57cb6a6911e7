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
