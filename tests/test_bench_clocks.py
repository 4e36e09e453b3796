"""bench.py's clock sampler: the summary it reports under "clocks" (no GPU needed)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import bench  # noqa: E402


def _row(sm, reasons=()):
    names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
    return [str(sm), "1965", "300.00"] + ["Active" if n in reasons else "Not Active" for n in names]


def test_summary_keeps_samples_inside_the_timed_region():
    c = bench.ClockSampler(0)
    c.nvml = object()  # as if NVML had opened
    c.rows = [(0.5, _row(900, ("hw_slowdown",))),  # before the region: dropped
              (1.0, _row(1965)), (1.1, _row(1950, ("sw_power_cap",))), (1.2, _row(1965)),
              (2.5, _row(800, ("hw_thermal_slowdown",)))]  # after the region: dropped
    c.t0, c.t1 = 1.0, 1.2
    s = c.summary()
    assert s["samples"] == 3 and s["sampler"] == "nvml 5 ms"
    assert s["sm_mhz"] == 1965.0 and s["sm_max_mhz"] == 1965.0
    assert s["reasons"] == ["sw_power_cap"]


def test_summary_without_samples_says_unsampled():
    c = bench.ClockSampler(0)
    c.t0, c.t1 = 1.0, 1.2
    assert c.summary()["reasons"] == ["unsampled"]
