"""bench.py's clock summary: only the samples taken during the timed region count, and
throttle reasons are reported by name (CPU test on a synthetic nvidia-smi log)."""

from __future__ import annotations

import tempfile

import bench


def _sampler(lines, before):
    s = bench.ClockSampler(0)
    s.out = tempfile.TemporaryFile("w+")
    s.out.write("\n".join(lines) + "\n")
    s.lines_before = before
    return s


def test_summary_uses_samples_of_the_timed_region():
    idle = "0, 600, 1965, 200.0, 0x1, Not Active, Not Active, Not Active, Not Active"
    busy = "0, 1965, 1965, 700.0, 0x0, Not Active, Not Active, Not Active, Not Active"
    capped = "0, 1620, 1965, 990.0, 0x4, Not Active, Not Active, Not Active, Active"
    s = _sampler([idle, idle, busy, busy, capped], before=2)
    r = s.summary()
    assert r["samples"] == 3 and r["sm_mhz"] == 1965.0 and r["sm_max_mhz"] == 1965.0
    assert r["reasons"] == ["sw_power_cap"]


def test_summary_falls_back_to_all_samples_for_a_short_region():
    busy = "0, 1965, 1965, 700.0, 0x0, Not Active, Not Active, Not Active, Not Active"
    r = _sampler([busy], before=1).summary()
    assert r["samples"] == 1 and r["sm_mhz"] == 1965.0
