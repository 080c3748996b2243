"""bench.py host logic without a GPU: the clock sampler keeps only samples taken
inside the timed region, and the default step counts keep that region long
enough for the 100 ms nvidia-smi period."""
import importlib.util
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _bench():
    spec = importlib.util.spec_from_file_location("bench_mod", os.path.join(ROOT, "bench.py"))
    mod = importlib.util.module_from_spec(spec)
    spec.loader.exec_module(mod)
    return mod


def _row(sm, reason="Not Active"):
    # index, clocks.sm, clocks.max.sm, power, active, hw, hw_thermal, sw_thermal, sw_power
    return ["0", str(sm), "1965", "700", "0x0", reason, "Not Active", "Not Active", "Not Active"]


def test_clock_sampler_keeps_only_in_region_samples():
    b = _bench()
    c = b.ClockSampler(0)
    c.t_start, c.t_end = 10.0, 11.0
    c.rows = [(9.9, _row(900)), (10.3, _row(1965)), (10.7, _row(1965, "Active")), (11.5, _row(300))]
    s = c.summary()
    assert s["samples"] == 2 and s["sm_mhz"] == 1965.0
    assert s["reasons"] == ["hw_slowdown"]  # the in-region row's reason; the idle row after is dropped
    assert "note" not in s


def test_clock_sampler_short_region_takes_first_sample_after_it():
    b = _bench()
    c = b.ClockSampler(0)
    c.t_start, c.t_end = 10.0, 10.04
    c.rows = [(9.9, _row(900)), (10.15, _row(1950)), (10.25, _row(1965))]
    s = c.summary()
    assert s["samples"] == 1 and s["sm_mhz"] == 1950.0 and "note" in s


def test_clock_sampler_unsampled():
    b = _bench()
    c = b.ClockSampler(0)
    assert c.summary()["reasons"] == ["unsampled"]


def test_default_steps(monkeypatch):
    b = _bench()
    for argv, want in [([], 200), (["--config", "C4"], 100), (["--config", "C5"], 20), (["--mode", "sim"], 60),
                       (["--impl", "reference"], 20), (["--steps", "7"], 7)]:
        monkeypatch.setattr(sys, "argv", ["bench.py", *argv])
        assert b.parse().steps == want, argv
