"""The benchmark's device-generated stimulus (gs_stim_synth) is the host
generator's stimulus (synth.stimulus), bit for bit, for any window range --
including ranges that start mid-run (a window shard) -- and the per-window
activity weights (gs_synth_window_counts) are its per-window toggle counts."""

import numpy as np
import pytest

from paper_2203_06117_b200 import _native, synth

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("name,lo,hi", [("C2", 0, 300), ("C2", 777, 1000), ("C3", 0, 40),
                                        ("C3", 5003, 5040), ("C4", 0, 16), ("C4", 2_000, 2_010),
                                        ("C5-avg-pct0", 12, 20)])
def test_device_stimulus_equals_host_generator(name, lo, hi):
    cfg = synth.config(name)
    m = synth.design(synth.config(name, gates=10_000, levels=4))  # same inputs, small netlist
    dev = m.device()
    ds = _native.SynthStimulus(dev, cfg, lo, hi)
    b, off, times, init = ds.download()
    ref = synth.stimulus(cfg, lo, hi)
    assert np.array_equal(b, ref.boundaries)
    assert np.array_equal(off, ref.pi_off)
    assert np.array_equal(times, ref.pi_times)
    assert np.array_equal(init, ref.pi_init)
    w = _native.synth_window_counts(cfg, lo, hi)
    per_window = np.diff(np.searchsorted(np.sort(ref.pi_times), ref.boundaries, side="left"))
    assert np.array_equal(w, per_window)


def test_device_stimulus_runs_like_the_host_stimulus():
    cfg = synth.config("C2", gates=20_000, windows=512)
    m = synth.design(cfg)
    dev = m.device()
    eng = _native.Engine(dev, 0)
    a = eng.run_stats(_native.SynthStimulus(dev, cfg, 100, 612), 0, 512, cfg.pct)
    b = eng.run_stats(_native.Stimulus(dev, synth.stimulus(cfg, 100, 612)), 0, 512, cfg.pct)
    for x, y in zip(a[:3], b[:3]):
        assert np.array_equal(x, y)
    assert a[3] == b[3]


def test_synth_rejects_bad_ranges():
    cfg = synth.config("C2", gates=1000, levels=2)
    dev = synth.design(cfg).device()
    with pytest.raises(ValueError):
        _native.SynthStimulus(dev, cfg, 10, 10)
    with pytest.raises(ValueError):
        _native.SynthStimulus(dev, synth.config("C2", gates=1000, levels=2, pi_hi=2_000_000),
                              0, 4)
