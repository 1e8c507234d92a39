"""Parity at BASELINE.json's full design sizes.

The CPU oracle cannot run 1M gates x 100k windows, but windows are
independent, so the exact check is made on sampled window ranges of the
full-size design -- including ranges that start mid-run (the stimulus
generator derives the window-start values from the toggle parity before the
range, as a window shard of a multi-GPU run does).  Per-net T0/T1/TC/IG and the
filter / discard totals must equal the oracle's bit for bit.
"""

import os

import numpy as np
import pytest

import paper_2203_06117_b200 as api
from paper_2203_06117_b200 import synth

pytestmark = pytest.mark.gpu


def _oracle_stats(oracle_lib, m, stim, pct):
    threads = os.cpu_count() or 4
    d = oracle_lib.Design.from_arrays(m.num_pis, m.order, m.level_starts, m.pin_off, m.pin_net,
                                      m.pin_ic, m.pin_arc, m.arc_rows, m.lut_off, m.lut_bits)
    st = oracle_lib.Stimulus.from_csr(stim.pi_off, stim.pi_times, stim.pi_init, stim.boundaries)
    a = oracle_lib.two_pass_simulate(d, st, pct=pct, threads=threads)
    return oracle_lib.compute_stats(d, st, a, threads=threads), a


@pytest.mark.parametrize("name,ranges", [
    ("C3", [(0, 3), (1001, 1003)]),
    ("C5-avg-pct0", [(0, 2)]),
    ("C4", [(0, 2), (777, 778)]),
])
def test_full_size_design_on_sampled_windows(oracle_lib, name, ranges):
    cfg = synth.config(name)
    m = synth.design(cfg)
    assert m.num_gates == cfg.gates
    for lo, hi in ranges:
        stim = synth.stimulus(cfg, lo, hi)
        stats, diag = api.simulate_streaming(m, stim, api.RunConfig(pathpulse_pct=cfg.pct))
        ref, a = _oracle_stats(oracle_lib, m, stim, cfg.pct)
        for f in ("t0", "t1", "tc", "ig"):
            assert np.array_equal(getattr(stats, f), ref[f]), f"{name} [{lo},{hi}) {f}"
        assert diag["discarded"] == int(a["discarded"].sum())
        assert diag["ic_filtered"] == int(a["ic_filtered"].sum())
        assert int(stats.tc.sum()) > 0


@pytest.mark.parametrize("name,lo,hi", [("C3", 2, 5), ("C4", 11, 12)])
def test_full_size_waveforms_on_device(oracle_lib, name, lo, hi):
    # every gate waveform of the full-size design (1M / 10M gates) on sampled
    # windows, checked on the device against the oracle's arena (K7) -- and a
    # perturbed reference is caught at the perturbed (gate, window)
    cfg = synth.config(name)
    m = synth.design(cfg)
    stim = synth.stimulus(cfg, lo, hi)
    _, a = _oracle_stats(oracle_lib, m, stim, cfg.pct)
    bad, first = api.compare_on_device(m, stim, a, pathpulse_pct=cfg.pct)
    assert (bad, first) == (0, None)
    counts = a["counts"]
    g, w = map(int, np.argwhere(counts > 0)[len(np.argwhere(counts > 0)) // 2])
    buf = a["buf"].copy()
    buf[a["offsets"][g, w]] += 1
    bad, first = api.compare_on_device(m, stim, dict(a, buf=buf), pathpulse_pct=cfg.pct)
    assert (bad, first) == (1, (g, w))
