"""Parity on the exact instances bench.py times (SURVEY §8(d) C2 / C3 / C4 /
C5), across several 128-window tiles, several window chunks and the tail
work items -- the paths the benchmark numbers come from -- against the CPU
oracle (oracle/port.py, pinned to the reference's golden vectors).

The stimulus is the benchmark's own: generated on the device
(gs_stim_synth, bit-identical to synth.stimulus, tests/test_synth_device.py),
as bench.py runs it.  Per-net T0/T1/TC/IG and the filter / discard totals must
be bit-exact; on sampled window ranges every gate waveform is compared on the
device (K7) against the oracle's arena.
"""

import os

import numpy as np
import pytest

import paper_2203_06117_b200 as api
from paper_2203_06117_b200 import _native, simcore, synth

pytestmark = pytest.mark.gpu

THREADS = os.cpu_count() or 4


def oracle_run(port, m, cfg, lo, hi, keep_arena=False):
    """The oracle over windows [lo, hi), in window segments that bound its
    host memory (~112 B per gate-window); per-net sums merge exactly
    (segmentation transparency, report.py:46-54)."""
    d = port.Design.from_arrays(m.num_pis, m.order, m.level_starts, m.pin_off, m.pin_net,
                                m.pin_ic, m.pin_arc, m.arc_rows, m.lut_off, m.lut_bits)
    seg = hi - lo if keep_arena else max(1, int(16e9 // (112 * max(1, m.num_gates))))
    N = m.num_nets
    ref = {"t1": np.zeros(N, np.int64), "tc": np.zeros(N, np.int64),
           "ig": np.zeros(N, np.int64)}
    tot = np.zeros(3, np.int64)
    a = s = None
    for x in range(lo, hi, seg):
        y = min(hi, x + seg)
        s = synth.stimulus(cfg, x, y)
        st = port.Stimulus.from_csr_fast(s.pi_off, s.pi_times, s.pi_init, s.boundaries)
        a = port.two_pass_simulate(d, st, pct=cfg.pct, threads=THREADS)
        r = port.compute_stats(d, st, a, threads=THREADS)
        for f in ("t1", "tc", "ig"):
            ref[f] += r[f]
        tot += [int(a["filtered"].sum()), int(a["ic_filtered"].sum()),
                int(a["discarded"].sum())]
        if not keep_arena:
            a = None
    ref["duration"] = (hi - lo) * cfg.period
    ref["t0"] = ref["duration"] - ref["t1"]
    ref["totals"] = tuple(int(v) for v in tot)
    return ref, a, s


def engine_stats(m, cfg, lo, hi, budget=0, items=None):
    dev = m.device()
    eng = _native.Engine(dev, budget)
    if items is not None:
        eng.set_items(*items)
    st = _native.SynthStimulus(dev, cfg, lo, hi)
    out = eng.run_stats(st, 0, hi - lo, cfg.pct)
    return out, eng.timing()


def check(got, ref, label):
    t1, tc, ig, tot = got
    assert np.array_equal(t1, ref["t1"]), f"{label}: t1"
    assert np.array_equal(ref["duration"] - t1, ref["t0"]), f"{label}: t0"
    assert np.array_equal(tc, ref["tc"]), f"{label}: tc"
    assert np.array_equal(ig, ref["ig"]), f"{label}: ig"
    assert tuple(tot) == ref["totals"], f"{label}: totals"
    assert int(tc.sum()) > 0


def test_c2_benched_instance_16_tiles(oracle_lib):
    # the full C2 design and the benchmark's stimulus, windows [0, 2048):
    # 16 tiles, 4 super-tiles per CTA step, head and tail items
    cfg = synth.config("C2")
    m = synth.design(cfg)
    ref, a, _ = oracle_run(oracle_lib, m, cfg, 0, 2048)
    got, tm = engine_stats(m, cfg, 0, 2048)
    check(got, ref, "C2 [0,2048)")
    got, tm = engine_stats(m, cfg, 0, 2048, items=(32, 2, 1))   # coarse head + re-cut tail
    check(got, ref, "C2 [0,2048) coarse items")


def test_c2_benched_instance_waveforms_on_device(oracle_lib):
    cfg = synth.config("C2")
    m = synth.design(cfg)
    ref, a, s = oracle_run(oracle_lib, m, cfg, 3000, 3300, keep_arena=True)
    bad, first = api.compare_on_device(m, s, a, pathpulse_pct=cfg.pct)
    assert (bad, first) == (0, None)


def test_c3_full_design_three_tiles_three_chunks(oracle_lib):
    # 1M gates over 300 windows (3 tiles, the last ragged) starting mid-run;
    # a small device budget splits them into 128-window chunks
    cfg = synth.config("C3")
    m = synth.design(cfg)
    ref, a, _ = oracle_run(oracle_lib, m, cfg, 5000, 5300)
    got, tm = engine_stats(m, cfg, 5000, 5300, budget=3 << 30, items=(64, 2, 1))
    assert tm["chunks"] >= 2
    check(got, ref, "C3 [5000,5300) chunked")
    got, tm = engine_stats(m, cfg, 5000, 5300)
    assert tm["chunks"] == 1
    check(got, ref, "C3 [5000,5300)")


@pytest.mark.parametrize("variant", ["C5", "C5-pct0", "C5-avg", "C5-avg-pct0"])
def test_c5_variants_full_design_two_tiles(oracle_lib, variant):
    cfg = synth.config(variant)
    m = synth.design(cfg)
    ref, a, s = oracle_run(oracle_lib, m, cfg, 777, 907)
    got, _ = engine_stats(m, cfg, 777, 907)
    check(got, ref, f"{variant} [777,907)")


def test_c4_full_design_two_tiles(oracle_lib):
    # 10M gates over 130 windows (two tiles, one of them a single window)
    cfg = synth.config("C4")
    m = synth.design(cfg)
    ref, a, _ = oracle_run(oracle_lib, m, cfg, 4000, 4130)
    got, _ = engine_stats(m, cfg, 4000, 4130)
    check(got, ref, "C4 [4000,4130)")


def test_device_accumulator_entry_equals_host_entry():
    # gs_run_stats_device (the timed entry of bench.py, NCCL all-reduce
    # buffer) adds exactly what gs_run_stats returns
    import torch
    cfg = synth.config("C2", gates=30_000, windows=1000)
    m = synth.design(cfg)
    dev = m.device()
    eng = _native.Engine(dev, 0)
    st = _native.SynthStimulus(dev, cfg, 0, 1000)
    t1, tc, ig, tot = eng.run_stats(st, 0, 1000, cfg.pct)
    N = m.num_nets
    acc = torch.full((3 * N + 3,), 5, dtype=torch.int64, device="cuda")
    eng.run_stats_device(st, 0, 1000, cfg.pct, acc.data_ptr())
    eng.run_stats_device(st, 0, 1000, cfg.pct, acc.data_ptr())
    v = acc.cpu().numpy() - 5
    assert np.array_equal(v[:N], 2 * t1) and np.array_equal(v[N:2 * N], 2 * tc)
    assert np.array_equal(v[2 * N:3 * N], 2 * ig)
    assert tuple(v[3 * N:]) == tuple(2 * x for x in tot)
