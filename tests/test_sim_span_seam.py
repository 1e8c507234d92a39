"""The sim_span-level seam (``gs_sim_span``): the reference's own per-level
driver (``simcore.py:295-463`` -- restated by ``oracle.port``'s count_pass /
store_pass) with each level's ``sim_span`` call (``_kernels.py:17-210``)
executed on the GPU instead of by the C restatement.  Both passes must
produce the oracle's arrays bit for bit: counts, offsets, the packed arena,
filter / discard counters and peaks.  The argument checks run on the host
and are covered without a GPU."""

import numpy as np
import pytest

import gen
import paper_2203_06117_b200 as api
from paper_2203_06117_b200 import _native
from oracle import port


def _gpu_level(d, stim, vals, gbuf, g_off, g_cap, g_cnt, filt, icf, disc, err, peak,
               lo, hi, w_lo, w_hi, pct, threads, cycle_parallelism):
    # same call the oracle's _sim_level makes, through the C-ABI seam
    _native.sim_span(lo, hi, w_lo, w_hi, w_lo, d.order, d.pin_off, d.pin_net, d.pin_ic,
                     d.pin_arc, d.arc_rows, d.lut_off, d.lut_bits, d.out_net, d.net_kind,
                     d.net_slot, stim.buf, stim.offsets, stim.counts, vals, stim.boundaries,
                     gbuf, g_off, g_cap, g_cnt, filt, icf, disc, err, peak, pct)


def _case(seed, **kw):
    docs = gen.make_docs(seed, **kw)
    nl, lv, delays, waves, duration, b, stim = gen.load(docs, api)
    d = port.Design(lv, delays)
    st = port.Stimulus(gen.oracle_inputs(nl, waves), b)
    return docs, d, st


def _both(d, st, pct, window_range, monkeypatch):
    vals = port.init_values(d, st)
    want_c = port.count_pass(d, st, vals, window_range, pct)
    want_a = port.store_pass(d, st, vals, want_c["peak"], window_range, pct)
    with monkeypatch.context() as m:
        m.setattr(port, "_sim_level", _gpu_level)
        got_c = port.count_pass(d, st, vals, window_range, pct)
        got_a = port.store_pass(d, st, vals, got_c["peak"], window_range, pct)
    return want_c, want_a, got_c, got_a


@pytest.mark.gpu
@pytest.mark.parametrize("seed", range(8))
def test_seam_matches_oracle_per_level(seed, monkeypatch):
    docs, d, st = _case(4000 + seed, max_k=3 + seed % 4, pct=(100, 60, 0, 100)[seed % 4],
                        max_toggles=40 + 20 * seed)
    W = st.num_windows
    rng = np.random.default_rng(seed)
    lo = int(rng.integers(0, W))
    for wr in ((0, W), (lo, W)):
        want_c, want_a, got_c, got_a = _both(d, st, docs.pct, wr, monkeypatch)
        for f in want_c:
            assert np.array_equal(got_c[f], want_c[f]), f
        for f in want_a:
            assert np.array_equal(got_a[f], want_a[f]), f


@pytest.mark.gpu
def test_seam_reports_overflow():
    # regions one short of the real count: err set, counting continues past
    # the region, nothing written outside it -- as the oracle does (first
    # level, whose fanins are all inputs)
    docs, d, st = _case(4100, n_gates=60, max_toggles=120)
    vals = port.init_values(d, st)
    c = port.count_pass(d, st, vals, None, docs.pct)
    if not (c["peak"] > 0).any():
        pytest.skip("no toggles")
    caps = np.maximum(c["peak"] - 1, 0)
    G, W = caps.shape
    # each region followed by a gap the overflowing (gate, window) reads but
    # nobody writes: sim_span reads its last stored edge at cnt - 1 >= cap,
    # which in a packed arena is a neighbour's region (order-dependent)
    span = c["peak"] + 1
    offsets = port.arena_offsets(span, d.order)
    lo, hi = int(d.level_starts[0]), int(d.level_starts[1])
    runs = []
    for level in (port._sim_level, _gpu_level):
        buf = np.full(int(span.sum()), -7, dtype=np.int64)
        z = [np.zeros((G, W), dtype=np.int64) for _ in range(6)]
        counts, filt, icf, disc, err, peak = z
        level(d, st, vals, buf, offsets, caps, counts, filt, icf, disc, err, peak,
              lo, hi, 0, W, docs.pct, 1, 32)
        runs.append((buf, *z))
    for x, y in zip(*runs):
        assert np.array_equal(x, y)
    err = runs[1][5]
    assert err[d.order[lo:hi]].any()


def test_seam_rejects_bad_ranges():
    try:
        _native.load()
    except RuntimeError:
        pytest.skip("libglsim_cuda.so not built")
    docs, d, st = _case(4200, n_gates=20)
    vals = port.init_values(d, st)
    G, W = d.num_gates, st.num_windows
    z = [np.zeros((G, W), dtype=np.int64) for _ in range(8)]
    g_off, g_cap, g_cnt, filt, icf, disc, err, peak = z
    gbuf = np.zeros(1, dtype=np.int64)
    args = lambda lo, hi, wl, wh, off: (lo, hi, wl, wh, off, d.order, d.pin_off, d.pin_net,  # noqa
                                        d.pin_ic, d.pin_arc, d.arc_rows, d.lut_off, d.lut_bits,
                                        d.out_net, d.net_kind, d.net_slot, st.buf, st.offsets,
                                        st.counts, vals, st.boundaries, gbuf, g_off, g_cap,
                                        g_cnt, filt, icf, disc, err, peak, 100)
    for bad in ((0, G + 1, 0, W, 0), (0, G, 0, W + 1, 0), (0, G, 1, W, 2), (-1, G, 0, W, 0)):
        with pytest.raises(ValueError):
            _native.sim_span(*args(*bad))
    g_cap[:] = 5  # regions past the end of gbuf
    with pytest.raises(ValueError):
        _native.sim_span(*args(0, G, 0, W, 0))
