"""GPU parity: the CUDA engine (through the public API and the C ABI) against
the reference's own outputs (golden fixtures) and the CPU oracle.

Bar: bit-exact on every integer array -- arena buffer, offsets, capacities,
counts, window-start values, filter/discard counters, per-net T0/T1/TC/IG --
and byte-identical SAIF.
"""

import json

import numpy as np
import pytest

import gen
import paper_2203_06117_b200 as api
from paper_2203_06117_b200 import simcore
from paper_2203_06117_b200.waveform import StimulusSet
from conftest import golden_names, load_golden

pytestmark = pytest.mark.gpu

ARENA_FIELDS = ("buf", "offsets", "caps", "counts", "pass1_counts", "initials", "filtered",
                "ic_filtered", "discarded")


def gpu_run(docs, **cfg):
    nl, lv, delays, waves, duration, b, stim = gen.load(docs, api)
    arena, diag = api.run(lv, stim, delays,
                          api.RunConfig(mem_cap=None, pathpulse_pct=docs.pct, **cfg))
    stats = api.compute_stats(arena, stim)
    return nl, lv, delays, stim, arena, diag, stats


@pytest.mark.parametrize("name", golden_names())
def test_arena_and_stats_match_reference(name):
    docs, ref = load_golden(name)
    nl, lv, delays, stim, arena, diag, stats = gpu_run(docs)
    for f in ARENA_FIELDS:
        assert np.array_equal(getattr(arena, f), ref[f]), f"{name}: arena.{f}"
    for f in ("t0", "t1", "tc", "ig"):
        assert np.array_equal(getattr(stats, f), ref[f]), f"{name}: stats.{f}"
    assert api.write_saif(stats, nl.name) == ref["saif"]
    rep = json.loads(json.dumps(api.run_report(stats, diag)))
    for k, v in ref["report"].items():
        assert rep[k] == v, f"{name}: report[{k}]"


@pytest.mark.parametrize("name", golden_names())
def test_streaming_stats_match_reference(name):
    docs, ref = load_golden(name)
    nl, lv, delays, waves, duration, b, stim = gen.load(docs, api)
    model = api.compile_design(lv, delays)
    stats, diag = api.simulate_streaming(model, stim, api.RunConfig(pathpulse_pct=docs.pct))
    for f in ("t0", "t1", "tc", "ig"):
        assert np.array_equal(getattr(stats, f), ref[f]), f"{name}: {f}"
    assert api.write_saif(stats, nl.name) == ref["saif"]
    assert diag["discarded"] == ref["report"]["discarded_events"]
    assert diag["ic_filtered"] == ref["report"]["interconnect_filtered"]
    assert diag["filtered"] == ref["report"]["total_filtered"]


@pytest.mark.parametrize("seed", range(12))
def test_random_instances_match_oracle(oracle_lib, seed):
    pct = (100, 0, 50, 100, 90, 100)[seed % 6]
    docs = gen.make_docs(5000 + seed, n_gates=int(200 + 150 * seed), windows=8 + 9 * seed,
                         max_toggles=40 + 30 * seed, duration_ps=4000 + 2500 * seed, pct=pct,
                         max_levels=4 + seed)
    nl, lv, delays, stim, arena, diag, stats = gpu_run(docs)
    waves = gen.load(docs, api)[3]
    d, st, oa, os_ = oracle_lib.simulate(lv, delays, gen.oracle_inputs(nl, waves),
                                         stim.boundaries, pct=docs.pct, threads=4)
    for f in ("buf", "offsets", "caps", "counts", "initials", "filtered", "ic_filtered",
              "discarded"):
        assert np.array_equal(getattr(arena, f), oa[f]), f"seed {seed}: arena.{f}"
    for f in ("t0", "t1", "tc", "ig"):
        assert np.array_equal(getattr(stats, f), os_[f]), f"seed {seed}: {f}"


def test_windowed_stimulus_form_matches_csr():
    # a StimulusSet built from the reference's windowed arrays goes through the
    # windowed K1 variant; results must equal the CSR (K1 segmentation) path
    docs, ref = load_golden("many_windows")
    nl, lv, delays, waves, duration, b, stim = gen.load(docs, api)
    win = StimulusSet(b, stim.buf.copy(), stim.offsets.copy(), stim.counts.copy(),
                      stim.initials.copy(), stim.duration)
    assert not win.is_csr
    arena, _ = api.run(lv, win, delays, api.RunConfig(mem_cap=None))
    for f in ARENA_FIELDS:
        assert np.array_equal(getattr(arena, f), ref[f]), f


def test_chunked_run_equals_single_chunk(monkeypatch):
    # a tiny device budget forces many window chunks (and pool regrowth);
    # windows are independent, so every array must come out identical
    docs, ref = load_golden("many_windows")
    monkeypatch.setattr(simcore, "ENGINE_MEM_BUDGET", 96 << 20)
    simcore._Session._cache.clear()
    nl, lv, delays, stim, arena, diag, stats = gpu_run(docs)
    for f in ARENA_FIELDS:
        assert np.array_equal(getattr(arena, f), ref[f]), f
    for f in ("t0", "t1", "tc", "ig"):
        assert np.array_equal(getattr(stats, f), ref[f]), f
    simcore._Session._cache.clear()


def test_window_subranges_merge_to_full_run():
    docs, ref = load_golden("many_windows")
    nl, lv, delays, waves, duration, b, stim = gen.load(docs, api)
    model = api.compile_design(lv, delays)
    W = stim.num_windows
    parts = [(0, 7), (7, 40), (40, 41), (41, W)]
    total = None
    for lo, hi in parts:
        s, _ = api.simulate_streaming(model, stim, window_range=(lo, hi))
        total = s if total is None else total.merge(s)
    for f in ("t0", "t1", "tc", "ig"):
        assert np.array_equal(getattr(total, f), ref[f]), f
    assert total.duration == int(ref["duration"])


def test_empty_stimulus_and_single_inverter():
    lib = api.parse_library('{"cells":[{"name":"INV","inputs":["A"],"output":"Y","truth":"10"}]}')
    nl = api.parse_netlist('{"name":"o","inputs":["p0"],"outputs":["z"],"gates":'
                           '[{"name":"u","cell":"INV","pins":{"A":"p0","Y":"z"}}]}', lib)
    lv = api.levelize(nl)
    stim = StimulusSet.build({"p0": api.Waveform(0, [])}, nl, [0, 100])
    arena = api.two_pass_simulate(lv, stim, api.zero_delays(nl))
    assert arena.buf.size == 0 and not arena.counts.any()
    stim = StimulusSet.build({"p0": api.Waveform(0, [40])}, nl, [0, 100])
    arena = api.two_pass_simulate(lv, stim, api.zero_delays(nl))
    assert arena.caps[0, 0] == 1
    assert arena.waveform(0, 0) == api.Waveform(1, [40])


def test_narrow_pulses_fully_filtered():
    # reference acceptance criterion 4 (test_acceptance.py:113-136)
    lib = api.parse_library('{"cells":[{"name":"BUF","inputs":["A"],"output":"Y","truth":"01"}]}')
    nl = api.parse_netlist('{"name":"p","inputs":["a"],"outputs":["y"],"gates":'
                           '[{"name":"u","cell":"BUF","pins":{"A":"a","Y":"y"}}]}', lib)
    lv = api.levelize(nl)
    dl = api.zero_delays(nl)
    dl.tables[0][0][:] = [[5000, 5000]]
    rng = np.random.default_rng(99)
    t, times = 1, []
    for _ in range(1000):
        w = int(rng.integers(1, 5000))
        times += [t, t + w]
        t += w + int(rng.integers(5001, 20000))
    stim = StimulusSet.build({"a": api.Waveform(0, np.array(times))}, nl, [0, t + 10_000])
    arena = api.two_pass_simulate(lv, stim, dl)
    stats = api.compute_stats(arena, stim)
    assert int(arena.counts.sum()) == 0 and int(stats.ig[nl.net_index["y"]]) == 1000


def test_window_joint_discard_keeps_settled_value():
    # reference test_report.py:133-150: an edge past the window end is dropped,
    # the next window opens at the zero-delay settled value
    lib = api.parse_library('{"cells":[{"name":"BUF","inputs":["A"],"output":"Y","truth":"01"}]}')
    nl = api.parse_netlist('{"name":"b","inputs":["a"],"outputs":[],"gates":'
                           '[{"name":"u","cell":"BUF","pins":{"A":"a","Y":"y"}}]}', lib)
    lv = api.levelize(nl)
    d = api.zero_delays(nl)
    d.tables[0][0][:] = [[30, 30]]
    stim = StimulusSet.build({"a": api.Waveform(0, [40])}, nl, [0, 50, 100])
    arena = api.two_pass_simulate(lv, stim, d)
    assert arena.waveform(0, 0).times.size == 0 and int(arena.discarded[0, 0]) == 1
    assert arena.waveform(0, 1).initial == 1
    back, _ = api.parse_vcd(api.write_vcd(arena, ["y"]), api.parse_netlist(
        '{"name":"t","inputs":["y"],"outputs":[],"gates":[]}', lib))
    assert back["y"] == api.Waveform(0, [50])


def test_zero_delay_degenerates_to_collapsed_evaluation():
    # reference acceptance criterion 7: with no delays every output toggles
    # exactly where its zero-delay value changes
    for seed in range(6):
        docs = gen.make_docs(700 + seed, with_sdf=False, windows=3)
        nl, lv, delays, stim, arena, diag, stats = gpu_run(docs)
        assert int(arena.filtered.sum()) == 0
        for w in range(stim.num_windows):
            pieces = [stim.window_waveform(p, w) for p in range(nl.num_pis)]
            ts = np.unique(np.concatenate([x.times for x in pieces] + [np.zeros(0, np.int64)]))
            vals = np.zeros((nl.num_nets, ts.size + 1), dtype=np.uint8)
            for p, x in enumerate(pieces):
                vals[p, 0] = x.initial
                vals[p, 1:] = x.initial ^ (np.searchsorted(x.times, ts, side="right") & 1)
            for g in lv.order:
                gate = nl.gates[g]
                idx = sum(vals[n].astype(np.int64) << p for p, n in enumerate(gate.pin_nets))
                vals[gate.out_net] = gate.cell.truth[idx]
            for g in range(nl.num_gates):
                v = vals[nl.num_pis + g]
                assert np.array_equal(arena.waveform(g, w).times, ts[v[1:] != v[:-1]])


def test_event_queue_simulator_agrees_with_engine():
    # the independent event-queue simulator (reference oracle.py semantics)
    from paper_2203_06117_b200 import eventsim
    for seed in range(8):
        docs = gen.make_docs(900 + seed, pct=(100, 50)[seed % 2], avg=seed % 3 == 2)
        nl, lv, delays, stim, arena, diag, stats = gpu_run(docs)
        for w in range(stim.num_windows):
            waves = eventsim.oracle_simulate(lv, delays,
                                             [stim.window_waveform(p, w) for p in range(nl.num_pis)],
                                             int(stim.boundaries[w + 1]), pathpulse_pct=docs.pct)
            assert eventsim.compare_waveforms(arena, waves, w, nl) is None


def test_c_abi_init_values_matches_oracle(oracle_lib):
    docs, ref = load_golden("rnd09")
    nl, lv, delays, waves, duration, b, stim = gen.load(docs, api)
    model = api.compile_design(lv, delays)
    vals = simcore.initial_values(model, stim)
    d = oracle_lib.Design(lv, delays)
    st = oracle_lib.Stimulus(gen.oracle_inputs(nl, waves), b)
    assert np.array_equal(vals, oracle_lib.init_values(d, st))
    assert np.array_equal(vals[nl.num_pis:], ref["initials"])


def test_config_c1_ripple_carry_adder_matches_oracle(oracle_lib):
    # 20-bit ripple-carry adder, 1k windows, full SDF (COND +
    # INTERCONNECT), documents through the text front-ends
    from paper_2203_06117_b200 import synth
    lib_t, net_t, sdf_t, vcd_t, period = synth.rca_docs()
    docs = gen.Docs(lib_t, net_t, sdf_t, vcd_t, period)
    nl, lv, delays, stim, arena, diag, stats = gpu_run(docs)
    assert nl.num_gates == 100 and stim.num_windows == 1000
    waves = gen.load(docs, api)[3]
    d, st, oa, os_ = oracle_lib.simulate(lv, delays, gen.oracle_inputs(nl, waves),
                                         stim.boundaries, threads=4)
    for f in ("buf", "offsets", "caps", "counts", "initials", "filtered", "ic_filtered",
              "discarded"):
        assert np.array_equal(getattr(arena, f), oa[f]), f
    for f in ("t0", "t1", "tc", "ig"):
        assert np.array_equal(getattr(stats, f), os_[f]), f
    assert int(stats.tc.sum()) > 0


@pytest.mark.parametrize("variant", ["C5", "C5-pct0", "C5-avg", "C5-avg-pct0"])
def test_config_c5_variants_match_oracle(oracle_lib, variant):
    # SURVEY §8(d) C5 feature ablation on the C3 netlist family (full/averaged
    # SDF x pathpulse 100/0), checked on a scaled-down design and 64 windows
    from paper_2203_06117_b200 import synth
    cfg = synth.config(variant, gates=20_000, levels=25, ppis=2_000, pis=100, windows=64)
    m = synth.design(cfg)
    stim = synth.stimulus(cfg, 0, 64)
    stats, diag = api.simulate_streaming(m, stim, api.RunConfig(pathpulse_pct=cfg.pct))
    d = oracle_lib.Design.from_arrays(m.num_pis, m.order, m.level_starts, m.pin_off, m.pin_net,
                                      m.pin_ic, m.pin_arc, m.arc_rows, m.lut_off, m.lut_bits)
    st = oracle_lib.Stimulus.from_csr(stim.pi_off, stim.pi_times, stim.pi_init, stim.boundaries)
    a = oracle_lib.two_pass_simulate(d, st, pct=cfg.pct, threads=8)
    ref = oracle_lib.compute_stats(d, st, a, threads=8)
    for f in ("t0", "t1", "tc", "ig"):
        assert np.array_equal(getattr(stats, f), ref[f]), f
    assert diag["discarded"] == int(a["discarded"].sum())
    assert diag["ic_filtered"] == int(a["ic_filtered"].sum())


def test_c_abi_rejects_malformed_stimulus_on_device():
    # gs_stim_create validates the uploaded stimulus with a device kernel
    # (K0); malformed input is a ValueError naming the problem, as before
    from paper_2203_06117_b200 import _native
    docs, _ = load_golden("many_windows")
    nl, lv, delays, waves, duration, b, stim = gen.load(docs, api)
    dev = api.compile_design(lv, delays).device()
    off, times, init = stim.pi_off.copy(), stim.pi_times.copy(), stim.pi_init.copy()
    _native.Stimulus(dev, StimulusSet.from_csr(b, off, times, init))  # well formed
    p = int(np.argmax(np.diff(off) >= 2))   # an input with two or more toggles
    bad = times.copy()
    bad[off[p] + 1] = bad[off[p]]           # repeated toggle time
    with pytest.raises(ValueError, match="strictly increasing"):
        _native.Stimulus(dev, StimulusSet.from_csr(b, off, bad, init))
    win = StimulusSet(b, stim.buf.copy(), stim.offsets.copy(), stim.counts.copy(),
                      stim.initials.copy(), stim.duration)
    _native.Stimulus(dev, win)
    i = int(np.argmax(win.counts.ravel() >= 1))
    shifted = win.buf.copy()
    shifted[win.offsets.ravel()[i]] = b[-1] + 5   # toggle past its window
    with pytest.raises(ValueError, match="outside its window"):
        _native.Stimulus(dev, StimulusSet(b, shifted, win.offsets, win.counts, win.initials,
                                          win.duration))
    cnt = win.counts.copy()
    cnt.ravel()[i] = win.buf.size + 1                # region past the buffer
    with pytest.raises(ValueError, match="out of range"):
        _native.Stimulus(dev, StimulusSet(b, win.buf, win.offsets, cnt, win.initials,
                                          win.duration))


def slab_words(k):
    """Staged words per warp of the K4 instance for k-input gates (narrow time)."""
    from paper_2203_06117_b200 import _native
    return int(_native.load().gs_slab_words(int(k), 1))


@pytest.mark.parametrize("seed,max_toggles,pct", [(1, 250, 100), (2, 700, 100), (3, 1500, 100),
                                                  (4, 4000, 100), (2, 700, 50), (3, 1500, 0)])
def test_busy_tiles_take_every_staging_path(oracle_lib, seed, max_toggles, pct):
    # Tiles with many fanin toggles leave the staged fast path (fanin segments
    # and outputs in the warp's shared-memory slab, about 2 UB words) and are
    # read in place with outputs staged in the pool.  All must agree with the
    # oracle; the instances are checked to actually leave the staged path.
    docs = gen.make_docs(9100 + seed, n_gates=240, n_pis=6, windows=6, duration_ps=60_000,
                         max_toggles=max_toggles, max_delay=1_500, max_levels=5, pct=pct)
    nl, lv, delays, stim, arena, diag, stats = gpu_run(docs)
    waves = gen.load(docs, api)[3]
    d, st, oa, os_ = oracle_lib.simulate(lv, delays, gen.oracle_inputs(nl, waves),
                                         stim.boundaries, pct=pct, threads=4)
    for f in ("buf", "offsets", "caps", "counts", "initials", "filtered", "ic_filtered",
              "discarded"):
        assert np.array_equal(getattr(arena, f), oa[f]), f"arena.{f}"
    for f in ("t0", "t1", "tc", "ig"):
        assert np.array_equal(getattr(stats, f), os_[f]), f
    # fanin toggles UB of each gate's (single, 6-window) tile -> staging path
    m = api.compile_design(lv, delays)
    net_tc = np.concatenate([stim.counts.sum(axis=1), arena.counts.sum(axis=1)])
    ub = np.array([net_tc[m.pin_net[m.pin_off[i]:m.pin_off[i + 1]]].sum()
                   for i in range(nl.num_gates)])
    slab = np.array([slab_words(int(x)) for x in np.diff(m.pin_off)])
    assert int((2 * ub > slab).sum()) > 0, "instance never leaves the staged path"


def test_stimulus_upload_overlaps_a_running_simulation():
    # gs_stim_create runs on its own stream: a stimulus created from a worker
    # thread while the engine simulates (the overlapped e2e pattern) must give
    # the same per-net sums as the serial sequence
    from concurrent.futures import ThreadPoolExecutor
    from paper_2203_06117_b200 import _native, synth
    cfg = synth.config("C2", gates=20_000, windows=512)
    m = synth.design(cfg)
    stim = synth.stimulus(cfg, 0, 512)
    dev = m.device()
    eng = _native.Engine(dev, 0)
    ref = eng.run_stats(_native.Stimulus(dev, stim), 0, 512, cfg.pct)
    with ThreadPoolExecutor(1) as ex:
        fut = ex.submit(_native.Stimulus, dev, stim)
        for _ in range(4):
            s = fut.result()
            fut = ex.submit(_native.Stimulus, dev, stim)
            got = eng.run_stats(s, 0, 512, cfg.pct)
            del s
            for a, b in zip(got[:3], ref[:3]):
                assert np.array_equal(a, b)
            assert got[3] == ref[3]
        fut.result()


@pytest.mark.parametrize("name", ["demo_pct50", "busy_pct0", "many_windows", "rnd04"])
def test_arena_comes_from_one_simulation(monkeypatch, name):
    # two_pass_simulate runs the GPU simulation once: the count pass keeps
    # every region's peak entries (K5) and the store pass only scatters them
    # -- and the arena, transient slots of pct < 100 included, is the
    # reference's byte for byte
    from paper_2203_06117_b200 import _native
    calls = []
    real = _native.Engine.run_arena

    def counting(self, *a, **k):
        calls.append(k.get("offsets") is not None)
        return real(self, *a, **k)

    monkeypatch.setattr(_native.Engine, "run_arena", counting)
    docs, ref = load_golden(name)
    nl, lv, delays, stim, arena, diag, stats = gpu_run(docs)
    assert calls and not any(calls), "a second (store) simulation ran"
    for f in ARENA_FIELDS:
        assert np.array_equal(getattr(arena, f), ref[f]), f"{name}: arena.{f}"


def test_store_pass_with_foreign_capacities_simulates_and_checks():
    # capacities that are not the count pass's own take the real store pass,
    # which still detects a region overflowing its capacity
    docs, ref = load_golden("many_windows")
    nl, lv, delays, waves, duration, b, stim = gen.load(docs, api)
    model = api.compile_design(lv, delays)
    counted = simcore.count_pass(model, stim)
    caps = counted.peak.copy()
    g, w = np.argwhere(caps > 0)[0]
    caps[g, w] -= 1
    arena = api.allocate_arena(caps, model.order, stim.boundaries, (0, stim.num_windows), lv)
    with pytest.raises(api.ConsistencyError):
        simcore.store_pass(model, stim, None, arena)


def test_stats_then_arena_on_one_engine_resizes_the_chunk():
    # a stats run sizes its window chunk for stats metadata; an arena run on
    # the same engine must size its own (arena metadata is ~50 B per
    # gate-window more) instead of reusing the stats chunk and running out of
    # its budget
    from paper_2203_06117_b200 import _native, synth
    cfg = synth.config("C2", gates=20_000, levels=8, windows=4096)
    m = synth.design(cfg)
    dev = m.device()
    budget = 256 << 20
    eng = _native.Engine(dev, budget)
    st = _native.SynthStimulus(dev, cfg, 0, 4096)
    ref = eng.run_stats(st, 0, 4096, cfg.pct)
    stats_chunks = eng.timing()["chunks"]
    r = eng.run_arena(st, 0, 4096, cfg.pct, want_stats=True)
    assert eng.timing()["chunks"] > stats_chunks
    for a, b in zip(r["stats"][:3], ref[:3]):
        assert np.array_equal(a, b)
    again = eng.run_stats(st, 0, 4096, cfg.pct)
    assert eng.timing()["chunks"] <= stats_chunks
    for a, b in zip(again[:3], ref[:3]):
        assert np.array_equal(a, b)
