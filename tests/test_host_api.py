"""Host-side API (no GPU): front-ends, windows, writers, scheduler planning and
the single-gate object layer, checked against the reference test suite's
known answers (``pkg/tests/test_{netlist,sdf,waveform,report,scheduler,
simcore,oracle}.py``)."""

import json

import numpy as np
import pytest
from hypothesis import given, settings
from hypothesis import strategies as st

import glsim
import paper_2203_06117_b200 as api
from paper_2203_06117_b200 import (ActivityStats, CapacityError, GateSimState, ParseError,
                                   RunConfig, SemanticError, StimulusSet, Waveform,
                                   emit_output, plan_segments, simulate_gate_window)

LIB3 = json.dumps({"cells": [
    {"name": "INV", "inputs": ["A"], "output": "Y", "truth": "10"},
    {"name": "AND2", "inputs": ["A", "B"], "output": "Y", "truth": "0001"},
    {"name": "MUX2", "inputs": ["A", "B", "S"], "output": "Y", "truth": "01010011"},
    {"name": "AND3", "inputs": ["A", "B", "C"], "output": "Y", "truth": "00000001"},
]})


def lib():
    return api.parse_library(LIB3)


def net(gates, inputs=("a", "b"), outputs=()):
    return api.parse_netlist(json.dumps({"name": "t", "inputs": list(inputs),
                                         "outputs": list(outputs), "gates": gates}), lib())


# ---------------------------------------------------------------- glsim alias

def test_glsim_alias_is_the_same_modules():
    import glsim.scheduler
    import glsim.simcore
    from glsim.oracle import compare_waveforms, oracle_simulate  # noqa: F401
    assert glsim.simcore is api.simcore
    assert glsim.scheduler.simcore is api.simcore
    assert glsim.simulate is api.simulate
    assert set(api.__all__) >= {"simulate", "two_pass_simulate", "write_saif", "parse_vcd",
                                "oracle_simulate", "StimulusSet", "WaveformArena"}


# ---------------------------------------------------------------- netlist

class TestNetlist:
    def test_lut_and_index_order(self):
        l = lib()
        assert api.eval_lut(l["AND2"], [1, 1]) == 1
        assert api.eval_lut(l["MUX2"], [0, 1, 1]) == int("01010011"[6])

    @pytest.mark.parametrize("doc,match", [
        ('{"cells":[{"name":"X","inputs":["A","B"],"output":"Y","truth":"001"}]}', "length 4"),
        ('{"cells":[{"name":"X","inputs":["A"],"output":"Y","truth":"0x"}]}', "only 0 and 1"),
        ('{"cells":[{"name":"X","inputs":["A","A"],"output":"Y","truth":"0011"}]}', "unique"),
        ("{nope", None),
    ])
    def test_library_parse_errors(self, doc, match):
        with pytest.raises(ParseError, match=match):
            api.parse_library(doc)

    def test_too_many_inputs(self):
        pins = [f"I{i}" for i in range(17)]
        with pytest.raises(ParseError, match="maximum"):
            api.parse_library(json.dumps({"cells": [{"name": "X", "inputs": pins, "output": "Y",
                                                     "truth": "0" * (1 << 17)}]}))

    def test_duplicate_cell(self):
        doc = {"cells": [{"name": "X", "inputs": ["A"], "output": "Y", "truth": "01"}] * 2}
        with pytest.raises(SemanticError, match="duplicate cell"):
            api.parse_library(json.dumps(doc))

    @pytest.mark.parametrize("gates,match", [
        ([{"name": "u1", "cell": "INV", "pins": {"A": "ghost", "Y": "y"}}], "undriven"),
        ([{"name": "u1", "cell": "INV", "pins": {"A": "a", "Y": "n1"}},
          {"name": "u2", "cell": "INV", "pins": {"A": "b", "Y": "n1"}}], "multiple drivers"),
        ([{"name": "u1", "cell": "NOPE", "pins": {"A": "a", "Y": "y"}}], "unknown cell"),
        ([{"name": "u1", "cell": "INV", "pins": {"A": "a", "Q": "x", "Y": "y"}}], "unknown pin"),
        ([{"name": "u1", "cell": "AND2", "pins": {"A": "a", "Y": "y"}}], "unbound"),
        ([{"name": "u1", "cell": "INV", "pins": {"A": "a", "Y": "n1"}},
          {"name": "u1", "cell": "INV", "pins": {"A": "b", "Y": "n2"}}], "duplicate gate"),
    ])
    def test_netlist_semantic_errors(self, gates, match):
        with pytest.raises(SemanticError, match=match):
            net(gates)

    def test_interning_and_round_trip(self):
        n = net([{"name": "u1", "cell": "INV", "pins": {"A": "a", "Y": "n1"}},
                 {"name": "u2", "cell": "INV", "pins": {"A": "n1", "Y": "n2"}}])
        assert n.net_names == ["a", "b", "n1", "n2"]
        assert n.driver_gate(n.net_index["n2"]) == 1
        n2 = api.parse_netlist(api.serialize_netlist(n), lib())
        assert n2.net_names == n.net_names
        assert [(g.name, g.pin_nets, g.out_net) for g in n2.gates] == \
               [(g.name, g.pin_nets, g.out_net) for g in n.gates]
        l2 = api.parse_library(api.serialize_library(lib()))
        assert set(l2.cells) == set(lib().cells)

    def test_levelize_chain_diamond_cycle(self):
        n = net([{"name": "u1", "cell": "INV", "pins": {"A": "a", "Y": "n1"}},
                 {"name": "u2", "cell": "INV", "pins": {"A": "n1", "Y": "n2"}},
                 {"name": "u3", "cell": "AND2", "pins": {"A": "n1", "B": "n2", "Y": "n3"}}])
        lv = api.levelize(n)
        assert list(lv.level_of) == [1, 2, 3]
        assert lv.order.tolist() == [0, 1, 2] and lv.level_starts.tolist() == [0, 1, 2, 3]
        cyc = net([{"name": "u1", "cell": "AND2", "pins": {"A": "a", "B": "n2", "Y": "n1"}},
                   {"name": "u2", "cell": "INV", "pins": {"A": "n1", "Y": "n2"}}])
        with pytest.raises(SemanticError, match="cycle through gate"):
            api.levelize(cyc)

    def test_levelize_soundness_random(self):
        import gen
        rng = np.random.default_rng(11)
        for _ in range(15):
            libd = gen.library_doc(rng)
            doc, _ = gen.netlist_doc(rng, libd, int(rng.integers(10, 150)), 6)
            n = api.parse_netlist(json.dumps(doc), api.parse_library(json.dumps(libd)))
            lv = api.levelize(n)
            for gi, g in enumerate(n.gates):
                fl = [int(lv.level_of[n.driver_gate(x)]) if n.driver_gate(x) >= 0 else 0
                      for x in g.pin_nets]
                assert lv.level_of[gi] == 1 + max(fl)
            for li, bucket in enumerate(lv.levels):
                assert list(bucket) == sorted(bucket)
                assert all(lv.level_of[g] == li + 1 for g in bucket)


# ---------------------------------------------------------------- sdf

def and2():
    return net([{"name": "u1", "cell": "AND2", "pins": {"A": "a", "B": "b", "Y": "y"}}])


class TestSdf:
    def test_units_cond_and_overwrite(self):
        inv = net([{"name": "u1", "cell": "INV", "pins": {"A": "a", "Y": "y"}}], inputs=["a"])
        d = api.parse_sdf('(DELAYFILE (TIMESCALE 1ns) (CELL (INSTANCE u1)'
                          ' (DELAY (ABSOLUTE (IOPATH A Y (0.3::) (0.5::))))))', inv)
        assert d.tables[0][0].tolist() == [[300_000, 500_000]]
        d = api.parse_sdf('(DELAYFILE (TIMESCALE 1ps) (CELL (INSTANCE u1) (DELAY (ABSOLUTE'
                          ' (IOPATH A Y (1.0) (1.0)) (COND !B (IOPATH A Y (7.0) (7.0)))))))',
                          and2())
        assert d.tables[0][0][:, 0].tolist() == [7000, 1000]

    def test_corners(self):
        inv = net([{"name": "u1", "cell": "INV", "pins": {"A": "a", "Y": "y"}}], inputs=["a"])
        body = '(CELL (INSTANCE u1) (DELAY (ABSOLUTE (IOPATH A Y (1.0:2.0:3.0) (1:2:3)))))'
        for corner, want in [("min", 1000), ("typ", 2000), ("max", 3000)]:
            d = api.parse_sdf(f"(DELAYFILE (TIMESCALE 1ps) {body})", inv, corner=corner)
            assert d.tables[0][0][0, 0] == want

    def test_cond_equality_literals(self):
        n = net([{"name": "u1", "cell": "AND3", "pins": {"A": "a", "B": "b", "C": "c", "Y": "y"}}],
                inputs=["a", "b", "c"])
        d = api.parse_sdf('(DELAYFILE (TIMESCALE 1ps) (CELL (INSTANCE u1) (DELAY (ABSOLUTE'
                          ' (COND B==1 && C==0 (IOPATH A Y (9.0) (9.0)))))))', n)
        assert d.tables[0][0][:, 0].tolist() == [0, 9000, 0, 0]

    def test_interconnect_and_errors(self):
        n = net([{"name": "u1", "cell": "INV", "pins": {"A": "a", "Y": "n1"}},
                 {"name": "u2", "cell": "AND2", "pins": {"A": "n1", "B": "b", "Y": "y"}}])
        d = api.parse_sdf('(DELAYFILE (TIMESCALE 1ps) (CELL (INSTANCE u2) (DELAY (ABSOLUTE'
                          ' (INTERCONNECT u1/Y u2/A (0.7)) (INTERCONNECT b u2/B (0.4))))))', n)
        assert d.interconnect[1].tolist() == [700, 400]
        with pytest.raises(SemanticError, match="connectivity"):
            api.parse_sdf('(DELAYFILE (CELL (INSTANCE u2) (DELAY (ABSOLUTE'
                          ' (INTERCONNECT a u2/A (0.7))))))', n)
        with pytest.raises(SemanticError, match="unknown instance"):
            api.parse_sdf('(DELAYFILE (CELL (INSTANCE zz) (DELAY (ABSOLUTE (IOPATH A Y (1))))))', n)
        with pytest.raises(SemanticError, match="switching pin"):
            api.parse_sdf('(DELAYFILE (CELL (INSTANCE u2) (DELAY (ABSOLUTE'
                          ' (COND A (IOPATH A Y (1) (1)))))))', n)
        with pytest.raises(ParseError, match="negative"):
            api.parse_sdf('(DELAYFILE (CELL (INSTANCE u2) (DELAY (ABSOLUTE (IOPATH A Y (-1))))))', n)
        with pytest.raises(ParseError) as e:
            api.parse_sdf("(DELAYFILE (CELL (INSTANCE u1)", n, path="x.sdf")
        assert "x.sdf" in str(e.value) and e.value.line is not None

    def test_unsupported_sections_warn(self):
        inv = net([{"name": "u1", "cell": "INV", "pins": {"A": "a", "Y": "y"}}], inputs=["a"])
        d = api.parse_sdf('(DELAYFILE (CELL (INSTANCE u1) (TIMINGCHECK (SETUP x y (1)))'
                          ' (DELAY (ABSOLUTE (IOPATH A Y (1) (1))))))', inv)
        assert any("TIMINGCHECK" in w for w in d.warnings)
        assert d.tables[0][0][0, 0] == d.timescale_fs

    def test_lookup_and_average(self):
        d = api.zero_delays(and2())
        d.tables[0][0][:] = [[100, 200], [300, 400]]
        assert api.lookup_delay(d, 0, [0], [1, 1], "rise") == 300
        avg = api.average_tables(d)
        assert avg.tables[0][0].tolist() == [[200, 300], [200, 300]]
        assert avg.delay_mode == "averaged"
        d.tables[0][0][:] = [[1, 1], [2, 2]]
        assert api.average_tables(d).tables[0][0][0].tolist() == [2, 2]  # half up

    @given(st.integers(1, 5))
    @settings(max_examples=20, deadline=None)
    def test_condition_index_bijective(self, k):
        seen = {api.condition_index(None, 0, [(r >> j) & 1 for j in range(k - 1)])
                for r in range(1 << (k - 1))}
        assert seen == set(range(1 << (k - 1)))


# ---------------------------------------------------------------- waveform

def pi_net(names):
    return api.parse_netlist(json.dumps({"name": "t", "inputs": list(names), "outputs": [],
                                         "gates": []}), lib())


VCD = ("$timescale 1 ps $end\n$scope module tb $end\n$var wire 1 ! a $end\n$upscope $end\n"
       "$enddefinitions $end\n")


class TestWaveform:
    def test_vcd_basics(self):
        w, dur = api.parse_vcd(VCD + "#0\n0!\n#10\n1!\n#25\n0!\n", pi_net(["a"]))
        assert w["a"] == Waveform(0, [10000, 25000]) and dur == 25000
        assert api.parse_vcd(VCD + "#0\nx!\n#5\n1!\n", pi_net(["a"]))[0]["a"] == Waveform(0, [5000])
        assert api.parse_vcd(VCD + "#0\n1!\n#7\n1!\n", pi_net(["a"]))[0]["a"] == Waveform(1, [])
        w, _ = api.parse_vcd(VCD + "#0\n0!\n#5\n1!\n0!\n#9\n1!\n", pi_net(["a"]))
        assert w["a"] == Waveform(0, [9000])

    @pytest.mark.parametrize("text,exc,match", [
        (VCD + "#0\n0!\n", SemanticError, "no scalar variable"),
        ("$timescale 1 ps $end\n$var wire 8 ! a $end\n$enddefinitions $end\n#0\n", SemanticError,
         "vector variable"),
        (VCD + "#10\n0!\n#5\n1!\n", ParseError, "non-monotonic"),
        ("$var wire 1 ! a $end\n$enddefinitions $end\n#0\n0!\n", ParseError, "timescale"),
    ])
    def test_vcd_errors(self, text, exc, match):
        names = ["a", "zz"] if match == "no scalar variable" else ["a"]
        with pytest.raises(exc, match=match):
            api.parse_vcd(text, pi_net(names))

    def test_slice_and_boundaries(self):
        parts = api.slice_windows(Waveform(0, [20]), [0, 20, 40])
        assert parts[0] == Waveform(0, []) and parts[1] == Waveform(0, [20])
        with pytest.raises(ValueError, match="ascending"):
            api.slice_windows(Waveform(0, []), [0, 20, 20])
        assert api.window_boundaries(100, period=30).tolist() == [0, 30, 60, 90, 100]
        assert api.window_boundaries(100, period=40, offset=15).tolist() == [0, 15, 55, 95, 100]
        assert api.window_boundaries(100, explicit=[0, 50, 120]).tolist() == [0, 50, 120]
        for kw, match in [({"explicit": [0, 50]}, "lasts"), ({"explicit": [10, 120]}, "start at 0")]:
            with pytest.raises(ValueError, match=match):
                api.window_boundaries(100, **kw)
        with pytest.raises(ValueError, match="positive"):
            api.window_boundaries(0)

    @given(st.lists(st.integers(0, 400), max_size=30, unique=True), st.integers(0, 1),
           st.lists(st.integers(1, 399), max_size=5, unique=True))
    @settings(max_examples=60, deadline=None)
    def test_slice_reconstructs(self, times, initial, cuts):
        w = Waveform(initial, sorted(times))
        b = [0] + sorted(cuts) + [400]
        for j, part in enumerate(api.slice_windows(w, b)):
            for t in range(b[j], b[j + 1], 7):
                assert part.value_at(t) == w.value_at(t)

    def test_stimulus_set_csr_matches_reference_windowing(self):
        n = pi_net(["a", "b"])
        waves = {"a": Waveform(0, [10, 25, 30]), "b": Waveform(1, [22])}
        s = StimulusSet.build(waves, n, [0, 20, 40])
        assert s.is_csr and s.num_windows == 2
        # windowed view equals slice_windows piece by piece (waveform.py:243-265)
        for pi, name in enumerate(["a", "b"]):
            for wi, piece in enumerate(api.slice_windows(waves[name], [0, 20, 40])):
                assert s.window_waveform(pi, wi) == piece
                o, c = s.offsets[pi, wi], s.counts[pi, wi]
                assert Waveform(int(s.initials[pi, wi]), s.buf[o:o + c]) == piece
        with pytest.raises(SemanticError, match="no stimulus"):
            StimulusSet.build({"a": Waveform(0, [])}, n, [0, 10])

    def test_allocate_arena(self):
        a = api.allocate_arena(np.array([[3], [0], [5]]), np.array([0, 1, 2]), np.array([0, 10]),
                               (0, 1))
        assert a.offsets[:, 0].tolist() == [0, 3, 3] and a.buf.size == 8
        a = api.allocate_arena(np.array([[2], [3], [4]]), np.array([2, 0, 1]), np.array([0, 10]),
                               (0, 1))
        assert a.offsets[:, 0].tolist() == [4, 6, 0]
        with pytest.raises(CapacityError) as e:
            api.allocate_arena(np.array([[1], [1]]), np.array([0, 1]), np.array([0, 10]), (0, 1),
                               mem_cap=1)
        assert e.value.required_bytes == 16


# ---------------------------------------------------------------- report

def one(t0, t1, tc, ig, dur):
    return ActivityStats(["n"], np.array([t0]), np.array([t1]), np.array([tc]), np.array([ig]),
                         dur, 1)


class TestReport:
    def test_saif_golden_single_net(self):
        assert api.write_saif(one(40, 60, 4, 0, 100), "demo") == (
            '(SAIFILE\n  (SAIFVERSION "2.0")\n  (DIRECTION "backward")\n  (DESIGN "demo")\n'
            "  (TIMESCALE 1 fs)\n  (DURATION 100)\n  (INSTANCE demo\n    (NET\n      (n\n"
            "        (T0 40) (T1 60) (TX 0)\n        (TC 4) (IG 0)\n      )\n    )\n  )\n)\n")

    def test_saif_variants(self):
        assert "(IG" not in api.write_saif(one(40, 60, 4, 2, 100), "x", include_ig=False)
        s = ActivityStats(["bus[3]"], np.array([1]), np.array([0]), np.array([0]),
                          np.array([0]), 1, 1)
        assert "bus\\[3\\]" in api.write_saif(s, "x")
        e = ActivityStats([], *(np.empty(0, np.int64) for _ in range(4)), 10, 1)
        assert "(NET\n    )" in api.write_saif(e, "void")

    def test_merge_and_factor(self):
        a = one(40, 60, 4, 1, 100)
        m = a.merge(one(10, 20, 2, 0, 30))
        assert (int(m.t0[0]), int(m.tc[0]), m.duration, m.windows) == (50, 6, 130, 2)
        assert a.activity_factor == 4.0

    def test_run_report_shape(self):
        r = api.run_report(one(40, 60, 4, 1, 100), {"timings": {"pass1": 0.5}, "discarded": 3})
        assert (r["duration"], r["total_tc"], r["total_filtered"], r["discarded_events"]) == \
               (100, 4, 1, 3)
        assert set(r["timings"]) == {"parse", "pass1", "alloc", "pass2", "report"}
        json.dumps(r)


# ---------------------------------------------------------------- scheduler

class TestScheduler:
    def test_plan_segments(self):
        assert plan_segments(np.ones((3, 4), dtype=np.int64), 10_000) == [(0, 4)]
        assert plan_segments(np.ones((1, 4), dtype=np.int64), 16) == [(0, 2), (2, 4)]
        assert plan_segments(np.ones((1, 4), dtype=np.int64), None) == [(0, 4)]
        with pytest.raises(CapacityError, match="alone"):
            plan_segments(np.array([[3, 1]]), 16)

    def test_run_config(self):
        for kw in ({"cycle_parallelism": 0}, {"pathpulse_pct": 101}, {"workers": -1}):
            with pytest.raises(ValueError):
                RunConfig(**kw)
        assert RunConfig(workers=0).resolved_workers >= 1
        assert RunConfig(workers=3).resolved_workers == 3


# ---------------------------------------------------------------- object layer

def cur(times, ic=0, initial=0):
    return api.PinCursor.from_waveform(Waveform(initial, times), ic)


class TestObjectLayer:
    def test_next_event_and_msi(self):
        assert api.next_event_time([cur([100], ic=10), cur([105])]) == 105
        a = cur([50, 52], ic=5)
        assert api.next_event_time([a]) is api.EXHAUSTED and a.filtered == 1
        assert api.next_event_time([cur([50, 55], ic=5)]) == 55  # width == delay survives
        a, b = cur([190], ic=10), cur([200])
        t = api.next_event_time([a, b])
        assert t == 200 and api.resolve_msi([a, b], t)[1] == [0, 1]

    def test_emit_output_kats(self):
        s = GateSimState(y=1)
        emit_output(s, 0, 10_000, 5_000, window_end=10**9)
        assert s.out_times == [15_000] and s.tc == 1
        s = GateSimState(y=0)
        emit_output(s, 1, 100, 5_000, window_end=10**9)
        emit_output(s, 0, 103, 5_000, window_end=10**9)
        assert s.out_times == [] and s.filtered == 1 and s.y == 0
        s = GateSimState(y=0)
        emit_output(s, 1, 90, 20, window_end=100)
        assert s.tc == 0 and s.discarded == 1 and s.y == 1
        s = GateSimState(y=0)
        emit_output(s, 1, 100, 50, window_end=10**9)
        emit_output(s, 0, 120, 0, window_end=10**9)
        assert s.out_times == [] and s.filtered == 1
        s = GateSimState(y=0, pathpulse_pct=50)
        emit_output(s, 1, 0, 1000, window_end=10**9)
        emit_output(s, 0, 600, 1000, window_end=10**9)
        assert s.out_times == [1000, 1600] and s.filtered == 0

    def test_simulate_gate_window_kats(self):
        n = api.parse_netlist(json.dumps({"name": "o", "inputs": ["p0", "p1"], "outputs": [],
                                          "gates": [{"name": "u", "cell": "AND2",
                                                     "pins": {"A": "p0", "B": "p1", "Y": "z"}}]}),
                              lib())
        cell = n.gates[0].cell
        s = simulate_gate_window(cell, [Waveform(0, [10]), Waveform(1, [])], [0, 0],
                                 api.zero_delays(n).tables[0], window_end=100)
        assert s.out_times == [10]

    def test_object_layer_matches_oracle_kernel(self, oracle_lib):
        # one gate, random waveforms: object layer == restated sim_span
        rng = np.random.default_rng(17)
        for trial in range(30):
            k = int(rng.integers(1, 5))
            pct = (100, 50, 75)[trial % 3]
            truth = "".join(map(str, rng.integers(0, 2, size=1 << k)))
            libd = api.parse_library(json.dumps({"cells": [
                {"name": "X", "inputs": [f"I{i}" for i in range(k)], "output": "Z",
                 "truth": truth}]}))
            n = api.parse_netlist(json.dumps({"name": "o", "inputs": [f"p{i}" for i in range(k)],
                                              "outputs": [], "gates": [{"name": "u", "cell": "X",
                                               "pins": {**{f"I{i}": f"p{i}" for i in range(k)},
                                                        "Z": "z"}}]}), libd)
            lv = api.levelize(n)
            d = api.zero_delays(n)
            for p in range(k):
                d.tables[0][p][:] = rng.integers(0, 800, size=d.tables[0][p].shape)
                d.interconnect[0][p] = int(rng.integers(0, 60))
            waves = [(int(rng.integers(0, 2)),
                      np.sort(rng.choice(np.arange(1, 6000), size=int(rng.integers(0, 30)),
                                         replace=False))) for _ in range(k)]
            _, _, arena, _ = oracle_lib.simulate(lv, d, waves, [0, 6100], pct=pct)
            s = simulate_gate_window(n.gates[0].cell, [Waveform(i, t) for i, t in waves],
                                     d.interconnect[0], d.tables[0], 6100, pathpulse_pct=pct)
            got = arena["buf"][arena["offsets"][0, 0]:arena["offsets"][0, 0] + arena["counts"][0, 0]]
            assert got.tolist() == s.out_times
            assert int(arena["filtered"][0, 0]) == s.filtered
            assert int(arena["ic_filtered"][0, 0]) == s.ic_filtered
            assert int(arena["discarded"][0, 0]) == s.discarded


# ---------------------------------------------------------------- event-queue simulator

def chain(n=3):
    gates, src = [], "a"
    for i in range(n):
        gates.append({"name": f"u{i}", "cell": "INV", "pins": {"A": src, "Y": f"n{i}"}})
        src = f"n{i}"
    nl = api.parse_netlist(json.dumps({"name": "c", "inputs": ["a"], "outputs": [src],
                                       "gates": gates}), lib())
    return nl, api.levelize(nl)


class TestEventSim:
    def test_chain_delays_and_time_zero(self):
        nl, lv = chain(3)
        d = api.zero_delays(nl)
        for g in range(3):
            d.tables[g][0][:] = [[1000, 1000]]
        w = api.oracle_simulate(lv, d, [Waveform(0, [0])], window_end=10_000)
        assert [w[nl.net_index[f"n{i}"]].times.tolist() for i in range(3)] == \
               [[1000], [2000], [3000]]
        nl, lv = chain(1)
        w = api.oracle_simulate(lv, api.zero_delays(nl), [Waveform(0, [0])], window_end=100)
        assert w[nl.net_index["n0"]] == Waveform(1, [0])

    def test_guard(self):
        import gen
        rng = np.random.default_rng(1)
        libd = gen.library_doc(rng, n_cells=2, max_k=2)
        doc, _ = gen.netlist_doc(rng, libd, 10_001, 4)
        nl = api.parse_netlist(json.dumps(doc), api.parse_library(json.dumps(libd)))
        lv = api.levelize(nl)
        sl = [Waveform(0, []) for _ in range(nl.num_pis)]
        with pytest.raises(SemanticError, match="refuses"):
            api.oracle_simulate(lv, api.zero_delays(nl), sl, window_end=100)

    def test_agrees_with_oracle_kernel_on_random_design(self, oracle_lib):
        import gen
        docs = gen.make_docs(2024, n_gates=200, windows=3)
        nl, lv, delays, waves, duration, b, stim = gen.load(docs, api)
        _, _, arena, _ = oracle_lib.simulate(lv, delays, gen.oracle_inputs(nl, waves), b)
        P = nl.num_pis
        for w in range(stim.num_windows):
            out = api.oracle_simulate(lv, delays, [stim.window_waveform(p, w) for p in range(P)],
                                      int(b[w + 1]))
            for g in range(nl.num_gates):
                o, c = arena["offsets"][g, w], arena["counts"][g, w]
                assert out[P + g].times.tolist() == arena["buf"][o:o + c].tolist()
