"""Native VCD writer (gs_vcdw_*) against the reference's own write_vcd bytes
(tests/golden/*.npz "vcd_out", made by running the reference:
tests/golden/make_golden.py) and against the Python formatter that restates
VcdWriter (pkg/src/glsim/report.py:144-214).  CPU only (host code): the
arenas are the reference's own, rebuilt from the fixtures."""

import io
import time

import numpy as np
import pytest

import gen
import paper_2203_06117_b200 as api
from paper_2203_06117_b200 import _native, report
from conftest import golden_names, load_golden


@pytest.fixture(scope="module", autouse=True)
def native_lib():
    try:
        _native.load()
    except RuntimeError:
        pytest.skip("libglsim_cuda.so not built")


def reference_arena(docs, ref):
    nl, lv, delays, waves, duration, b, stim = gen.load(docs, api)
    W = int(ref["windows"])
    a = api.WaveformArena(ref["buf"], ref["offsets"], ref["caps"], b, (0, W), lv)
    a.counts, a.initials = ref["counts"], ref["initials"]
    a.stimuli = stim
    return nl, a, stim


def dump(arena, names, python=False, segments=None):
    out = io.StringIO()
    w = report.VcdWriter(out, arena.levelized.netlist.name, names)
    if python:
        w._vcd = None
        w.ids = {n: report._id_code(i) for i, n in enumerate(names)}
        w.last = {}
        out.seek(0)
        out.truncate()
        hdr = ["$timescale 1 fs $end", f"$scope module {arena.levelized.netlist.name} $end"]
        hdr += [f"$var wire 1 {w.ids[n]} {n} $end" for n in names]
        out.write("\n".join(hdr + ["$upscope $end", "$enddefinitions $end"]) + "\n")
    w.feed(arena)
    w.finish(int(arena.boundaries[arena.window_range[1]]))
    return out.getvalue()


@pytest.mark.parametrize("name", golden_names())
def test_reference_golden_vcd_bytes(name):
    docs, ref = load_golden(name)
    nl, arena, stim = reference_arena(docs, ref)
    want = bytes(ref["vcd_out"]).decode()
    assert report.write_vcd(arena, stimuli=stim) == want
    assert dump(arena, list(nl.net_names), python=True) == want


@pytest.mark.parametrize("name", ["demo", "rnd03", "many_windows", "busy_pct0"])
def test_subsets_duplicates_and_segments(name):
    # reordered subsets with repeated names (a name keeps its last id and one
    # shared last value), and a run fed as two window segments
    docs, ref = load_golden(name)
    nl, arena, stim = reference_arena(docs, ref)
    rng = np.random.default_rng(7)
    names = list(nl.net_names)
    pick = [names[i] for i in rng.integers(0, len(names), size=max(3, len(names) // 2))]
    assert dump(arena, pick) == dump(arena, pick, python=True)
    W = arena.window_range[1]
    if W >= 2:
        outs = []
        for py in (False, True):
            out = io.StringIO()
            w = report.VcdWriter(out, nl.name, names)
            if py:
                w._vcd = None
                w.ids = {n: report._id_code(i) for i, n in enumerate(names)}
                w.last = {}
            for lo, hi in ((0, W // 2), (W // 2, W)):
                seg = api.WaveformArena(arena.buf, arena.offsets[:, lo:hi], arena.caps[:, lo:hi],
                                        arena.boundaries, (lo, hi), arena.levelized)
                seg.counts, seg.initials = arena.counts[:, lo:hi], arena.initials[:, lo:hi]
                w.feed(seg, stim)
            w.finish(int(arena.boundaries[W]))
            outs.append(out.getvalue())
        assert outs[0].split("$enddefinitions $end\n")[1] == \
            outs[1].split("$enddefinitions $end\n")[1]
        assert outs[0].endswith(bytes(ref["vcd_out"]).decode().split("$enddefinitions $end\n")[1])


def test_unknown_net_is_rejected():
    docs, ref = load_golden("demo")
    nl, arena, stim = reference_arena(docs, ref)
    with pytest.raises(api.SemanticError, match="unknown net 'nope'"):
        report.write_vcd(arena, net_names=["nope"], stimuli=stim)


def test_large_dump_is_fast():
    # 1M nets x 4 windows through the native writer (the Python formatter
    # handles ~1e5 events/s; this is ~4e6 events)
    G, W = 1_000_000, 4
    rng = np.random.default_rng(3)
    cnt = rng.integers(0, 2, size=(G, W)).astype(np.int64)
    off = np.concatenate(([0], np.cumsum(cnt.ravel())[:-1])).reshape(G, W)
    b = np.arange(W + 1, dtype=np.int64) * 1000
    buf = (np.repeat(b[:-1][None, :], G, 0) + 500).ravel()[cnt.ravel() > 0]
    ini = rng.integers(0, 2, size=(G, W)).astype(np.uint8)
    names = [f"g{i}" for i in range(G)]
    t0 = time.perf_counter()
    v = _native.VcdText(names, "big")
    z = np.zeros((0, W), dtype=np.int64)
    v.feed(np.ones(G, np.uint8), np.arange(G), (np.zeros(0, np.int64), z, z,
                                               np.zeros((0, W), np.uint8), 0),
           (buf, off, cnt, ini, 0), b, 0, W)
    v.finish(int(b[-1]))
    text = v.take()
    dt = time.perf_counter() - t0
    assert text.count("\n") > 5 * G
    assert dt < 30, dt
