"""Native netlist JSON reader (gs_netlist_parse, csrc/netlist_reader.h)
against the Python reader that restates the reference's parse_netlist
(pkg/src/glsim/netlist.py:190-275), and the whole array-native front end
(netlist + SDF readers, levelize, compile_design, StimulusSet.build) against
the reference's own flattened arrays stored in the golden fixtures (made by
running the reference: tests/golden/make_golden.py).  CPU only (host code)."""

import json

import numpy as np
import pytest

import gen
import paper_2203_06117_b200 as api
from paper_2203_06117_b200 import _native, netlist
from paper_2203_06117_b200.errors import ParseError, SemanticError
from conftest import golden_names, load_golden


@pytest.fixture(scope="module", autouse=True)
def native_lib():
    try:
        _native.load()
    except RuntimeError:
        pytest.skip("libglsim_cuda.so not built")


def same_netlist(a, b):
    assert a.name == b.name
    assert a.pi_names == b.pi_names and a.po_names == b.po_names
    assert a.net_names == b.net_names
    assert a.net_index == b.net_index and a.gate_index == b.gate_index
    assert len(a.gates) == len(b.gates)
    for x, y in zip(a.gates, b.gates):
        assert (x.name, x.cell.name, x.pin_nets, x.out_net) == \
            (y.name, y.cell.name, y.pin_nets, y.out_net)


@pytest.mark.parametrize("name", golden_names())
def test_golden_documents(name):
    docs, _ = load_golden(name)
    lib = api.parse_library(docs.lib)
    nat = api.parse_netlist(docs.net, lib)
    assert nat._gates is None, "golden netlist fell back to the Python reader"
    same_netlist(nat, netlist._parse_netlist_py(docs.net, lib))


@pytest.mark.parametrize("name", golden_names())
def test_front_end_arrays_equal_the_references(name):
    # the reference's own CompiledDesign arrays (order, level starts, pins,
    # interconnect delays, condition rows) from our readers + compile_design,
    # and the windowed stimulus arrays of its StimulusSet.build
    docs, ref = load_golden(name)
    nl, lv, delays, waves, duration, b, stim = gen.load(docs, api)
    m = api.compile_design(lv, delays)
    for f in ("order", "level_starts", "pin_off", "pin_net", "pin_ic", "pin_arc"):
        assert np.array_equal(getattr(m, f), ref[f]), f
    assert np.array_equal(m.arc_rows.reshape(-1, 2), ref["arc_rows"].reshape(-1, 2))
    for f, g in (("buf", "stim_buf"), ("offsets", "stim_offsets"), ("counts", "stim_counts"),
                 ("initials", "stim_initials")):
        assert np.array_equal(getattr(stim, f), ref[g]), f


@pytest.mark.parametrize("seed", range(10))
def test_random_documents(seed):
    docs = gen.make_docs(500 + seed, n_gates=50 + 60 * seed, max_k=3 + seed % 4)
    lib = api.parse_library(docs.lib)
    nat = api.parse_netlist(docs.net, lib)
    assert nat._gates is None
    same_netlist(nat, netlist._parse_netlist_py(docs.net, lib))


LIB = {"cells": [{"name": "AND2", "inputs": ["A", "B"], "output": "Y", "truth": "0001"},
                 {"name": "INV", "inputs": ["A"], "output": "Y", "truth": "10"}]}


def doc(gates, inputs=("a", "b"), outputs=("y",), **extra):
    return json.dumps({"name": "t", "inputs": list(inputs), "outputs": list(outputs),
                       "gates": gates, **extra})


G_OK = [{"name": "u1", "cell": "AND2", "pins": {"A": "a", "B": "n", "Y": "y"}},
        {"name": "u2", "cell": "INV", "pins": {"A": "b", "Y": "n"}}]
E_ACUTE = "é"
SMILE = "\U0001F600"

EDGE = [
    doc(G_OK),                                                   # forward reference
    doc(G_OK, extra_key={"x": [1, 2.5e3, None, True, False, "s"]}),
    doc([]), doc([], inputs=()), '{"name": "t"}',
    '{"name": "t", "inputs": ["a"], "name": "u", "gates": [], "outputs": []}',  # last key wins
    '{"name":"t","inputs":["a","b"],"outputs":["y"],"gates":[{"name":"u1","cell":"AND2",'
    '"pins":{"A":"a","B":"b","Y":"q","Y":"y"}}]}',                # repeated pin key
    doc([{"name": "g\\u00e9", "cell": "INV", "pins": {"A": "a", "Y": "y"}}]),
    doc([{"name": "x" + E_ACUTE + SMILE, "cell": "INV", "pins": {"A": E_ACUTE, "Y": "y"}}],
        inputs=(E_ACUTE,)),
    json.dumps({"name": "t", "inputs": [SMILE], "outputs": [], "gates": []}, ensure_ascii=False),
    '  \n{"name":"t","inputs":[],"outputs":[],"gates":[]}\n  ',
    '{"name":"t","gates":[],"z":NaN,"w":-Infinity}',
    # everything below is rejected by the reference: the Python reader raises
    doc(G_OK, outputs=("zz",)),                                   # undriven output
    doc([{"name": "u", "cell": "INV", "pins": {"A": "zz", "Y": "y"}}]),  # undriven input
    doc([{"name": "u", "cell": "INV", "pins": {"A": "a", "Y": "a"}}]),   # two drivers
    doc([{"name": "u", "cell": "INV", "pins": {"A": "a", "Y": "y"}}] * 2),  # duplicate gate
    doc([{"name": "u", "cell": "NOPE", "pins": {"A": "a", "Y": "y"}}]),
    doc([{"name": "u", "cell": "INV", "pins": {"A": "a", "B": "b", "Y": "y"}}]),
    doc([{"name": "u", "cell": "INV", "pins": {"Y": "y"}}]),
    doc([{"name": "u", "cell": "INV", "pins": {"A": 3, "Y": "y"}}]),
    doc([{"name": "", "cell": "INV", "pins": {"A": "a", "Y": "y"}}]),
    doc([["u"]]), '{"name": ""}', '[]', '{"name": "t", "inputs": [1]}',
    '{"name": "t",}', '{"name": "t"', '{"name": "t\\x"}', '{"name": "t", "inputs": "a"}',
    '{"name": 5}', '{"name": "t", "gates": [1,]}', '{"name": "t"} x',
]


@pytest.mark.parametrize("i", range(len(EDGE)))
def test_edge_documents(i):
    lib = api.parse_library(json.dumps(LIB))
    text = EDGE[i]

    def run(f):
        try:
            return f()
        except (ParseError, SemanticError) as e:
            return (type(e).__name__, str(e))
    got = run(lambda: api.parse_netlist(text, lib))
    want = run(lambda: netlist._parse_netlist_py(text, lib))
    if isinstance(want, tuple):
        assert got == want
    else:
        same_netlist(got, want)


def test_large_netlist_reads_fast():
    # 1M gates of random 1-2 input cells: native read + levelize in seconds
    import time
    rng = np.random.default_rng(0)
    G, P = 1_000_000, 1000
    gates = []
    for i in range(G):
        a = f"n{int(rng.integers(0, P + i))}" if i else "n0"
        if i % 2:
            gates.append({"name": f"u{i}", "cell": "INV", "pins": {"A": a, "Y": f"n{P + i}"}})
        else:
            b = f"n{int(rng.integers(0, P + i))}" if i else "n1"
            gates.append({"name": f"u{i}", "cell": "AND2",
                          "pins": {"A": a, "B": b, "Y": f"n{P + i}"}})
    text = json.dumps({"name": "big", "inputs": [f"n{i}" for i in range(P)], "outputs": [],
                       "gates": gates})
    lib = api.parse_library(json.dumps(LIB))
    t0 = time.perf_counter()
    nl = api.parse_netlist(text, lib)
    lv = api.levelize(nl)
    dt = time.perf_counter() - t0
    assert nl.num_gates == G and nl._gates is None
    assert lv.order.size == G
    assert dt < 30, dt
