"""Native SDF reader (gs_sdf_parse, csrc/sdf_reader.h) against the Python
reader restating the reference's parse_sdf (pkg/src/glsim/sdf.py:229-503).

CPU only (host code).  Every case runs both readers on the same text and
requires identical delay tables, interconnect delays, timescale and warnings,
or the identical error (type and message).
"""

import json

import numpy as np
import pytest

import gen
import paper_2203_06117_b200 as api
from paper_2203_06117_b200 import _native, sdf
from paper_2203_06117_b200.errors import ParseError, SemanticError
from conftest import golden_names, load_golden


@pytest.fixture(scope="module", autouse=True)
def native_lib():
    try:
        _native.load()
    except RuntimeError:
        pytest.skip("libglsim_cuda.so not built")


def run_both(text, nl, corner="typ"):
    def run(f):
        try:
            return f()
        except (ParseError, SemanticError) as e:
            return (type(e).__name__, str(e))
    nat = run(lambda: _native.sdf_parse(text, nl, corner, "<sdf>"))
    py = run(lambda: sdf._parse_sdf_py(text, nl, corner, "<sdf>"))
    return nat, py


def assert_same(text, nl, corner="typ", allow_fallback=False):
    nat, py = run_both(text, nl, corner)
    if nat is None:
        assert allow_fallback, "native reader declined an ASCII document"
        return "fallback"
    if isinstance(py, tuple):
        assert nat == py
        return "error"
    arc, ic, ts, warns = nat
    assert ts == py.timescale_fs
    assert warns == py.warnings
    flat = [t for per in py.tables for t in per]
    ref_arc = np.concatenate(flat) if flat else np.zeros((0, 2), dtype=np.int64)
    assert np.array_equal(arc, ref_arc)
    ref_ic = np.concatenate(py.interconnect) if py.interconnect else np.zeros(0, np.int64)
    assert np.array_equal(ic, ref_ic)
    return "ok"


@pytest.mark.parametrize("name", golden_names())
def test_golden_documents(name):
    docs, _ = load_golden(name)
    if not docs.sdf:
        pytest.skip("zero-delay fixture")
    nl = api.parse_netlist(docs.net, api.parse_library(docs.lib))
    for corner in ("min", "typ", "max"):
        assert assert_same(docs.sdf, nl, corner) == "ok"


@pytest.mark.parametrize("seed", range(12))
def test_random_documents(seed):
    docs = gen.make_docs(800 + seed, n_gates=60 + 40 * seed, max_k=4 + seed % 3)
    nl = api.parse_netlist(docs.net, api.parse_library(docs.lib))
    assert assert_same(docs.sdf, nl) == "ok"


LIB = {"cells": [{"name": "AND2", "inputs": ["A", "B"], "output": "Y", "truth": "0001"},
                 {"name": "AO3", "inputs": ["A", "B", "C"], "output": "Z", "truth": "00010111"},
                 {"name": "INV", "inputs": ["A"], "output": "Y", "truth": "10"}]}
NET = {"name": "t", "inputs": ["a", "b", "c"], "outputs": ["y"],
       "gates": [{"name": "u1", "cell": "AND2", "pins": {"A": "a", "B": "b", "Y": "n1"}},
                 {"name": "u2", "cell": "AO3", "pins": {"A": "n1", "B": "c", "C": "a", "Z": "n2"}},
                 {"name": "u3", "cell": "INV", "pins": {"A": "n2", "Y": "y"}}]}


def nl():
    return api.parse_netlist(json.dumps(NET), api.parse_library(json.dumps(LIB)))


def doc(body, head="(TIMESCALE 1ps)"):
    return f"(DELAYFILE (SDFVERSION \"3.0\") {head}\n{body}\n)\n"


def cell(inst, entries, kind="AND2"):
    return f'(CELL (CELLTYPE "{kind}") (INSTANCE {inst}) (DELAY (ABSOLUTE {entries})))'


CASES = [
    doc(cell("u1", "(IOPATH A Y (10) (12)) (IOPATH B Y (1:2:3) (4:5:6))")),
    doc(cell("u2", "(COND B == 1 && !C (IOPATH A Z (7) (8))) (COND (C==1'b0) (IOPATH B Z (3)))"
             " (COND A==1'b1&&B (IOPATH C Z (9) (9)))", "AO3")),
    doc(cell("u2", "(COND B && !B (IOPATH A Z (7)))", "AO3")),          # contradictory
    doc(cell("u2", "(IOPATH A Z (1) (2) (3))", "AO3")),                # extra values
    doc(cell("u1", "(IOPATH (posedge A) Y (5))")),                      # edge-qualified
    doc(cell("u1", "(IOPATH A Y (:4:) (::6))") + cell("u3", "(IOPATH A Y () (2::))", "INV")),
    doc("(CELL (INSTANCE u1) (TIMINGCHECK (SETUP A B (1))) (LABEL x) (FOO) bar"
        " (DELAY (INCREMENT (IOPATH A Y (1))) (PATHPULSE A Y (1)) (ABSOLUTE"
        " (PATHPULSEPERCENT A Y (5)) (DEVICE (1)) (IOPATH A Y (1.5)))))"),
    doc("(CELL (INSTANCE u2) (DELAY (ABSOLUTE (INTERCONNECT n1 u2/A (3)) (INTERCONNECT u1/Y u2/A"
        " (4)) (INTERCONNECT c u2/B (1e3)) (INTERCONNECT a u2/C (0.0015)))))", "(TIMESCALE 10 ns)"),
    doc("(DIVIDER .)" + "(CELL (INSTANCE u3) (DELAY (ABSOLUTE (INTERCONNECT u2.Z u3.A (2)))))"),
    doc("// comment line\n" + cell("u1", "(IOPATH \"A\" Y (2.5) (3.5)) // trailing")),
    doc(cell("u1", "(IOPATH A Y (0.5) (1.5)) (IOPATH A Y (2.5) (3.5))"), "(TIMESCALE 1 ns)"),
    doc(cell("u1", "(IOPATH A Y (1))"), "(TIMESCALE 100fs) (DESIGN \"t\") (VOLTAGE 1:1:1)"),
    # errors
    doc(cell("u1", "(IOPATH A Y (1:2))")),
    doc(cell("u1", "(IOPATH A Y (x))"), ""),
    doc(cell("u9", "(IOPATH A Y (1))")),
    doc(cell("u1", "(IOPATH A Q (1))")),
    doc(cell("u1", "(IOPATH D Y (1))")),
    doc(cell("u1", "(IOPATH A Y)")),
    doc(cell("u1", "(IOPATH A (Y) (1))")),
    doc(cell("u1", "(IOPATH A Y 1)")),
    doc(cell("u2", "(COND (IOPATH A Z (1)))", "AO3")),
    doc(cell("u2", "(COND B (FOO A Z (1)))", "AO3")),
    doc(cell("u2", "(COND B && && C (IOPATH A Z (1)))", "AO3")),
    doc(cell("u2", "(COND B == 2 (IOPATH A Z (1)))", "AO3")),
    doc(cell("u2", "(COND D (IOPATH A Z (1)))", "AO3")),
    doc(cell("u2", "(COND A (IOPATH A Z (1)))", "AO3")),
    doc("(CELL (DELAY (ABSOLUTE (IOPATH A Y (1)))))"),
    doc("(CELL (INSTANCE) (DELAY (ABSOLUTE (IOPATH A Y (1)))))"),
    doc("(CELL (INSTANCE u2) (DELAY (ABSOLUTE (INTERCONNECT a u2/A (3)))))"),
    doc("(CELL (INSTANCE u2) (DELAY (ABSOLUTE (INTERCONNECT zz u2/A (3)))))"),
    doc("(CELL (INSTANCE u2) (DELAY (ABSOLUTE (INTERCONNECT u1/A u2/A (3)))))"),
    doc("(CELL (INSTANCE u2) (DELAY (ABSOLUTE (INTERCONNECT n1 u2 (3)))))"),
    doc("(CELL (INSTANCE u2) (DELAY (ABSOLUTE (INTERCONNECT n1 u2/Q (3)))))"),
    doc("(CELL (INSTANCE u2) (DELAY (ABSOLUTE (INTERCONNECT n1 u2/A))))"),
    doc("(CELL (INSTANCE u2) (DELAY (ABSOLUTE (INTERCONNECT (n1) u2/A (1)))))"),
    doc(cell("u1", "(IOPATH A Y (1))"), "(TIMESCALE 1 NS)"),
    doc(cell("u1", "(IOPATH A Y (1))"), "(TIMESCALE 2ps)"),
    doc(cell("u1", "(IOPATH A Y (1))"), "()"),
    doc(cell("u1", "(IOPATH A Y (1))"), "stray"),
    "(DELAYFILE (TIMESCALE 1ps)) (DELAYFILE)",
    "(FOO)",
    "(DELAYFILE (CELL (INSTANCE u1)",
    "(DELAYFILE (CELL (INSTANCE u1))))",
    "(DELAYFILE (CELL (INSTANCE \"u1)))",
    "",
]


@pytest.mark.parametrize("i", range(len(CASES)))
def test_edge_cases(i):
    assert assert_same(CASES[i], nl()) in ("ok", "error")


def test_warnings_and_errors_read_like_the_reference():
    nat, py = run_both(doc(cell("u9", "(IOPATH A Y (1))")), nl())
    assert nat == py == ("SemanticError", "<sdf>:2: unknown instance 'u9'")
    nat, py = run_both(doc(cell("u1", "(IOPATH A Y (1:2))")), nl())
    assert nat == py and nat[0] == "ParseError" and "bad delay value '1:2'" in nat[1]
    arc, ic, ts, warns = _native.sdf_parse(doc("(CELL (INSTANCE u1) (LABEL x))"), nl(), "typ",
                                           "<sdf>")
    assert warns == ["<sdf>:2: skipping unsupported LABEL section"]


@pytest.mark.parametrize("text", [
    doc(cell("u1", "(IOPATH A Y (-1))")),           # negative: Python float in the message
    doc(cell("u1", "(IOPATH A Y (inf))")),
    doc(cell("u1", "(IOPATH A Y (1_0))")),
    doc(cell("u1", "(IOPATH A Y ((1)))")),
    doc("(DIVIDER \"\")" + cell("u1", "(IOPATH A Y (1))")),
    doc(cell("u1", "(IOPATH A Y (1))") + "\"(\""),
    doc(cell("u1", "(IOPATH A Y (1))")) + "// café\n",
])
def test_unsupported_text_falls_back_to_python(text):
    # the native reader declines; the public entry then answers exactly as the
    # Python reader does (a result, or the same exception -- for "(inf)" the
    # reference itself stops with OverflowError)
    assert _native.sdf_parse(text, nl(), "typ", "<sdf>") is None

    def outcome(f):
        try:
            d = f()
            return [t.tolist() for per in d.tables for t in per], d.warnings
        except Exception as e:  # noqa: BLE001 -- compared, not swallowed
            return type(e).__name__, str(e)
    assert outcome(lambda: api.parse_sdf(text, nl())) == \
        outcome(lambda: sdf._parse_sdf_py(text, nl()))


def test_public_entry_matches_python_reader():
    docs, _ = load_golden("demo")
    n = api.parse_netlist(docs.net, api.parse_library(docs.lib))
    a, b = api.parse_sdf(docs.sdf, n), sdf._parse_sdf_py(docs.sdf, n)
    assert a.timescale_fs == b.timescale_fs and a.warnings == b.warnings
    for ta, tb in zip(a.tables, b.tables):
        for x, y in zip(ta, tb):
            assert np.array_equal(x, y)
    for x, y in zip(a.interconnect, b.interconnect):
        assert np.array_equal(x, y)
