"""Native VCD reader (gs_vcd_parse, csrc/vcd_reader.h) against the Python
reader restating the reference's parse_vcd (pkg/src/glsim/waveform.py:101-198).

CPU only: the reader is host code in libglsim_cuda.so and needs no device.
Every case runs both readers on the same text and requires identical
waveforms, duration, or the identical error (type, message, line).
"""

import json

import numpy as np
import pytest

import gen
import paper_2203_06117_b200 as api
from paper_2203_06117_b200 import _native, waveform
from paper_2203_06117_b200.errors import ParseError, SemanticError
from conftest import golden_names, load_golden

LIB = api.parse_library('{"cells":[{"name":"BUF","inputs":["A"],"output":"Y","truth":"01"}]}')


def nets(names):
    return api.parse_netlist(json.dumps({"name": "t", "inputs": list(names), "outputs": [],
                                         "gates": []}), LIB)


def both(text, nl):
    """(native result or exception, python result or exception)"""
    def run(f):
        try:
            return f()
        except (ParseError, SemanticError) as e:
            return (type(e).__name__, str(e))
    nat = run(lambda: _native.vcd_parse(text, nl.pi_names, "<vcd>"))
    py = run(lambda: waveform._parse_vcd_py(text, nl, "<vcd>"))
    return nat, py


def assert_same(text, nl):
    nat, py = both(text, nl)
    assert nat is not None, "native reader declined an ASCII document"
    if isinstance(py, tuple) and isinstance(py[0], str):
        assert nat == py
        return
    waves, dur = py
    pi_off, pi_times, pi_init, ndur = nat
    assert ndur == dur
    for i, name in enumerate(nl.pi_names):
        w = waves[name]
        assert int(pi_init[i]) == w.initial, name
        assert np.array_equal(pi_times[pi_off[i]:pi_off[i + 1]], w.times), name


@pytest.fixture(scope="module", autouse=True)
def native_lib():
    try:
        _native.load()
    except RuntimeError:
        pytest.skip("libglsim_cuda.so not built")


@pytest.mark.parametrize("name", golden_names())
def test_golden_documents(name):
    docs, _ = load_golden(name)
    nl = api.parse_netlist(docs.net, api.parse_library(docs.lib))
    assert_same(docs.vcd, nl)


@pytest.mark.parametrize("seed", range(20))
def test_random_documents(seed):
    docs = gen.make_docs(700 + seed, max_toggles=30 + 40 * seed)
    nl = api.parse_netlist(docs.net, api.parse_library(docs.lib))
    assert_same(docs.vcd, nl)


HEAD = "$timescale 1 ps $end\n$scope module tb $end\n$var wire 1 ! a $end\n$var wire 1 \" b $end\n" \
       "$upscope $end\n$enddefinitions $end\n"

CASES = [
    HEAD + "#0\n0!\n1\"\n#10\n1!\n#25\n0!\n0\"\n",                 # basics
    HEAD + "#0\nx!\nz\"\n#5\n1!\nX!\n#6\nZ\"\n",                    # x/z read as 0
    HEAD + "#5\n1!\n0!\n1!\n#7\n1!\n#9\n0!\n1!\n",                   # same-mark changes
    HEAD + "0!\n1\"\n#3\n1!\n",                                      # before any time mark
    HEAD + "#-4\n1!\n#-4\n#0\n0!\n#2\n1!\n",                         # negative marks
    HEAD + "#+5\n1!\n#1_000\n0!\n#0010_0\n",                         # Python int() forms
    HEAD + "#3\nb101 !\n1!\nr1.5 \"\n1\"\nb1\n!\n#4\n0!\n",           # vector / real skips
    HEAD.replace("\n", "\r\n") + "#2\r\n1!\r\n#4\r\n0!\r\n",        # CRLF
    HEAD.replace("\n", "\r") + "#2\r1!\r#4\r0!\r",                  # lone CR
    "$timescale\n 10\n ns\n $end $var wire 1 ! a $end $var reg 1 \" b $end\n#1 1! 1\" #2 0!\n",
    "$timescale 100fs $end\n$var wire 1 ! a $end\n$var wire 1 # a $end\n$var wire 1 \" b $end\n"
    "#1\n1#\n1!\n#2\n0\"\n",                                         # alias of a bound input
    "$timescale 1us $end\n$var wire 1 ! b $end\n$var wire 1 ! a $end\n$var wire 1 ? b $end\n"
    "#1\n1!\n1?\n",                                                  # identifier rebound
    "$comment $end $date x $end\n$timescale 1 s $end\n$var wire 1 ! a $end\n"
    "$var wire 1 \" b $end $dumpvars 0! 1\" $end\n#1\n1!\n",
    "$end\n$timescale 1ps\n$end $var wire 1 ! a $end $var wire 1 \" b $end\n#1\n",  # stray $end
    "",                                                              # missing inputs
    HEAD + "#1\n1!\n",                                               # no trailing mark
    # errors
    HEAD + "#abc\n",
    HEAD + "#1__0\n",
    HEAD + "#10_\n",
    HEAD + "#5\n#4\n",
    "$var wire 1 ! a $end\n#1\n",
    "$timescale 1 NS $end\n",
    "$timescale 2 ns $end\n",
    "$timescale $end\n",
    "$timescale 1 ns $end\n$var wire 1 ! $end\n",
    "$timescale 1 ns $end\n$var wire 4 ! a $end\n",
    "$timescale 1 ns $end\n$var wire 1 ! a $end\n",
    HEAD + "$dumpvars\n1!\n#3\n",
    "$timescale 1 ns $end\n$var wire 1 'q a $end\n$var wire 1 \" b $end\n#1\n1'q\n",
]


@pytest.mark.parametrize("i", range(len(CASES)))
def test_edge_cases(i):
    assert_same(CASES[i], nets(["a", "b"]))


def test_errors_carry_reference_messages():
    nat, py = both(HEAD + "#5\n#4\n", nets(["a", "b"]))
    assert nat == py == ("ParseError", "<vcd>:8: non-monotonic time mark #4")
    nat, py = both("$timescale 1 ns $end\n$var wire 1 ! a $end\n", nets(["a", "b"]))
    assert nat == py == ("SemanticError", "VCD declares no scalar variable for input net 'b'")


def test_unsupported_text_falls_back_to_python():
    text = HEAD + "#1\n1!\n$comment café $end\n#2\n0!\n"
    assert _native.vcd_parse(text, ["a", "b"]) is None
    w, dur = api.parse_vcd(text, nets(["a", "b"]))
    assert w["a"] == api.Waveform(0, [1000, 2000]) and dur == 2000


def test_csr_feeds_the_stimulus_set():
    docs, _ = load_golden("many_windows")
    nl = api.parse_netlist(docs.net, api.parse_library(docs.lib))
    pi_off, pi_times, pi_init, dur = waveform.parse_vcd_csr(docs.vcd, nl)
    waves, dur2 = api.parse_vcd(docs.vcd, nl)
    b = api.window_boundaries(dur, period=docs.period)
    a = api.StimulusSet.from_csr(b, pi_off, pi_times, pi_init)
    c = api.StimulusSet.build(waves, nl, b)
    for f in ("buf", "offsets", "counts", "initials"):
        assert np.array_equal(getattr(a, f), getattr(c, f)), f
