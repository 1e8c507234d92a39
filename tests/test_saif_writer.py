"""Native SAIF writer (gs_saif_format) against the Python formatter that
restates the reference's write_saif (pkg/src/glsim/report.py:94-131), and
against the reference's own golden SAIF bytes.  CPU only (host code)."""

import numpy as np
import pytest

from paper_2203_06117_b200 import _native, report
from paper_2203_06117_b200.report import ActivityStats
from conftest import golden_names, load_golden


@pytest.fixture(scope="module", autouse=True)
def native_lib():
    try:
        _native.load()
    except RuntimeError:
        pytest.skip("libglsim_cuda.so not built")


def stats(names, seed=0, duration=10**12):
    rng = np.random.default_rng(seed)
    n = len(names)
    t1 = rng.integers(0, duration, n)
    return ActivityStats(list(names), duration - t1, t1, rng.integers(0, 10**6, n),
                         rng.integers(0, 50, n), duration, 7)


@pytest.mark.parametrize("include_ig", [True, False])
def test_native_equals_python_formatter(include_ig):
    names = ["a", "u1/Z", "bus[3]", "x\\y", "", "ünïcode/[1]", "n" * 300, "tab\there", "[]/\\"]
    s = stats(names, 1)
    assert report.write_saif(s, "top", include_ig) == report._write_saif_py(s, "top", include_ig)
    big = stats([f"u{i}/q[{i % 5}]" for i in range(20000)], 2)
    assert report.write_saif(big, "chip", include_ig) == \
        report._write_saif_py(big, "chip", include_ig)


def test_empty_design():
    s = stats([], 3, duration=0)
    assert report.write_saif(s, "e") == report._write_saif_py(s, "e")


@pytest.mark.parametrize("name", golden_names())
def test_reference_golden_bytes(name):
    # the reference's own SAIF for the fixture, re-formatted from its stats
    import paper_2203_06117_b200 as api
    docs, ref = load_golden(name)
    nl = api.parse_netlist(docs.net, api.parse_library(docs.lib))
    s = ActivityStats(list(nl.net_names), ref["t0"], ref["t1"], ref["tc"], ref["ig"],
                      int(ref["report"]["duration"]), int(ref["report"]["windows"]))
    assert report.write_saif(s, nl.name) == ref["saif"]
