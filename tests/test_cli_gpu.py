"""``glsim`` command line end to end on the GPU: golden SAIF bytes, exit codes,
environment fallbacks, oracle cross-check and fault injection (the behaviours
reference ``pkg/tests/test_cli.py`` pins)."""

import json

import pytest

from conftest import load_golden
from paper_2203_06117_b200 import cli

pytestmark = pytest.mark.gpu


@pytest.fixture()
def demo(tmp_path):
    docs, ref = load_golden("demo")
    paths = {}
    for key, text in (("lib", docs.lib), ("netlist", docs.net), ("sdf", docs.sdf),
                      ("vcd", docs.vcd)):
        p = tmp_path / f"demo.{key}"
        p.write_text(text)
        paths[key] = str(p)
    paths["golden"] = ref["saif"]
    return paths


def args(d, tmp_path, *extra):
    return ["--netlist", d["netlist"], "--lib", d["lib"], "--sdf", d["sdf"], "--vcd", d["vcd"],
            "--window-period", "20000", "--saif", str(tmp_path / "out.saif"), *extra]


def test_golden_saif(demo, tmp_path):
    assert cli.main(args(demo, tmp_path)) == 0
    assert (tmp_path / "out.saif").read_text() == demo["golden"]


def test_usage_and_parse_errors(demo, tmp_path, capsys):
    assert cli.main(["--lib", demo["lib"], "--vcd", demo["vcd"]]) == 1
    assert "--netlist" in capsys.readouterr().err
    bad = tmp_path / "bad.json"
    bad.write_text("{nope")
    a = args(demo, tmp_path)
    a[a.index("--netlist") + 1] = str(bad)
    assert cli.main(a) == 2
    a = args(demo, tmp_path)
    a[a.index("--vcd") + 1] = str(tmp_path / "missing.vcd")
    assert cli.main(a) == 2


def test_semantic_and_capacity_errors(demo, tmp_path):
    bad = tmp_path / "undriven.json"
    bad.write_text(json.dumps({"name": "u", "inputs": ["a"], "outputs": [],
                               "gates": [{"name": "g", "cell": "INV",
                                          "pins": {"A": "ghost", "Y": "y"}}]}))
    a = args(demo, tmp_path)
    a[a.index("--netlist") + 1] = str(bad)
    assert cli.main(a) == 3
    a = args(demo, tmp_path, "--mem-cap", "8")
    a.remove("--window-period")
    a.remove("20000")
    assert cli.main(a) == 4


def test_segmented_fallback_same_bytes(demo, tmp_path):
    assert cli.main(args(demo, tmp_path, "--mem-cap", "100")) == 0
    assert (tmp_path / "out.saif").read_text() == demo["golden"]


def test_oracle_and_fault_injection(demo, tmp_path, monkeypatch):
    assert cli.main(args(demo, tmp_path, "--oracle")) == 0
    assert cli.main(args(demo, tmp_path, "--pathpulse-pct", "50", "--oracle")) == 0
    assert cli.main(args(demo, tmp_path, "--delay-mode", "avg", "--oracle")) == 0
    from paper_2203_06117_b200 import scheduler, simcore
    original = scheduler.simcore.two_pass_simulate

    def corrupted(*a, **k):
        arena = original(*a, **k)
        if arena.buf.size:
            arena.buf[0] += 1
        return arena

    monkeypatch.setattr(scheduler.simcore, "two_pass_simulate", corrupted)
    assert cli.main(args(demo, tmp_path, "--oracle")) == 5
    monkeypatch.undo()

    def broken(model, arena):
        from paper_2203_06117_b200.errors import ConsistencyError
        raise ConsistencyError("two-pass mismatch (injected)")

    monkeypatch.setattr(simcore, "verify_two_pass", broken)
    assert cli.main(args(demo, tmp_path)) == 5


def test_env_report_dump_and_flags(demo, tmp_path, monkeypatch):
    for k, v in (("NETLIST", demo["netlist"]), ("LIB", demo["lib"]), ("SDF", demo["sdf"]),
                 ("VCD", demo["vcd"]), ("WINDOW_PERIOD", "20000"),
                 ("SAIF", str(tmp_path / "env.saif"))):
        monkeypatch.setenv("GLSIM_" + k, v)
    assert cli.main([]) == 0
    assert (tmp_path / "env.saif").read_text() == demo["golden"]
    a = args(demo, tmp_path, "--report", str(tmp_path / "r.json"), "--dump-vcd",
             str(tmp_path / "d.vcd"), "--dump-nets", "y,n1")
    assert cli.main(a) == 0
    rep = json.loads((tmp_path / "r.json").read_text())
    assert rep["nets"] == 7 and rep["windows"] == 2
    assert rep["total_tc"] == 21 and rep["total_filtered"] == 1
    assert " y $end" in (tmp_path / "d.vcd").read_text()
    assert cli.main(args(demo, tmp_path, "--no-ig")) == 0
    assert "(IG" not in (tmp_path / "out.saif").read_text()


def test_zero_delay_windows_file_and_bad_values(demo, tmp_path):
    a = args(demo, tmp_path)
    i = a.index("--sdf")
    del a[i:i + 2]
    assert cli.main(a) == 0
    assert "(DURATION 40000)" in (tmp_path / "out.saif").read_text()
    wf = tmp_path / "w.txt"
    wf.write_text("0\n20000\n40000\n")
    a = args(demo, tmp_path)
    i = a.index("--window-period")
    del a[i:i + 2]
    assert cli.main(a + ["--windows-file", str(wf)]) == 0
    assert (tmp_path / "out.saif").read_text() == demo["golden"]
    assert cli.main(args(demo, tmp_path, "--windows-file", str(wf))) == 1
    for bad in (("--mem-cap", "lots"), ("--pathpulse-pct", "150"), ("--cycle-parallelism", "0")):
        assert cli.main(args(demo, tmp_path, *bad)) == 1
