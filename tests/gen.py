"""Random design/stimulus instances for the parity tests.

Instances are emitted as *documents* (library JSON, netlist JSON, SDF text,
VCD text) so that every consumer -- the GPU engine under test, the CPU oracle
and, in ``golden/make_golden.py``, the reference package itself -- starts from
the same bytes and runs its own parsers.

Shapes follow the reference test generator's spirit (``pkg/tests/gen.py``):
random truth tables with up to ``max_k`` inputs, a levelized DAG where every
gate anchors one input on the previous level, SDF with COND rows and
INTERCONNECT entries, VCD stimulus with random toggles.  The RNG streams are
this file's own.
"""

import json
from dataclasses import dataclass

import numpy as np

PS = 1000  # documents use 1 ps time units


def library_doc(rng, n_cells=8, max_k=4, min_k=1):
    cells = []
    for i in range(n_cells):
        k = int(rng.integers(min_k, max_k + 1))
        bits = rng.integers(0, 2, size=1 << k)
        cells.append({"name": f"X{i}_{k}", "inputs": [f"A{j}" for j in range(k)],
                      "output": "Z", "truth": "".join(map(str, bits.tolist()))})
    return {"cells": cells}


def netlist_doc(rng, lib, n_gates, n_pis, max_levels=8, name="rnd"):
    pis = [f"in{i}" for i in range(n_pis)]
    by_level = {0: list(pis)}
    gates, driver = [], {}
    top = 0
    for j in range(n_gates):
        lvl = int(rng.integers(1, min(max_levels, top + 1) + 1))
        cell = lib["cells"][int(rng.integers(len(lib["cells"])))]
        k = len(cell["inputs"])
        pool = [n for lv in range(lvl) for n in by_level.get(lv, [])]
        anchor = int(rng.integers(k))
        pins = {}
        for p, pin in enumerate(cell["inputs"]):
            src = by_level[lvl - 1] if p == anchor else pool
            pins[pin] = src[int(rng.integers(len(src)))]
        out = f"w{j}"
        pins[cell["output"]] = out
        gates.append({"name": f"u{j}", "cell": cell["name"], "pins": pins})
        by_level.setdefault(lvl, []).append(out)
        driver[out] = f"u{j}/Z"
        top = max(top, lvl)
    outs = [g["pins"]["Z"] for g in gates]
    pos = sorted(rng.choice(outs, size=min(len(outs), max(1, n_gates // 8)), replace=False)
                 .tolist()) if outs else []
    return {"name": name, "inputs": pis, "outputs": pos, "gates": gates}, driver


def _ps(fs):
    return f"{fs / PS:.3f}"


def sdf_text(rng, net, lib, driver, max_delay=10_000, p_cond=0.6, p_ic=0.4):
    cells = {c["name"]: c for c in lib["cells"]}
    out = ["(DELAYFILE", ' (SDFVERSION "3.0")', " (DIVIDER /)", " (TIMESCALE 1ps)"]
    for g in net["gates"]:
        cell = cells[g["cell"]]
        ent = []
        for pin in cell["inputs"]:
            r, f = (int(x) for x in rng.integers(0, max_delay + 1, size=2))
            ent.append(f"(IOPATH {pin} Z ({_ps(r)}::) ({_ps(f)}::))")
            side = [q for q in cell["inputs"] if q != pin]
            if side and rng.random() < p_cond:
                for _ in range(int(rng.integers(1, 3))):
                    lits = rng.choice(side, size=int(rng.integers(1, len(side) + 1)),
                                      replace=False)
                    expr = " && ".join(q if rng.random() < 0.5 else f"!{q}" for q in lits)
                    r, f = (int(x) for x in rng.integers(0, max_delay + 1, size=2))
                    ent.append(f"(COND {expr} (IOPATH {pin} Z ({_ps(r)}::) ({_ps(f)}::)))")
            if rng.random() < p_ic:
                src = g["pins"][pin]
                d = int(rng.integers(0, max_delay // 4 + 1))
                ent.append(f"(INTERCONNECT {driver.get(src, src)} {g['name']}/{pin} "
                           f"({_ps(d)}::))")
        out.append(f' (CELL (CELLTYPE "{cell["name"]}") (INSTANCE {g["name"]})'
                   f" (DELAY (ABSOLUTE {' '.join(ent)})))")
    out.append(")")
    return "\n".join(out)


def vcd_text(rng, pis, duration_ps, max_toggles=64):
    ids = {n: f"v{i}" for i, n in enumerate(pis)}
    events = {}
    lines = ["$timescale 1 ps $end", "$scope module tb $end"]
    lines += [f"$var wire 1 {ids[n]} {n} $end" for n in pis]
    lines += ["$upscope $end", "$enddefinitions $end", "#0"]
    for n in pis:
        v = int(rng.integers(2))
        lines.append(f"{v}{ids[n]}")
        cnt = int(rng.integers(0, max_toggles + 1))
        if cnt and duration_ps > 1:
            for t in np.unique(rng.integers(1, duration_ps, size=cnt)).tolist():
                v ^= 1
                events.setdefault(t, []).append(f"{v}{ids[n]}")
    for t in sorted(events):
        lines.append(f"#{t}")
        lines += events[t]
    lines.append(f"#{duration_ps}")
    return "\n".join(lines) + "\n"


@dataclass
class Docs:
    """One instance as documents plus its window period (None = one window)."""

    lib: str
    net: str
    sdf: str
    vcd: str
    period: object
    pct: int = 100
    avg: bool = False


def make_docs(seed, n_gates=None, n_pis=None, windows=None, with_sdf=True, max_levels=8,
              max_toggles=64, max_delay=10_000, max_k=4, duration_ps=None, pct=100, avg=False):
    rng = np.random.default_rng(seed)
    n_gates = int(rng.integers(10, 400)) if n_gates is None else n_gates
    n_pis = int(rng.integers(2, 12)) if n_pis is None else n_pis
    windows = int(rng.integers(1, 9)) if windows is None else windows
    duration_ps = int(rng.integers(200, 2000)) if duration_ps is None else duration_ps
    lib = library_doc(rng, max_k=max_k)
    net, driver = netlist_doc(rng, lib, n_gates, n_pis, max_levels)
    sdf = sdf_text(rng, net, lib, driver, max_delay) if with_sdf else None
    vcd = vcd_text(rng, net["inputs"], duration_ps, max_toggles)
    period = (duration_ps * PS) // windows if windows > 1 else None
    return Docs(json.dumps(lib), json.dumps(net), sdf, vcd, period, pct, avg)


def load(docs, api):
    """Parse ``docs`` with a glsim-compatible ``api`` module ->
    (netlist, levelized, delays, waves, duration, boundaries, stimuli)."""
    lib = api.parse_library(docs.lib)
    nl = api.parse_netlist(docs.net, lib)
    lv = api.levelize(nl)
    delays = api.parse_sdf(docs.sdf, nl) if docs.sdf else api.zero_delays(nl)
    if docs.avg:
        delays = api.average_tables(delays)
    waves, duration = api.parse_vcd(docs.vcd, nl)
    b = api.window_boundaries(duration, period=docs.period)
    stim = api.StimulusSet.build(waves, nl, b)
    return nl, lv, delays, waves, duration, b, stim


def oracle_inputs(nl, waves):
    """Per-input (initial, times) list in input order, for ``oracle.port``."""
    return [(waves[n].initial, np.asarray(waves[n].times, dtype=np.int64)) for n in nl.pi_names]
