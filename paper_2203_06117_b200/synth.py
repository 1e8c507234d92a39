"""Array-native synthetic workloads for the benchmark configs.

Designs are built directly as :class:`~.simcore.CompiledDesign` arrays (no
per-gate Python objects, so 10M-gate netlists take seconds), stimuli directly
as CSR :class:`~.waveform.StimulusSet`.  Stimulus uses a counter-based RNG
(splitmix64 of (seed, input, window)), so any window range of any config can be
regenerated independently -- each GPU rank generates only its own shard, and
the CPU baseline regenerates exactly the windows it samples.

Configs
  C1  20-bit ripple-carry adder (text documents through the parsers), 1k windows
  C2  100k gates, 20 levels x 5,000, 2,048 inputs, 10k windows, conditional SDF
      + interconnect, pct 100                                   (bench default)
  C3  1M gates, 25 levels x 40,000, 50,000 PPIs + 1,000 PIs, 100k windows
  C4  10M gates, 40 levels x 250,000, 16,384 PPIs, 1M windows
  C5  C3 with (full|averaged SDF) x (pct 100|0)
"""

import json
from dataclasses import dataclass

import numpy as np

from .simcore import CompiledDesign

# (name, truth table string, k): the cell mix of SURVEY §8(d) C2
CELLS = [
    ("INV", "10", 1), ("BUF", "01", 1),
    ("AND2", "0001", 2), ("OR2", "0111", 2), ("NAND2", "1110", 2), ("NOR2", "1000", 2),
    ("XOR2", "0110", 2),
    # AOI21: !((A&B)|C); OAI21: !((A|B)&C); MUX2: S ? B : A  (pins A,B,S)
    ("AOI21", "".join(str(int(not ((i & 1 and i >> 1 & 1) or i >> 2 & 1))) for i in range(8)), 3),
    ("OAI21", "".join(str(int(not ((i & 1 or i >> 1 & 1) and i >> 2 & 1))) for i in range(8)), 3),
    ("MUX2", "".join(str((i >> 1 & 1) if (i >> 2 & 1) else (i & 1)) for i in range(8)), 3),
    ("AOI22", "".join(str(int(not ((i & 1 and i >> 1 & 1) or (i >> 2 & 1 and i >> 3 & 1))))
                      for i in range(16)), 4),
    ("AND4", "0" * 15 + "1", 4),
]


@dataclass
class Config:
    name: str
    gates: int
    levels: int
    ppis: int           # register outputs (pseudo-primary inputs)
    pis: int            # primary inputs
    windows: int
    period: int
    ppi_alpha: float
    ppi_lo: int
    ppi_hi: int
    pi_alpha: float
    pi_lo: int
    pi_hi: int
    seed: int
    ic_frac: float = 0.4
    ic_max: int = 2000
    dly_lo: int = 2000
    dly_hi: int = 20000
    pct: int = 100
    averaged: bool = False
    description: str = ""

    @property
    def num_inputs(self):
        return self.ppis + self.pis


CONFIGS = {
    "C2": Config("C2", 100_000, 20, 0, 2048, 10_000, 1_000_000, 0.0, 0, 1, 0.5, 1, 200_000, 2,
                 description="synthetic levelized 100k-gate netlist, 10k cycles, conditional "
                             "SDF + inertial filtering"),
    "C3": Config("C3", 1_000_000, 25, 50_000, 1_000, 100_000, 1_000_000, 0.25, 10_000, 40_000,
                 0.5, 1, 200_000, 3,
                 description="synthetic 1M-gate sequential-style netlist, 100k cycles, full SDF"),
    "C4": Config("C4", 10_000_000, 40, 16_384, 0, 1_000_000, 1_000_000, 0.1, 10_000, 40_000,
                 0.0, 1, 2, 4,
                 description="synthetic 10M-gate industrial-scale netlist, 1M cycles"),
}


def config(name, **over):
    """A named config, optionally with fields overridden (e.g. windows=1024)."""
    if name.startswith("C5"):
        # C5[-avg][-pct0]: feature ablation on the C3 netlist
        c = CONFIGS["C3"]
        over.setdefault("averaged", "avg" in name)
        over.setdefault("pct", 0 if "pct0" in name else 100)
        over.setdefault("description", "C3 feature ablation: "
                        f"{'averaged' if over['averaged'] else 'full'} SDF, pct {over['pct']}")
        return Config(**{**c.__dict__, "name": name, **over})
    c = CONFIGS[name]
    return Config(**{**c.__dict__, **over})


def _splitmix64(x):
    x = (x + np.uint64(0x9E3779B97F4A7C15)) & np.uint64(0xFFFFFFFFFFFFFFFF)
    z = x
    z = (z ^ (z >> np.uint64(30))) * np.uint64(0xBF58476D1CE4E5B9)
    z = (z ^ (z >> np.uint64(27))) * np.uint64(0x94D049BB133111EB)
    return z ^ (z >> np.uint64(31))


def design(cfg):
    """Balanced levelized netlist as a CompiledDesign.

    Level ``l`` gates take one input (random pin position) from level ``l-1``
    (the inputs for ``l = 0``) and the others uniformly from every lower net,
    so a gate's longest-path level is exactly ``l + 1``.  Delays: an
    independent U[dly_lo, dly_hi) value per (arc, condition row, edge), i.e.
    a fully conditional SDF; interconnect U[0, ic_max] on ``ic_frac`` of the
    pins.  ``averaged`` collapses each arc to its mean row (average_tables).
    """
    rng = np.random.default_rng(cfg.seed)
    P, G, L = cfg.num_inputs, cfg.gates, cfg.levels
    with np.errstate(over="ignore"):
        cell = rng.integers(0, len(CELLS), size=G)
    ks = np.array([c[2] for c in CELLS], dtype=np.int64)
    k = ks[cell]
    sizes = np.full(L, G // L, dtype=np.int64)
    sizes[-1] += G - sizes.sum()
    level_starts = np.concatenate(([0], np.cumsum(sizes))).astype(np.int64)
    pin_off = np.concatenate(([0], np.cumsum(k))).astype(np.int64)
    n_pins = int(pin_off[-1])
    gate_of_pin = np.repeat(np.arange(G, dtype=np.int64), k)
    pin_pos = np.arange(n_pins, dtype=np.int64) - pin_off[gate_of_pin]
    lvl_of_gate = np.repeat(np.arange(L, dtype=np.int64), sizes)
    lvl = lvl_of_gate[gate_of_pin]
    below = P + level_starts[lvl]                       # nets strictly below the level
    prev_lo = np.where(lvl == 0, 0, P + level_starts[np.maximum(lvl - 1, 0)])
    prev_n = np.where(lvl == 0, P, sizes[np.maximum(lvl - 1, 0)])
    anchor = (rng.random(G) * k).astype(np.int64)
    is_anchor = pin_pos == anchor[gate_of_pin]
    u = rng.random(n_pins)
    pin_net = np.where(is_anchor, prev_lo + (u * prev_n).astype(np.int64),
                       (u * below).astype(np.int64))
    pin_ic = np.where(rng.random(n_pins) < cfg.ic_frac,
                      rng.integers(0, cfg.ic_max + 1, size=n_pins), 0).astype(np.int64)
    rows = np.left_shift(1, k[gate_of_pin] - 1)
    pin_arc = (np.cumsum(rows) - rows).astype(np.int64)
    R = int(rows.sum())
    arc = rng.integers(cfg.dly_lo, cfg.dly_hi, size=(R, 2), dtype=np.int64)
    if cfg.averaged:
        # per-arc mean row, rounded half up (sdf.average_tables semantics)
        seg = np.repeat(np.arange(n_pins), rows)
        s = np.zeros((n_pins, 2), dtype=np.int64)
        np.add.at(s, seg, arc)
        mean = (s + (rows // 2)[:, None]) // rows[:, None]
        arc = mean[seg]
    lut_bits = np.concatenate([np.frombuffer(c[1].encode(), np.uint8) - 48 for c in CELLS])
    cell_off = np.concatenate(([0], np.cumsum([len(c[1]) for c in CELLS])[:-1]))
    lut_off = cell_off[cell].astype(np.int64)
    return CompiledDesign.from_arrays(P, np.arange(G, dtype=np.int64), level_starts, pin_off,
                                      pin_net, pin_ic, pin_arc, arc, lut_off,
                                      lut_bits.astype(np.uint8))


def stimulus_arrays(cfg, w_lo, w_hi):
    """Per-input CSR toggles for windows [w_lo, w_hi): (pi_off, times, init).

    Input ``p`` toggles in window ``w`` with probability alpha at offset
    U[lo, hi) -- drawn from splitmix64(seed, p, w), independent of the range.
    Initial values are drawn per input from splitmix64(seed, p).
    """
    P = cfg.num_inputs
    W = w_hi - w_lo
    p = np.arange(P, dtype=np.uint64)[:, None]
    w = np.arange(w_lo, w_hi, dtype=np.uint64)[None, :]
    key = (np.uint64(cfg.seed) << np.uint64(56)) ^ (p << np.uint64(32)) ^ w
    with np.errstate(over="ignore"):
        h1 = _splitmix64(key)
        h2 = _splitmix64(h1 ^ np.uint64(0xD1B54A32D192ED03))
    u = (h1 >> np.uint64(11)).astype(np.float64) * (1.0 / (1 << 53))
    is_ppi = (np.arange(P) < cfg.ppis)[:, None]
    alpha = np.where(is_ppi, cfg.ppi_alpha, cfg.pi_alpha)
    lo = np.where(is_ppi, cfg.ppi_lo, cfg.pi_lo).astype(np.uint64)
    span = np.where(is_ppi, cfg.ppi_hi - cfg.ppi_lo, cfg.pi_hi - cfg.pi_lo).astype(np.uint64)
    mask = u < alpha
    off = (lo + h2 % np.maximum(span, np.uint64(1))).astype(np.int64)
    times = (w.astype(np.int64) * cfg.period + off)
    counts = mask.sum(axis=1)
    pi_off = np.concatenate(([0], np.cumsum(counts))).astype(np.int64)
    sel = times[mask]  # row-major: per input, in window order
    with np.errstate(over="ignore"):
        init = (_splitmix64(np.uint64(cfg.seed) * np.uint64(1000003) + np.arange(P, dtype=np.uint64))
                & np.uint64(1)).astype(np.uint8)
    return pi_off, sel.astype(np.int64), init


def boundaries(cfg, w_lo, w_hi):
    return np.arange(w_lo, w_hi + 1, dtype=np.int64) * cfg.period


def stimulus(cfg, w_lo=0, w_hi=None, rebase=True):
    """CSR :class:`~.waveform.StimulusSet` for windows [w_lo, w_hi).

    With ``rebase`` the set's window indices start at 0 (absolute times are
    kept): a rank simulating a shard sees an ordinary stimulus.
    """
    from .waveform import StimulusSet
    w_hi = cfg.windows if w_hi is None else w_hi
    pi_off, times, init = stimulus_arrays(cfg, w_lo, w_hi)
    b = boundaries(cfg, w_lo, w_hi)
    # window-start values of the shard: toggles before w_lo flip the initial
    # value; parity of the toggle count in [0, w_lo) is derived per input
    if w_lo > 0:
        init = init ^ _parity_before(cfg, w_lo)
    return StimulusSet.from_csr(b, pi_off, times, init)


def _parity_before(cfg, w_lo, block=2048):
    """Per input, parity of its toggle count over windows [0, w_lo): only the
    toggle decision of stimulus_arrays (u < alpha, as the integer test
    h1 >> 11 < ceil(alpha * 2^53)) is evaluated."""
    P = cfg.num_inputs
    par = np.zeros(P, dtype=np.uint64)
    p = np.arange(P, dtype=np.uint64)[:, None]
    is_ppi = (np.arange(P) < cfg.ppis)[:, None]
    alpha = np.where(is_ppi, cfg.ppi_alpha, cfg.pi_alpha)
    thr = np.ceil(alpha * float(1 << 53)).astype(np.uint64)
    base = (np.uint64(cfg.seed) << np.uint64(56)) ^ (p << np.uint64(32))
    for a in range(0, w_lo, block):
        w = np.arange(a, min(w_lo, a + block), dtype=np.uint64)[None, :]
        with np.errstate(over="ignore"):
            h1 = _splitmix64(base ^ w)
        par ^= ((h1 >> np.uint64(11)) < thr).sum(axis=1, dtype=np.uint64) & np.uint64(1)
    return par.astype(np.uint8)


def work_units(cfg, windows):
    """Gate-cycle evaluations of ``windows`` windows."""
    return cfg.gates * windows


# ---------------------------------------------------------------------------
# C1: 20-bit ripple-carry adder through the text front-ends

def rca_docs(bits=20, windows=1000, period=2_000_000, seed=1, alpha=0.5, t_hi=400_000):
    """Library / netlist / SDF / VCD documents of the C1 adder."""
    rng = np.random.default_rng(seed)
    lib = {"cells": [{"name": "XOR2", "inputs": ["A", "B"], "output": "Y", "truth": "0110"},
                     {"name": "AND2", "inputs": ["A", "B"], "output": "Y", "truth": "0001"},
                     {"name": "OR2", "inputs": ["A", "B"], "output": "Y", "truth": "0111"}]}
    pis = [f"a{i}" for i in range(bits)] + [f"b{i}" for i in range(bits)] + ["cin"]
    gates, carry = [], "cin"
    for i in range(bits):
        a, b = f"a{i}", f"b{i}"
        gates += [
            {"name": f"x1_{i}", "cell": "XOR2", "pins": {"A": a, "B": b, "Y": f"p{i}"}},
            {"name": f"x2_{i}", "cell": "XOR2", "pins": {"A": f"p{i}", "B": carry, "Y": f"s{i}"}},
            {"name": f"g1_{i}", "cell": "AND2", "pins": {"A": a, "B": b, "Y": f"g{i}"}},
            {"name": f"g2_{i}", "cell": "AND2", "pins": {"A": f"p{i}", "B": carry, "Y": f"t{i}"}},
            {"name": f"o_{i}", "cell": "OR2", "pins": {"A": f"g{i}", "B": f"t{i}", "Y": f"c{i}"}},
        ]
        carry = f"c{i}"
    net = {"name": "rca", "inputs": pis, "outputs": [f"s{i}" for i in range(bits)] + [carry],
           "gates": gates}
    drv = {g["pins"]["Y"]: f"{g['name']}/Y" for g in gates}
    sdf = ["(DELAYFILE", ' (SDFVERSION "3.0")', " (DIVIDER /)", " (TIMESCALE 1fs)"]
    for g in gates:
        ent = []
        for pin, other in (("A", "B"), ("B", "A")):
            r, f = rng.integers(5_000, 20_001, size=2)
            ent.append(f"(IOPATH {pin} Y ({r}) ({f}))")
            if rng.random() < 0.6:
                for val in (0, 1):
                    r, f = rng.integers(5_000, 20_001, size=2)
                    lit = other if val else f"!{other}"
                    ent.append(f"(COND {lit} (IOPATH {pin} Y ({r}) ({f})))")
            src = g["pins"][pin]
            ent.append(f"(INTERCONNECT {drv.get(src, src)} {g['name']}/{pin} "
                       f"({int(rng.integers(0, 3_001))}))")
        sdf.append(f' (CELL (CELLTYPE "{g["cell"]}") (INSTANCE {g["name"]})'
                   f" (DELAY (ABSOLUTE {' '.join(ent)})))")
    sdf.append(")")
    ids = {n: f"i{j}" for j, n in enumerate(pis)}
    vcd = ["$timescale 1 fs $end", "$scope module tb $end"]
    vcd += [f"$var wire 1 {ids[n]} {n} $end" for n in pis]
    vcd += ["$upscope $end", "$enddefinitions $end", "#0"]
    val = {n: int(rng.integers(0, 2)) for n in pis}
    vcd += [f"{val[n]}{ids[n]}" for n in pis]
    for w in range(windows):
        ev = []
        for n in pis:
            if rng.random() < alpha:
                ev.append((w * period + int(rng.integers(1, t_hi)), n))
        for t, n in sorted(ev):
            val[n] ^= 1
            vcd += [f"#{t}", f"{val[n]}{ids[n]}"]
    vcd.append(f"#{windows * period}")
    return json.dumps(lib), json.dumps(net), "\n".join(sdf), "\n".join(vcd) + "\n", period
