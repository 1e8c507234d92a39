"""CPU oracle for the CUDA engine: the reference algorithm, restated.

TEST INFRASTRUCTURE ONLY -- the parity checker of ``tests/`` and the CPU
baseline of ``bench.py``.  The product package never imports this module.

The orchestration below follows reference ``simcore.py`` / ``waveform.py`` /
``report.py`` step by step (file:line on each function); the inner loops are
the C restatements in ``glsim_oracle.c`` (built to ``oracle/liboracle.so`` by
``oracle/Makefile`` or ``__graft_entry__.build()``).  Inputs are plain
arrays, so the oracle shares no code with the engine under test.

Pinning: ``tests/test_oracle_pinning.py`` checks this port against golden
vectors produced by running the reference itself (numba, in the build
container) -- ``tests/golden/make_golden.py`` -- and against the reference
test-suite's known-answer values (demo SAIF bytes, report totals, KATs).
"""

import ctypes as C
import os
import subprocess

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
LIB = os.path.join(HERE, "liboracle.so")

_i64p = C.POINTER(C.c_int64)
_u8p = C.POINTER(C.c_uint8)
_lib = None


def build(force=False):
    """Compile ``liboracle.so`` with gcc (OpenMP)."""
    src = os.path.join(HERE, "glsim_oracle.c")
    if force or not os.path.exists(LIB) or os.path.getmtime(LIB) < os.path.getmtime(src):
        subprocess.check_call(["gcc", "-O2", "-fopenmp", "-shared", "-fPIC", "-o", LIB, src])
    return LIB


def _load():
    global _lib
    if _lib is None:
        if not os.path.exists(LIB):
            build()
        _lib = C.CDLL(LIB)
        _lib.or_max_threads.restype = C.c_int
    return _lib


def _p64(a):
    assert a.dtype == np.int64 and a.flags.c_contiguous
    return a.ctypes.data_as(_i64p)


def _p8(a):
    assert a.dtype == np.uint8 and a.flags.c_contiguous
    return a.ctypes.data_as(_u8p)


def max_threads():
    return int(_load().or_max_threads())


class Design:
    """Flat design arrays, restating ``CompiledDesign`` (``simcore.py:203-272``):
    one truth table per gate concatenated in gate order, one condition table
    per pin concatenated in pin order."""

    def __init__(self, levelized, delays):
        nl = levelized.netlist
        G, P = len(nl.gates), len(nl.pi_names)
        self.num_pis, self.num_gates, self.num_nets = P, G, len(nl.net_names)
        self.order = np.asarray(levelized.order, dtype=np.int64)
        self.level_starts = np.asarray(levelized.level_starts, dtype=np.int64)
        pin_off = [0]
        lut_off, luts, out_net = [], [], []
        pin_net, pin_ic, pin_arc, arcs = [], [], [], []
        top_lut = top_arc = 0
        for gi, g in enumerate(nl.gates):
            k = len(g.pin_nets)
            pin_off.append(pin_off[-1] + k)
            lut_off.append(top_lut)
            luts.append(np.asarray(g.cell.truth, dtype=np.uint8))
            top_lut += 1 << k
            out_net.append(g.out_net)
            for p, n in enumerate(g.pin_nets):
                pin_net.append(n)
                pin_ic.append(int(delays.interconnect[gi][p]))
                pin_arc.append(top_arc)
                rows = np.asarray(delays.tables[gi][p], dtype=np.int64)
                arcs.append(rows)
                top_arc += rows.shape[0]
        self.pin_off = np.array(pin_off, dtype=np.int64)
        self.lut_off = np.array(lut_off, dtype=np.int64)
        self.lut_bits = np.concatenate(luts) if luts else np.zeros(0, np.uint8)
        self.out_net = np.array(out_net, dtype=np.int64)
        self.pin_net = np.array(pin_net, dtype=np.int64)
        self.pin_ic = np.array(pin_ic, dtype=np.int64)
        self.pin_arc = np.array(pin_arc, dtype=np.int64)
        self.arc_rows = np.ascontiguousarray(np.vstack(arcs) if arcs else
                                             np.zeros((0, 2), np.int64), dtype=np.int64)
        self.net_kind = np.zeros(self.num_nets, dtype=np.uint8)
        self.net_slot = np.zeros(self.num_nets, dtype=np.int64)
        for n in range(self.num_nets):
            if n < P:
                self.net_slot[n] = n
            else:
                self.net_kind[n] = 1
                self.net_slot[n] = n - P

    @classmethod
    def from_arrays(cls, num_pis, order, level_starts, pin_off, pin_net, pin_ic, pin_arc,
                    arc_rows, lut_off, lut_bits):
        """Flat arrays given directly (array-native synthetic designs); gate g
        drives net num_pis + g."""
        self = cls.__new__(cls)
        c64 = lambda a: np.ascontiguousarray(a, dtype=np.int64)  # noqa: E731
        self.num_pis = int(num_pis)
        self.num_gates = len(pin_off) - 1
        self.num_nets = self.num_pis + self.num_gates
        self.order, self.level_starts = c64(order), c64(level_starts)
        self.pin_off, self.pin_net, self.pin_ic = c64(pin_off), c64(pin_net), c64(pin_ic)
        self.pin_arc, self.arc_rows = c64(pin_arc), c64(arc_rows).reshape(-1, 2)
        self.lut_off = c64(lut_off)
        self.lut_bits = np.ascontiguousarray(lut_bits, dtype=np.uint8)
        self.out_net = np.arange(self.num_pis, self.num_nets, dtype=np.int64)
        self.net_kind = np.zeros(self.num_nets, dtype=np.uint8)
        self.net_kind[self.num_pis:] = 1
        self.net_slot = np.concatenate([np.arange(self.num_pis),
                                        np.arange(self.num_gates)]).astype(np.int64)
        return self

    @property
    def num_levels(self):
        return self.level_starts.size - 1


class Stimulus:
    """Windowed stimulus arrays (``StimulusSet``, ``waveform.py:227-274``),
    built from per-input waveforms exactly as ``StimulusSet.build``
    (``waveform.py:243-265``: searchsorted cuts, slices in window order)."""

    def __init__(self, waves, boundaries):
        """``waves``: list of (initial, int64 times) per input, in input order."""
        b = np.asarray(boundaries, dtype=np.int64)
        P, W = len(waves), b.size - 1
        self.boundaries = b
        self.offsets = np.zeros((P, W), dtype=np.int64)
        self.counts = np.zeros((P, W), dtype=np.int64)
        self.initials = np.zeros((P, W), dtype=np.uint8)
        chunks, top = [], 0
        for p, (init, times) in enumerate(waves):
            times = np.asarray(times, dtype=np.int64)
            cuts = np.searchsorted(times, b, side="left")
            for j in range(W):
                self.offsets[p, j] = top
                self.counts[p, j] = cuts[j + 1] - cuts[j]
                self.initials[p, j] = int(init) ^ (int(cuts[j]) & 1)
                chunks.append(times[cuts[j]:cuts[j + 1]])
                top += cuts[j + 1] - cuts[j]
        self.buf = np.concatenate(chunks).astype(np.int64) if chunks else np.zeros(0, np.int64)

    @classmethod
    def from_csr(cls, pi_off, pi_times, pi_init, boundaries):
        waves = [(int(pi_init[p]), pi_times[pi_off[p]:pi_off[p + 1]])
                 for p in range(len(pi_off) - 1)]
        return cls(waves, boundaries)

    @classmethod
    def from_csr_fast(cls, pi_off, pi_times, pi_init, boundaries):
        """The same arrays as :meth:`from_csr`, with the per-window loop of
        each input done by numpy (one searchsorted per input) -- for parity
        tests on large window ranges; the CPU baseline times :meth:`from_csr`,
        the reference's own loop."""
        self = cls.__new__(cls)
        b = np.asarray(boundaries, dtype=np.int64)
        P, W = len(pi_off) - 1, b.size - 1
        self.boundaries = b
        self.offsets = np.zeros((P, W), dtype=np.int64)
        self.counts = np.zeros((P, W), dtype=np.int64)
        self.initials = np.zeros((P, W), dtype=np.uint8)
        parts, top = [], 0
        for p in range(P):
            times = np.asarray(pi_times[pi_off[p]:pi_off[p + 1]], dtype=np.int64)
            cuts = np.searchsorted(times, b, side="left")
            self.offsets[p] = top + cuts[:-1] - cuts[0]
            self.counts[p] = np.diff(cuts)
            self.initials[p] = (int(pi_init[p]) ^ (cuts[:-1] & 1)).astype(np.uint8)
            parts.append(times[cuts[0]:cuts[-1]])
            top += int(cuts[-1] - cuts[0])
        self.buf = np.concatenate(parts).astype(np.int64) if parts else np.zeros(0, np.int64)
        return self

    @property
    def num_windows(self):
        return self.boundaries.size - 1


def init_values(d, stim):
    """``init_values`` (``_kernels.py:213-231``, caller ``simcore.py:279-283``)."""
    W = stim.num_windows
    vals = np.zeros((d.num_nets, W), dtype=np.uint8)
    vals[:d.num_pis] = stim.initials
    _load().or_init_values(C.c_int64(d.num_gates), _p64(d.order), _p64(d.pin_off),
                           _p64(d.pin_net), _p64(d.lut_off), _p8(d.lut_bits), _p64(d.out_net),
                           _p8(vals), C.c_int64(W))
    return vals


def _sim_level(d, stim, vals, gbuf, g_off, g_cap, g_cnt, filt, icf, disc, err, peak,
               lo, hi, w_lo, w_hi, pct, threads, cycle_parallelism):
    # one level of _run_level (simcore.py:295-325); the join is the barrier
    _load().or_sim_span_mt(
        C.c_int(threads), C.c_int64(cycle_parallelism), C.c_int64(lo), C.c_int64(hi),
        C.c_int64(w_lo), C.c_int64(w_hi), C.c_int64(w_lo), _p64(d.order), _p64(d.pin_off),
        _p64(d.pin_net), _p64(d.pin_ic), _p64(d.pin_arc), _p64(d.arc_rows), _p64(d.lut_off),
        _p8(d.lut_bits), _p64(d.out_net), _p8(d.net_kind), _p64(d.net_slot), _p64(stim.buf),
        _p64(stim.offsets), _p64(stim.counts), C.c_int64(stim.num_windows), _p8(vals),
        C.c_int64(stim.num_windows), _p64(stim.boundaries), _p64(gbuf), _p64(g_off),
        _p64(g_cap), _p64(g_cnt), C.c_int64(w_hi - w_lo), _p64(filt), _p64(icf), _p64(disc),
        _p64(err), _p64(peak), C.c_int64(pct))


def count_pass(d, stim, vals, window_range=None, pct=100, threads=1, cycle_parallelism=32):
    """Pass 1 (``simcore.py:328-379``): exact counts via ub-sized scratch."""
    w_lo, w_hi = window_range if window_range is not None else (0, stim.num_windows)
    Ws, G = w_hi - w_lo, d.num_gates
    z = lambda: np.zeros((G, Ws), dtype=np.int64)  # noqa: E731
    g_off, g_cap, g_cnt, filt, icf, disc, err, peak = (z() for _ in range(8))
    gbuf = np.empty(4096, dtype=np.int64)
    top = 0
    for li in range(d.num_levels):
        lo, hi = int(d.level_starts[li]), int(d.level_starts[li + 1])
        ub = np.empty((hi - lo, Ws), dtype=np.int64)
        _load().or_level_ub(_p64(d.order), C.c_int64(lo), C.c_int64(hi), _p64(d.pin_off),
                            _p64(d.pin_net), _p8(d.net_kind), _p64(d.net_slot),
                            _p64(stim.counts), C.c_int64(stim.num_windows), _p64(g_cnt),
                            C.c_int64(Ws), C.c_int64(w_lo), C.c_int64(w_hi), C.c_int64(w_lo),
                            _p64(ub))
        need = int(ub.sum())
        if top + need > gbuf.size:  # simcore.py:362-365
            grown = np.empty(max(gbuf.size * 2, top + need), dtype=np.int64)
            grown[:top] = gbuf[:top]
            gbuf = grown
        flat = np.concatenate(([0], np.cumsum(ub.ravel())[:-1])) + top
        sel = d.order[lo:hi]
        g_off[sel] = flat.reshape(hi - lo, Ws)
        g_cap[sel] = ub
        top += need
        _sim_level(d, stim, vals, gbuf, g_off, g_cap, g_cnt, filt, icf, disc, err, peak,
                   lo, hi, w_lo, w_hi, pct, threads, cycle_parallelism)
        if err[sel].any():
            raise AssertionError("oracle: counting pass overran its output bound")
    return {"tc": g_cnt, "peak": peak, "filtered": filt, "ic_filtered": icf, "discarded": disc}


def arena_offsets(caps, order):
    """``allocate_arena`` offsets (``waveform.py:340-344``)."""
    offsets = np.zeros_like(caps)
    if caps.size:
        ordered = caps[order]
        flat = np.concatenate(([0], np.cumsum(ordered.ravel())[:-1]))
        offsets[order] = flat.reshape(ordered.shape)
    return offsets


def store_pass(d, stim, vals, caps, window_range=None, pct=100, threads=1,
               cycle_parallelism=32):
    """Pass 2 (``simcore.py:382-410``) into the packed arena."""
    w_lo, w_hi = window_range if window_range is not None else (0, stim.num_windows)
    Ws, G = w_hi - w_lo, d.num_gates
    caps = np.ascontiguousarray(caps, dtype=np.int64)
    offsets = arena_offsets(caps, d.order)
    buf = np.zeros(int(caps.sum()), dtype=np.int64)
    z = lambda: np.zeros((G, Ws), dtype=np.int64)  # noqa: E731
    counts, filt, icf, disc, err, peak = (z() for _ in range(6))
    for li in range(d.num_levels):
        lo, hi = int(d.level_starts[li]), int(d.level_starts[li + 1])
        _sim_level(d, stim, vals, buf, offsets, caps, counts, filt, icf, disc, err, peak,
                   lo, hi, w_lo, w_hi, pct, threads, cycle_parallelism)
        if err[d.order[lo:hi]].any():
            raise AssertionError("oracle: store pass overran the counting pass")
    return {"buf": buf, "offsets": offsets, "caps": caps, "counts": counts, "filtered": filt,
            "ic_filtered": icf, "discarded": disc}


def two_pass_simulate(d, stim, pct=100, window_range=None, threads=1):
    """``two_pass_simulate`` (``simcore.py:424-463``) -> arena dict.  Asserts
    the two-pass postcondition (``simcore.py:413-421``)."""
    w_lo, w_hi = window_range if window_range is not None else (0, stim.num_windows)
    vals = init_values(d, stim)
    c = count_pass(d, stim, vals, (w_lo, w_hi), pct, threads)
    a = store_pass(d, stim, vals, c["peak"], (w_lo, w_hi), pct, threads)
    assert np.array_equal(a["counts"], c["tc"]), "oracle: two-pass mismatch"
    a["pass1_counts"] = c["tc"]
    a["initials"] = np.ascontiguousarray(vals[d.num_pis:, w_lo:w_hi])
    a["window_range"] = (w_lo, w_hi)
    return a


def compute_stats(d, stim, arena, threads=1):
    """``compute_stats`` (``report.py:57-91``) -> dict t0, t1, tc, ig, duration."""
    w_lo, w_hi = arena["window_range"]
    N = d.num_nets
    t0, t1, tc = (np.zeros(N, dtype=np.int64) for _ in range(3))
    _load().or_dwell_sweep(C.c_int64(N), _p8(d.net_kind), _p64(d.net_slot), _p64(stim.buf),
                           _p64(stim.offsets), _p64(stim.counts), _p8(stim.initials),
                           C.c_int64(stim.num_windows), _p64(arena["buf"]),
                           _p64(arena["offsets"]), _p64(arena["counts"]),
                           _p8(arena["initials"]), C.c_int64(w_hi - w_lo),
                           _p64(stim.boundaries), C.c_int64(w_lo), C.c_int64(w_hi),
                           C.c_int64(w_lo), _p64(t0), _p64(t1), _p64(tc), C.c_int(threads))
    ig = np.zeros(N, dtype=np.int64)
    if d.num_gates:
        ig[d.num_pis:] = arena["filtered"].sum(axis=1)
    duration = int(stim.boundaries[w_hi] - stim.boundaries[w_lo])
    return {"t0": t0, "t1": t1, "tc": tc, "ig": ig, "duration": duration,
            "windows": w_hi - w_lo}


def escape(name):
    """SAIF name escaping (``report.py:94-100``)."""
    return "".join("\\" + c if c in "[]/\\" else c for c in name)


def saif_text(stats, net_names, design_name, include_ig=True):
    """SAIF bytes (``report.py:103-131``)."""
    lines = ["(SAIFILE", '  (SAIFVERSION "2.0")', '  (DIRECTION "backward")',
             f'  (DESIGN "{design_name}")', "  (TIMESCALE 1 fs)",
             f"  (DURATION {stats['duration']})", f"  (INSTANCE {design_name}", "    (NET"]
    for i, name in enumerate(net_names):
        lines.append(f"      ({escape(name)}")
        lines.append(f"        (T0 {int(stats['t0'][i])}) (T1 {int(stats['t1'][i])}) (TX 0)")
        if include_ig:
            lines.append(f"        (TC {int(stats['tc'][i])}) (IG {int(stats['ig'][i])})")
        else:
            lines.append(f"        (TC {int(stats['tc'][i])})")
        lines.append("      )")
    lines += ["    )", "  )", ")"]
    return "\n".join(lines) + "\n"


def simulate(levelized, delays, waves, boundaries, pct=100, threads=1):
    """End to end: (design, stimulus, arena, stats)."""
    d = Design(levelized, delays)
    stim = Stimulus(waves, boundaries)
    arena = two_pass_simulate(d, stim, pct=pct, threads=threads)
    return d, stim, arena, compute_stats(d, stim, arena, threads)
