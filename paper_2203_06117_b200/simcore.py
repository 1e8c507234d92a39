"""Per-(gate, window) simulation: the readable object layer and the GPU engine.

Two forms of one semantics, as in reference ``simcore.py`` (``SC:1-463``):

* the object layer (:class:`PinCursor`, :func:`next_event_time`,
  :func:`resolve_msi`, :class:`GateSimState`, :func:`emit_output`,
  :func:`simulate_gate_window`) -- plain Python for one gate and one window,
  the executable statement of Algo. 1 that unit tests poke at;
* the array engine (:func:`compile_design`, :func:`count_pass`,
  :func:`store_pass`, :func:`two_pass_simulate`, :func:`simulate_stats`) --
  flat arrays handed to ``libglsim_cuda.so``.  Every simulation here runs on
  the GPU (kernels K1/K4 of ``csrc/kernels.cuh``); nothing falls back to the
  CPU.

Two-pass contract (``SC:11-16``): the counting pass yields exact per-(gate,
window) counts and the high-water ``peak`` that sizes the arena regions; the
store pass re-simulates into the arena; :func:`verify_two_pass` checks they
agree.  On the GPU each pass is one chunked sweep over all logic levels.
"""

import time
from dataclasses import dataclass, field

import numpy as np

from . import _native
from .errors import ConsistencyError
from .netlist import eval_lut
from .sdf import condition_row
from .waveform import allocate_arena

EXHAUSTED = None


# ---------------------------------------------------------------------------
# object layer (reference SC:32-197): the names, fields and results of the
# reference's per-gate Python model, organised around a waveform view that
# drops narrow pairs and an output edge log

@dataclass
class PinCursor:
    """One input pin's view of its driver's window waveform: every toggle
    arrives ``ic_delay`` later, and a toggle pair closer together than
    ``ic_delay`` never arrives (``filtered`` counts such pairs)."""

    times: np.ndarray
    ic_delay: int
    value: int
    pos: int = 0
    filtered: int = 0

    @classmethod
    def from_waveform(cls, w, ic_delay=0):
        return cls(w.times, int(ic_delay), int(w.initial))

    def _drop_narrow_pairs(self):
        t, d, i = self.times, self.ic_delay, self.pos
        while i + 1 < len(t) and t[i + 1] - t[i] < d:
            i += 2
        self.filtered += (i - self.pos) // 2
        self.pos = i

    def peek(self):
        """Arrival time of the pin's next surviving toggle, or
        :data:`EXHAUSTED`."""
        self._drop_narrow_pairs()
        if self.pos < len(self.times):
            return int(self.times[self.pos]) + self.ic_delay
        return EXHAUSTED

    def consume(self):
        self.pos += 1
        self.value ^= 1


def next_event_time(cursors):
    """Earliest pending arrival over all pins (the time only)."""
    arrivals = [t for t in map(PinCursor.peek, cursors) if t is not EXHAUSTED]
    return min(arrivals, default=EXHAUSTED)


def resolve_msi(cursors, t):
    """Apply every arrival at exactly ``t`` (multiple simultaneous inputs);
    returns the input vector after them and the switching pin indices."""
    switching = [p for p, c in enumerate(cursors) if c.peek() == t]
    for p in switching:
        cursors[p].consume()
    return tuple(c.value for c in cursors), switching


@dataclass
class GateSimState:
    """Output side of one (gate, window) simulation."""

    y: int
    mode: str = "store"
    pathpulse_pct: int = 100
    tc: int = 0
    filtered: int = 0
    ic_filtered: int = 0
    discarded: int = 0
    t_last: object = None
    d_last: int = 0
    last_stored: bool = False
    out_times: list = field(default_factory=list)

    def previous_edge(self):
        """The edge a new one is compared with: the newest edge (stored or
        discarded), else the newest stored edge left after withdrawals."""
        if self.t_last is not None:
            return self.t_last
        return self.out_times[-1] if self.out_times else None

    def withdraw_previous(self):
        """The new edge cancels the previous one: both vanish."""
        if self.t_last is not None and not self.last_stored:
            self.discarded -= 1          # it had been discarded, nothing stored
        else:
            self.out_times.pop()
            self.tc -= 1
        self.filtered += 1
        self.t_last = None

    def record(self, t_out, delay, window_end):
        self.last_stored = t_out < window_end
        if self.last_stored:
            self.out_times.append(t_out)
            self.tc += 1
        else:
            self.discarded += 1
        self.t_last, self.d_last = t_out, delay


def emit_output(state, new_y, t_event, delay, window_end):
    """Schedule an output edge through the inertial filter (``SC:117-160``).

    The edge lands at ``t_event + delay``.  At or before the previous edge, or
    closer to it than ``delay * pct // 100``, it withdraws that edge and is
    not emitted (the output returns to its pre-pulse value); the newest
    remaining stored edge is then the next comparison target.  Edges at or
    past ``window_end`` are discarded but still set the logical value.
    """
    if new_y == state.y:
        return state
    t_out = t_event + delay
    prev = state.previous_edge()
    if prev is not None and (t_out <= prev or t_out - prev < delay * state.pathpulse_pct // 100):
        state.withdraw_previous()
    else:
        state.record(t_out, delay, window_end)
    state.y = new_y
    return state


def _event_delay(arc_tables, k, switching, values, col):
    """Delay of an output edge: the largest conditioned arc delay over the
    switching pins (``SC:139-151``)."""
    return max((int(arc_tables[p][condition_row(k, p, values), col]) for p in switching),
               default=0)


def simulate_gate_window(cell, pin_waveforms, ic_delays, arc_tables, window_end,
                         mode="store", pathpulse_pct=100):
    """One gate over one window from explicit fanin waveforms (``SC:163-197``)."""
    pins = [PinCursor.from_waveform(w, d) for w, d in zip(pin_waveforms, ic_delays)]
    state = GateSimState(y=eval_lut(cell, [c.value for c in pins]), mode=mode,
                         pathpulse_pct=pathpulse_pct)
    t = next_event_time(pins)
    while t is not EXHAUSTED:
        values, switching = resolve_msi(pins, t)
        y = eval_lut(cell, values)
        if y != state.y:
            emit_output(state, y, t, _event_delay(arc_tables, len(pins), switching, values,
                                                  0 if y else 1), window_end)
        t = next_event_time(pins)
    state.ic_filtered = sum(c.filtered for c in pins)
    return state


# ---------------------------------------------------------------------------
# array engine

class CompiledDesign:
    """Flat (SoA) design: the arrays of reference ``SC:203-272``.

    ``pin_off [G+1]``, ``pin_net``/``pin_ic``/``pin_arc [sum k]``,
    ``arc_rows [R, 2]``, ``lut_off [G]`` into ``lut_bits`` (one truth table
    per distinct cell), ``out_net [G]``, ``net_kind``/``net_slot [N]``,
    ``order``/``level_starts``.  The device copy is created on first use.
    """

    def __init__(self, levelized, delays):
        nl = levelized.netlist
        if delays.netlist is not nl:
            raise ValueError("delay annotation was built for a different netlist")
        self.levelized = levelized
        self.netlist = nl
        # array-native: the netlist's pin and cell arrays and the delays'
        # flat tables (no per-gate Python objects on this path)
        pin_off, pin_net = nl.pin_arrays()
        cells, gate_cell = nl.cell_arrays()
        # one truth table per distinct (name, truth) cell, in order of first use
        first_use = np.full(len(cells), -1, dtype=np.int64)
        if gate_cell.size:
            u, at = np.unique(gate_cell, return_index=True)
            first_use[u] = at
        keys, lut_parts, cell_lut, top = {}, [], np.zeros(len(cells), dtype=np.int64), 0
        for c in sorted(range(len(cells)), key=lambda c: (first_use[c] < 0, first_use[c])):
            cell = cells[c]
            truth = np.asarray(cell.truth, dtype=np.uint8)
            key = (cell.name, truth.tobytes())
            if key not in keys:
                keys[key] = top
                lut_parts.append(truth)
                top += truth.size
            cell_lut[c] = keys[key]
        lut_off = cell_lut[gate_cell] if gate_cell.size else np.zeros(0, dtype=np.int64)
        arc_rows, pin_ic = delays.arrays()
        k = np.diff(pin_off)
        rows = np.repeat(np.left_shift(np.int64(1), k - 1), k) if k.size else np.zeros(0, np.int64)
        pin_arc = np.cumsum(rows) - rows
        self._set(levelized.order, levelized.level_starts, nl.num_pis, pin_off.copy(),
                  pin_net.copy(), pin_ic.copy(), pin_arc, arc_rows.copy(),
                  lut_off, np.concatenate(lut_parts) if lut_parts else np.zeros(0, np.uint8))

    def _set(self, order, level_starts, num_pis, pin_off, pin_net, pin_ic, pin_arc, arc_rows,
             lut_off, lut_bits):
        G = pin_off.size - 1
        self.order = np.asarray(order, dtype=np.int64)
        self.level_starts = np.asarray(level_starts, dtype=np.int64)
        self.num_pis = int(num_pis)
        self.pin_off, self.pin_net, self.pin_ic = pin_off, pin_net, pin_ic
        self.pin_arc, self.arc_rows = pin_arc, arc_rows.reshape(-1, 2)
        self.lut_off, self.lut_bits = lut_off, lut_bits
        self.out_net = np.arange(self.num_pis, self.num_pis + G, dtype=np.int64)
        N = self.num_pis + G
        self.net_kind = np.zeros(N, dtype=np.uint8)
        self.net_kind[self.num_pis:] = 1
        self.net_slot = np.concatenate([np.arange(self.num_pis), np.arange(G)]).astype(np.int64)
        self._device = None

    @classmethod
    def from_arrays(cls, num_pis, order, level_starts, pin_off, pin_net, pin_ic, pin_arc,
                    arc_rows, lut_off, lut_bits, levelized=None):
        """Array-native construction (no per-gate Python objects)."""
        self = cls.__new__(cls)
        self.levelized = levelized
        self.netlist = levelized.netlist if levelized is not None else None
        self._set(order, level_starts, num_pis, np.asarray(pin_off, np.int64),
                  np.asarray(pin_net, np.int64), np.asarray(pin_ic, np.int64),
                  np.asarray(pin_arc, np.int64), np.asarray(arc_rows, np.int64),
                  np.asarray(lut_off, np.int64), np.asarray(lut_bits, np.uint8))
        return self

    @property
    def num_gates(self):
        return self.pin_off.size - 1

    @property
    def num_nets(self):
        return self.num_pis + self.num_gates

    @property
    def num_levels(self):
        return self.level_starts.size - 1

    def device(self):
        """The ``gs_design`` device copy (uploaded once)."""
        if self._device is None:
            self._device = _native.Design(self)
        return self._device


def compile_design(levelized, delays):
    return CompiledDesign(levelized, delays)


def initial_values(model, stimuli):
    """Zero-delay window-start value of every net, ``uint8 [N, W]`` (GPU K2)."""
    return _native.init_values(model, stimuli.initials)


@dataclass
class PassResult:
    tc: np.ndarray
    peak: np.ndarray
    filtered: np.ndarray
    ic_filtered: np.ndarray
    discarded: np.ndarray
    initials: np.ndarray = None
    stats: tuple = None


ENGINE_MEM_BUDGET = 0  # device bytes per engine for window-chunk workspace; 0 = 75% of free
# K4 work-item sizing of new engines (workers, tail_div, tail_frac); None =
# the engine's defaults.  Tests force the coarse-item and tail paths with it.
ENGINE_ITEMS = None


class _Session:
    """Device design + stimulus + engine for one (model, stimuli) pair."""

    _cache = {}

    def __init__(self, model, stimuli):
        self.design = model.device()
        self.stim = _native.Stimulus(self.design, stimuli)
        self.engine = _native.Engine(self.design, ENGINE_MEM_BUDGET)
        if ENGINE_ITEMS is not None:
            self.engine.set_items(*ENGINE_ITEMS)

    @classmethod
    def get(cls, model, stimuli):
        key = (id(model), id(stimuli), ENGINE_MEM_BUDGET, ENGINE_ITEMS)
        s = cls._cache.get(key)
        if s is None or s.model_ref is not model or s.stim_ref is not stimuli:
            cls._cache.clear()  # one live session: device memory is released promptly
            s = cls(model, stimuli)
            s.model_ref, s.stim_ref = model, stimuli
            cls._cache[key] = s
        return s


def compare_on_device(model, stimuli, reference, window_range=None, pathpulse_pct=100):
    """Simulate ``window_range`` on the GPU and check every gate waveform
    against ``reference`` -- an arena in the reference layout (``buf``,
    ``offsets``, ``counts``, ``initials`` as attributes or keys, [G, Ws],
    absolute times; e.g. the oracle's) -- on the device (``gs_run_compare``,
    SURVEY §8(f) item 4), without copying the engine's waveforms back.
    Returns ``(mismatching (gate, window) pairs, first (gate, window) or None)``.
    """
    def get(k):
        return reference[k] if isinstance(reference, dict) else getattr(reference, k)
    w_lo, w_hi = window_range if window_range is not None else (0, stimuli.num_windows)
    s = _Session.get(model, stimuli)
    return s.engine.run_compare(s.stim, w_lo, w_hi, pathpulse_pct, get("buf"), get("offsets"),
                                get("counts"), get("initials"))


def _trace(model, task_trace, task_counts, w_lo):
    # one entry per level launch, in level order: the level barrier is the
    # kernel boundary (what the reference's task_trace ramps assert)
    for li in range(model.num_levels):
        lo = int(model.level_starts[li])
        if task_trace is not None:
            task_trace.append((li + 1, lo, int(w_lo)))
        if task_counts is not None:
            task_counts.append(1)


def count_pass(model, stimuli, init_vals=None, *, window_range=None, cycle_parallelism=32,
               pathpulse_pct=100, executor=None, workers=1, task_trace=None,
               task_counts=None):
    """Pass 1 on the GPU: exact per-(gate, window) counts, ``peak``, filter
    counters and window-start values (``SC:328-379``).  ``init_vals`` is
    accepted for signature compatibility; the kernel derives them itself."""
    w_lo, w_hi = window_range if window_range is not None else (0, stimuli.num_windows)
    s = _Session.get(model, stimuli)
    r = s.engine.run_arena(s.stim, w_lo, w_hi, int(pathpulse_pct), want_stats=True)
    s.last_count = (w_lo, w_hi, int(pathpulse_pct), r)
    _trace(model, task_trace, task_counts, w_lo)
    return PassResult(r["counts"], r["peak"], r["filtered"], r["ic_filtered"], r["discarded"],
                      r["initials"], r["stats"])


def store_pass(model, stimuli, init_vals, arena, *, cycle_parallelism=32, pathpulse_pct=100,
               executor=None, workers=1, task_trace=None, task_counts=None):
    """Pass 2 (``SC:382-410``): every region of the arena.

    When the engine's last count pass was this run (same stimulus, window
    range, pct, and the arena sized by its ``peak``), that single simulation
    already holds every region's contents -- K5 packed them per window chunk
    -- and they are scattered into ``arena.buf`` without simulating again.
    Otherwise (e.g. capacities from elsewhere) the identical simulation runs
    again, writing the regions on the GPU, and a region overflowing its
    capacity raises :class:`ConsistencyError`."""
    w_lo, w_hi = arena.window_range
    s = _Session.get(model, stimuli)
    last = getattr(s, "last_count", None)
    if (last is not None and last[:3] == (w_lo, w_hi, int(pathpulse_pct))
            and np.array_equal(arena.caps, last[3]["peak"])):
        # the count pass of this very run kept its waveforms (K5): the arena
        # is filled without simulating again -- same contents, same counters
        r = last[3]
        if s.engine.arena_fill(s.stim, w_lo, w_hi, int(pathpulse_pct), arena.buf,
                               arena.offsets):
            for f in ("counts", "filtered", "ic_filtered", "discarded", "initials"):
                getattr(arena, f)[:] = r[f]
            _trace(model, task_trace, task_counts, w_lo)
            return
    r = s.engine.run_arena(s.stim, w_lo, w_hi, int(pathpulse_pct), offsets=arena.offsets,
                           n_buf=arena.buf.size, caps=arena.caps)
    arena.buf[:] = r["buf"]
    arena.counts[:] = r["counts"]
    arena.filtered[:] = r["filtered"]
    arena.ic_filtered[:] = r["ic_filtered"]
    arena.discarded[:] = r["discarded"]
    arena.initials[:] = r["initials"]
    _trace(model, task_trace, task_counts, w_lo)


def verify_two_pass(model, arena):
    """Defining postcondition: stored counts equal pass-1 counts (``SC:413-421``)."""
    expect = arena.pass1_counts if arena.pass1_counts is not None else arena.caps
    if not np.array_equal(arena.counts, expect):
        g, j = np.argwhere(arena.counts != expect)[0]
        w = arena.window_range[0] + int(j)
        name = model.netlist.gates[int(g)].name if model.netlist is not None else int(g)
        raise ConsistencyError(
            f"two-pass mismatch at gate {name!r}, window {w}: "
            f"counted {int(expect[g, j])}, stored {int(arena.counts[g, j])}")


def two_pass_simulate(levelized, stimuli, delays, *, cycle_parallelism=32, pathpulse_pct=100,
                      mem_cap=None, workers=1, executor=None, task_trace=None, timings=None,
                      task_counts=None):
    """Count, allocate, store, verify (``SC:424-463``); returns the arena.

    :class:`~.errors.CapacityError` when the arena exceeds ``mem_cap``;
    :class:`~.errors.ConsistencyError` on any pass disagreement.
    """
    t0 = time.perf_counter()
    model = compile_design(levelized, delays)
    t1 = time.perf_counter()
    counted = count_pass(model, stimuli, None, pathpulse_pct=pathpulse_pct,
                         task_trace=task_trace, task_counts=task_counts)
    t2 = time.perf_counter()
    arena = allocate_arena(counted.peak, model.order, stimuli.boundaries,
                           (0, stimuli.num_windows), levelized, mem_cap=mem_cap)
    arena.pass1_counts = counted.tc
    arena.initials[:] = counted.initials
    arena.stimuli = stimuli
    t3 = time.perf_counter()
    store_pass(model, stimuli, None, arena, pathpulse_pct=pathpulse_pct,
               task_trace=task_trace, task_counts=task_counts)
    verify_two_pass(model, arena)
    t4 = time.perf_counter()
    if timings is not None:
        for key, dt in (("compile", t1 - t0), ("pass1", t2 - t1), ("alloc", t3 - t2),
                        ("pass2", t4 - t3)):
            timings[key] = timings.get(key, 0.0) + dt
    return arena


def simulate_stats(model, stimuli, *, window_range=None, pathpulse_pct=100, timings=None):
    """Streaming GPU run: per-net statistics without materializing an arena.

    One sweep of K1 + per-level K4 with the dwell/toggle reduction fused in,
    over window chunks sized to device memory.  Returns ``(t1, tc, ig, totals)``
    as int64 arrays over all nets plus ``(filtered, ic_filtered, discarded)``.
    """
    w_lo, w_hi = window_range if window_range is not None else (0, stimuli.num_windows)
    t0 = time.perf_counter()
    s = _Session.get(model, stimuli)
    out = s.engine.run_stats(s.stim, w_lo, w_hi, int(pathpulse_pct))
    if timings is not None:
        timings["kernel"] = timings.get("kernel", 0.0) + time.perf_counter() - t0
        timings["device"] = s.engine.timing()
    return out
