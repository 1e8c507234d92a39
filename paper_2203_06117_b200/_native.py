"""ctypes binding of ``libglsim_cuda.so`` (C ABI in ``include/glsim_cuda.h``).

This is the only door to the GPU.  There is no CPU fallback: if the library is
missing or no CUDA device is visible, every entry point raises.  Status codes
map onto the package's error types (``GS_ERR_CAPACITY`` -> ``CapacityError``,
``GS_ERR_CONSISTENCY`` -> ``ConsistencyError``).
"""

import ctypes as C
import os
import weakref

import numpy as np

from .errors import CapacityError, ConsistencyError

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_NAME = "libglsim_cuda.so"
LIB_PATH = os.path.join(_HERE, os.environ.get("GLSIM_LIB", LIB_NAME))

(GS_OK, GS_ERR_ARG, GS_ERR_CUDA, GS_ERR_NODEVICE, GS_ERR_CAPACITY, GS_ERR_CONSISTENCY,
 GS_ERR_PARSE, GS_ERR_SEMANTIC, GS_ERR_UNSUPPORTED) = range(9)

_i64p = C.POINTER(C.c_int64)
_u8p = C.POINTER(C.c_uint8)


class DesignDesc(C.Structure):
    _fields_ = [("num_pis", C.c_int64), ("num_gates", C.c_int64), ("num_levels", C.c_int64),
                ("order", _i64p), ("level_starts", _i64p), ("pin_off", _i64p),
                ("pin_net", _i64p), ("pin_ic", _i64p), ("pin_arc", _i64p),
                ("arc_rows", _i64p), ("num_arc_rows", C.c_int64),
                ("lut_off", _i64p), ("lut_bits", _u8p), ("num_lut_bits", C.c_int64)]


class StimDesc(C.Structure):
    _fields_ = [("num_pis", C.c_int64), ("num_windows", C.c_int64), ("boundaries", _i64p),
                ("pi_off", _i64p), ("pi_times", _i64p), ("pi_init", _u8p),
                ("buf", _i64p), ("n_buf", C.c_int64), ("offsets", _i64p),
                ("counts", _i64p), ("initials", _u8p)]


class SynthDesc(C.Structure):
    _fields_ = [("num_pis", C.c_int64), ("num_ppis", C.c_int64), ("seed", C.c_uint64),
                ("period", C.c_int64), ("ppi_thr", C.c_uint64), ("pi_thr", C.c_uint64),
                ("ppi_lo", C.c_int64), ("ppi_span", C.c_int64), ("pi_lo", C.c_int64),
                ("pi_span", C.c_int64), ("w_lo", C.c_int64), ("w_hi", C.c_int64)]


class StatsOut(C.Structure):
    _fields_ = [("t1", _i64p), ("tc", _i64p), ("ig", _i64p), ("totals", C.c_int64 * 3)]


class ArenaOut(C.Structure):
    _fields_ = [("counts", _i64p), ("peak", _i64p), ("filtered", _i64p),
                ("ic_filtered", _i64p), ("discarded", _i64p), ("initials", _u8p),
                ("offsets", _i64p), ("buf", _i64p), ("n_buf", C.c_int64), ("caps", _i64p)]


class SdfDesign(C.Structure):
    _fields_ = [("num_gates", C.c_int64), ("num_nets", C.c_int64), ("num_cells", C.c_int64),
                ("gate_names", C.c_char_p), ("gate_name_off", _i64p),
                ("net_names", C.c_char_p), ("net_name_off", _i64p),
                ("pin_names", C.c_char_p), ("pin_name_off", _i64p),
                ("cell_pin_first", _i64p),
                ("cell_outputs", C.c_char_p), ("cell_output_off", _i64p),
                ("gate_cell", _i64p), ("pin_off", _i64p), ("pin_net", _i64p),
                ("out_net", _i64p)]


class WaveSrc(C.Structure):
    _fields_ = [("buf", _i64p), ("n_buf", C.c_int64), ("offsets", _i64p), ("counts", _i64p),
                ("initials", _u8p), ("cols", C.c_int64), ("col0", C.c_int64)]


class ArenaRef(C.Structure):
    _fields_ = [("buf", _i64p), ("n_buf", C.c_int64), ("offsets", _i64p), ("counts", _i64p),
                ("initials", _u8p), ("cols", C.c_int64)]


class Timing(C.Structure):
    _fields_ = [("ms_total", C.c_float), ("ms_gate_eval", C.c_float), ("ms_stim", C.c_float),
                ("launches", C.c_int64), ("gate_eval_launches", C.c_int64),
                ("chunks", C.c_int64), ("data_bytes_peak", C.c_int64),
                ("input_toggles", C.c_int64), ("output_toggles", C.c_int64),
                ("graph_builds", C.c_int64), ("graph_replays", C.c_int64)]


# every symbol include/glsim_cuda.h declares, with its ctypes signature
SIGNATURES = {
    "gs_version": (C.c_int, []),
    "gs_last_error": (C.c_char_p, []),
    "gs_device_count": (C.c_int, [C.POINTER(C.c_int)]),
    "gs_design_create": (C.c_int, [C.POINTER(DesignDesc), C.c_int, C.POINTER(C.c_void_p)]),
    "gs_design_destroy": (C.c_int, [C.c_void_p]),
    "gs_stim_create": (C.c_int, [C.c_void_p, C.POINTER(StimDesc), C.POINTER(C.c_void_p)]),
    "gs_stim_destroy": (C.c_int, [C.c_void_p]),
    "gs_stim_synth": (C.c_int, [C.c_void_p, C.POINTER(SynthDesc), C.POINTER(C.c_void_p)]),
    "gs_synth_window_counts": (C.c_int, [C.POINTER(SynthDesc), C.c_int, _i64p]),
    "gs_stim_sizes": (C.c_int, [C.c_void_p, _i64p, _i64p]),
    "gs_stim_download": (C.c_int, [C.c_void_p, _i64p, _i64p, _i64p, _u8p]),
    "gs_engine_create": (C.c_int, [C.c_void_p, C.c_int64, C.c_void_p, C.POINTER(C.c_void_p)]),
    "gs_engine_destroy": (C.c_int, [C.c_void_p]),
    "gs_engine_set_items": (C.c_int, [C.c_void_p, C.c_int64, C.c_int, C.c_int]),
    "gs_slab_words": (C.c_int, [C.c_int, C.c_int]),
    "gs_run_stats": (C.c_int, [C.c_void_p, C.c_void_p, C.c_int64, C.c_int64, C.c_int,
                               C.POINTER(StatsOut)]),
    "gs_run_arena": (C.c_int, [C.c_void_p, C.c_void_p, C.c_int64, C.c_int64, C.c_int,
                               C.POINTER(ArenaOut), C.POINTER(StatsOut)]),
    "gs_last_timing": (C.c_int, [C.c_void_p, C.POINTER(Timing)]),
    "gs_arena_fill": (C.c_int, [C.c_void_p, C.c_void_p, C.c_int64, C.c_int64, C.c_int, _i64p,
                                C.c_int64, _i64p, C.c_int64, C.POINTER(C.c_int)]),
    "gs_run_stats_device": (C.c_int, [C.c_void_p, C.c_void_p, C.c_int64, C.c_int64, C.c_int,
                                      C.c_void_p]),
    "gs_run_compare": (C.c_int, [C.c_void_p, C.c_void_p, C.c_int64, C.c_int64, C.c_int,
                                 C.POINTER(ArenaRef), _i64p, _i64p, _i64p]),
    "gs_dwell_sweep": (C.c_int, [C.c_int64, _u8p, _i64p, _i64p, C.c_int64, _i64p, _i64p, _u8p,
                                 C.c_int64, C.c_int64, _i64p, C.c_int64, _i64p, _i64p, _u8p,
                                 C.c_int64, C.c_int64, _i64p, C.c_int64, C.c_int64, C.c_int64,
                                 _i64p, _i64p, _i64p]),
    "gs_init_values": (C.c_int, [C.POINTER(DesignDesc), _u8p, C.c_int64, _u8p]),
    "gs_sim_span": (C.c_int, [C.c_int64] * 5 + [_i64p, C.c_int64, _i64p, _i64p, _i64p, _i64p,
                                                _i64p, C.c_int64, _i64p, _u8p, C.c_int64,
                                                _i64p, _u8p, _i64p, C.c_int64, _i64p,
                                                C.c_int64, _i64p, _i64p, C.c_int64, C.c_int64,
                                                _u8p, C.c_int64, _i64p, _i64p, C.c_int64,
                                                _i64p, _i64p, _i64p, C.c_int64, _i64p, _i64p,
                                                _i64p, _i64p, _i64p, C.c_int64]),
    "gs_vcd_parse": (C.c_int, [C.c_char_p, C.c_int64, C.POINTER(C.c_char_p), C.c_int64,
                               C.POINTER(C.c_void_p)]),
    "gs_vcd_sizes": (C.c_int, [C.c_void_p, _i64p, _i64p]),
    "gs_vcd_copy": (C.c_int, [C.c_void_p, _i64p, _i64p, _u8p]),
    "gs_vcd_destroy": (C.c_int, [C.c_void_p]),
    "gs_last_error_line": (C.c_int64, []),
    "gs_last_error_col": (C.c_int64, []),
    "gs_sdf_parse": (C.c_int, [C.c_char_p, C.c_int64, C.POINTER(SdfDesign), C.c_int,
                               C.c_char_p, C.POINTER(C.c_void_p)]),
    "gs_sdf_sizes": (C.c_int, [C.c_void_p, _i64p, _i64p, _i64p, _i64p]),
    "gs_sdf_copy": (C.c_int, [C.c_void_p, _i64p, _i64p]),
    "gs_sdf_warning": (C.c_char_p, [C.c_void_p, C.c_int64]),
    "gs_sdf_destroy": (C.c_int, [C.c_void_p]),
    "gs_vcdw_create": (C.c_int, [C.c_char_p, _i64p, C.c_int64, C.c_char_p,
                                 C.POINTER(C.c_void_p)]),
    "gs_vcdw_feed": (C.c_int, [C.c_void_p, _u8p, _i64p, C.POINTER(WaveSrc), _i64p, C.c_int64,
                               C.c_int64]),
    "gs_vcdw_finish": (C.c_int, [C.c_void_p, C.c_int64]),
    "gs_vcdw_take": (C.c_int, [C.c_void_p, C.c_char_p, C.c_int64, _i64p]),
    "gs_vcdw_destroy": (C.c_int, [C.c_void_p]),
    "gs_netlist_parse": (C.c_int, [C.c_char_p, C.c_int64, C.c_char_p, _i64p, C.c_int64,
                                   C.c_char_p, _i64p, _i64p, C.c_char_p, _i64p,
                                   C.POINTER(C.c_void_p)]),
    "gs_netlist_sizes": (C.c_int, [C.c_void_p, _i64p, _i64p]),
    "gs_netlist_copy": (C.c_int, [C.c_void_p, C.c_char_p, C.c_char_p, _i64p, C.c_char_p, _i64p,
                                  C.c_char_p, _i64p, C.c_char_p, _i64p, _i64p, _i64p, _i64p]),
    "gs_netlist_destroy": (C.c_int, [C.c_void_p]),
    "gs_nccl_unique_id": (C.c_int, [C.c_char_p]),
    "gs_nccl_comm_create": (C.c_int, [C.c_char_p, C.c_int, C.c_int, C.c_int,
                                      C.POINTER(C.c_void_p)]),
    "gs_nccl_comm_destroy": (C.c_int, [C.c_void_p]),
    "gs_allreduce_stats": (C.c_int, [C.c_void_p, C.c_int64, C.c_void_p, C.c_void_p]),
    "gs_saif_format": (C.c_int, [C.c_char_p, _i64p, C.c_int64, _i64p, _i64p, _i64p, _i64p,
                                 C.c_int64, C.c_char_p, C.c_char_p, C.c_int, C.c_char_p,
                                 C.c_int64, _i64p]),
}

_lib = None


def load(path=LIB_PATH):
    """Load the library (once).  Raises if it has not been built."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(path):
        raise RuntimeError(f"{LIB_NAME} is not built ({path} missing); run "
                           "`python -c 'import __graft_entry__ as g; g.build()'` first. "
                           "There is no CPU fallback.")
    lib = C.CDLL(path)
    for name, (res, args) in SIGNATURES.items():
        fn = getattr(lib, name)
        fn.restype = res
        fn.argtypes = args
    _lib = lib
    return lib


def _check(rc):
    if rc == GS_OK:
        return
    msg = (_lib.gs_last_error() or b"").decode(errors="replace")
    if rc == GS_ERR_CAPACITY:
        raise CapacityError(f"device memory: {msg}")
    if rc == GS_ERR_CONSISTENCY:
        raise ConsistencyError(msg)
    if rc == GS_ERR_ARG:
        raise ValueError(msg)
    raise RuntimeError(f"libglsim_cuda: {msg}")


def vcd_parse(text, pi_names, path=None):
    """Native VCD reader (``gs_vcd_parse``): -> ``(pi_off, pi_times, pi_init,
    duration)``, or None when the library is not built or the text is outside
    the native reader's byte-exact subset (the caller then uses the Python
    reader).  Raises the reference's ParseError / SemanticError."""
    from .errors import ParseError, SemanticError
    try:
        lib = load()
    except RuntimeError:
        return None
    try:
        raw = text.encode("ascii") if isinstance(text, str) else bytes(text)
    except UnicodeEncodeError:
        return None
    names = [n.encode("ascii", errors="surrogateescape") if n.isascii() else None
             for n in pi_names]
    if any(n is None for n in names):
        return None
    arr = (C.c_char_p * max(1, len(names)))(*names)
    h = C.c_void_p()
    rc = lib.gs_vcd_parse(raw, len(raw), arr, len(names), C.byref(h))
    if rc == GS_ERR_UNSUPPORTED:
        return None
    if rc in (GS_ERR_PARSE, GS_ERR_SEMANTIC):
        msg = (lib.gs_last_error() or b"").decode()
        if rc == GS_ERR_PARSE:
            raise ParseError(msg, path, int(lib.gs_last_error_line()))
        raise SemanticError(msg)
    _check(rc)
    try:
        n, dur = C.c_int64(), C.c_int64()
        _check(lib.gs_vcd_sizes(h, C.byref(n), C.byref(dur)))
        P = len(names)
        pi_off = np.empty(P + 1, dtype=np.int64)
        pi_times = np.empty(n.value, dtype=np.int64)
        pi_init = np.empty(P, dtype=np.uint8)
        _check(lib.gs_vcd_copy(h, _p64(pi_off), _p64(pi_times), _p8(pi_init)))
    finally:
        lib.gs_vcd_destroy(h)
    return pi_off, pi_times, pi_init, int(dur.value)


def _names(blob, off):
    """UTF-8 blob + byte offsets -> list of str."""
    if not off.size or off[-1] == 0:
        return [""] * (off.size - 1)
    raw = bytes(blob)
    if raw.isascii() and b"\0" not in raw:
        # one split at C speed: a separator at every boundary
        sep = np.frombuffer(raw, dtype=np.uint8)
        parts = np.insert(sep, off[1:-1], 0).tobytes()
        return parts.decode("ascii").split("\0")
    return [raw[off[i]:off[i + 1]].decode("utf-8", errors="surrogatepass")
            for i in range(off.size - 1)]


def netlist_parse(text, lib):
    """Native netlist reader (``gs_netlist_parse``): -> dict of the design
    name, name lists and flat arrays (gate_cell, pin_off, pin_net), or None
    when the library is not built or the document is outside the reader's
    scope (every document the reference rejects: the Python reader then
    raises its exact error)."""
    try:
        lib_ = load()
    except RuntimeError:
        return None
    try:
        raw = text.encode("utf-8") if isinstance(text, str) else bytes(text)
    except UnicodeEncodeError:
        return None
    cells = list(lib.cells.values())
    cn, cno = _blob(c.name for c in cells)
    pn, pno = _blob(p for c in cells for p in c.input_pins)
    first = np.zeros(len(cells) + 1, dtype=np.int64)
    np.cumsum([len(c.input_pins) for c in cells], out=first[1:])
    co, coo = _blob(c.output_pin for c in cells)
    h = C.c_void_p()
    rc = lib_.gs_netlist_parse(raw, len(raw), cn, _p64(cno), len(cells), pn, _p64(pno),
                               _p64(first), co, _p64(coo), C.byref(h))
    if rc == GS_ERR_UNSUPPORTED:
        return None
    _check(rc)
    try:
        cnt = np.zeros(4, dtype=np.int64)
        nb = np.zeros(5, dtype=np.int64)
        _check(lib_.gs_netlist_sizes(h, _p64(cnt), _p64(nb)))
        P, O, G, NP = (int(x) for x in cnt)
        bufs = [C.create_string_buffer(max(1, int(b))) for b in nb]
        offs = [np.zeros(n + 1, dtype=np.int64) for n in (P, O, G, G)]
        gate_cell = np.zeros(G, dtype=np.int64)
        pin_off = np.zeros(G + 1, dtype=np.int64)
        pin_net = np.zeros(NP, dtype=np.int64)
        _check(lib_.gs_netlist_copy(h, bufs[0], bufs[1], _p64(offs[0]), bufs[2], _p64(offs[1]),
                                    bufs[3], _p64(offs[2]), bufs[4], _p64(offs[3]),
                                    _p64(gate_cell), _p64(pin_off), _p64(pin_net)))
    finally:
        lib_.gs_netlist_destroy(h)
    name = bufs[0].raw[:int(nb[0])].decode("utf-8", errors="surrogatepass")
    pis, pos, gates, outs = (_names(bufs[i + 1].raw[:int(nb[i + 1])], offs[i])
                             for i in range(4))
    return {"name": name, "pis": pis, "pos": pos, "gates": gates, "outs": outs,
            "cells": cells, "gate_cell": gate_cell, "pin_off": pin_off, "pin_net": pin_net}


def _blob(strings):
    """ASCII/UTF-8 strings -> (bytes, int64 byte offsets [n+1])."""
    strings = list(strings)
    joined = "".join(strings)
    if joined.isascii():
        lens = np.fromiter(map(len, strings), dtype=np.int64, count=len(strings))
        blob = joined.encode("ascii")
    else:
        enc = [x.encode("utf-8", errors="surrogatepass") for x in strings]
        lens = np.fromiter(map(len, enc), dtype=np.int64, count=len(enc))
        blob = b"".join(enc)
    off = np.zeros(len(strings) + 1, dtype=np.int64)
    np.cumsum(lens, out=off[1:])
    return blob, off


def _sdf_context(netlist):
    """Flat netlist description for gs_sdf_parse, cached on the netlist."""
    ctx = getattr(netlist, "_gs_sdf_ctx", None)
    if ctx is not None:
        return ctx
    cells, gate_cell = netlist.cell_arrays()
    pin_off, pin_net = netlist.pin_arrays()
    G = gate_cell.size
    out_net = np.arange(netlist.num_pis, netlist.num_pis + G, dtype=np.int64)
    pins = [p for c in cells for p in c.input_pins]
    first = np.zeros(len(cells) + 1, dtype=np.int64)
    np.cumsum([len(c.input_pins) for c in cells], out=first[1:])
    keep = {"gn": _blob(netlist.gate_names), "nn": _blob(netlist.net_names),
            "pn": _blob(pins), "co": _blob(c.output_pin for c in cells),
            "first": first, "gate_cell": gate_cell, "pin_off": pin_off, "pin_net": pin_net,
            "out_net": out_net}
    d = SdfDesign(num_gates=G, num_nets=len(netlist.net_names), num_cells=len(cells))
    d.gate_names, d.gate_name_off = keep["gn"][0], _p64(keep["gn"][1])
    d.net_names, d.net_name_off = keep["nn"][0], _p64(keep["nn"][1])
    d.pin_names, d.pin_name_off = keep["pn"][0], _p64(keep["pn"][1])
    d.cell_pin_first = _p64(first)
    d.cell_outputs, d.cell_output_off = keep["co"][0], _p64(keep["co"][1])
    d.gate_cell, d.pin_off = _p64(gate_cell), _p64(pin_off)
    d.pin_net, d.out_net = _p64(pin_net), _p64(out_net)
    ctx = (d, keep)
    try:
        netlist._gs_sdf_ctx = ctx
    except AttributeError:
        pass
    return ctx


def sdf_parse(text, netlist, corner, path):
    """Native SDF reader (``gs_sdf_parse``): -> ``(arc_rows [R, 2], pin_ic,
    timescale_fs, warnings)`` or None (library not built / text outside the
    native subset).  Raises the reference's ParseError / SemanticError."""
    from .errors import ParseError, SemanticError
    try:
        lib = load()
    except RuntimeError:
        return None
    try:
        raw = text.encode("ascii") if isinstance(text, str) else bytes(text)
    except UnicodeEncodeError:
        return None
    d, keep = _sdf_context(netlist)
    h = C.c_void_p()
    rc = lib.gs_sdf_parse(raw, len(raw), C.byref(d), ("min", "typ", "max").index(corner),
                          str(path).encode("utf-8", errors="surrogatepass"), C.byref(h))
    if rc == GS_ERR_UNSUPPORTED:
        return None
    if rc in (GS_ERR_PARSE, GS_ERR_SEMANTIC):
        msg = (lib.gs_last_error() or b"").decode("utf-8", errors="surrogatepass")
        if rc == GS_ERR_PARSE:
            line, col = int(lib.gs_last_error_line()), int(lib.gs_last_error_col())
            raise ParseError(msg, path, line or None, col or None)
        raise SemanticError(msg)
    _check(rc)
    try:
        r, p, ts, nw = (C.c_int64() for _ in range(4))
        _check(lib.gs_sdf_sizes(h, C.byref(r), C.byref(p), C.byref(ts), C.byref(nw)))
        arc = np.empty((r.value, 2), dtype=np.int64)
        ic = np.empty(p.value, dtype=np.int64)
        _check(lib.gs_sdf_copy(h, _p64(arc), _p64(ic)))
        warns = [lib.gs_sdf_warning(h, i).decode("utf-8", errors="surrogatepass")
                 for i in range(nw.value)]
    finally:
        lib.gs_sdf_destroy(h)
    return arc, ic, int(ts.value), warns


def saif_format(net_names, t0, t1, tc, ig, duration, design_name, version, include_ig):
    """Native SAIF text (``gs_saif_format``), or None if the library is not
    built (the caller then formats in Python)."""
    try:
        lib = load()
    except RuntimeError:
        return None
    names = list(net_names)
    joined = "".join(names)
    lens = np.fromiter(map(len, names), dtype=np.int64, count=len(names))
    if joined.isascii():  # one encode; byte offsets = character offsets
        blob = joined.encode("ascii")
    else:
        enc = [n.encode("utf-8", errors="surrogatepass") for n in names]
        lens = np.fromiter(map(len, enc), dtype=np.int64, count=len(enc))
        blob = b"".join(enc)
    off = np.zeros(len(names) + 1, dtype=np.int64)
    np.cumsum(lens, out=off[1:])
    arrs = [_c64(a) for a in (t0, t1, tc, ig)]
    dname = str(design_name).encode("utf-8", errors="surrogatepass")
    args = (blob, _p64(off), len(names), *[_p64(a) for a in arrs], int(duration), dname,
            version.encode(), int(bool(include_ig)))
    need = C.c_int64()
    lib.gs_saif_format(*args, None, 0, C.byref(need))
    buf = np.empty(need.value, dtype=np.uint8)
    n = C.c_int64()
    _check(lib.gs_saif_format(*args, buf.ctypes.data_as(C.c_char_p), need.value, C.byref(n)))
    return buf[:n.value].tobytes().decode("utf-8", errors="surrogatepass")


class VcdText:
    """Native VCD writer handle (``gs_vcdw_*``): header on creation, windows
    appended by :meth:`feed`; :meth:`take` returns the pending text."""

    def __init__(self, names, design_name):
        lib = load()
        blob, off = _blob(names)
        h = C.c_void_p()
        _check(lib.gs_vcdw_create(blob, _p64(off), len(off) - 1,
                                  str(design_name).encode("utf-8", errors="surrogatepass"),
                                  C.byref(h)))
        self.handle = h
        self._fin = weakref.finalize(self, lib.gs_vcdw_destroy, h)

    @staticmethod
    def _src(buf, offsets, counts, initials, col0):
        keep = (_c64(buf), _c64(offsets), _c64(counts), _c8(initials))
        b, o, c, i = keep
        cols = o.shape[1] if o.ndim == 2 else 0
        s = WaveSrc(buf=_p64(b) if b.size else None, n_buf=b.size, offsets=_p64(o),
                    counts=_p64(c), initials=_p8(i), cols=cols, col0=int(col0))
        return s, keep

    def feed(self, net_src, net_row, inputs, gates, boundaries, w_lo, w_hi):
        """``inputs`` / ``gates``: (buf, offsets, counts, initials, col0) windowed
        arrays; net i is row net_row[i] of inputs (net_src 0) or gates (1)."""
        s0, k0 = self._src(*inputs)
        s1, k1 = self._src(*gates)
        srcs = (WaveSrc * 2)(s0, s1)
        ns, nr, b = _c8(net_src), _c64(net_row), _c64(boundaries)
        _check(load().gs_vcdw_feed(self.handle, _p8(ns), _p64(nr), srcs, _p64(b), int(w_lo),
                                   int(w_hi)))

    def finish(self, end_time):
        _check(load().gs_vcdw_finish(self.handle, int(end_time)))

    def take(self):
        lib = load()
        n = C.c_int64()
        _check(lib.gs_vcdw_take(self.handle, None, 0, C.byref(n)))
        buf = C.create_string_buffer(max(1, n.value))
        _check(lib.gs_vcdw_take(self.handle, buf, n.value, C.byref(n)))
        return buf.raw[:n.value].decode("utf-8", errors="surrogatepass")


def _p64(a):
    return a.ctypes.data_as(_i64p) if a is not None else None


def _p8(a):
    return a.ctypes.data_as(_u8p) if a is not None else None


def _c64(a):
    return np.ascontiguousarray(a, dtype=np.int64)


def _c8(a):
    return np.ascontiguousarray(a, dtype=np.uint8)


def device_count():
    lib = load()
    n = C.c_int(0)
    _check(lib.gs_device_count(C.byref(n)))
    return n.value


_device = None


def current_device():
    """Device index this process drives: ``set_device`` > ``LOCAL_RANK`` > 0."""
    if _device is not None:
        return _device
    return int(os.environ.get("LOCAL_RANK", "0"))


def set_device(i):
    global _device
    _device = int(i)


def _design_desc(m):
    keep = dict(order=_c64(m.order), level_starts=_c64(m.level_starts), pin_off=_c64(m.pin_off),
                pin_net=_c64(m.pin_net), pin_ic=_c64(m.pin_ic), pin_arc=_c64(m.pin_arc),
                arc_rows=_c64(m.arc_rows).reshape(-1), lut_off=_c64(m.lut_off),
                lut_bits=_c8(m.lut_bits))
    d = DesignDesc(num_pis=m.num_pis, num_gates=m.num_gates, num_levels=m.num_levels,
                   order=_p64(keep["order"]), level_starts=_p64(keep["level_starts"]),
                   pin_off=_p64(keep["pin_off"]), pin_net=_p64(keep["pin_net"]),
                   pin_ic=_p64(keep["pin_ic"]), pin_arc=_p64(keep["pin_arc"]),
                   arc_rows=_p64(keep["arc_rows"]), num_arc_rows=keep["arc_rows"].size // 2,
                   lut_off=_p64(keep["lut_off"]), lut_bits=_p8(keep["lut_bits"]),
                   num_lut_bits=keep["lut_bits"].size)
    return d, keep


class Design:
    """Device copy of a compiled design (``gs_design``)."""

    def __init__(self, model, device=None):
        lib = load()
        self.device = current_device() if device is None else device
        desc, keep = _design_desc(model)
        h = C.c_void_p()
        _check(lib.gs_design_create(C.byref(desc), self.device, C.byref(h)))
        self.handle = h
        self.num_nets = model.num_pis + model.num_gates
        self.num_pis = model.num_pis
        self.num_gates = model.num_gates
        self._fin = weakref.finalize(self, lib.gs_design_destroy, h)


class Stimulus:
    """Device copy of a stimulus set (``gs_stim``), CSR or windowed form."""

    def __init__(self, design, stimuli):
        lib = load()
        b = _c64(stimuli.boundaries)
        keep = {"b": b}
        d = StimDesc(num_pis=stimuli.num_pis, num_windows=b.size - 1, boundaries=_p64(b))
        if stimuli.is_csr:
            keep.update(off=_c64(stimuli.pi_off), t=_c64(stimuli.pi_times), i=_c8(stimuli.pi_init))
            d.pi_off, d.pi_times, d.pi_init = _p64(keep["off"]), _p64(keep["t"]), _p8(keep["i"])
        else:
            keep.update(buf=_c64(stimuli.buf), off=_c64(stimuli.offsets),
                        cnt=_c64(stimuli.counts), ini=_c8(stimuli.initials))
            d.buf, d.n_buf = _p64(keep["buf"]), keep["buf"].size
            d.offsets, d.counts = _p64(keep["off"]), _p64(keep["cnt"])
            d.initials = _p8(keep["ini"])
        h = C.c_void_p()
        _check(lib.gs_stim_create(design.handle, C.byref(d), C.byref(h)))
        self.handle = h
        self.design = design
        self.num_windows = b.size - 1
        self._fin = weakref.finalize(self, lib.gs_stim_destroy, h)


def _synth_desc(cfg, w_lo, w_hi):
    import math

    def thr(a):  # u < alpha, as the integer test (h1 >> 11) < ceil(alpha * 2^53)
        return math.ceil(a * float(1 << 53))
    return SynthDesc(num_pis=cfg.num_inputs, num_ppis=cfg.ppis, seed=cfg.seed,
                     period=cfg.period, ppi_thr=thr(cfg.ppi_alpha), pi_thr=thr(cfg.pi_alpha),
                     ppi_lo=cfg.ppi_lo, ppi_span=cfg.ppi_hi - cfg.ppi_lo, pi_lo=cfg.pi_lo,
                     pi_span=cfg.pi_hi - cfg.pi_lo, w_lo=int(w_lo), w_hi=int(w_hi))


def synth_window_counts(cfg, w_lo, w_hi, device=None):
    """Per-window input toggles of a config's synthetic stimulus over
    [w_lo, w_hi), counted on the device (``gs_synth_window_counts``)."""
    out = np.empty(int(w_hi) - int(w_lo), dtype=np.int64)
    d = _synth_desc(cfg, w_lo, w_hi)
    _check(load().gs_synth_window_counts(C.byref(d), current_device() if device is None
                                         else int(device), _p64(out)))
    return out


class SynthStimulus(Stimulus):
    """A benchmark config's stimulus generated on the device
    (``gs_stim_synth``; identical to :func:`synth.stimulus` for the same
    window range)."""

    def __init__(self, design, cfg, w_lo, w_hi):  # noqa: D107 (no super().__init__: no host arrays)
        lib = load()
        d = _synth_desc(cfg, w_lo, w_hi)
        h = C.c_void_p()
        _check(lib.gs_stim_synth(design.handle, C.byref(d), C.byref(h)))
        self.handle = h
        self.design = design
        self.num_windows = int(w_hi) - int(w_lo)
        self._fin = weakref.finalize(self, lib.gs_stim_destroy, h)

    def download(self, pinned=False):
        """Host CSR arrays (boundaries, pi_off, pi_times, pi_init); page-locked
        (torch pinned memory) when ``pinned``."""
        lib = load()
        W, T = C.c_int64(), C.c_int64()
        _check(lib.gs_stim_sizes(self.handle, C.byref(W), C.byref(T)))
        P = self.design.num_pis
        shapes = ((W.value + 1, np.int64), (P + 1, np.int64), (T.value, np.int64), (P, np.uint8))
        if pinned:
            import torch
            arrs = [torch.empty(n, dtype=torch.int64 if t is np.int64 else torch.uint8)
                    .pin_memory().numpy() for n, t in shapes]
        else:
            arrs = [np.empty(n, dtype=t) for n, t in shapes]
        b, off, tm, ini = arrs
        _check(lib.gs_stim_download(self.handle, _p64(b), _p64(off), _p64(tm) if tm.size else None,
                                    _p8(ini) if ini.size else None))
        return b, off, tm, ini


class Engine:
    """Per-device engine (``gs_engine``): chunk workspace, stream, timers."""

    def __init__(self, design, mem_budget=0, stream=None):
        lib = load()
        h = C.c_void_p()
        _check(lib.gs_engine_create(design.handle, int(mem_budget),
                                    C.c_void_p(stream) if stream else None, C.byref(h)))
        self.handle = h
        self.design = design
        self._fin = weakref.finalize(self, lib.gs_engine_destroy, h)

    def set_items(self, workers=0, tail_div=2, tail_frac=2):
        """K4 work-item sizing (``gs_engine_set_items``); results never depend on it."""
        _check(load().gs_engine_set_items(self.handle, int(workers), int(tail_div),
                                          int(tail_frac)))

    def run_stats(self, stim, w_lo, w_hi, pct):
        """Stats over [w_lo, w_hi): (t1, tc, ig [N] int64, totals (filt, icf, disc))."""
        N = self.design.num_nets
        t1, tc, ig = (np.zeros(N, dtype=np.int64) for _ in range(3))
        out = StatsOut(t1=_p64(t1), tc=_p64(tc), ig=_p64(ig))
        _check(load().gs_run_stats(self.handle, stim.handle, int(w_lo), int(w_hi), int(pct),
                                   C.byref(out)))
        return t1, tc, ig, tuple(int(x) for x in out.totals)

    def run_stats_device(self, stim, w_lo, w_hi, pct, acc_ptr):
        """Add stats of [w_lo, w_hi) into a device int64 buffer [3N+3] at acc_ptr."""
        _check(load().gs_run_stats_device(self.handle, stim.handle, int(w_lo), int(w_hi),
                                          int(pct), C.c_void_p(acc_ptr)))

    def run_compare(self, stim, w_lo, w_hi, pct, buf, offsets, counts, initials):
        """Simulate [w_lo, w_hi) and compare every gate waveform with a
        reference arena on the device (``gs_run_compare``): -> (mismatching
        (gate, window) pairs, first (gate, window) or None)."""
        buf, offsets, counts = _c64(buf), _c64(offsets), _c64(counts)
        initials = _c8(initials)
        ref = ArenaRef(buf=_p64(buf), n_buf=buf.size, offsets=_p64(offsets),
                       counts=_p64(counts), initials=_p8(initials), cols=offsets.shape[1])
        n, g, w = C.c_int64(), C.c_int64(), C.c_int64()
        _check(load().gs_run_compare(self.handle, stim.handle, int(w_lo), int(w_hi), int(pct),
                                     C.byref(ref), C.byref(n), C.byref(g), C.byref(w)))
        return int(n.value), ((int(g.value), int(w.value)) if n.value else None)

    def run_arena(self, stim, w_lo, w_hi, pct, offsets=None, n_buf=0, want_stats=False,
                  caps=None):
        """Count pass (offsets None) or store pass over [w_lo, w_hi).

        Returns dict of [G, Ws] arrays (counts, peak, filtered, ic_filtered,
        discarded, initials), ``buf`` for a store pass, and ``stats`` (as
        :meth:`run_stats`) when requested.
        """
        G = self.design.num_gates
        Ws = int(w_hi) - int(w_lo)
        res = {k: np.zeros((G, Ws), dtype=np.int64)
               for k in ("counts", "peak", "filtered", "ic_filtered", "discarded")}
        res["initials"] = np.zeros((G, Ws), dtype=np.uint8)
        a = ArenaOut(counts=_p64(res["counts"]), peak=_p64(res["peak"]),
                     filtered=_p64(res["filtered"]), ic_filtered=_p64(res["ic_filtered"]),
                     discarded=_p64(res["discarded"]), initials=_p8(res["initials"]))
        if offsets is not None:
            off = _c64(offsets)
            buf = np.empty(int(n_buf), dtype=np.int64)
            res["buf"] = buf
            a.offsets, a.buf, a.n_buf = _p64(off), (_p64(buf) if buf.size else
                                                    C.cast(C.c_void_p(8), _i64p)), buf.size
            if caps is not None:
                cp = _c64(caps)
                res["_caps"] = cp
                a.caps = _p64(cp)
        st = None
        if want_stats:
            N = self.design.num_nets
            t1, tc, ig = (np.zeros(N, dtype=np.int64) for _ in range(3))
            st = StatsOut(t1=_p64(t1), tc=_p64(tc), ig=_p64(ig))
        _check(load().gs_run_arena(self.handle, stim.handle, int(w_lo), int(w_hi), int(pct),
                                   C.byref(a), C.byref(st) if st is not None else None))
        if want_stats:
            res["stats"] = (t1, tc, ig, tuple(int(x) for x in st.totals))
        return res

    def arena_fill(self, stim, w_lo, w_hi, pct, buf, offsets):
        """Fill ``buf`` at ``offsets`` [G, Ws] from this engine's last count
        pass of (stim, [w_lo, w_hi), pct) (``gs_arena_fill``); False (nothing
        written) when that pass is not the last one run."""
        off = _c64(offsets)
        f = C.c_int(0)
        _check(load().gs_arena_fill(self.handle, stim.handle, int(w_lo), int(w_hi), int(pct),
                                    _p64(buf) if buf.size else None, buf.size, _p64(off),
                                    off.shape[1] if off.ndim == 2 else int(w_hi) - int(w_lo),
                                    C.byref(f)))
        return bool(f.value)

    def timing(self):
        t = Timing()
        _check(load().gs_last_timing(self.handle, C.byref(t)))
        return {f: getattr(t, f) for f, _ in Timing._fields_}


NCCL_ID_BYTES = 128


def nccl_unique_id():
    """A new NCCL unique id (``gs_nccl_unique_id``), as bytes."""
    buf = C.create_string_buffer(NCCL_ID_BYTES)
    _check(load().gs_nccl_unique_id(buf))
    return buf.raw


class NcclComm:
    """NCCL communicator of this rank (``gs_nccl_comm_create``); ``uid`` from
    :func:`nccl_unique_id` on one rank, shared with all."""

    def __init__(self, uid, nranks, rank, device=None):
        lib = load()
        h = C.c_void_p()
        dev = current_device() if device is None else int(device)
        _check(lib.gs_nccl_comm_create(bytes(uid), int(nranks), int(rank), dev, C.byref(h)))
        self.handle = h
        self._fin = weakref.finalize(self, lib.gs_nccl_comm_destroy, h)

    def allreduce_stats(self, acc_ptr, n, stream=None):
        """In-place int64 sum of the device accumulator at ``acc_ptr`` [n]
        across the ranks (``gs_allreduce_stats``), on ``stream``."""
        _check(load().gs_allreduce_stats(C.c_void_p(acc_ptr), int(n), self.handle,
                                         C.c_void_p(stream) if stream else None))


def dwell_sweep(arena, stimuli, boundaries, num_pis, num_gates):
    """GPU dwell_sweep (``_kernels.py:254-295``) over an arena: per-net (t1, tc, ig)."""
    lib = load()
    N = num_pis + num_gates
    net_kind = np.zeros(N, dtype=np.uint8)
    net_kind[num_pis:] = 1
    net_slot = np.concatenate([np.arange(num_pis), np.arange(num_gates)]).astype(np.int64)
    w_lo, w_hi = arena.window_range
    sbuf, soff, scnt, sini = (_c64(stimuli.buf), _c64(stimuli.offsets), _c64(stimuli.counts),
                              _c8(stimuli.initials))
    gbuf, goff, gcnt, gini = (_c64(arena.buf), _c64(arena.offsets), _c64(arena.counts),
                              _c8(arena.initials))
    b = _c64(boundaries)
    t0, t1, tc = (np.zeros(N, dtype=np.int64) for _ in range(3))
    W = b.size - 1
    _check(lib.gs_dwell_sweep(N, _p8(net_kind), _p64(net_slot), _p64(sbuf), sbuf.size,
                              _p64(soff), _p64(scnt), _p8(sini), num_pis, W,
                              _p64(gbuf), gbuf.size, _p64(goff), _p64(gcnt), _p8(gini),
                              num_gates, goff.shape[1] if goff.ndim == 2 else w_hi - w_lo,
                              _p64(b), w_lo, w_hi, w_lo, _p64(t0), _p64(t1), _p64(tc)))
    ig = np.zeros(N, dtype=np.int64)
    if num_gates:
        ig[num_pis:] = np.asarray(arena.filtered, dtype=np.int64).sum(axis=1)
    return t1, tc, ig


def sim_span(oi_lo, oi_hi, w_lo, w_hi, w_off, order, pin_off, pin_net, pin_ic, pin_arc,
             arc_rows, lut_off, lut_bits, out_net, net_kind, net_slot, stim_buf, stim_off,
             stim_cnt, init_vals, boundaries, gbuf, g_off, g_cap, g_cnt, out_filt, out_icf,
             out_disc, out_err, out_peak, pct):
    """The reference kernel ``sim_span`` (``_kernels.py:17-210``) with its own
    argument list, on the GPU (``gs_sim_span``): arrays as the reference
    passes them (numpy, int64 / uint8, 2-D row-major); outputs written in
    place."""
    c = [_c64(a) for a in (order, pin_off, pin_net, pin_ic, pin_arc, arc_rows, lut_off, out_net,
                           net_slot, stim_buf, stim_off, stim_cnt, boundaries, g_off, g_cap)]
    order, pin_off, pin_net, pin_ic, pin_arc, arc_rows, lut_off, out_net, net_slot, \
        stim_buf, stim_off, stim_cnt, boundaries, g_off, g_cap = c
    u = [_c8(a) for a in (lut_bits, net_kind, init_vals)]
    lut_bits, net_kind, init_vals = u
    outs = (gbuf, g_cnt, out_filt, out_icf, out_disc, out_err, out_peak)
    for a in outs:
        if a.dtype != np.int64 or not a.flags.c_contiguous:
            raise ValueError("sim_span outputs must be C-contiguous int64 arrays")
    G = order.size
    _check(load().gs_sim_span(
        int(oi_lo), int(oi_hi), int(w_lo), int(w_hi), int(w_off), _p64(order), G,
        _p64(pin_off), _p64(pin_net), _p64(pin_ic), _p64(pin_arc), _p64(arc_rows),
        arc_rows.size // 2, _p64(lut_off), _p8(lut_bits), lut_bits.size, _p64(out_net),
        _p8(net_kind), _p64(net_slot), net_kind.size, _p64(stim_buf), stim_buf.size,
        _p64(stim_off), _p64(stim_cnt), stim_off.shape[0], stim_off.shape[1],
        _p8(init_vals), init_vals.shape[1], _p64(boundaries), _p64(gbuf), gbuf.size,
        _p64(g_off), _p64(g_cap), _p64(g_cnt), g_off.shape[1], _p64(out_filt), _p64(out_icf),
        _p64(out_disc), _p64(out_err), _p64(out_peak), int(pct)))


def init_values(model, stim_init):
    """GPU init_values (``_kernels.py:213-231``): uint8 [N, W]."""
    lib = load()
    desc, keep = _design_desc(model)
    si = _c8(stim_init)
    W = si.shape[1] if si.ndim == 2 else 0
    out = np.zeros((model.num_pis + model.num_gates, W), dtype=np.uint8)
    _check(lib.gs_init_values(C.byref(desc), _p8(si), W, _p8(out)))
    return out
