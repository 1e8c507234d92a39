"""Generate the golden fixtures by running the REFERENCE package itself.

Run in the build container (where /root/reference exists):

    python tests/golden/make_golden.py

The reference ``glsim`` (numba) is copied to a temp directory and imported from
there (numba's ``cache=True`` must not write into /root/reference).  For every
case the script stores the input documents and the reference outputs --
arena arrays, per-net statistics, SAIF text, run-report totals, and the
reference's flattened design / windowed stimulus arrays -- into
``tests/golden/<case>.npz``.  The GPU box never needs /root/reference: tests
read only these files.
"""

import json
import os
import shutil
import sys
import tempfile

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(HERE))  # tests/ (for gen)
import gen  # noqa: E402

REF = "/root/reference/pkg"


def import_reference():
    tmp = tempfile.mkdtemp(prefix="glsim_ref_")
    shutil.copytree(os.path.join(REF, "src", "glsim"), os.path.join(tmp, "glsim"))
    sys.path.insert(0, tmp)
    import glsim  # noqa: F401  (the reference, from the temp copy)
    assert glsim.__file__.startswith(tmp)
    return glsim


def demo_docs(period=20000, **kw):
    rd = lambda n: open(os.path.join(REF, "tests", "data", n)).read()  # noqa: E731
    return gen.Docs(rd("demo.lib.json"), rd("demo.netlist.json"), rd("demo.sdf"),
                    rd("demo.vcd"), period, **kw)


def cases():
    yield "demo", demo_docs()
    yield "demo_pct50", demo_docs(pct=50)
    yield "demo_avg", demo_docs(avg=True)
    yield "demo_one_window", demo_docs(period=None)
    d = demo_docs()
    yield "demo_zero_delay", gen.Docs(d.lib, d.net, None, d.vcd, d.period)
    pcts = (100, 100, 50, 0, 75, 100, 25, 100)
    for s in range(32):
        yield f"rnd{s:02d}", gen.make_docs(1000 + s, pct=pcts[s % len(pcts)], avg=(s % 11 == 5),
                                           with_sdf=(s % 13 != 7))
    # wider cells (generic k path, k > 6 truth tables in packed words)
    yield "wide_k", gen.make_docs(77, n_gates=60, n_pis=9, windows=4, max_k=8, max_toggles=40)
    # delays long against the windows: many window-end discards
    yield "discards", gen.make_docs(78, n_gates=200, windows=8, max_delay=60_000,
                                    duration_ps=1200)
    # heavy activity, low filter threshold: retractions of stored edges
    yield "busy_pct0", gen.make_docs(79, n_gates=300, n_pis=6, windows=3, max_toggles=200,
                                     pct=0, duration_ps=1500)
    # many windows (several 32-window tiles, ragged last tile)
    yield "many_windows", gen.make_docs(80, n_gates=150, n_pis=8, windows=75,
                                        max_toggles=300, duration_ps=30000)
    # one window longer than 2^32 fs (64-bit timestamp path)
    yield "long_window", gen.make_docs(81, n_gates=80, n_pis=5, windows=1,
                                       duration_ps=6_000_000, max_delay=2_000_000,
                                       max_toggles=30)


def run_case(ref, docs):
    nl, lv, delays, waves, duration, b, stim = gen.load(docs, ref)
    arena, diag = ref.run(lv, stim, delays, ref.RunConfig(workers=2, mem_cap=None,
                                                          pathpulse_pct=docs.pct))
    stats = ref.compute_stats(arena, stim)
    model = ref.simcore.compile_design(lv, delays)
    out = dict(
        buf=arena.buf, offsets=arena.offsets, caps=arena.caps, counts=arena.counts,
        pass1_counts=arena.pass1_counts, initials=arena.initials, filtered=arena.filtered,
        ic_filtered=arena.ic_filtered, discarded=arena.discarded,
        t0=stats.t0, t1=stats.t1, tc=stats.tc, ig=stats.ig,
        duration=np.int64(stats.duration), windows=np.int64(stats.windows),
        boundaries=np.asarray(b, dtype=np.int64),
        stim_buf=stim.buf, stim_offsets=stim.offsets, stim_counts=stim.counts,
        stim_initials=stim.initials,
        order=model.order, level_starts=model.level_starts, pin_off=model.pin_off,
        pin_net=model.pin_net, pin_ic=model.pin_ic, pin_arc=model.pin_arc,
        arc_rows=model.arc_rows,
        saif=np.frombuffer(ref.write_saif(stats, nl.name).encode(), dtype=np.uint8),
        vcd_out=np.frombuffer(ref.write_vcd(arena, stimuli=stim).encode(), dtype=np.uint8),
        report=np.frombuffer(json.dumps({k: v for k, v in ref.run_report(stats, diag).items()
                                         if k not in ("timings", "tasks")}).encode(),
                             dtype=np.uint8),
    )
    return out


def main():
    ref = import_reference()
    index = {}
    for name, docs in cases():
        out = run_case(ref, docs)
        meta = {"lib": docs.lib, "net": docs.net, "sdf": docs.sdf, "vcd": docs.vcd,
                "period": docs.period, "pct": docs.pct, "avg": docs.avg}
        np.savez_compressed(os.path.join(HERE, f"{name}.npz"),
                            meta=np.frombuffer(json.dumps(meta).encode(), dtype=np.uint8), **out)
        index[name] = {"gates": int(out["counts"].shape[0]), "windows": int(out["windows"]),
                       "toggles": int(out["counts"].sum()), "pct": docs.pct}
        print(name, index[name])
    with open(os.path.join(HERE, "index.json"), "w") as f:
        json.dump(index, f, indent=1, sort_keys=True)


if __name__ == "__main__":
    main()
