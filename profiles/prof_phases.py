"""Dev probe: per-phase split of K4 (GS_PROF build) on a config slice.

    python profiles/prof_phases.py C3 4096

Needs paper_2203_06117_b200/libglsim_cuda_prof.so, built with
    python -c "import __graft_entry__ as g; g.build_native(force=True,
        out='paper_2203_06117_b200/libglsim_cuda_prof.so', defines=['GS_PROF'])"
Cycle shares are summed SM clocks of all warps in each phase (clock64 deltas,
lane 0), so they weight phases by the time warps spend in them.
"""
import ctypes as C
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
os.environ.setdefault("GLSIM_LIB", "libglsim_cuda_prof.so")
from paper_2203_06117_b200 import synth, _native  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "C3"
W = int(sys.argv[2]) if len(sys.argv) > 2 else 4096
cfg = synth.config(name)
m = synth.design(cfg)
stim = synth.stimulus(cfg, 0, W)
dev = m.device()
eng = _native.Engine(dev, 0)
s = _native.Stimulus(dev, stim)
lib = _native.load()
lib.gs_prof_read.argtypes = [C.POINTER(C.c_uint64)]
buf = (C.c_uint64 * 16)()
eng.run_stats(s, 0, W, cfg.pct)
lib.gs_prof_read(buf)
eng.run_stats(s, 0, W, cfg.pct)
lib.gs_prof_read(buf)
v = list(buf)
names = ["(A) counts, staging, inline windows", "(unused)", "(M) pooled worklists",
         "(C) compaction, sums"]
tot = sum(v[:4]) or 1
print(f"config {name} x {W} windows, {cfg.gates} gates")
for i, n in enumerate(names):
    print(f"  {n:40s} {v[i] / tot * 100:5.1f}% of warp-cycles")
tiles = max(v[8], 1)
print(f"  tiles {v[8]}, two-transition windows {v[9]} "
      f"({v[9] / (tiles * 128) * 100:.1f}% of tile windows), loop windows {v[7]} "
      f"({v[7] / (tiles * 128) * 100:.1f}%)")
print(f"  device ms (gate_eval) {eng.timing()['ms_gate_eval']:.2f}")
