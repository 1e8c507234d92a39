"""Dev probe: per-phase cycle split of K4 on C2 (GS_PROF build: python -c "import __graft_entry__ as g; g.build_native(force=True, out='paper_2203_06117_b200/libglsim_cuda_prof.so', defines=['GS_PROF'])")."""
import ctypes as C, os, sys
import numpy as np
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
os.environ.setdefault("GLSIM_LIB", "libglsim_cuda_prof.so")
from paper_2203_06117_b200 import synth, _native
cfg = synth.config("C2")
W = int(sys.argv[1]) if len(sys.argv) > 1 else 2048
m = synth.design(cfg); stim = synth.stimulus(cfg, 0, W)
dev = m.device(); eng = _native.Engine(dev, 0); s = _native.Stimulus(dev, stim)
lib = _native.load(); lib.gs_prof_read.argtypes = [C.POINTER(C.c_uint64)]
buf = (C.c_uint64 * 16)()
eng.run_stats(s, 0, W, 100); lib.gs_prof_read(buf)
eng.run_stats(s, 0, W, 100); lib.gs_prof_read(buf)
v = list(buf)
names = ["phase1", "closed+worklist", "event loop", "phase3"]
tot = sum(v[:4])
for i, n in enumerate(names):
    print(f"{n:16s} {v[i]/tot*100:5.1f}% of warp-cycles")
print(f"tiles {v[8]}, slow(global) tiles {v[10]}, trivial windows {v[9]}, loop windows {v[7]}")
print(f"loop iterations {v[4]}, avg busy lanes/iter {v[5]/max(v[4],1):.2f}, iters per tile {v[4]/max(v[8],1):.1f}")
print(f"slow tile cycles {v[11]/tot*100:.1f}% of warp-cycles, avg UB {v[12]/max(v[10],1):.0f}")
print(f"device ms {eng.timing()['ms_gate_eval']:.2f}")
