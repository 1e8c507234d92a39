"""Front-end scale probe (CPU): a synthetic netlist JSON of G gates through
parse_library -> parse_netlist -> levelize -> zero_delays / parse_sdf ->
compile_design, timed per stage.

    python profiles/frontend_scale.py 10000000 [--sdf]
"""
import json
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2203_06117_b200 as api  # noqa: E402
from paper_2203_06117_b200 import synth  # noqa: E402

G = int(sys.argv[1]) if len(sys.argv) > 1 else 1_000_000
with_sdf = "--sdf" in sys.argv
cfg = synth.config("C2", gates=G, levels=20)
m = synth.design(cfg)  # the arrays of a random levelized netlist of the C-config shape
P = m.num_pis
names = [c[0] for c in synth.CELLS]
pins = {1: ["A"], 2: ["A", "B"], 3: ["A", "B", "C"], 4: ["A", "B", "C", "D"]}
lib = {"cells": [{"name": n, "inputs": pins[k], "output": "Y", "truth": t}
                 for n, t, k in synth.CELLS]}
cell_of = {}
for i, (n, t, k) in enumerate(synth.CELLS):
    cell_of[t, k] = n
t0 = time.perf_counter()
k = np.diff(m.pin_off)
luts = {}
parts = ['{"name": "scale", "inputs": [', ",".join(f'"i{p}"' for p in range(P)),
         '], "outputs": [], "gates": [']
lut_cells = {int(o): None for o in np.unique(m.lut_off)}
off_name = {}
top = 0
for n, t, kk in synth.CELLS:
    off_name[top] = (n, kk)
    top += len(t)
net = lambda x: f"i{x}" if x < P else f"n{x - P}"  # noqa: E731
pin_net = m.pin_net.tolist()
po = m.pin_off.tolist()
lo = m.lut_off.tolist()
gates = []
for g in range(G):
    n, kk = off_name[lo[g]]
    pn = ",".join(f'"{pins[kk][q]}":"{net(pin_net[po[g] + q])}"' for q in range(kk))
    gates.append(f'{{"name":"u{g}","cell":"{n}","pins":{{{pn},"Y":"n{g}"}}}}')
parts.append(",".join(gates))
parts.append("]}")
text = "".join(parts)
del gates, parts
t_gen = time.perf_counter() - t0
print(f"G={G}: JSON {len(text) / 1e6:.0f} MB generated in {t_gen:.1f} s")

stages = {}
t = time.perf_counter()
L = api.parse_library(json.dumps(lib))
nl = api.parse_netlist(text, L)
stages["parse_netlist"] = time.perf_counter() - t
assert nl._gates is None and nl.num_gates == G
t = time.perf_counter()
lv = api.levelize(nl)
stages["levelize"] = time.perf_counter() - t
t = time.perf_counter()
d = api.zero_delays(nl)
stages["zero_delays"] = time.perf_counter() - t
t = time.perf_counter()
cm = api.compile_design(lv, d)
stages["compile_design"] = time.perf_counter() - t
assert np.array_equal(cm.pin_net, m.pin_net) and np.array_equal(cm.pin_off, m.pin_off)
print("  " + ", ".join(f"{k} {v:.2f} s" for k, v in stages.items()),
      f"-> total {sum(stages.values()):.2f} s")
