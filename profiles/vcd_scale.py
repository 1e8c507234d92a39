"""VCD writer scale probe (CPU, native gs_vcdw_*): G nets x W windows of
random waveforms (0 or 1 toggle per net-window) through report's native
writer path; prints the time and the output size.

    python profiles/vcd_scale.py 10000000 4
"""
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2203_06117_b200 import _native  # noqa: E402

G = int(sys.argv[1]) if len(sys.argv) > 1 else 10_000_000
W = int(sys.argv[2]) if len(sys.argv) > 2 else 4
rng = np.random.default_rng(3)
cnt = rng.integers(0, 2, size=(G, W)).astype(np.int64)
off = np.concatenate(([0], np.cumsum(cnt.ravel())[:-1])).reshape(G, W)
b = np.arange(W + 1, dtype=np.int64) * 1000
buf = (np.repeat(b[:-1][None, :], G, 0) + 500).ravel()[cnt.ravel() > 0]
ini = rng.integers(0, 2, size=(G, W)).astype(np.uint8)
names = [f"g{i}" for i in range(G)]
z = np.zeros((0, W), dtype=np.int64)
t0 = time.perf_counter()
v = _native.VcdText(names, "big")
t1 = time.perf_counter()
v.feed(np.ones(G, np.uint8), np.arange(G), (np.zeros(0, np.int64), z, z,
                                           np.zeros((0, W), np.uint8), 0),
       (buf, off, cnt, ini, 0), b, 0, W)
v.finish(int(b[-1]))
text = v.take()
t2 = time.perf_counter()
print(f"{G} nets x {W} windows, {int(cnt.sum())} toggles: header {t1 - t0:.2f} s, "
      f"events {t2 - t1:.2f} s, total {t2 - t0:.2f} s, {len(text) / 1e6:.0f} MB of VCD text")
