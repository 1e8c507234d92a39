"""Per-source-line warp instructions per 128-window tile of one K4 launch,
from an ncu report (needs -lineinfo and --import-source on).

    python profiles/k4_lines.py REPORT LAUNCH_INDEX TILES [min_per_tile]
"""
import csv
import io
import subprocess
import sys

rep, idx, tiles = sys.argv[1], int(sys.argv[2]), float(sys.argv[3])
lo = float(sys.argv[4]) if len(sys.argv) > 4 else 1.0
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source",
                      "cuda,sass", "--launch-skip", str(idx), "--launch-count", "1"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
fname, hdr, tot, per = "", None, 0, []
for r in rows:
    if len(r) >= 2 and r[0] == "File Path":
        fname = r[1].split("/")[-1]
    if r and r[0] == "Line No":
        hdr = r
        continue
    if hdr and r and r[0].isdigit() and len(r) > 7 and r[7] not in ("-", ""):
        try:
            n = int(r[7])
        except ValueError:
            continue
        tot += n
        per.append((fname, int(r[0]), r[1].strip(), n))
print(f"total {tot:,} warp instructions = {tot / tiles:.0f} per tile = {tot / tiles / 128:.2f} per gate-window")
for f, ln, src, n in per:
    if n / tiles >= lo:
        print(f"{f[:16]:16s} {ln:4d} {n / tiles:7.1f}  {src[:90]}")

# per-function totals (kernels_lean.cuh line ranges)
import re as _re
src = open(__file__.replace("profiles/k4_lines.py", "paper_2203_06117_b200/csrc/kernels_lean.cuh")).read().splitlines()
marks = [(i + 1, m.group(1)) for i, l in enumerate(src)
         for m in [_re.match(r"(?:__global__ void|__device__ __forceinline__ \w+ )\s*(\w+)\(|^gate_eval_lean\(", l)] if m]
def _fn(ln):
    name = "?"
    for a, nme in marks:
        if a <= ln:
            name = nme or "gate_eval_lean"
    return name
agg = {}
for f, ln, s_, n in per:
    k = _fn(ln) if f == "kernels_lean.cuh" else f
    agg[k] = agg.get(k, 0) + n
print("per function (warp inst per tile):")
for k, v in sorted(agg.items(), key=lambda x: -x[1]):
    print(f"  {k:28s} {v / tiles:7.1f}")
