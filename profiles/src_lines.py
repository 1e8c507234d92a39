"""Aggregate an ncu source page (--print-source cuda,sass --csv) by CUDA line:
instructions executed and warp-stall samples per source line.

    ncu -i rep --page source --csv --print-source cuda,sass > src.csv
    python profiles/src_lines.py src.csv [top]
"""
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
top = int(sys.argv[2]) if len(sys.argv) > 2 else 40
hdr = None
lines = []
fname = ""
for r in rows:
    if len(r) >= 2 and r[0] == "File Path":
        fname = r[1].split("/")[-1]
    if r and r[0] == "Line No":
        hdr = r
        continue
    if hdr and r and r[0] not in ("", "Line No") and r[0].isdigit() and len(r) > 7:
        try:
            samples = int(r[4]) if r[4] not in ("-", "") else 0
            inst = int(r[7]) if r[7] not in ("-", "") else 0
        except ValueError:
            continue
        lines.append((fname, int(r[0]), r[1].strip()[:70], inst, samples))
ti = sum(x[3] for x in lines) or 1
ts = sum(x[4] for x in lines) or 1
print(f"total instructions {ti:,}  stall samples {ts:,}")
print("by instructions:")
for f, ln, src, i, s in sorted(lines, key=lambda x: -x[3])[:top]:
    print(f"  {f}:{ln:5d} inst {i / ti * 100:5.1f}%  samples {s / ts * 100:5.1f}%  {src}")
print("by stall samples:")
for f, ln, src, i, s in sorted(lines, key=lambda x: -x[4])[:top]:
    print(f"  {f}:{ln:5d} inst {i / ti * 100:5.1f}%  samples {s / ts * 100:5.1f}%  {src}")
