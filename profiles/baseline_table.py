"""BASELINE.md §4 table rows from a measurement pass's bench lines.

    python profiles/baseline_table.py [prefix]      (default profiles/r02/final_bench_)
"""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
prefix = sys.argv[1] if len(sys.argv) > 1 else os.path.join(ROOT, "profiles", "r02", "final_bench_")
ROWS = [("c1", "C1", "100 x 1,000"), ("c2", "C2", "100,000 x 10,000"),
        ("default", "**C3**", "1,000,000 x 100,000"), ("c4", "C4", "10,000,000 x 16,384"),
        ("C5", "C5 full SDF, pct 100", "1,000,000 x 16,384"),
        ("C5-pct0", "C5 full SDF, pct 0", "1,000,000 x 16,384"),
        ("C5-avg", "C5 averaged SDF, pct 100", "1,000,000 x 16,384"),
        ("C5-avg-pct0", "C5 averaged SDF, pct 0", "1,000,000 x 16,384")]
print("| Config | GPUs | Gates x windows | Gate-cycles/s | ms per step | End to end (ms per step) "
      "| K4 HBM (of 6,529 / 8,000 GB/s) | CPU baseline | Parity |")
print("|---|---|---|---|---|---|---|---|---|")
for key, name, shape in ROWS:
    path = f"{prefix}{key}.jsonl"
    if not os.path.exists(path):
        continue
    x = json.loads(open(path).read().splitlines()[0])
    r, e, cb = x["roofline"], x["e2e"], x["cpu_baseline"]
    bold = name.startswith("**")
    v = f"{x['value']:.3g}".replace("e+", "e+")
    ev = f"{e['value']:.3g}"
    frac = f"{r['frac'] * 100:.1f} %"
    print(f"| {name} | 1 | {shape} | {'**' + v + '**' if bold else v} | {x['ms_per_step']:.1f} ms "
          f"| {'**' + ev + '**' if bold else ev} ({e['ms_per_step']:.1f} ms) "
          f"| {r['achieved']:.0f} GB/s = {'**' + frac + '**' if bold else frac} / "
          f"{r['achieved'] / 8000 * 100:.1f} % | {cb['value']:.3g} ({cb['cores']} threads, oracle port) "
          f"| {x.get('parity', {}).get('result', '?')} |")
    if key == "c4":
        print("| C4 | 2 / 4 / 8 | 16,384 per GPU | not measured (one GPU per call in this "
              "environment) | | | | | |")
