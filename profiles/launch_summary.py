"""K4 launch-list summaries and profiles/k4_traffic.json from a measurement
pass's ncu launch lists (gpu__time_duration, dram bytes, instructions).

    python profiles/launch_summary.py PREFIX     (e.g. gpurun_out/m3_)
"""
import collections
import csv
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
prefix = sys.argv[1]


def agg(path):
    rows = [r for r in csv.reader(open(path)) if len(r) > 10]
    hdr = [r for r in rows if r[0] == "ID"][0]
    ix = {n: i for i, n in enumerate(hdr)}
    per, names = collections.defaultdict(dict), {}
    for r in rows:
        if not r[0].isdigit():
            continue
        per[r[0]][r[ix["Metric Name"]]] = float(r[ix["Metric Value"]].replace(",", ""))
        names[r[0]] = r[ix["Kernel Name"]].split("(")[0].replace("void ", "")
    return per, names


out = []
for cfg, csvf, windows, lps, bench, flag in (
        ("C3", "launches_c3.csv", 100000, 900, "final_bench_default.jsonl", ""),
        ("C2", "launches_c2.csv", 10000, 80, "final_bench_c2.jsonl", " --config C2")):
    per, names = agg(prefix + csvf)
    n = len(per)
    dram_of = lambda v: v.get("dram__bytes_read.sum", 0) + v.get("dram__bytes_write.sum", 0)  # noqa
    dram = sum(dram_of(v) for v in per.values()) / n
    t = sum(v["gpu__time_duration.sum"] for v in per.values()) / n
    alg = json.loads(open(os.path.join(ROOT, "profiles", "r02", bench)).read())
    alg = alg["roofline"]["algorithmic_bytes_per_step"] / lps
    out.append({"config": cfg, "windows": windows, "kernel": "gate_eval_lean (K4)",
                "launches_per_step": lps, "dram_bytes_per_launch": dram,
                "algorithmic_bytes_per_launch": alg,
                "source": f"ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum over the "
                          f"first {n} K4 launches (one window chunk, all levels and fanin groups) "
                          f"of python bench.py{flag} --steps 1 --warmup 0 (round 2, final kernel)"})
    by = collections.defaultdict(list)
    for k, v in per.items():
        by[names[k]].append(v)
    lines = [f"{cfg} x {windows} windows: first {n} K4 launches (one chunk): mean {t / 1e3:.1f} us, "
             f"{dram / 1e6:.1f} MB DRAM per launch (ncu, cold, serialized); algorithmic "
             f"{alg / 1e6:.1f} MB per launch -> traffic/algorithmic {dram / alg:.2f}"]
    for nm, vs in sorted(by.items()):
        m = len(vs)
        lines.append(f"   {nm:38s} launches {m:3d}  us/launch "
                     f"{sum(v['gpu__time_duration.sum'] for v in vs) / m / 1e3:9.1f}  dram MB/launch "
                     f"{sum(dram_of(v) for v in vs) / m / 1e6:9.1f}  Minst/launch "
                     f"{sum(v.get('smsp__inst_executed.sum', 0) for v in vs) / m / 1e6:8.1f}")
    print("\n".join(lines))
    with open(os.path.join(ROOT, "profiles", "r02", f"launches_k4_final_{cfg}.txt"), "w") as f:
        f.write("\n".join(lines) + "\n")
with open(os.path.join(ROOT, "profiles", "k4_traffic.json"), "w") as f:
    json.dump(out, f, indent=1)
