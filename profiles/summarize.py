"""Summarise a round's raw ncu output into the tracked text files.

python profiles/summarize.py launches <launches.csv> <windows> <alg_bytes_per_step> <out.txt>
python profiles/summarize.py full <report.ncu-rep> <out.txt>
"""
import collections
import csv
import subprocess
import sys


def launches(path, windows, alg_bytes, out):
    rows = [r for r in csv.reader(open(path)) if len(r) > 10]
    hdr = [r for r in rows if r[0] == "ID"][0]
    ix = {n: i for i, n in enumerate(hdr)}
    agg = collections.defaultdict(lambda: collections.defaultdict(float))
    seen = collections.defaultdict(set)
    for r in rows:
        if not r[0].isdigit():
            continue
        name = r[ix["Kernel Name"]].split("(")[0].replace("void ", "")
        agg[name][r[ix["Metric Name"]]] += float(r[ix["Metric Value"]].replace(",", ""))
        seen[name].add(r[0])
    lines = ["kernel                                                      launches  us/launch"
             "   dram_MB/launch  Minst/launch"]
    k4_t = k4_b = k4_n = 0.0
    for name, a in sorted(agg.items(), key=lambda x: -x[1]["gpu__time_duration.sum"]):
        n = len(seen[name])
        dram = (a.get("dram__bytes_read.sum", 0) + a.get("dram__bytes_write.sum", 0)) / n
        lines.append(f"{name[:58]:58s} {n:9d} {a['gpu__time_duration.sum'] / n / 1e3:10.1f}"
                     f" {dram / 1e6:16.1f} {a.get('smsp__inst_executed.sum', 0) / n / 1e6:13.1f}")
        if "gate_eval" in name:
            k4_t += a["gpu__time_duration.sum"]
            k4_b += dram * n
            k4_n += n
    per_launch = k4_b / k4_n
    step_launches = 80
    lines.append("")
    lines.append(f"K4 gate_eval: mean {k4_t / k4_n / 1e3:.1f} us and {per_launch / 1e6:.1f} MB DRAM per "
                 f"launch; x{step_launches} launches per step = {per_launch * step_launches / 1e9:.2f} GB "
                 f"vs algorithmic {alg_bytes / 1e9:.2f} GB per step "
                 f"({per_launch * step_launches / alg_bytes:.2f}x)")
    open(out, "w").write("\n".join(lines) + "\n")
    print("\n".join(lines))
    return per_launch


def full(rep, out):
    raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True,
                         text=True).stdout
    r = list(csv.reader(raw.splitlines()))
    d = dict(zip(r[0], r[2]))
    keys = ["Kernel Name", "gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
            "launch__grid_size", "launch__block_size", "launch__registers_per_thread",
            "launch__occupancy_limit_registers", "launch__occupancy_limit_shared_mem",
            "sm__warps_active.avg.pct_of_peak_sustained_active", "smsp__inst_executed.sum",
            "smsp__issue_active.avg.pct_of_peak_sustained_active",
            "smsp__thread_inst_executed_per_inst_executed.ratio",
            "sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active",
            "l1tex__data_pipe_lsu_wavefronts.avg.pct_of_peak_sustained_elapsed",
            "lts__t_sector_hit_rate.pct", "l1tex__t_sector_hit_rate.pct",
            "sm__cycles_active.avg", "gpc__cycles_elapsed.max"]
    lines = [f"{k:70s} {d.get(k)}" for k in keys]
    st = {k: float(v) for k, v in d.items()
          if k.startswith("smsp__average_warps_issue_stalled_") and k.endswith("_per_issue_active.ratio")}
    lines.append("")
    lines.append("stall reasons (warps stalled per issued instruction):")
    for k, v in sorted(st.items(), key=lambda t: -t[1])[:10]:
        lines.append(f"  {k.replace('smsp__average_warps_issue_stalled_', '').replace('_per_issue_active.ratio', ''):24s} {v:.2f}")
    open(out, "w").write("\n".join(lines) + "\n")
    print("\n".join(lines))


if __name__ == "__main__":
    if sys.argv[1] == "launches":
        launches(sys.argv[2], int(sys.argv[3]), float(sys.argv[4]), sys.argv[5])
    else:
        full(sys.argv[2], sys.argv[3])
