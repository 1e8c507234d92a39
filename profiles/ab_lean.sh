# A/B of lean-kernel build variants (paper_2203_06117_b200/libglsim_cuda_<v>.so),
# interleaved rounds; one JSON line per run into gpurun_out/ab_lean.jsonl
mkdir -p gpurun_out
: > gpurun_out/ab_lean.jsonl
for r in 1 2 3; do
  for v in $VARIANTS; do
    for c in "C3 --windows 8192" "C2"; do
      line=$(GLSIM_LIB=libglsim_cuda_$v.so timeout 300 python bench.py --config $c --steps 5 --warmup 3 --no-cpu-baseline --e2e-steps 1 2>/dev/null | grep '^{')
      echo "{\"variant\": \"$v\", \"round\": $r, \"run\": $line}" >> gpurun_out/ab_lean.jsonl
    done
  done
done
python - <<'PY'
import json, collections, statistics
d = collections.defaultdict(list)
for l in open("gpurun_out/ab_lean.jsonl"):
    try:
        x = json.loads(l)
    except Exception:
        continue
    r = x["run"]
    d[(x["variant"], r["config"]["workload"][:2])].append((r["roofline"]["k4_ms_per_step"], r["ms_per_step"]))
for k, v in sorted(d.items()):
    k4 = [a for a, _ in v]
    st = [b for _, b in v]
    print(k, "k4 ms", [round(a, 2) for a in k4], "median", round(statistics.median(k4), 2),
          "| step ms median", round(statistics.median(st), 2))
PY
