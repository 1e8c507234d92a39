# A/B of build variants on the full C3 bench (100k windows, all chunks), 2 interleaved rounds
mkdir -p gpurun_out
: > gpurun_out/ab_full.jsonl
for r in 1 2; do
  for v in $VARIANTS; do
    line=$(GLSIM_LIB=libglsim_cuda_$v.so timeout 600 python bench.py --steps 4 --warmup 3 --no-cpu-baseline --e2e-steps 1 2>/dev/null | grep '^{')
    echo "{\"variant\": \"$v\", \"round\": $r, \"run\": $line}" >> gpurun_out/ab_full.jsonl
  done
done
python - <<'PY'
import json, collections, statistics
d = collections.defaultdict(list)
for l in open("gpurun_out/ab_full.jsonl"):
    try:
        x = json.loads(l)
    except Exception:
        continue
    r = x["run"]
    d[x["variant"]].append((r["ms_per_step"], r["roofline"]["k4_ms_per_step"], r["activity"].get("chunks_per_step")))
for k, v in sorted(d.items()):
    print(k, "step ms", [round(a, 1) for a, _, _ in v], "k4 ms", [round(b, 1) for _, b, _ in v], "chunks", v[0][2])
PY
