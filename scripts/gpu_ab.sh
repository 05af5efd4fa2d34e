# A/B of env settings on configs 2 and 4 (per-op profile totals), alternating, RUNS times.
# VARS="QSG_TC_PF=0 QSG_TC_PF=4" RUNS=2
mkdir -p gpurun_out
for r in $(seq 1 ${RUNS:-2}); do
  for v in $VARS; do
    tag=$(echo $v | tr '=' '_')
    env $v python bench.py --config 4 --steps 1 --warmup 1 --no-cpu-baseline --profile-out gpurun_out/ab_c4_${tag}_$r.jsonl > /dev/null 2>&1
    env $v python bench.py --steps 1 --warmup 2 --no-cpu-baseline --profile-out gpurun_out/ab_c2_${tag}_$r.jsonl > /dev/null 2>&1
    python - <<PY
import json
for c in ("c4", "c2"):
    rows = [json.loads(l) for l in open("gpurun_out/ab_%s_${tag}_$r.jsonl" % c)]
    tot = sum(x["ms_total"] for x in rows)
    n256 = [x for x in rows if x["kind"] == 1 and x["n"] == 256 and x["k"] == 256]
    top = max(rows, key=lambda x: x["ms_total"])
    print("$v run $r", c, "total %.1f  top %.1f  n256 avg %.2f" % (tot, top["ms_total"] / top["executions"],
          sum(x["ms_total"] / x["executions"] for x in n256) / max(1, len(n256))))
PY
  done
done
