"""Per-op profile (bench.py --profile-out) grouped by GEMM class (k, n): time share, Eq.1 TF/s, GB/s."""
import collections
import json
import sys

for f in sys.argv[1:]:
    rows = [json.loads(line) for line in open(f)]
    tot = sum(r["ms_total"] for r in rows)
    g = collections.defaultdict(lambda: [0, 0.0, 0, 0.0])
    for r in rows:
        key = ("gemm", r["k"], r["n"]) if r["kind"] == 1 else (("permute" if r["kind"] == 0 else "other"), 0, 0)
        g[key][0] += r["executions"]
        g[key][1] += r["ms_total"]
        g[key][2] += r["flops"] * r["executions"]
        g[key][3] += r["bytes"] * r["executions"]
    print(f, "total %.1f ms" % tot)
    for k, v in sorted(g.items(), key=lambda kv: -kv[1][1])[:8]:
        print("   %-8s k=%-6d n=%-5d ops %3d  ms %7.1f  share %5.1f%%  TF %4.0f  GB/s %5.0f" %
              (k[0], k[1], k[2], v[0], v[1], 100 * v[1] / tot, v[2] / v[1] / 1e9, v[3] / v[1] / 1e6))
