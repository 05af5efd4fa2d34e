"""Print the per-op profile written by bench.py --profile-out (top N ops)."""
import json
import sys


def main():
    f = sys.argv[1]
    top = int(sys.argv[2]) if len(sys.argv) > 2 else 16
    rows = [json.loads(line) for line in open(f)]
    tot = sum(r["ms_total"] for r in rows)
    print(f"{f}: total {tot:.1f} ms over {len(rows)} ops")
    for r in rows[:top]:
        ms = r["ms_total"] / r["executions"]
        tf = r["flops"] / (ms / 1e3) / 1e12 if r["kind"] == 1 else 0.0
        gbs = r["bytes"] / (ms / 1e3) / 1e9
        print(f"  s{r['step']:03d} kind={r['kind']} m={r['m']} n={r['n']} k={r['k']} tc={r['tensor_cores']} "
              f"x{r['executions']} ms={ms:8.2f} share={100 * r['ms_total'] / tot:5.1f}% TF={tf:6.1f} GB/s={gbs:7.1f}")


if __name__ == "__main__":
    main()
