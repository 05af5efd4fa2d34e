"""Pick the longest launch of a kernel from an ncu launch-list CSV and print
its index among launches of that kernel (the value for `ncu -k regex:NAME -s`).
Also prints a per-kernel summary of one batch when --summary is given."""
import csv
import sys
from collections import defaultdict


def rows(path):
    with open(path) as f:
        lines = [ln for ln in f if ln.startswith('"')]
    return list(csv.DictReader(lines))


def main():
    path, name = sys.argv[1], sys.argv[2]
    rs = [r for r in rows(path) if r["Metric Name"] == "gpu__time_duration.sum"]
    hits = [(i, float(r["Metric Value"])) for i, r in enumerate(x for x in rs if name in x["Kernel Name"])]
    rng = [float(a.split("=")[1]) * 1e6 for a in sys.argv if a.startswith("--ms=")]  # --ms=LO --ms=HI (ms)
    variant = [a.split("=", 1)[1] for a in sys.argv if a.startswith("--variant=")]
    if variant:  # index among all `name` launches (ncu -k regex:name -s IDX), longest of one template variant
        names = [x["Kernel Name"] for x in rs if name in x["Kernel Name"]]
        cand = [(i, v) for i, v in hits if variant[0] in names[i]]
        if len(rng) == 2:  # --ms window too: the first launch of the variant inside it (after --skip=N others)
            skip = int(next((a.split("=")[1] for a in sys.argv if a.startswith("--skip=")), "0"))
            print(sorted(i for i, v in cand if rng[0] <= v <= rng[1])[skip])
        else:
            top = max(v for _, v in cand)
            print(min(i for i, v in cand if v >= 0.95 * top))
    elif len(rng) == 2:
        print(min(i for i, v in hits if rng[0] <= v <= rng[1]))  # first launch in the duration window
    else:
        top = max(v for _, v in hits)
        print(min(i for i, v in hits if v >= 0.95 * top))  # first launch of the longest step
    if "--summary" in sys.argv:
        tot = defaultdict(float)
        for r in rs:
            tot[r["Kernel Name"].split("(")[0].replace("void ", "").replace("unnamed>::", "")] += float(r["Metric Value"])
        s = sum(tot.values())
        for k, v in sorted(tot.items(), key=lambda t: -t[1]):
            print(f"{k:50s} {v / 1e6:10.2f} ms {100 * v / s:6.2f}%", file=sys.stderr)


if __name__ == "__main__":
    main()
