"""Authors the Bristlecone-70 / -60 (1+32+1) contraction plans (configs 3/4).

The reference has no Bristlecone geometry; the circuit is the
masked 11x12 embedding (generate_rqc_masked + bristlecone_mask: idle cells
carry only the outer H layers and fold to scalars).  Its plan must keep
every intermediate at rank <= 32 (32 GiB complex64) using cut bonds, with
K >= 2^12 (BC-70) / 2^10 (BC-60) slices of which a fixed subset runs.

Search: sweep orders of the active cells (columns / rows / diagonals, both
directions, snake or not) chained onto one accumulator after all idle
scalars are folded into the first active node; bonds are then cut greedily
(the bond whose removal most reduces the over-budget fronts, ties by Eq.(1)
flops) until max rank <= the budget, then the remaining K is padded up to
the required slice count with the cheapest extra cuts.  The result is
annotated by our planner (plan_json) and, when oracle/_ref exists, by the
reference's own plan_from_json + annotate_plan (proj/src/plan.cpp:122-210,
481-552), which must agree on flops, peak and max rank.

    python scripts/bristlecone_plan.py --active 70 --out configs/config4_bristlecone70_plan.json
"""
from __future__ import annotations

import argparse
import json
import os
import sys
from collections import defaultdict

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

ROWS, COLS = 11, 12


def network(text: str):
    """(labels per qubit, active qubits) from the circuit's CZ gates: bond
    b_{cycle}_{q0}_{q1} (src/network.cpp:32-49) on both endpoints."""
    labels = defaultdict(list)
    for ln in text.splitlines()[1:]:
        f = ln.split()
        if len(f) == 4 and f[1] == "cz":
            c, a, b = int(f[0]), int(f[2]), int(f[3])
            a, b = min(a, b), max(a, b)
            lab = f"b_{c:03d}_{a:03d}_{b:03d}"
            labels[a].append(lab)
            labels[b].append(lab)
    return {q: sorted(v) for q, v in labels.items()}


def evaluate(order, labels, cut):
    """Chain `order` onto one accumulator: (max rank, Eq.(1) flops, ranks)."""
    front = set()
    flops, mx, ranks = 0, 0, []
    for i, q in enumerate(order):
        lab = [x for x in labels[q] if x not in cut]
        if i == 0:
            front = set(lab)
            ranks.append(len(front))
            continue
        s = set(lab)
        shared = front & s
        m = len(front) - len(shared)
        n = len(s) - len(shared)
        k = len(shared)
        flops += 8 * (1 << (m + n + k))
        front = front ^ s
        ranks.append(len(front))
        mx = max(mx, len(front))
    return mx, flops, ranks


def cell(q):
    return divmod(q, COLS)


def sweep_orders(active):
    """Candidate sweeps: columns / rows / anti-diagonals / diagonals, each in
    both directions, plain or snake within a line."""
    cells = {q: cell(q) for q in active}
    out = {}
    keys = {
        "col": lambda rc: (rc[1], rc[0]),
        "row": lambda rc: (rc[0], rc[1]),
        "diag": lambda rc: (rc[0] + rc[1], rc[0]),
        "adiag": lambda rc: (rc[0] - rc[1], rc[0]),
    }
    for name, key in keys.items():
        for rev in (False, True):
            base = sorted(active, key=lambda q: key(cells[q]), reverse=rev)
            out[f"{name}{'-rev' if rev else ''}"] = base
            lines = defaultdict(list)
            for q in base:
                lines[key(cells[q])[0]].append(q)
            snake = []
            for i, ln in enumerate(lines.values()):
                snake.extend(ln if i % 2 == 0 else ln[::-1])
            out[f"{name}{'-rev' if rev else ''}-snake"] = snake
    return out


def greedy_cut(order, labels, budget, min_bonds):
    cut = set()
    all_labels = sorted({x for q in order for x in labels[q]})
    while True:
        mx, fl, ranks = evaluate(order, labels, cut)
        if mx <= budget and len(cut) >= min_bonds:
            return cut, mx, fl
        best = None
        for lab in all_labels:
            if lab in cut:
                continue
            c2 = cut | {lab}
            m2, f2, r2 = evaluate(order, labels, c2)
            excess = sum(max(0, r - budget) for r in r2)
            key = (excess, m2, f2) if mx > budget else (f2,)
            if best is None or key < best[0]:
                best = (key, lab)
        cut.add(best[1])


def build_plan(text, order, idle, cut):
    """Plan JSON draft: idle scalars chained first, then the sweep."""
    seq = list(idle) + list(order)
    steps, acc = [], f"n_{seq[0]:03d}"
    for i, q in enumerate(seq[1:]):
        steps.append([acc, f"n_{q:03d}"])
        acc = f"s{i:03d}"
    return {"version": 1, "open_qubits": [], "cut": {"labels": sorted(cut), "group": 1}, "order": steps}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--active", type=int, default=70)
    ap.add_argument("--budget", type=int, default=32)
    ap.add_argument("--min-bonds", type=int, default=0, help="at least this many cut bonds (K >= 2^min_bonds)")
    ap.add_argument("--orders", default="", help="comma list of sweep names (default: all)")
    ap.add_argument("--out", default="")
    args = ap.parse_args()
    import paper_1905_00444_b200 as Q
    mask = Q.bristlecone_mask(args.active)
    text = Q.generate_rqc_masked(ROWS, COLS, mask, 32, 0)
    labels = network(text)
    active = [q for q in range(ROWS * COLS) if mask[q] == "1"]
    idle = [q for q in range(ROWS * COLS) if mask[q] != "1"]
    min_bonds = args.min_bonds or (12 if args.active == 70 else 10)
    orders = sweep_orders(active)
    if args.orders:
        orders = {k: v for k, v in orders.items() if k in args.orders.split(",")}
    results = []
    for name, order in orders.items():
        mx0, fl0, _ = evaluate(order, labels, set())
        cut, mx, fl = greedy_cut(order, labels, args.budget, min_bonds)
        results.append((len(cut), fl, name, cut, mx))
        print(f"{name:18s} uncut max rank {mx0:3d}  -> cut {len(cut):2d} bonds, max rank {mx}, "
              f"{fl:.3e} flop/slice", flush=True)
    results.sort(key=lambda r: (r[0], r[1]))
    ncut, fl, name, cut, mx = results[0]
    print(f"best: {name}: K = 2^{ncut}, max rank {mx}, {fl:.4e} flop/slice")
    if args.out:
        draft = build_plan(text, orders[name], idle, cut)
        plan = Q.plan_json(text, [], Q.PLAN_JSON, json.dumps(draft))
        pj = json.loads(plan)
        print("annotated:", pj["slices"], "slices,", pj["per_slice"])
        with open(args.out, "w") as f:
            f.write(plan)


if __name__ == "__main__":
    main()
