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
the required slice count with the cheapest extra cuts.  A device time
model (tensor-core rate vs HBM passes) then drives (a) an optimal bundling
of the sweep into small pre-contracted clusters (cluster_dp: no pass-through
cell costs a full HBM pass over a 32 GiB accumulator) and (b) an exchange
search over the cut bonds at fixed K.  The result is
annotated by our planner (plan_json) and, when oracle/_ref exists, by the
reference's own plan_from_json + annotate_plan (proj/src/plan.cpp:122-210,
481-552), which must agree on flops, peak and max rank.

    python scripts/bristlecone_plan.py --active 70 --orders col-snake --anneal-cuts 3000 --seeds 3 \
        --out configs/config4_bristlecone70_plan.json
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


# Device time model of one step (B200, measured r2): tensor-core GEMMs at
# ~480 TF/s Eq.(1), memory-bound steps at ~4 TB/s over the operand and
# result bytes (the m=2^28 x 16 x 16 and outer-product steps of a naive
# sweep run at 0.5-3.3 TB/s and dominated the first Bristlecone-70 plan).
RATE_FLOPS, RATE_BYTES = 4.8e14, 4.0e12


def step_time(m, n, k):
    flops = 8.0 * 2.0 ** (m + n + k)
    byts = 8.0 * (2.0 ** (m + k) + 2.0 ** (k + n) + 2.0 ** (m + n))
    return max(flops / RATE_FLOPS, byts / RATE_BYTES)


def evaluate(order, labels, cut, with_time=False):
    """Chain `order` onto one accumulator: (max rank, Eq.(1) flops, ranks[, modelled seconds])."""
    front = set()
    flops, mx, ranks, secs = 0, 0, [], 0.0
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
        if with_time:
            secs += step_time(m, n, k)
        front = front ^ s
        ranks.append(len(front))
        mx = max(mx, len(front))
    if with_time:
        return mx, flops, ranks, secs
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


def anneal(order, labels, cut, budget, iters, seed):
    """Local search at a FIXED number of cut bonds (the slice count K): swap
    nearby cells of the order and exchange one cut bond for another,
    keeping max rank <= budget, minimising the modelled device time."""
    import math
    import random
    rng = random.Random(seed)
    all_labels = sorted({x for q in order for x in labels[q]})
    cur_o, cur_c = list(order), set(cut)
    mx, fl, _, t = evaluate(cur_o, labels, cur_c, True)
    assert mx <= budget
    cur_t = best_t = t
    best = (list(cur_o), set(cur_c))
    temp = 0.05 * t
    for it in range(iters):
        o, c = list(cur_o), set(cur_c)
        if rng.random() < 0.6:
            i = rng.randrange(len(o) - 1)
            j = min(len(o) - 1, i + rng.randint(1, 6))
            o[i], o[j] = o[j], o[i]
        else:
            c.remove(rng.choice(sorted(c)))
            c.add(rng.choice([x for x in all_labels if x not in c]))
        mx, fl, _, t = evaluate(o, labels, c, True)
        if mx > budget:
            continue
        if t < cur_t or rng.random() < math.exp((cur_t - t) / temp):
            cur_o, cur_c, cur_t = o, c, t
            if t < best_t:
                best_t, best = t, (list(o), set(c))
        temp = max(1e-4 * best_t, temp * 0.9995)
    return best[0], best[1], best_t


def _labset(q, labels, cut):
    return frozenset(x for x in labels[q] if x not in cut)


def cluster_dp(order, labels, cut, budget, jmax=4):
    """Optimal bundling of a fixed sweep order: the accumulator absorbs the
    order in consecutive clusters of up to jmax cells, each cluster first
    contracted on its own (a small chain).  A pass-through cell at the rank
    budget (one shared and one new edge: m = 2^28, n = k = 16, a pure HBM
    pass over a 32 GiB tensor) merged with its neighbour costs one pass
    instead of two; a cell that shares no uncut bond with the accumulator
    stops being an outer product.  Returns (clusters, modelled seconds, max rank)."""
    n = len(order)
    sets = [_labset(q, labels, cut) for q in order]
    fronts = [frozenset()]
    for s_ in sets:
        fronts.append(fronts[-1] ^ s_)
    INF = float("inf")
    best = [(INF, None)] * (n + 1)

    def chain(cells):  # contract cells left to right; (labels, seconds, max rank) or None
        acc, secs, mx = sets[cells[0]], 0.0, len(sets[cells[0]])
        for c in cells[1:]:
            sh = acc & sets[c]
            secs += step_time(len(acc) - len(sh), len(sets[c]) - len(sh), len(sh))
            acc = acc ^ sets[c]
            mx = max(mx, len(acc))
        return (acc, secs, mx) if mx <= budget else None

    for j in range(1, jmax + 1):  # the first cluster is the initial accumulator
        if j <= n:
            r = chain(list(range(j)))
            if r is not None and len(fronts[j]) <= budget:
                best[j] = (r[1], (0, j))
    for i in range(1, n):
        if best[i][0] == INF:
            continue
        for j in range(1, jmax + 1):
            if i + j > n or len(fronts[i + j]) > budget:
                continue
            r = chain(list(range(i, i + j)))
            if r is None:
                continue
            cl, secs, _ = r
            f = fronts[i]
            sh = f & cl
            t = best[i][0] + secs + step_time(len(f) - len(sh), len(cl) - len(sh), len(sh))
            if t < best[i + j][0]:
                best[i + j] = (t, (i, j))
    if best[n][0] == INF:
        return [], INF, max(len(f) for f in fronts)
    clusters, i = [], n
    while i > 0:
        a, j = best[i][1]
        clusters.append(order[a:a + j])
        i = a
    clusters.reverse()
    mx = max(len(f) for f in fronts)
    return clusters, best[n][0], mx


def anneal_cuts(order, labels, cut, budget, iters, seed):
    """Exchange cut bonds (count fixed: K stays 2^|cut|) to minimise the
    clustered plan's modelled time (cluster_dp); infeasible sets rejected."""
    import math
    import random
    rng = random.Random(seed)
    all_labels = sorted({x for q in order for x in labels[q]})
    cur = set(cut)
    cur_t = cluster_dp(order, labels, cur, budget)[1]
    best_t, best = cur_t, set(cur)
    temp = 0.05 * cur_t
    for _ in range(iters):
        c = set(cur)
        c.remove(rng.choice(sorted(c)))
        c.add(rng.choice([x for x in all_labels if x not in c]))
        t = cluster_dp(order, labels, c, budget)[1]
        if t == float("inf"):
            continue
        if t < cur_t or rng.random() < math.exp((cur_t - t) / temp):
            cur, cur_t = c, t
            if t < best_t:
                best_t, best = t, set(c)
        temp = max(1e-4 * best_t, temp * 0.998)
    return best, best_t


def build_plan(text, order, idle, cut, clusters=None):
    """Plan JSON draft: idle scalars chained first (into the first active
    cell), then the sweep, cluster by cluster (each cluster chained on its
    own, then absorbed by the accumulator)."""
    clusters = clusters or [[q] for q in order]
    steps = []

    def name_of(i):
        return f"s{i:03d}"

    acc = f"n_{idle[0]:03d}" if idle else None
    for q in list(idle[1:]) + [clusters[0][0]]:
        if acc is None:
            acc = f"n_{q:03d}"
            continue
        steps.append([acc, f"n_{q:03d}"])
        acc = name_of(len(steps) - 1)
    for q in clusters[0][1:]:
        steps.append([acc, f"n_{q:03d}"])
        acc = name_of(len(steps) - 1)
    for cl in clusters[1:]:
        part = f"n_{cl[0]:03d}"
        for q in cl[1:]:
            steps.append([part, f"n_{q:03d}"])
            part = name_of(len(steps) - 1)
        steps.append([acc, part])
        acc = name_of(len(steps) - 1)
    return {"version": 1, "open_qubits": [], "cut": {"labels": sorted(cut), "group": 1}, "order": steps}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--active", type=int, default=70)
    ap.add_argument("--budget", type=int, default=32)
    ap.add_argument("--min-bonds", type=int, default=0, help="at least this many cut bonds (K >= 2^min_bonds)")
    ap.add_argument("--orders", default="", help="comma list of sweep names (default: all)")
    ap.add_argument("--anneal", type=int, default=0, help="local-search iterations at the found cut count")
    ap.add_argument("--seeds", type=int, default=1)
    ap.add_argument("--anneal-cuts", type=int, default=0,
                    help="cut-exchange iterations against the clustered time model (K fixed)")
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
    order = orders[name]
    print(f"best: {name}: K = 2^{ncut}, max rank {mx}, {fl:.4e} flop/slice, "
          f"model {evaluate(order, labels, cut, True)[3] * 1e3:.1f} ms")
    if args.anneal:
        best = None
        for seed in range(args.seeds):
            for nm, o0 in orders.items():
                c0, m0, _ = greedy_cut(o0, labels, args.budget, min_bonds)
                if len(c0) != ncut:
                    continue
                o, c, t = anneal(o0, labels, c0, args.budget, args.anneal, seed)
                print(f"  anneal {nm} seed {seed}: model {t * 1e3:.1f} ms", flush=True)
                if best is None or t < best[2]:
                    best = (o, c, t)
        order, cut = best[0], best[1]
        mx, fl, _, t = evaluate(order, labels, cut, True)
        print(f"annealed: K = 2^{len(cut)}, max rank {mx}, {fl:.4e} flop/slice, model {t * 1e3:.1f} ms")
    if args.anneal_cuts:
        best = None
        for seed in range(args.seeds):
            c, t = anneal_cuts(order, labels, cut, args.budget, args.anneal_cuts, seed)
            print(f"  cut exchange seed {seed}: model {t * 1e3:.1f} ms", flush=True)
            if best is None or t < best[1]:
                best = (c, t)
        cut = best[0]
    clusters, t_dp, _ = cluster_dp(order, labels, cut, args.budget)
    print(f"clustered: {sum(len(c) > 1 for c in clusters)} multi-cell clusters, model {t_dp * 1e3:.1f} ms")
    if args.out:
        draft = build_plan(text, order, idle, cut, clusters)
        plan = Q.plan_json(text, [], Q.PLAN_JSON, json.dumps(draft))
        pj = json.loads(plan)
        print("annotated:", pj["slices"], "slices,", pj["per_slice"])
        with open(args.out, "w") as f:
            f.write(plan)


if __name__ == "__main__":
    main()
