"""CPU restatement of the reference's amplitude path, in numpy.

TEST INFRASTRUCTURE ONLY -- the checker for tests/, __graft_entry__.smoke()
and bench.py's cpu_baseline leg.  The product (paper_1905_00444_b200) never
imports this module.

Parity status: PINNED.  tests/test_oracle.py checks every function here
against golden vectors produced by the UNMODIFIED reference library
(oracle/_ref, built from /root/reference/proj/src by oracle/Makefile) and
committed under tests/golden/ by oracle/gen_golden.py.

Restated functions (reference file:line, relative to proj/):
  gate_matrix          src/circuit.cpp:25-46
  parse_circuit        src/circuit.cpp:128-193 (well-formed input only)
  evolve               src/oracle.cpp:22-66   (double state vector, q <-> bit n-1-q)
  fold_worldlines      src/network.cpp:58-149
  cut_digits/apply_cut src/plan.cpp:89-115
  execute_slice        src/engine.cpp:182-245 (here: complex128 tensordot)
  amplitude_batch      src/sampler.cpp:17-36, 111-120 (+ merge_bits :41-52)
  mix_seed             include/qsim/types.hpp:25-30
  select_slices        src/engine.cpp:285-298
  flop_count           include/qsim/contraction.hpp:46-56
"""
from __future__ import annotations

import json
import math

import numpy as np

M64 = (1 << 64) - 1


def mix_seed(seed: int, stream: int) -> int:
    z = (seed + 0x9E3779B97F4A7C15 * (stream + 1)) & M64
    z = ((z ^ (z >> 30)) * 0xBF58476D1CE4E5B9) & M64
    z = ((z ^ (z >> 27)) * 0x94D049BB133111EB) & M64
    return z ^ (z >> 31)


class MT19937_64:
    """std::mt19937_64 (the reference's RNG, src/circuit.cpp:250, src/sampler.cpp:155)."""

    def __init__(self, seed: int):
        self.mt = [0] * 312
        self.mt[0] = seed & M64
        for i in range(1, 312):
            self.mt[i] = (6364136223846793005 * (self.mt[i - 1] ^ (self.mt[i - 1] >> 62)) + i) & M64
        self.idx = 312

    def __call__(self) -> int:
        if self.idx >= 312:
            mt = self.mt
            for i in range(312):
                x = (mt[i] & 0xFFFFFFFF80000000) | (mt[(i + 1) % 312] & 0x7FFFFFFF)
                xa = x >> 1
                if x & 1:
                    xa ^= 0xB5026F5AA96619E9
                mt[i] = mt[(i + 156) % 312] ^ xa
            self.idx = 0
        y = self.mt[self.idx]
        self.idx += 1
        y ^= (y >> 29) & 0x5555555555555555
        y ^= (y << 17) & 0x71D67FFFEDA60000
        y ^= (y << 37) & 0xFFF7EEE000000000
        y ^= y >> 43
        return y & M64


def draw_x1(n: int, open_qubits, seed: int, index: int):
    """Random x1 for task `index`: mt19937_64(mix_seed(seed, index)), one bit per
    closed qubit from successive 64-bit words, LSB first (src/sampler.cpp:70-82)."""
    rng = MT19937_64(mix_seed(seed, index))
    x1, word, left = [-1] * n, 0, 0
    opn = set(open_qubits)
    for q in range(n):
        if q in opn:
            continue
        if left == 0:
            word, left = rng(), 64
        x1[q] = word & 1
        word >>= 1
        left -= 1
    return x1


def select_slices(num: int, den: int, num_slices: int, seed: int):
    if den != num_slices:
        raise ValueError("fraction denominator does not match the plan's slices")
    off = mix_seed(seed, 0x51CE) % num_slices
    return sorted((off + i) % num_slices for i in range(num))


def flop_count(v0: int, v1: int, v2: int) -> int:
    prod = v0 * v1 * v2
    r = math.isqrt(prod)
    if r * r != prod:
        raise ValueError("flop_count: volume product is not a perfect square")
    return 8 * r


def gate_matrix(name: str) -> np.ndarray:
    s = 1.0 / math.sqrt(2.0)
    if name == "h":
        return np.array([[s, s], [s, -s]], dtype=np.complex128)
    if name == "t":
        return np.array([[1, 0], [0, np.exp(1j * math.pi / 4)]], dtype=np.complex128)
    if name == "x_1_2":
        return 0.5 * np.array([[1 + 1j, 1 - 1j], [1 - 1j, 1 + 1j]], dtype=np.complex128)
    if name == "y_1_2":
        return 0.5 * np.array([[1 + 1j, -1 - 1j], [1 + 1j, 1 + 1j]], dtype=np.complex128)
    raise ValueError(name)


def parse_circuit(text: str):
    """(rows, cols, gates) with gates sorted (cycle, q0, q1); q1 = -1 for 1-qubit gates."""
    n, gr, gc, gates = None, 0, 0, []
    for raw in text.splitlines():
        line = raw.strip()
        if not line:
            continue
        if line.startswith("#"):
            parts = line[1:].split()
            if len(parts) == 2 and parts[0] == "grid" and "x" in parts[1]:
                gr, gc = (int(x) for x in parts[1].split("x"))
            continue
        tok = line.split()
        if n is None:
            n = int(tok[0])
            continue
        cyc, name, q0 = int(tok[0]), tok[1], int(tok[2])
        q1 = int(tok[3]) if name == "cz" else -1
        if name == "cz" and q0 > q1:
            q0, q1 = q1, q0
        gates.append((cyc, name, q0, q1))
    if gr and gc:
        rows, cols = gr, gc
    else:
        side = int(round(math.sqrt(n)))
        rows, cols = (side, side) if side * side == n else (1, n)
    gates.sort(key=lambda g: (g[0], g[2], g[3]))
    return rows, cols, gates


def evolve(text: str) -> np.ndarray:
    rows, cols, gates = parse_circuit(text)
    n = rows * cols
    psi = np.zeros(1 << n, dtype=np.complex128)
    psi[0] = 1.0
    psi = psi.reshape([2] * n)  # axis q <-> qubit q <-> bit n-1-q of the flat index
    for cyc, name, q0, q1 in gates:
        if name == "cz":
            idx = [slice(None)] * n
            idx[q0] = 1
            idx[q1] = 1
            psi[tuple(idx)] *= -1
        else:
            psi = np.moveaxis(np.tensordot(gate_matrix(name), psi, axes=([1], [q0])), 0, q0)
    return psi.reshape(-1)


def bitstring_index(bits: str) -> int:
    return int(bits, 2)


def bond_label(cycle, q0, q1):
    if q0 > q1:
        q0, q1 = q1, q0
    return f"b_{cycle:03d}_{q0:03d}_{q1:03d}"


def open_label(q):
    return f"o_{q:03d}"


def fold_worldlines(text: str, out_bits, in_bits=None):
    """List of (labels, complex64 ndarray) per qubit, fold layout (axis 0 = open label if any)."""
    rows, cols, gates = parse_circuit(text)
    n = rows * cols
    in_bits = in_bits or [0] * n
    nodes = []
    for q in range(n):
        nodes.append((["w"], np.array([1.0 if in_bits[q] == 0 else 0.0, 1.0 if in_bits[q] == 1 else 0.0],
                                      dtype=np.complex64)))
    for cyc, name, q0, q1 in gates:
        if name == "cz":
            b = bond_label(cyc, q0, q1)
            for q, phase in ((q0, True), (q1, False)):
                labels, t = nodes[q]
                flat = t.reshape(2, -1)
                out = np.zeros(flat.shape + (2,), dtype=np.complex64)
                if phase:
                    out[0, :, 0] = flat[0]
                    out[0, :, 1] = flat[0]
                    out[1, :, 0] = flat[1]
                    out[1, :, 1] = -flat[1]
                else:
                    out[0, :, 0] = flat[0]
                    out[1, :, 1] = flat[1]
                nodes[q] = (labels + [b], out.reshape(t.shape + (2,)))
        else:
            u = gate_matrix(name).astype(np.complex64)
            labels, t = nodes[q0]
            flat = t.reshape(2, -1)
            a, bb = flat[0].copy(), flat[1].copy()
            nodes[q0] = (labels, np.stack([u[0, 0] * a + u[0, 1] * bb, u[1, 0] * a + u[1, 1] * bb]).reshape(t.shape))
    out = []
    for q in range(n):
        labels, t = nodes[q]
        if out_bits[q] < 0:
            out.append(([open_label(q)] + labels[1:], t))
        else:
            out.append((labels[1:], t[out_bits[q]]))
    return out


def cut_fixed_count(cut_labels, group, extent=lambda l: 2):
    if group <= 1:
        return len(cut_labels)
    acc, i = 1, len(cut_labels)
    while i > 0 and acc < group:
        i -= 1
        acc *= extent(cut_labels[i])
    if acc != group:
        raise ValueError("cut group does not divide the trailing multi-index")
    return i


def cut_digits(cut_labels, group, slice_id):
    fixed = cut_fixed_count(cut_labels, group)
    total = 2 ** fixed
    if not 0 <= slice_id < total:
        raise IndexError("apply_cut: slice_id out of range")
    return [(slice_id >> (fixed - 1 - i)) & 1 for i in range(fixed)]


def apply_cut(nodes, cut_labels, group, slice_id):
    digits = cut_digits(cut_labels, group, slice_id)
    fixed = dict(zip(cut_labels[: len(digits)], digits))
    out = []
    for labels, t in nodes:
        idx = tuple(fixed.get(l, slice(None)) for l in labels)
        kept = [l for l in labels if l not in fixed]
        out.append((kept, np.asarray(t[idx])))
    return out


def execute_slice(nodes, order):
    """Contract node tensors following plan `order` (list of [lhs, rhs]) in complex128.

    Returns (labels sorted, tensor) of the final result (src/engine.cpp:182-245;
    intermediates in sorted label order as annotate_plan prescribes)."""
    live = {f"n_{q:03d}": (labels, t.astype(np.complex128)) for q, (labels, t) in enumerate(nodes)}
    for i, (lhs, rhs) in enumerate(order):
        (la, a), (lb, b) = live.pop(lhs), live.pop(rhs)
        shared = [l for l in la if l in lb]
        c = np.tensordot(a, b, axes=([la.index(l) for l in shared], [lb.index(l) for l in shared]))
        lc = [l for l in la if l not in shared] + [l for l in lb if l not in shared]
        perm = sorted(range(len(lc)), key=lambda j: lc[j])
        live[f"s{i:03d}"] = ([lc[j] for j in perm], np.transpose(c, perm) if lc else c)
    if len(live) != 1:
        raise ValueError("plan left multiple tensors")
    return next(iter(live.values()))


def merge_bits(x1, open_sorted, idx):
    s = ["1" if b == 1 else "0" for b in x1]
    k = len(open_sorted)
    for r, q in enumerate(open_sorted):
        s[q] = str((idx >> (k - 1 - r)) & 1)
    return "".join(s)


def amplitude_batch(text: str, plan_text: str, x1, slice_ids):
    """(bitstrings, complex128 batch) summed over slice_ids in ascending order."""
    plan = json.loads(plan_text)
    cut = plan.get("cut", {"labels": [], "group": 1})
    nodes = fold_worldlines(text, x1)
    open_sorted = sorted(q for q, b in enumerate(x1) if b < 0)
    acc = np.zeros(1 << len(open_sorted), dtype=np.complex128)
    for sid in slice_ids:
        labels, t = execute_slice(apply_cut(nodes, cut["labels"], cut.get("group", 1), sid), plan["order"])
        acc += np.asarray(t).reshape(-1)
    bits = [merge_bits(x1, open_sorted, i) for i in range(len(acc))]
    return bits, acc
