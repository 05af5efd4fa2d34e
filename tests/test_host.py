"""Host model of libqsg.so (no GPU needed) is bit-exact with the reference:
generator text, canonical form and errors, plans and annotations, fold,
slice selection and x1 draws.  Mirrors proj/tests/test_circuit.cpp and the
SPEC acceptance #3 / #9 checks."""
import hashlib
import json
import os

import numpy as np
import pytest

import paper_1905_00444_b200 as Q
import qsim_oracle as O
from conftest import GOLDEN, ROOT


def sha(b):
    return hashlib.sha256(b).hexdigest()


def test_generate_rqc_bit_exact(golden):
    for c in golden["circuits"]:
        text = Q.generate_rqc(c["rows"], c["cols"], c["m"], c["seed"])
        assert sha(text.encode()) == c["sha256"], c
        if c["text"]:
            assert text == c["text"]
            assert Q.canonical_circuit(text) == text  # byte-identical round trip


def test_generate_determinism_and_m0():
    assert Q.generate_rqc(4, 4, 8, 987) == Q.generate_rqc(4, 4, 8, 987)
    assert Q.generate_rqc(4, 4, 8, 987) != Q.generate_rqc(4, 4, 8, 988)
    text = Q.generate_rqc(2, 2, 0, 12345)
    assert text.splitlines()[1:] == ["0 h 0", "0 h 1", "0 h 2", "0 h 3", "1 h 0", "1 h 1", "1 h 2", "1 h 3"]


def test_parse_errors_carry_line_numbers():
    # proj/tests/test_circuit.cpp:55-93
    with pytest.raises(Q.CircuitError) as e:
        Q.canonical_circuit("2\n0 h 0\nnonsense\n")
    assert e.value.line == 3
    with pytest.raises(Q.CircuitError) as e:
        Q.canonical_circuit("2\n0 h 0\n0 h 7\n")
    assert e.value.line == 3
    with pytest.raises(Q.CircuitError):
        Q.canonical_circuit("2\n0 q 0\n")
    with pytest.raises(Q.CircuitError, match="two gates on qubit"):
        Q.canonical_circuit("2\n0 h 0\n0 h 0\n")
    with pytest.raises(Q.CircuitError, match="non-adjacent"):
        Q.canonical_circuit("4\n0 h 0\n0 h 1\n0 h 2\n0 h 3\n1 cz 0 3\n2 h 0\n2 h 1\n2 h 2\n2 h 3\n")
    with pytest.raises(Q.CircuitError, match="every qubit"):
        Q.canonical_circuit("2\n0 h 0\n")
    with pytest.raises(Q.CircuitError, match="Hadamard"):
        Q.canonical_circuit("2\n0 h 0\n0 h 1\n1 t 0\n")


def test_grid_comment_and_inference():
    text = Q.generate_rqc(4, 5, 6, 3)
    assert "# grid 4x5" in text
    info = Q.circuit_info(text)
    assert (info["rows"], info["cols"]) == (4, 5)
    assert Q.circuit_info("4\n0 h 0\n0 h 1\n0 h 2\n0 h 3\n") == {"rows": 2, "cols": 2, "qubits": 4, "cycles": 1}
    assert Q.canonical_circuit("2\n0 h 1\n0 h 0\n1 cz 0 1\n2 h 1\n2 h 0\n") == "2\n0 h 0\n0 h 1\n1 cz 0 1\n2 h 0\n2 h 1\n"


def test_config_plans_match_reference_annotations(golden):
    for name, g in golden["plans"].items():
        r, c, m, s = g["circuit"]
        text = Q.generate_rqc(r, c, m, s)
        plan_text = open(os.path.join(ROOT, "configs", f"{name}_plan.json")).read()
        pj = json.loads(Q.plan_json(text, kind=Q.PLAN_JSON, plan_text=plan_text))
        assert pj["per_slice"] == g["per_slice"], name
        assert pj["slices"] == g["slices"]
        assert [st["flops"] for st in pj["steps"]] == g["step_flops"]
        assert sha(json.dumps([st["out_labels"] for st in pj["steps"]]).encode()) == g["out_labels_sha"]
        # SPEC #3: per-slice flops are exactly the sum of Eq.(1) over steps
        assert sum(g["step_flops"]) == g["per_slice"]["flops"]


def test_reference_7x7_plan_structure(golden):
    # SPEC acceptance #9: 1024 slices, max rank <= 30
    text = Q.generate_rqc(7, 7, 40, 0)
    pj = json.loads(Q.plan_json(text, kind=Q.PLAN_REF7X7))
    assert pj["slices"] == 1024
    assert pj["per_slice"]["max_rank"] <= 30
    assert pj["per_slice"] == golden["plans"]["config5"]["per_slice"]


def test_greedy_planner_matches_reference():
    meta = json.load(open(os.path.join(GOLDEN, "amplitudes.json")))
    for case in meta["cases"]:
        text = Q.generate_rqc(case["rows"], case["cols"], case["m"], case["seed"])
        budget = 0 if meta["cases"].index(case) % 3 else 4096
        mine = json.loads(Q.plan_json(text, case["open"], Q.PLAN_GREEDY, "", budget))
        ref = json.loads(case["plan"])
        assert mine["order"] == ref["order"]
        assert mine["cut"] == ref["cut"]
        assert mine["per_slice"] == ref["per_slice"]


def test_greedy_planner_rejects_overflow():
    """the reference greedy wraps int64 volumes / uint64
    flops on large grids (7x7 (1+32+1): 'rank 90, 1.6e14 flop').  Here the
    candidate ordering stays defined past 2^60 and annotation refuses plans
    whose sizes overflow, with the reference's error type for volume overflow."""
    text = Q.generate_rqc(7, 7, 32, 0)
    with pytest.raises(Q.LengthError, match="overflow"):
        Q.plan_json(text, [0, 1], Q.PLAN_GREEDY)


def test_fold_bit_exact(golden):
    for f in golden["folds"]:
        r, c, m, s = f["circuit"]
        text = Q.generate_rqc(r, c, m, s)
        h = hashlib.sha256()
        for labels, dims, ls, data in Q.fold_worldlines(text, f["x1"]):
            h.update(("|".join(labels) + ";" + ",".join(map(str, dims))).encode())
            h.update(np.ascontiguousarray(data).tobytes())
        assert h.hexdigest() == f["sha256"]


def test_fold_matches_oracle_restatement():
    text = Q.generate_rqc(4, 5, 8, 2)
    x1 = [0, 1] * 10
    x1[3] = x1[7] = -1
    mine = Q.fold_worldlines(text, x1)
    ora = O.fold_worldlines(text, x1)
    for (l1, d1, ls, t1), (l2, t2) in zip(mine, ora):
        assert l1 == l2
        assert np.allclose(t1, t2, atol=1e-6)


def test_cut_slices_and_errors():
    meta = json.load(open(os.path.join(GOLDEN, "amplitudes.json")))
    cut_case = next(c for c in meta["cases"] if c["slices"] > 1)
    text = Q.generate_rqc(cut_case["rows"], cut_case["cols"], cut_case["m"], cut_case["seed"])
    with pytest.raises(Q.OutOfRange):
        Q.fold_worldlines(text, cut_case["x1"], cut_case["plan"], cut_case["slices"])


def test_selection_and_seeds(golden):
    for s, t, want in golden["mix_seed"]:
        assert Q.mix_seed(s, t) == want
    for k, K, seed, ids in golden["select_slices"]:
        assert Q.select_slices(k, K, K, seed) == ids
    with pytest.raises(Q.InvalidArgument, match="does not match the plan"):
        Q.select_slices(1, 3, 4, 0)


def test_draw_x1_matches_oracle():
    for i in range(10):
        opn = [32, 33, 34, 39, 40, 41, 45, 46, 47, 48]
        assert Q.draw_x1(49, opn, 5, i) == O.draw_x1(49, opn, 5, i)


def test_flop_count():
    assert Q.flop_count(4, 4, 4) == 64
    assert Q.flop_count(2**30, 2**30, 2**30) == 8 << 45
    with pytest.raises(Q.InvalidArgument):
        Q.flop_count(2, 3, 5)


def test_masked_generator_and_bristlecone_masks():
    """masked-grid RQCs.  All-ones mask = generate_rqc
    (bit-exact text); inactive cells carry only the two H layers; CZs only
    join active neighbours; the Bristlecone diamond masks have 72/70/60 cells."""
    assert Q.generate_rqc_masked(5, 5, "1" * 25, 20, 3) == Q.generate_rqc(5, 5, 20, 3)
    counts = {a: Q.bristlecone_mask(a).count("1") for a in (72, 70, 60)}
    assert counts == {72: 72, 70: 70, 60: 60}
    mask = Q.bristlecone_mask(70)
    text = Q.generate_rqc_masked(11, 12, mask, 32, 0)
    lines = [l.split() for l in text.splitlines()[2:]]
    for f in lines:
        qs = [int(x) for x in f[2:]]
        if f[1] != "h":
            assert all(mask[q] == "1" for q in qs), f
        if f[1] == "cz":
            a, b = qs
            assert abs(a - b) in (1, 12)
    inactive = [q for q in range(132) if mask[q] == "0"]
    assert all(sum(1 for f in lines if int(f[2]) == q) == 2 for q in inactive[:10])
    with pytest.raises(Q.InvalidArgument):
        Q.generate_rqc_masked(3, 3, "101", 8, 0)
