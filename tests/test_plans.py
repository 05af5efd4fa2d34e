"""Authored plans for the BASELINE configs (configs/*.json): the Bristlecone-
60/70 plans (configs 3/4) and the rectangular stand-ins / config 2.

Each plan re-annotates identically under our planner (annotate_plan
semantics, proj/src/plan.cpp:122-210) and matches the reference's own
annotation recorded by oracle/validate_plans.py (plan_from_json +
annotate_plan of the unmodified reference, tests/golden/plan_validation.json);
with oracle/_ref present the reference re-annotates live as well."""
import json
import os

import pytest

import paper_1905_00444_b200 as Q
from conftest import GOLDEN, ROOT

VALID = json.load(open(os.path.join(GOLDEN, "plan_validation.json")))


def test_bristlecone_circuit_fixtures_match_generator():
    for active in (60, 70):
        text = Q.generate_rqc_masked(11, 12, Q.bristlecone_mask(active), 32, 0)
        with open(os.path.join(GOLDEN, f"bristlecone{active}_circuit.txt")) as f:
            assert f.read() == text


def _circuit(name):
    if "bristlecone" in name:
        active = 60 if "60" in name else 70
        return open(os.path.join(GOLDEN, f"bristlecone{active}_circuit.txt")).read()
    spec = {"config3_standin_6x10": (6, 10), "config4_standin_7x10": (7, 10), "config2": (7, 7)}[name]
    return Q.generate_rqc(spec[0], spec[1], 32, 0)


@pytest.mark.parametrize("name", sorted(VALID))
def test_plan_annotation_matches_reference(name):
    rec = VALID[name]
    plan_text = open(os.path.join(ROOT, rec["plan"])).read()
    committed = json.loads(plan_text)
    ours = json.loads(Q.plan_json(_circuit(name), committed["open_qubits"], Q.PLAN_JSON, plan_text))
    assert rec["identical_annotation"]
    assert ours["slices"] == committed["slices"] == rec["reference_slices"]
    assert ours["per_slice"] == committed["per_slice"] == rec["reference_per_slice"]
    assert len(ours["steps"]) == rec["steps"]
    assert ours["per_slice"]["max_rank"] <= 32


def test_bristlecone_plans_slice_budget():
    """BC-70: K >= 2^12 (the fixed 2^12 subset runs), BC-60: K >= 2^10; both
    keep every intermediate at rank <= 32 (32 GiB complex64)."""
    for path, need in (("configs/config4_bristlecone70_plan.json", 1 << 12),
                       ("configs/config3_bristlecone60_plan.json", 1 << 10)):
        p = json.load(open(os.path.join(ROOT, path)))
        assert p["slices"] >= need
        assert max(len(s["out_labels"]) for s in p["steps"]) <= 32


def test_reference_reannotates_live():
    import reflib
    if not reflib.available():
        pytest.skip("oracle/_ref not built")
    for name in ("config4_bristlecone70", "config3_bristlecone60"):
        rec = VALID[name]
        plan_text = open(os.path.join(ROOT, rec["plan"])).read()
        ref = json.loads(reflib.plan_json(_circuit(name), [], reflib.PLAN_JSON, plan_text))
        assert ref["per_slice"] == rec["reference_per_slice"] and ref["slices"] == rec["reference_slices"]
