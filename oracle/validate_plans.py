"""Validates authored plan files with the UNMODIFIED reference planner.

TEST INFRASTRUCTURE.  For each (circuit, plan file) the reference's own
load path -- plan_from_json + annotate_plan (proj/src/plan.cpp:122-210,
481-552), reached through oracle/_ref's ref_plan_json -- re-annotates the
plan; its slices, per-slice Eq.(1) flops, peak memory and max rank must
equal the committed file's (written by our planner).  Writes
tests/golden/plan_validation.json.

    python oracle/validate_plans.py
"""
from __future__ import annotations

import json
import os
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
sys.path.insert(0, HERE)
import reflib as R  # noqa: E402

# (name, circuit generator spec, plan file)
PLANS = [
    ("config3_bristlecone60", ("masked", 60), "configs/config3_bristlecone60_plan.json"),
    ("config4_bristlecone70", ("masked", 70), "configs/config4_bristlecone70_plan.json"),
    ("config3_standin_6x10", ("rect", 6, 10), "configs/config3_standin_6x10_plan.json"),
    ("config4_standin_7x10", ("rect", 7, 10), "configs/config4_standin_7x10_plan.json"),
    ("config2", ("rect", 7, 7), "configs/config2_plan.json"),
]


def circuit(spec, depth=32):
    if spec[0] == "rect":
        return R.generate_rqc(spec[1], spec[2], depth, 0)
    # The reference has no masked generator: the circuit text comes from the
    # committed fixture written by our generator (tests/golden/), parsed and
    # validated by the reference's own parse_circuit inside ref_plan_json.
    with open(os.path.join(ROOT, "tests", "golden", f"bristlecone{spec[1]}_circuit.txt")) as f:
        return f.read()


def main():
    out = {}
    for name, spec, path in PLANS:
        plan_text = open(os.path.join(ROOT, path)).read()
        ours = json.loads(plan_text)
        text = circuit(spec)
        ref = json.loads(R.plan_json(text, ours["open_qubits"], R.PLAN_JSON, plan_text))
        same = (ref["slices"] == ours["slices"] and ref["per_slice"] == ours["per_slice"]
                and [s["flops"] for s in ref["steps"]] == [s["flops"] for s in ours["steps"]]
                and [s["out_labels"] for s in ref["steps"]] == [s["out_labels"] for s in ours["steps"]])
        out[name] = {"plan": path, "reference_slices": ref["slices"], "reference_per_slice": ref["per_slice"],
                     "steps": len(ref["steps"]), "identical_annotation": same}
        print(name, ref["slices"], ref["per_slice"], "identical" if same else "DIFFERENT")
        if not same:
            raise SystemExit(f"{name}: reference annotation differs from the committed plan")
    with open(os.path.join(ROOT, "tests", "golden", "plan_validation.json"), "w") as f:
        json.dump(out, f, indent=1)


if __name__ == "__main__":
    main()
