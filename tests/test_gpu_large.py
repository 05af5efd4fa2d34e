"""Full-size parity of the BASELINE configs.

Three independent answers per amplitude, at the real sizes:
  * the reference's own fp32 amplitude_batch, one slice at a time
    (tests/golden/large_*.npz from oracle/gen_golden_large.py, run on the
    unmodified reference in oracle/_ref);
  * an fp64 contraction of the same folded node tensors with torch
    complex128 on the GPU (cuBLAS ZGEMM; test infrastructure, the plan's
    own order, oracle fold + cut) -- the truth for the fp32 problem;
  * our engines: tcgen05 3xFP16 and FP32 FFMA (C ABI).
Every amplitude is checked (no magnitude filter).  Bars: fidelity >= 1 -
1e-6 and rel-L2 <= 5e-5 vs fp64 for every fp32 answer; max relative |amp|
error <= 1e-4 over all amplitudes for our engines, and never more than 2x
the reference's own fp32 error on the same batch (so any small-amplitude
floor is one the reference shares, reported in the JSON written to
gpurun_out/)."""
import json
import os

import numpy as np
import pytest

from conftest import GOLDEN, ROOT

pytestmark = pytest.mark.gpu

OUT = os.path.join(ROOT, "gpurun_out")


def fp64_slice(text, plan, x1, slice_id):
    """complex128 contraction of one slice on the GPU (oracle fold + cut, the
    plan's pairwise order); returns the final tensor in sorted open order."""
    import torch
    import qsim_oracle as O
    cut = plan.get("cut", {"labels": [], "group": 1})
    nodes = O.apply_cut(O.fold_worldlines(text, x1), cut["labels"], cut.get("group", 1), slice_id)
    live = {f"n_{q:03d}": (lab, torch.from_numpy(np.ascontiguousarray(t)).to("cuda", torch.complex128))
            for q, (lab, t) in enumerate(nodes)}
    for i, (lhs, rhs) in enumerate(plan["order"]):
        (la, a), (lb, b) = live.pop(lhs), live.pop(rhs)
        shared = [x for x in la if x in lb]
        lc = [x for x in la if x not in shared] + [x for x in lb if x not in shared]
        if a.dim() == 0 or b.dim() == 0:  # scalar factor (idle Bristlecone cells): torch.tensordot adds a dim
            c = a * b
        else:
            c = torch.tensordot(a, b, dims=([la.index(x) for x in shared], [lb.index(x) for x in shared]))
        c = c.reshape([2] * len(lc))
        del a, b
        live[f"s{i:03d}"] = (lc, c)
    (lab, t), = live.values()
    perm = sorted(range(len(lab)), key=lambda j: lab[j])
    out = t.permute(perm).reshape(-1) if lab else t.reshape(-1)
    res = out.cpu().numpy()
    del live, t, out
    torch.cuda.empty_cache()
    return res


def stats(got, truth):
    got, truth = np.asarray(got).reshape(-1), np.asarray(truth).reshape(-1)
    nz = truth != 0  # structurally vanishing contributions (inconsistent cut digits) must come out ~0
    rel = np.abs(np.abs(got[nz]) - np.abs(truth[nz])) / np.abs(truth[nz])
    ng, nt = np.vdot(got, got).real, np.vdot(truth, truth).real
    fid = abs(np.vdot(got, truth)) ** 2 / (ng * nt) if ng > 0 and nt > 0 else float(ng == nt)
    scale = np.linalg.norm(truth) if nt > 0 else 1.0
    return {"rel_l2": float(np.linalg.norm(got - truth) / scale),
            "max_rel_abs": float(rel.max()) if nz.any() else 0.0, "fidelity_deficit": float(1 - fid),
            "zero_entries": int((~nz).sum()), "max_abs_at_zeros": float(np.abs(got[~nz]).max()) if (~nz).any() else 0.0,
            "min_abs_over_rms": float(np.abs(truth[nz]).min() / np.sqrt(np.mean(np.abs(truth) ** 2)))
            if nz.any() else 0.0}


def engine_per_slice(gpu, text, plan_text, x1, slices, tc):
    with gpu.Engine(text, plan_text, tensor_cores=tc) as e:
        e.prepare(x1)
        e.run(slices, reset=True, per_slice=True)
        amps, per = e.results(per_slice=True)
    return amps, per


CASES = {
    # name: (circuit spec, plan, open-x1 draw or closed bitstrings, slices, fixture)
    "config2": ((7, 7, 32, 0), "configs/config2_plan.json", [0, 1], "large_config2"),
    "config5": ((7, 7, 40, 0), "configs/config5_plan.json", [5], "large_config5"),
    "config3s": ((6, 10, 32, 0), "configs/config3_standin_6x10_plan.json", [0, 1], "large_config3s"),
    # Bristlecone-60 (masked 11x12 embedding, circuit text committed)
    "bc60": (("mask", 60), "configs/config3_bristlecone60_plan.json", [0, 1], "large_bc60"),
    "bc70": (("mask", 70), "configs/config4_bristlecone70_plan.json", [2, 6], "large_bc70"),
}


def circuit(gpu, spec):
    if spec[0] == "mask":
        return open(os.path.join(GOLDEN, f"bristlecone{spec[1]}_circuit.txt")).read(), 132
    return gpu.generate_rqc(*spec), spec[0] * spec[1]


@pytest.mark.parametrize("name", sorted(CASES))
def test_full_size_vs_fp64_and_reference(gpu, name):
    spec, plan_path, slices, fixture = CASES[name]
    text, n = circuit(gpu, spec)
    plan_text = open(os.path.join(ROOT, plan_path)).read()
    plan = json.loads(plan_text)
    fx_path = os.path.join(GOLDEN, fixture + ".npz")
    ref = np.load(fx_path) if os.path.exists(fx_path) else None
    meta = json.load(open(os.path.join(GOLDEN, fixture + ".json"))) if ref is not None else None
    if plan["open_qubits"]:
        x1s = [gpu.draw_x1(n, plan["open_qubits"], 0, 0)]
    else:
        if meta is None:
            pytest.skip(f"{fixture} not generated (oracle/gen_golden_large.py)")
        x1s = meta["x1"]
    if meta is not None:
        assert meta["x1"] == x1s and meta["slices"] == slices
    report, fails = {}, []
    for xi, x1 in enumerate(x1s):
        truth = np.stack([fp64_slice(text, plan, x1, s) for s in slices])
        res = {tc: engine_per_slice(gpu, text, plan_text, x1, slices, tc) for tc in (True, False)}
        for tc, (amps, per) in res.items():
            key = "tc" if tc else "simt"
            # cut completeness: the K3 batch is the ascending sum of the rows
            acc = np.zeros_like(amps)
            for row in per:
                acc = acc + row
            assert np.array_equal(acc, amps)
            st = stats(per, truth)
            report[f"x1#{xi} {key}"] = st
            if not (st["fidelity_deficit"] <= 1e-6 and st["rel_l2"] <= 5e-5):
                fails.append((xi, key, "fidelity/rel_l2"))
        st_ref = None
        if ref is not None:
            rp = ref[f"per_slice{xi}"]
            st_ref = stats(rp, truth)
            report[f"x1#{xi} reference"] = st_ref
            if st_ref["fidelity_deficit"] > 1e-6:
                fails.append((xi, "reference", "fidelity"))
            for tc in (True, False):
                report[f"x1#{xi} {'tc' if tc else 'simt'} vs reference"] = stats(res[tc][1], rp)
        bound = max(1e-4, 2 * st_ref["max_rel_abs"]) if st_ref else 1e-4
        for key in ("tc", "simt"):
            if report[f"x1#{xi} {key}"]["max_rel_abs"] > bound:
                fails.append((xi, key, f"max_rel_abs > {bound:.2e}"))
    os.makedirs(OUT, exist_ok=True)
    with open(os.path.join(OUT, f"parity_{name}.json"), "w") as f:
        json.dump(report, f, indent=1)
    assert not fails, (fails, report)
