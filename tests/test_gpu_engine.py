"""End-to-end parity of the device executor (Engine, C ABI) against the
reference's amplitude_batch outputs and the double-precision state vector.

SPEC acceptance (proj/../SPEC.md:499-510) restated here:
  #1 oracle equivalence: 20 circuits <= 4x5, depth (1+8+1)..(1+16+1),
     relative L2 error vs the state vector <= 1e-4 (amplitudes above floor);
  #2 cut completeness: per-slice contributions sum to the full amplitude
     and match the reference's per-slice values (1e-5);
  #8 determinism: bit-identical results across runs and across slice
     partitions (the multi-GPU ordered merge).
Tolerance vs the reference's own fp32 TTGT: relative L2 <= 1e-5."""
import json
import os

import numpy as np
import pytest

from conftest import GOLDEN, ROOT, sweep_plan

pytestmark = pytest.mark.gpu


def rel(a, b):
    nb = np.linalg.norm(b)
    if nb == 0:
        return float(np.linalg.norm(a))  # exact zero contribution (e.g. a cut slice that vanishes)
    return float(np.linalg.norm(a - b) / nb)


@pytest.fixture(scope="module")
def cases():
    am = np.load(os.path.join(GOLDEN, "amplitudes.npz"))
    meta = json.load(open(os.path.join(GOLDEN, "amplitudes.json")))
    return am, meta


@pytest.mark.parametrize("tc", [True, False])
def test_twenty_circuits_vs_reference_and_state_vector(gpu, cases, tc):
    am, meta = cases
    for i, case in enumerate(meta["cases"]):
        text = gpu.generate_rqc(case["rows"], case["cols"], case["m"], case["seed"])
        with gpu.Engine(text, case["plan"], tensor_cores=tc) as e:
            bits, amps = e.amplitude_batch(case["x1"], range(case["slices"]))
        import hashlib
        assert hashlib.sha256("".join(bits).encode()).hexdigest() == case["bits_sha"]
        assert rel(amps, am[f"amps{i}"]) < 1e-5, i
        exact = am[f"exact{i}"]
        assert rel(amps, exact) < 1e-4, i


def test_cut_completeness_per_slice(gpu, cases):
    am, meta = cases
    checked = 0
    for i, case in enumerate(meta["cases"]):
        if case["slices"] < 2:
            continue
        text = gpu.generate_rqc(case["rows"], case["cols"], case["m"], case["seed"])
        with gpu.Engine(text, case["plan"]) as e:
            e.prepare(case["x1"])
            e.run(range(case["slices"]), reset=True, per_slice=True)
            amps, per = e.results()
        ref_per = am[f"per_slice{i}"]
        for s in range(case["slices"]):
            assert rel(per[s], ref_per[s]) < 1e-5
        # the ascending-order sum of contributions IS the batch (bit-exact)
        acc = np.zeros_like(amps)
        for s in range(case["slices"]):
            acc = acc + per[s]
        assert np.array_equal(acc, amps)
        checked += 1
    assert checked >= 3


def test_config1_batches(gpu, cases):
    am, meta = cases
    text = gpu.generate_rqc(4, 4, 16, 0)
    plan = open(os.path.join(ROOT, "configs", "config1_plan.json")).read()
    sv = am["cfg1_state"]
    with gpu.Engine(text, plan) as e:
        for i, c in enumerate(meta["config1"]):
            x1 = gpu.draw_x1(16, list(range(10, 16)), 0, i)
            assert x1 == c["x1"]
            bits, amps = e.amplitude_batch(x1, [0])
            assert rel(amps, am[f"cfg1_amps{i}"]) < 1e-5
            exact = np.array([sv[int(b, 2)] for b in bits])
            assert rel(amps, exact) < 1e-4


def test_determinism_and_partition_invariance(gpu, cases):
    am, meta = cases
    case = max(meta["cases"], key=lambda c: c["slices"])
    text = gpu.generate_rqc(case["rows"], case["cols"], case["m"], case["seed"])
    ids = list(range(case["slices"]))
    with gpu.Engine(text, case["plan"]) as e:
        _, a1 = e.amplitude_batch(case["x1"], ids)
        _, a2 = e.amplitude_batch(case["x1"], ids)
        assert np.array_equal(a1, a2)
        # G-way contiguous partition, per-slice contributions merged in slice order
        for g in (2, 4):
            blocks = np.array_split(np.array(ids), g)
            pers = []
            for blk in blocks:
                e.prepare(case["x1"])
                e.run(list(blk), reset=True, per_slice=True)
                pers.append(e.results()[1])
            merged = np.zeros_like(a1)
            for p in np.concatenate(pers):
                merged = merged + p
            assert np.array_equal(merged, a1)


def test_run_amplitudes_closed_plan(gpu):
    text = gpu.generate_rqc(4, 4, 10, 5)
    plan = gpu.plan_json(text, [], gpu.PLAN_GREEDY, "", 2048)
    pj = json.loads(plan)
    assert pj["slices"] > 1
    import qsim_oracle as O
    sv = O.evolve(text)
    rng = np.random.default_rng(0)
    bits = ["".join(str(int(b)) for b in rng.integers(0, 2, 16)) for _ in range(5)]
    with gpu.Engine(text, plan) as e:
        amps, ids, flops = e.run_amplitudes(bits)
        assert ids == list(range(pj["slices"]))
        assert flops == pj["per_slice"]["flops"] * pj["slices"] * len(bits)  # SPEC #3, exact
        exact = np.array([sv[int(b, 2)] for b in bits])
        assert rel(amps, exact) < 1e-4
        # fractional path: k of K slices, seeded offset (engine.cpp:285-298)
        k = pj["slices"] // 2
        part, ids2, _ = e.run_amplitudes(bits, (k, pj["slices"]), seed=3)
        assert ids2 == gpu.select_slices(k, pj["slices"], pj["slices"], 3)


_JOB_CHILD = r"""
import json, sys
sys.path.insert(0, sys.argv[1])
import paper_1905_00444_b200 as Q
text = Q.generate_rqc(4, 4, 10, 5)
plan = Q.plan_json(text, [], Q.PLAN_GREEDY, "", 2048)
bits = ["0" * 16, "1" * 16]
with Q.Engine(text, plan) as e:
    try:
        e.run_amplitudes(bits)
        print(json.dumps({"raised": None}))
    except Q.JobError as err:
        print(json.dumps({"raised": "JobError", "slice": err.slice_id, "msg": str(err)}))
"""


def test_run_amplitudes_failure_names_lowest_failing_slice(gpu):
    """SURVEY 5 failure detection / SPEC "worker panic -> job fails with the
    offending slice_id": a run_amplitudes job whose slices 3 and 1 fail
    (fault injection, QSG_FAIL_SLICES, in a fresh process) raises JobError
    for slice 1 -- the lowest failing task, as the reference's schedule()
    reports it (src/engine.cpp:247-283) -- with " (slice 1)" in the message."""
    import subprocess
    import sys
    env = dict(os.environ, QSG_FAIL_SLICES="3,1")
    res = subprocess.run([sys.executable, "-c", _JOB_CHILD, ROOT], env=env, capture_output=True, text=True,
                         timeout=300)
    assert res.returncode == 0, res.stderr[-2000:]
    got = json.loads(res.stdout.strip().splitlines()[-1])
    assert got["raised"] == "JobError" and got["slice"] == 1, got
    assert got["msg"].endswith("(slice 1)"), got


def test_engine_rejects_bad_inputs(gpu, cases):
    am, meta = cases
    case = meta["cases"][0]
    text = gpu.generate_rqc(case["rows"], case["cols"], case["m"], case["seed"])
    with gpu.Engine(text, case["plan"]) as e:
        with pytest.raises(gpu.OutOfRange):
            e.amplitude_batch(case["x1"], [case["slices"]])
        bad = list(case["x1"])
        bad[case["open"][0]] = 0
        with pytest.raises(gpu.InvalidArgument):
            e.prepare(bad)


def test_config2_full_size_tensor_core_vs_simt(gpu):
    """BASELINE config 2 at full size (7x7, 1+32+1, 1024-amplitude batch, 2
    slices, 2.15e14 flop): the tcgen05 (3xFP16 split) engine and the FP32-FFMA
    engine are independent GEMM implementations; they must agree to rel-L2
    1e-4 and batch fidelity >= 1 - 1e-6 (per-amplitude bars against fp64 and
    the reference: tests/test_gpu_large.py).  Also
    checks the size-independent properties: Porter-Thomas scale of the batch
    norm and cut completeness (per-slice contributions sum to the batch)."""
    text = gpu.generate_rqc(7, 7, 32, 0)
    plan = open(os.path.join(ROOT, "configs", "config2_plan.json")).read()
    opn = json.loads(plan)["open_qubits"]
    x1 = gpu.draw_x1(49, opn, 0, 0)
    res = {}
    for tc in (True, False):
        with gpu.Engine(text, plan, tensor_cores=tc) as e:
            e.prepare(x1)
            e.run([0, 1], reset=True, per_slice=True)
            res[tc] = e.results()
    (a, pa), (b, pb) = res[True], res[False]
    assert np.array_equal(pa[0] + pa[1], a) and np.array_equal(pb[0] + pb[1], b)
    # every amplitude against fp64 and the reference: tests/test_gpu_large.py
    assert rel(a, b) < 1e-4
    fid = abs(np.vdot(a, b)) ** 2 / (np.vdot(a, a).real * np.vdot(b, b).real)
    assert fid >= 1 - 1e-6
    # Porter-Thomas: E[2^n |a|^2] = 1 over random bitstrings (loose, 1024 samples)
    assert 0.8 < np.mean(np.abs(a) ** 2) * 2.0**49 < 1.25


def test_config5_slice_tensor_core_vs_simt(gpu):
    """Config 5 (7x7, 1+40+1, reference_plan_7x7) at full size, one slice
    (7.2e14 flop, rank-30 intermediates, 2^15 x 2^15 x 2^15 GEMMs): the
    tcgen05 3xFP16 engine (split hand-offs, pre-split A, K-sync) vs the
    FP32-FFMA engine -- north-star tolerance on |amp| and fidelity."""
    text = gpu.generate_rqc(7, 7, 40, 0)
    plan = open(os.path.join(ROOT, "configs", "config5_plan.json")).read()
    x1 = gpu.draw_x1(49, json.loads(plan)["open_qubits"], 0, 0)
    res = {}
    for tc in (True, False):
        with gpu.Engine(text, plan, tensor_cores=tc) as e:
            e.prepare(x1)
            e.run([5], reset=True)
            res[tc] = e.results()
    a, b = res[True], res[False]
    # every amplitude against fp64 and the reference: tests/test_gpu_large.py
    fid = abs(np.vdot(a, b)) ** 2 / (np.vdot(a, a).real * np.vdot(b, b).real)
    assert fid >= 1 - 1e-6
    assert rel(a, b) < 1e-4


def test_split_handoffs_match_fp32_storage(gpu, monkeypatch):
    """GEMM -> GEMM hand-offs in fp16 hi|lo split storage (config 2 has 13
    chained ones, up to five in a row): same amplitudes as fp32 storage to
    FP32-level accuracy, i.e. the bound-based output scaling does not lose
    precision along chains."""
    text = gpu.generate_rqc(7, 7, 32, 0)
    plan = open(os.path.join(ROOT, "configs", "config2_plan.json")).read()
    x1 = gpu.draw_x1(49, json.loads(plan)["open_qubits"], 0, 1)
    res = {}
    for split in ("1", "0"):
        monkeypatch.setenv("QSG_TC_CSPLIT", split)
        with gpu.Engine(text, plan, tensor_cores=True) as e:
            desc = e.describe()
            e.prepare(x1)
            e.run([0], reset=True)
            res[split] = e.results()
        assert (desc.count("split-in") >= 10) == (split == "1")
    assert rel(res["1"], res["0"]) < 5e-6


def test_lane_store_epilogue_matches_staged(gpu, monkeypatch):
    """The lane-per-row STG.256 split-output epilogue (default) and the staged
    smem-slab one (QSG_TC_LANESTORE=0) write the same hi | lo planes; on a
    config-2 slice (13 chained split hand-offs) the amplitudes agree to
    FP32-level accuracy (only the max |c|^2 bookkeeping is computed
    differently: on the split values, rescaled once per tile)."""
    text = gpu.generate_rqc(7, 7, 32, 0)
    plan = open(os.path.join(ROOT, "configs", "config2_plan.json")).read()
    x1 = gpu.draw_x1(49, json.loads(plan)["open_qubits"], 0, 1)
    res = {}
    for lane in ("1", "0"):
        monkeypatch.setenv("QSG_TC_LANESTORE", lane)
        with gpu.Engine(text, plan, tensor_cores=True) as e:
            e.prepare(x1)
            e.run([0], reset=True)
            res[lane] = e.results()
    assert rel(res["1"], res["0"]) < 1e-6


@pytest.mark.parametrize("lane", ["1", "0"])
def test_tensor_core_paths_forced_small_vs_oracle(gpu, monkeypatch, lane):
    """Forces every supported GEMM onto the tcgen05 path (QSG_TC_MIN_FLOPS=0)
    on a 7x7 (1+20+1) circuit with the config-2 region order and cut, so the
    CTA-pair kernel, its narrow-N variants and the fused output permutation
    (lookahead layouts) all run at a size the numpy oracle checks exactly --
    with the lane-store epilogue and with the staged one."""
    import qsim_oracle as O
    monkeypatch.setenv("QSG_TC_MIN_FLOPS", "0")
    monkeypatch.setenv("QSG_TC_LANESTORE", lane)
    text = gpu.generate_rqc(7, 7, 20, 0)
    order = json.load(open(os.path.join(ROOT, "configs", "config2_plan.json")))["order"]
    opn = [32, 33, 34, 39, 40, 41, 45, 46, 47, 48]
    plan = json.dumps({"version": 1, "open_qubits": opn, "cut": {"labels": ["b_007_003_004"], "group": 1},
                       "order": order})
    listing = gpu.program_listing(text, plan)
    assert "fused-store" in listing and " tc " in listing
    x1 = gpu.draw_x1(49, opn, 3, 0)
    with gpu.Engine(text, plan) as e:
        bits, amps = e.amplitude_batch(x1, [0, 1])
    obits, oamps = O.amplitude_batch(text, plan, x1, [0, 1])
    assert bits == obits
    assert rel(amps, oamps) < 1e-5
    with gpu.Engine(text, plan, tensor_cores=False) as e:
        _, samps = e.amplitude_batch(x1, [0, 1])
    assert rel(amps, samps) < 1e-5


def _small_config2_like(gpu, depth=20):
    text = gpu.generate_rqc(7, 7, depth, 0)
    order = json.load(open(os.path.join(ROOT, "configs", "config2_plan.json")))["order"]
    opn = [32, 33, 34, 39, 40, 41, 45, 46, 47, 48]
    plan = json.dumps({"version": 1, "open_qubits": opn, "cut": {"labels": ["b_007_003_004"], "group": 1},
                       "order": order})
    return text, plan, opn


@pytest.mark.parametrize("tc", [True, False])
def test_out_of_core_matches_in_core(gpu, tc):
    """SURVEY 8f row 1 (ExecOptions::memory_budget, src/engine.cpp:216-222):
    steps whose working set exceeds the budget run as m/n pieces through the
    depth-2 copy/compute pipeline with their tensors in pinned host memory;
    the amplitudes equal the in-HBM run (every output element keeps its full
    K loop), the device arena shrinks, and the oracle agrees."""
    import qsim_oracle as O
    text, plan, opn = _small_config2_like(gpu)
    budget = 1 << 20  # 31 of 48 steps out of core, 231 pieces
    listing = gpu.program_listing(text, plan, tensor_cores=tc, memory_budget=budget)
    head = listing.splitlines()[0]
    assert "host arena" in head and listing.count(" ooc pieces ") >= 5
    full = int(gpu.program_listing(text, plan, tensor_cores=tc).splitlines()[0].split()[1])
    assert int(head.split()[1]) < full
    x1 = gpu.draw_x1(49, opn, 5, 0)
    with gpu.Engine(text, plan, tensor_cores=tc) as e:
        _, ref = e.amplitude_batch(x1, [0, 1])
    for depth in (1, 2, 3):
        with gpu.Engine(text, plan, tensor_cores=tc, memory_budget=budget, pipeline_depth=depth) as e:
            bits, amps = e.amplitude_batch(x1, [0, 1])
        assert rel(amps, ref) < 1e-6, depth
    obits, oamps = O.amplitude_batch(text, plan, x1, [0, 1])
    assert bits == obits and rel(amps, oamps) < 1e-5


def test_out_of_core_config2_full_size(gpu):
    """Config 2 at full size under an 8 GiB contraction budget: 18 of 48
    steps (including s026, whose operands alone are 17 GiB) run out of core
    with ~36 GB of tensors in host memory; amplitudes match the in-HBM run."""
    text = gpu.generate_rqc(7, 7, 32, 0)
    plan = open(os.path.join(ROOT, "configs", "config2_plan.json")).read()
    x1 = gpu.draw_x1(49, json.loads(plan)["open_qubits"], 0, 2)
    with gpu.Engine(text, plan) as e:
        e.prepare(x1)
        e.run([0], reset=True)
        ref = e.results()
    with gpu.Engine(text, plan, memory_budget=8 << 30) as e:
        assert "ooc" in e.describe()
        e.prepare(x1)
        e.run([0], reset=True)
        got = e.results()
    assert rel(got, ref) < 1e-6


def test_out_of_core_indivisible(gpu):
    """The reference's error when no piece fits (src/plan.cpp:437)."""
    text, plan, _ = _small_config2_like(gpu, depth=12)
    with pytest.raises(gpu.QsgError, match="indivisible contraction still over budget"):
        gpu.Engine(text, plan, memory_budget=64)


def test_amplitude_batches_widened_plan(gpu):
    """Many x1 draws in one contraction: config 1's plan with every x1 qubit
    opened (same order / cut) serves 64 draws x 64 amplitudes at once;
    each draw's list equals the per-draw amplitude_batch (bit-exact
    bitstrings, amplitudes to FP32 level) and the oracle."""
    import qsim_oracle as O
    text = gpu.generate_rqc(4, 4, 16, 0)
    plan = open(os.path.join(ROOT, "configs", "config1_plan.json")).read()
    base = json.loads(plan)["open_qubits"]
    closed = [q for q in range(16) if q not in base]
    wide = gpu.widen_plan(text, plan, closed)
    draws = [gpu.draw_x1(16, base, 0, i) for i in range(64)]
    with gpu.Engine(text, wide) as e:
        got = e.amplitude_batches(base, draws, [0])
        # pipelined form: two batches in flight, collected in order, bit-identical
        halves = [draws[:32], draws[32:]]
        e.amplitude_batches_submit(base, halves[0], [0], slot=0)
        e.amplitude_batches_submit(base, halves[1], [0], slot=1)
        late = e.amplitude_batches_collect(1, bitstrings=True)
        early = e.amplitude_batches_collect(0, bitstrings=True)
        for (b1, a1), (b2, a2) in zip(early + late, got):
            assert b1 == b2 and np.array_equal(a1, a2)
    with gpu.Engine(text, plan) as e:
        for x1, (bits, amps) in zip(draws[:8], got[:8]):
            rbits, ramps = e.amplitude_batch(x1, [0])
            assert bits == rbits
            assert rel(amps, ramps) < 1e-5
    for x1, (bits, amps) in zip(draws[:4], got[:4]):
        obits, oamps = O.amplitude_batch(text, plan, x1, [0])
        assert bits == obits and rel(amps, oamps) < 1e-5
    with pytest.raises(gpu.InvalidArgument, match="closed"):
        with gpu.Engine(text, gpu.widen_plan(text, plan, closed[:2])) as e:
            e.amplitude_batches(base, draws, [0])


def test_masked_grid_amplitudes_vs_state_vector(gpu):
    """A masked 4x5 grid (3 idle cells, depth 1+12+1) through the greedy plan:
    amplitudes match the double state vector; an idle cell's output 1 has
    amplitude 0 (its worldline is H.H = I)."""
    import qsim_oracle as O
    mask = "11111" "10111" "11101" "01111"
    text = gpu.generate_rqc_masked(4, 5, mask, 12, 7)
    opn = [0, 5, 6, 7, 12]  # qubit 6 is an idle cell (mask row 1 = 10111)
    plan = gpu.plan_json(text, opn, gpu.PLAN_GREEDY)
    sv = O.evolve(text)
    x1 = [-1 if q in opn else (q * 7 + 3) % 2 for q in range(20)]
    x1 = [b if mask[q] == "1" or b < 0 else 0 for q, b in enumerate(x1)]  # idle closed cells read 0
    with gpu.Engine(text, plan) as e:
        bits, amps = e.amplitude_batch(x1, [0])
    exact = np.array([sv[int(b, 2)] for b in bits])
    assert rel(amps, exact) < 1e-4
    idle_one = np.array([b[6] == "1" for b in bits])
    assert np.all(np.abs(amps[idle_one]) < 1e-7 * np.abs(amps).max())


def test_load_nodes_rebinds_circuit_instance(gpu, cases):
    """Another gate draw of the same layout through fold_nodes + load_nodes
    gives bit-identical amplitudes to a fresh engine on that circuit; a
    different layout is rejected."""
    import torch
    _, meta = cases
    case = meta["cases"][0]
    a = gpu.generate_rqc(case["rows"], case["cols"], case["m"], case["seed"])
    b = gpu.generate_rqc(case["rows"], case["cols"], case["m"], case["seed"] + 17)
    with gpu.Engine(b, case["plan"]) as fresh:
        want_bits, want = fresh.amplitude_batch(case["x1"], range(case["slices"]))
    with gpu.Engine(a, case["plan"]) as e:
        assert np.array_equal(e.export_nodes(), e.fold_nodes(a))
        host = torch.empty(e.info.node_bytes // 8, dtype=torch.complex64, pin_memory=True)
        e.fold_nodes(b, out=host)
        assert e.load_nodes(host) == e.info.node_bytes
        bits, got = e.amplitude_batch(case["x1"], range(case["slices"]))
        assert bits == want_bits and np.array_equal(got, want)
        assert np.array_equal(e.export_nodes(), host.numpy())
        other = gpu.generate_rqc(case["rows"], case["cols"], case["m"] + 1, case["seed"])
        with pytest.raises(gpu.QsgError):
            e.fold_nodes(other)
        with pytest.raises(gpu.QsgError):
            e.load_nodes(np.zeros(4, dtype=np.complex64))


@pytest.mark.parametrize("tc", [True, False])
def test_reassociated_plan_same_amplitudes(gpu, tc, monkeypatch):
    """A sweep plan and its reassociated tree give the same batch (1e-5) and
    both match the double state vector (1e-4)."""
    import qsim_oracle as O
    if tc:
        monkeypatch.setenv("QSG_TC_MIN_FLOPS", "0")
    text, plan, opn = sweep_plan(gpu, 4, 5, 16, 3, 4)
    new, k = gpu.reassociate_plan(text, plan)
    assert k > 0
    x1 = [-1 if q in opn else (q * 5 + 1) % 2 for q in range(20)]
    with gpu.Engine(text, plan, tensor_cores=tc) as e:
        bits, want = e.amplitude_batch(x1, [0])
    with gpu.Engine(text, new, tensor_cores=tc) as e:
        bits2, got = e.amplitude_batch(x1, [0])
    assert bits == bits2
    assert rel(got, want) < 1e-5
    sv = O.evolve(text)
    exact = np.array([sv[int(b, 2)] for b in bits])
    assert rel(got, exact) < 1e-4


def test_repeated_runs_replay_as_graph(gpu, cases, monkeypatch):
    """A run repeated with the same slices and x1 is captured once and replayed
    as a CUDA graph: bit-identical results, same kernel count per run, and a
    new x1 / slice list falls back to eager launches."""
    _, meta = cases
    case = next(c for c in meta["cases"] if c["slices"] >= 2)
    text = gpu.generate_rqc(case["rows"], case["cols"], case["m"], case["seed"])
    monkeypatch.setenv("QSG_TC_MIN_FLOPS", "0")
    out, counts = [], []
    with gpu.Engine(text, case["plan"]) as e:
        e.prepare(case["x1"])
        for _ in range(4):
            n0 = e.launches()
            e.run(range(case["slices"]), reset=True, per_slice=True)
            out.append(e.results())
            counts.append(e.launches() - n0)
        e.run([0], reset=True)
        single = e.results()
    assert len(set(counts)) == 1 and counts[0] > 0
    for amps, per in out[1:]:
        assert np.array_equal(amps, out[0][0]) and np.array_equal(per, out[0][1])
    assert rel(single, out[0][1][0]) < 1e-12
