"""The executor's compiled device program (no GPU needed): heavy steps run on
the tcgen05 path, the static arena fits HBM, and flops match the plan."""
import json
import os

import pytest

import paper_1905_00444_b200 as Q
from conftest import ROOT, sweep_plan

HBM_BYTES = 180e9


def listing(cfg, r, c, m, s, tensor_cores=True):
    text = Q.generate_rqc(r, c, m, s)
    plan = open(os.path.join(ROOT, "configs", f"{cfg}_plan.json")).read()
    return json.loads(plan), Q.program_listing(text, plan, tensor_cores=tensor_cores).splitlines()


@pytest.mark.parametrize("cfg,shape", [("config2", (7, 7, 32, 0)), ("config5", (7, 7, 40, 0)),
                                       ("config3_standin_6x10", (6, 10, 32, 0)),
                                       ("config4_standin_7x10", (7, 10, 32, 0))])
def test_heavy_steps_on_tensor_cores_and_arena_fits(cfg, shape):
    plan, lines = listing(cfg, *shape)
    arena = int(lines[0].split()[1])
    assert arena < 0.6 * HBM_BYTES
    gemm = [l.split() for l in lines if l.split()[0] == "gemm"]
    assert len(gemm) == len(plan["steps"])
    assert sum(int(f[10]) for f in gemm) == plan["per_slice"]["flops"]  # SPEC #3, exact
    heavy = [f for f in gemm if int(f[10]) >= 0.01 * plan["per_slice"]["flops"]]
    assert heavy and all("tc" in f for f in heavy), [" ".join(f) for f in heavy if "tc" not in f]
    tc_flops = sum(int(f[10]) for f in gemm if "tc" in f)
    assert tc_flops >= 0.99 * plan["per_slice"]["flops"]


def test_no_tensor_core_program_uses_simt_everywhere():
    plan, lines = listing("config2", 7, 7, 32, 0, tensor_cores=False)
    assert all("simt" in l.split() for l in lines if l.split()[0] == "gemm")


def test_out_of_core_placement():
    """memory_budget (ExecOptions): oversized steps and every step reading
    their host-resident results go out of core; the device arena shrinks to
    what the in-core steps need, the rest is the pinned host arena."""
    text = Q.generate_rqc(7, 7, 32, 0)
    plan = open(os.path.join(ROOT, "configs", "config2_plan.json")).read()
    full = Q.program_listing(text, plan).splitlines()
    lines = Q.program_listing(text, plan, memory_budget=8 << 30).splitlines()
    head = lines[0].split()
    assert int(head[1]) < 0.2 * int(full[0].split()[1])
    assert "host" in lines[0]
    ooc = [l.split() for l in lines if " ooc pieces " in l]
    assert any(f[2] == "26" and int(f[-1]) >= 2 for f in ooc)  # s026 (17 GiB of operands) is split
    assert sum(int(f[10]) for f in (l.split() for l in lines) if f[0] == "gemm") == json.loads(plan)["per_slice"]["flops"]
    with pytest.raises(Q.QsgError, match="indivisible"):
        Q.program_listing(text, plan, memory_budget=4096)


def test_out_of_core_automatic_budget():
    """memory_budget=-1: in HBM when the program fits the device, else the
    largest power-of-two contraction budget whose out-of-core program fits."""
    text = Q.generate_rqc(7, 7, 32, 0)
    plan = open(os.path.join(ROOT, "configs", "config2_plan.json")).read()
    big = Q.program_listing(text, plan, memory_budget=-1, device_memory=180 << 30).splitlines()
    assert "host arena" not in big[0] and not any(" ooc " in l for l in big)
    for dev in (30 << 30, 12 << 30):
        head = Q.program_listing(text, plan, memory_budget=-1, device_memory=dev).splitlines()[0].split()
        arena, slot = int(head[1]), int(head[head.index("scratch") + 1])
        assert arena + 2 * slot <= 0.92 * dev


def test_reassociate_plan_sweeps():
    """The opt-in tree rewrite keeps cut, slices, open qubits and peak bounds,
    lowers the Eq.(1) flops of sweep plans, and is idempotent."""
    text, plan, _ = sweep_plan(Q, 4, 5, 16, 3, 4)
    new, k = Q.reassociate_plan(text, plan)
    a, b = json.loads(plan), json.loads(new)
    assert k > 0 and len(b["order"]) == len(a["order"])
    assert b["per_slice"]["flops"] < 0.6 * a["per_slice"]["flops"]
    assert b["per_slice"]["max_rank"] <= a["per_slice"]["max_rank"]
    assert Q.reassociate_plan(text, new)[1] == 0
    c3 = Q.generate_rqc(6, 10, 32, 0)
    p3 = open(os.path.join(ROOT, "configs", "config3_standin_6x10_plan.json")).read()
    n3, k3 = Q.reassociate_plan(c3, p3)
    a3, b3 = json.loads(p3), json.loads(n3)
    assert k3 > 0 and b3["slices"] == a3["slices"] and b3["cut"] == a3["cut"]
    assert b3["per_slice"]["flops"] < a3["per_slice"]["flops"]
    assert b3["per_slice"]["peak_memory"] <= a3["per_slice"]["peak_memory"]
    assert "gemm" in Q.program_listing(c3, n3)


@pytest.mark.skipif(not os.path.exists(os.path.join(ROOT, "oracle", "_ref", "libqsim_ref.so")),
                    reason="oracle/_ref not built")
def test_bench_reference_arm_prints_exactly_one_json_line():
    """The driver parses bench.py's stdout: one JSON line, nothing else
    (library banners go to stderr)."""
    import subprocess
    import sys
    res = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--impl", "reference", "--config", "1",
                          "--steps", "1", "--warmup", "1", "--cpu-budget-flops", "1e9", "--help"],
                         capture_output=True, text=True, timeout=600, cwd=ROOT)
    assert res.returncode == 0 and res.stdout == ""  # --help text is not the result line
    res = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--impl", "reference", "--config", "1",
                          "--steps", "1", "--warmup", "1", "--cpu-budget-flops", "1e9"],
                         capture_output=True, text=True, timeout=600, cwd=ROOT)
    assert res.returncode == 0, res.stderr[-2000:]
    lines = res.stdout.splitlines()
    assert len(lines) == 1
    d = json.loads(lines[0])
    assert d["impl"] == "reference" and d["value"] > 0 and d["e2e"]["h2d_bytes_per_step"] == 0
