"""The executor's compiled device program (no GPU needed): heavy steps run on
the tcgen05 path, the static arena fits HBM, and flops match the plan."""
import json
import os

import pytest

import paper_1905_00444_b200 as Q
from conftest import ROOT

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
