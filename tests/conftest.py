import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "oracle"))
GOLDEN = os.path.join(ROOT, "tests", "golden")


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200); run with -m gpu")
    config.addinivalue_line("markers", "slow: long-running parity case")


def has_gpu() -> bool:
    try:
        import paper_1905_00444_b200 as Q
        return Q.device_count() > 0
    except Exception:
        return False


@pytest.fixture(scope="session")
def golden():
    import json
    with open(os.path.join(GOLDEN, "golden.json")) as f:
        return json.load(f)


@pytest.fixture(scope="session")
def gpu():
    if not has_gpu():
        pytest.fail("GPU test selected but no CUDA device is visible")
    import paper_1905_00444_b200 as Q
    return Q


def sweep_plan(Q, rows, cols, m, seed, nopen):
    """Column-major sweep chained onto one accumulator (the config 3/4 plan
    shape) on a small grid, with the first `nopen` qubits of the last row open:
    (circuit text, plan JSON, open qubits)."""
    import json
    text = Q.generate_rqc(rows, cols, m, seed)
    nodes = [r * cols + c for c in range(cols) for r in range(rows)]
    order, acc = [], f"n_{nodes[0]:03d}"
    for i, q in enumerate(nodes[1:]):
        order.append([acc, f"n_{q:03d}"])
        acc = f"s{i:03d}"
    opn = sorted((rows - 1) * cols + c for c in range(nopen))
    draft = {"version": 1, "open_qubits": opn, "cut": {"labels": [], "group": 1}, "order": order}
    return text, Q.plan_json(text, opn, Q.PLAN_JSON, json.dumps(draft)), opn


def tc_gemm(Q, a_ptr, b_ptr, c_ptr, m, n, k, trans_b=0):
    """qsg_cgemm_tc_dev with a caller-owned workspace (the C ABI allocates
    nothing and does not synchronise); synchronises here for the check."""
    import torch
    nbytes = int(Q.lib().qsg_cgemm_tc_workspace_bytes(m, n, k, trans_b))
    assert nbytes >= 0, "shape not eligible for the tensor-core path"
    ws = torch.empty(max(nbytes, 16), dtype=torch.uint8, device="cuda")
    Q._check(Q.lib().qsg_cgemm_tc_dev(a_ptr, b_ptr, c_ptr, m, n, k, trans_b, ws.data_ptr(), nbytes, None))
    torch.cuda.synchronize()
