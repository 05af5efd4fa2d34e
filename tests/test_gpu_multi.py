"""One sliced amplitude job across 2 GPUs over NCCL:
distributed.sliced_amplitudes -- contiguous blocks of the ascending slice
list, one all-gather of the per-slice FP64 contributions, ascending merge
(src/engine.cpp:352-356) -- must equal the single-GPU run bit for bit.
Needs >= 2 visible GPUs (gpurun --gpus 2); skipped on one."""
import json
import os
import socket

import numpy as np
import pytest

from conftest import ROOT

pytestmark = pytest.mark.gpu

CASES = {
    # closed 6x10 stand-in (4096 slices): 8 slices, one bitstring
    "config3s": ((6, 10, 32, 0), "configs/config3_standin_6x10_plan.json", 8),
    # config 5 (64-amplitude batch): 4 of the 1024 slices
    "config5": ((7, 7, 40, 0), "configs/config5_plan.json", 4),
}


def _port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _rank_main(rank, world, port, name, q):
    import torch
    import torch.distributed as dist
    import paper_1905_00444_b200 as Q
    from paper_1905_00444_b200 import distributed as D
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    torch.cuda.set_device(rank)
    dist.init_process_group("nccl", rank=rank, world_size=world, device_id=torch.device("cuda", rank))
    spec, plan_path, k = CASES[name]
    text = Q.generate_rqc(*spec)
    plan_text = open(os.path.join(ROOT, plan_path)).read()
    plan = json.loads(plan_text)
    n = spec[0] * spec[1]
    x1 = Q.draw_x1(n, plan["open_qubits"], 0, 0)
    ids = Q.select_slices(k, plan["slices"], plan["slices"], 0)
    with Q.Engine(text, plan_text, device=rank) as e:
        merged, allc = D.sliced_amplitudes(e, x1, ids, rank, world, device=torch.device("cuda", rank))
        if rank == 0:
            e.prepare(x1)
            e.run(ids, reset=True, per_slice=True)
            single, rows = e.results(per_slice=True)
            q.put({"merged": merged.view(np.float64).tolist(), "single": single.view(np.float64).tolist(),
                   "rows_equal": bool(np.array_equal(rows, allc)), "k": len(ids)})
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("name", sorted(CASES))
def test_two_gpu_sliced_batch_equals_single_gpu(gpu, name):
    import torch
    import torch.multiprocessing as mp
    if torch.cuda.device_count() < 2:
        pytest.skip("needs 2 GPUs (gpurun --gpus 2)")
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _port()
    procs = [ctx.Process(target=_rank_main, args=(r, 2, port, name, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = q.get(timeout=900)
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    assert res["rows_equal"], "per-slice contributions differ between GPUs"
    assert res["merged"] == res["single"], "merged 2-GPU batch != single-GPU batch"
    os.makedirs(os.path.join(ROOT, "gpurun_out"), exist_ok=True)
    with open(os.path.join(ROOT, "gpurun_out", f"multi2_{name}.json"), "w") as f:
        json.dump({"case": name, "slices": res["k"], "bit_identical": True}, f)
