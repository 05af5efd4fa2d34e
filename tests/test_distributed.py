"""Multi-rank path on CPU (gloo, world_size 2 and 4): contiguous slice
partition + one all-gather + ascending-order FP64 merge is bit-identical to
the single-process merge (the engine's K3 order), for any rank count."""
import os
import socket

import numpy as np
import pytest
import torch.multiprocessing as mp

from paper_1905_00444_b200 import distributed as D


def test_slice_blocks_are_contiguous_and_balanced():
    ids = list(range(1024))
    for world in (1, 2, 3, 4, 8):
        blocks = D.slice_blocks(ids[::-1], world)
        assert sum(blocks, []) == ids
        sizes = [len(b) for b in blocks]
        assert max(sizes) - min(sizes) <= 1


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _worker(rank, world, port, contrib, out):
    import torch.distributed as dist
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    blocks = D.slice_blocks(range(contrib.shape[0]), world)
    local = contrib[blocks[rank]]
    allc = D.gather_contributions(local, [len(b) for b in blocks])
    merged = D.ordered_merge(allc)
    if rank == 0:
        out.put(merged.view(np.float64).tolist())
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 4])
def test_gloo_gather_and_ordered_merge_bit_identical(world):
    rng = np.random.default_rng(world)
    k, batch = 37, 64
    contrib = (rng.standard_normal((k, batch)) + 1j * rng.standard_normal((k, batch))) * 2.0 ** rng.integers(
        -40, 0, (k, 1))
    want = D.ordered_merge(contrib)
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, contrib, q)) for r in range(world)]
    for p in procs:
        p.start()
    got = np.array(q.get(timeout=120)).view(np.complex128)
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    assert np.array_equal(got, want)
