"""Multi-GPU partitioning and the single end-of-job collective.

Slices (and x1 batches) are independent with identical shapes and cost
(reference src/plan.cpp:72-87), so ranks never exchange data while
computing.  Each rank takes a contiguous block of the ascending slice list
(or its own x1 batches); at the end ONE all-gather brings every rank's
per-slice FP64 contributions to all ranks, and the sum runs in ascending
slice order -- the reference's fixed merge order (src/engine.cpp:352-356,
src/sampler.cpp:28-34), so results are bit-identical for any GPU count.

torch.distributed is only the transport (NCCL on GPUs, gloo in the CPU
tests); the numbers come from the engine (libqsg.so).
"""
from __future__ import annotations

import numpy as np


def slice_blocks(slice_ids, world: int):
    """Contiguous, balanced blocks of the ascending slice list, one per rank."""
    ids = sorted(int(s) for s in slice_ids)
    base, extra = divmod(len(ids), world)
    out, pos = [], 0
    for r in range(world):
        n = base + (1 if r < extra else 0)
        out.append(ids[pos:pos + n])
        pos += n
    return out


def ordered_merge(contributions: np.ndarray) -> np.ndarray:
    """Sum per-slice contributions [k, batch] (complex128) in ascending slice
    order, starting from zero -- the same sequence of FP64 additions the
    engine's K3 kernel performs on one GPU."""
    acc = np.zeros(contributions.shape[1:], dtype=np.complex128)
    for c in contributions:
        acc = acc + c
    return acc


def gather_contributions(local: np.ndarray, counts, group=None, device=None) -> np.ndarray:
    """All-gather every rank's per-slice contributions (rank order = slice
    order for contiguous blocks) with one collective.  `counts[r]` is rank
    r's number of slices; blocks are padded to the maximum for the
    equal-size all_gather."""
    import torch
    import torch.distributed as dist

    world = dist.get_world_size(group)
    kmax = max(counts)
    batch = local.shape[1] if local.ndim == 2 else 0
    pad = np.zeros((kmax, batch), dtype=np.complex128)
    pad[: local.shape[0]] = local
    t = torch.from_numpy(pad.view(np.float64).copy())
    if device is not None:
        t = t.to(device)
    bufs = [torch.empty_like(t) for _ in range(world)]
    dist.all_gather(bufs, t, group=group)
    parts = [b.cpu().numpy().view(np.complex128)[: counts[r]] for r, b in enumerate(bufs)]
    return np.concatenate(parts, axis=0) if parts else np.zeros((0, batch), np.complex128)


def sliced_amplitudes(engine, x1_bits, slice_ids, rank: int, world: int, group=None, device=None):
    """One amplitude batch over `slice_ids` split across `world` ranks:
    each rank runs its contiguous block on its own engine/GPU, then one
    all-gather + ordered merge.  Returns (amplitudes, per-slice contributions)."""
    blocks = slice_blocks(slice_ids, world)
    mine = blocks[rank]
    engine.prepare(x1_bits)
    batch = engine.info.batch_size
    if mine:
        engine.run(mine, reset=True, per_slice=True)
        _, per = engine.results()
    else:
        per = np.zeros((0, batch), dtype=np.complex128)
    allc = gather_contributions(per, [len(b) for b in blocks], group=group, device=device)
    return ordered_merge(allc), allc
