"""Population sharding across ranks (one process per GPU) — SURVEY.md §8e.

Trees are independent units: each rank evaluates a contiguous block of
slots, balanced by opcode bytes (work is proportional to nodes), and the
per-individual records {fitness, hits, size, depth} are all-gathered so every
rank holds the whole population's records for tournament selection. There
is no other data-path exchange (no floating-point reduction crosses ranks),
so records are identical for any world size.

The collective is torch.distributed (NCCL on GPUs, gloo on CPU for tests);
the per-rank evaluation is the engine's C ABI.
"""
from __future__ import annotations

import numpy as np

RECORD_BYTES = 16


def shard_ranges(sizes, world: int):
    """Contiguous slot ranges [(first, count)] per rank, balanced by bytes.

    Same rule as the engine's in-process partition (ltgp_engine.cu
    ``partition``): rank g takes slots while the running byte total stays
    below g+1 shares, counting a slot when half of it fits."""
    sizes = np.asarray(sizes, dtype=np.uint64)
    M = len(sizes)
    total = int(sizes.sum())
    out = []
    i = 0
    acc = 0
    for g in range(world):
        first = i
        goal = total * (g + 1) // world
        while i < M and (g == world - 1 or acc + int(sizes[i]) // 2 < goal):
            acc += int(sizes[i])
            i += 1
        out.append((first, i - first))
    return out


def gather_records(local, ranges, group=None, device=None):
    """All-gather per-rank record blocks into the full population array.

    ``local``: torch uint8 tensor of count*16 bytes (this rank's records, on
    ``device``). Returns a numpy RECORD array of all slots in slot order."""
    import torch
    import torch.distributed as dist

    from . import RECORD_DTYPE

    world = dist.get_world_size(group)
    cmax = max(c for _, c in ranges)
    dev = device if device is not None else local.device
    send = torch.zeros(cmax * RECORD_BYTES, dtype=torch.uint8, device=dev)
    send[: local.numel()] = local
    recv = torch.empty(world * cmax * RECORD_BYTES, dtype=torch.uint8, device=dev)
    dist.all_gather_into_tensor(recv, send, group=group)
    flat = recv.cpu().numpy().reshape(world, cmax * RECORD_BYTES)
    parts = [flat[g, : ranges[g][1] * RECORD_BYTES] for g in range(world)]
    return np.concatenate(parts).view(RECORD_DTYPE)


class DeviceRecords:
    """Zero-copy view of an engine shard's device record array, exposed
    through __cuda_array_interface__ so torch can wrap it (torch.as_tensor)."""

    def __init__(self, ptr: int, count: int):
        self.__cuda_array_interface__ = {
            "shape": (count * RECORD_BYTES,),
            "typestr": "|u1",
            "data": (ptr, False),
            "version": 3,
            "strides": None,
        }
