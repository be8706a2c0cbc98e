"""Host-side plumbing of the multi-GPU path (one process per GPU).

Works with any torch.distributed backend (NCCL on the GPU box, gloo in the CPU
tests).  The data-path collective itself (the all-reduce of partial aggregates)
runs inside liblmfao_gpu over NCCL; these helpers only move the communicator id,
mirror the library's shard formula and reduce timings.
"""
from __future__ import annotations


def shard_range(n_rows: int, part: int, nparts: int):
    """Contiguous shard of the sorted root kept by `part` (same formula as
    lmfao_prepare: [N*r/G, N*(r+1)/G))."""
    return n_rows * part // nparts, n_rows * (part + 1) // nparts


def broadcast_bytes(dist, payload: bytes | None, nbytes: int, rank: int, device="cpu") -> bytes:
    """Broadcast rank 0's `payload` (e.g. the NCCL unique id) to every rank."""
    import torch
    t = torch.zeros(nbytes, dtype=torch.uint8, device=device)
    if rank == 0:
        t.copy_(torch.frombuffer(bytearray(payload), dtype=torch.uint8))
    dist.broadcast(t, 0)
    return bytes(t.cpu().numpy().tobytes())


def max_over_ranks(dist, values, device="cpu"):
    """Element-wise max over ranks (multi-GPU timings are the slowest rank's)."""
    import torch
    t = torch.tensor(list(values), dtype=torch.float64, device=device)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return [float(x) for x in t]
