"""Host plumbing for row-sharded training (one process per GPU): the row partition and the
exchange of the opaque peer-mapping handles.  No arithmetic of the method lives here; the
per-iteration exchange runs inside the CUDA kernel over NVLink peer memory (csrc/smo.cu)."""
from __future__ import annotations


def shard_bounds(n: int, world: int, rank: int) -> tuple[int, int]:
    """Contiguous row block [r0, r1) of `rank` (rank r holds [r n / P, (r+1) n / P))."""
    if not (0 <= rank < world):
        raise ValueError("rank out of range")
    return rank * n // world, (rank + 1) * n // world


def all_gather_bytes(blob: bytes, group=None) -> list[bytes]:
    """Every rank's handle blob in rank order (torch.distributed.all_gather_object)."""
    import torch.distributed as dist
    out = [None] * dist.get_world_size(group)
    dist.all_gather_object(out, blob, group=group)
    return out
