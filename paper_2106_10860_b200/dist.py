"""Row sharding and the one-time model/LUT broadcast (torch.distributed plumbing).

MADDNESS rows are independent ("embarrassingly parallel with respect to rows
of the input"), so the multi-GPU path has exactly one exchange:
rank 0 builds the tables once (h(B), the "set_operator" step) and broadcasts
the serialized model + LUT bytes; every rank then runs the fused kernel on its
own contiguous row shard. No collective sits on the data path.
"""
from __future__ import annotations

import torch
import torch.distributed as dist


def shard_rows(rank: int, world: int, rows_per_rank: int, chunk_rows: int):
    """Weak scaling: rank r owns global rows [r * rows_per_rank, (r+1) * rows_per_rank).
    Returns (first_row, n_rows, first_generator_chunk). rows_per_rank must be a
    multiple of the generator chunk so shards start on chunk boundaries."""
    if rows_per_rank % chunk_rows:
        raise ValueError("rows_per_rank must be a multiple of the generator chunk")
    if not (0 <= rank < world):
        raise ValueError("bad rank")
    first = rank * rows_per_rank
    return first, rows_per_rank, first // chunk_rows


def broadcast_blobs(blobs: list[bytes] | None, src: int = 0, device=None) -> list[bytes]:
    """Broadcast a list of byte strings from `src` to every rank (one size
    exchange + one payload broadcast). `device` is the tensor device the
    process group's backend needs (cuda for NCCL, cpu for gloo)."""
    rank = dist.get_rank()
    if device is None:
        device = torch.device("cuda", torch.cuda.current_device()) \
            if dist.get_backend() == "nccl" else torch.device("cpu")
    n = torch.zeros(1, dtype=torch.int64, device=device)
    if rank == src:
        n[0] = len(blobs)
    dist.broadcast(n, src)
    sizes = torch.zeros(int(n.item()), dtype=torch.int64, device=device)
    if rank == src:
        sizes.copy_(torch.tensor([len(b) for b in blobs], dtype=torch.int64))
    dist.broadcast(sizes, src)
    total = int(sizes.sum().item())
    buf = torch.empty(total, dtype=torch.uint8, device=device)
    if rank == src:
        buf.copy_(torch.frombuffer(bytearray(b"".join(blobs)), dtype=torch.uint8))
    dist.broadcast(buf, src)
    host = buf.cpu().numpy().tobytes()
    out, off = [], 0
    for s in sizes.tolist():
        out.append(host[off:off + s])
        off += s
    return out
