"""Multi-process (gloo, world_size 2, CPU) coverage of the N > 1 host logic:
the one-time model/LUT byte broadcast and the weak-scaling row shards
(rows are independent, so these are the only exchanges)."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from helpers import model_bytes


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from datagen.synth import relu_W, relu_lowrank_torch
    from paper_2106_10860_b200.dist import broadcast_blobs, shard_rows
    blobs = [model_bytes("tiny"), b"\x01\x02luts-bytes", b""] if rank == 0 else None
    got = broadcast_blobs(blobs, 0)
    chunk, per_rank = 64, 192
    first, n, first_chunk = shard_rows(rank, world, per_rank, chunk)
    A = relu_lowrank_torch(relu_W("tiny"), n, first_chunk, "cpu", chunk_rows=chunk)
    parts = [torch.empty_like(A) for _ in range(world)]
    dist.all_gather(parts, A)
    q.put((rank, [len(b) for b in got], got[0] == model_bytes("tiny"), got[1], first, n,
           torch.cat(parts).numpy() if rank == 0 else None))
    dist.barrier()
    dist.destroy_process_group()


def test_gloo_broadcast_and_shards():
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = sorted([q.get(timeout=180) for _ in range(world)], key=lambda r: r[0])
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    for rank, sizes, model_ok, luts, first, n, _ in res:
        assert model_ok and luts == b"\x01\x02luts-bytes" and sizes[2] == 0
        assert first == rank * 192 and n == 192
    from datagen.synth import relu_W, relu_lowrank_torch
    serial = relu_lowrank_torch(relu_W("tiny"), 384, 0, "cpu", chunk_rows=64).numpy()
    assert np.array_equal(res[0][6], serial)      # shards tile the serial matrix exactly


def test_shard_rows_rules():
    from paper_2106_10860_b200.dist import shard_rows
    assert shard_rows(3, 8, 1 << 21, 1 << 20) == (3 << 21, 1 << 21, 6)
    with pytest.raises(ValueError):
        shard_rows(0, 2, 100, 64)
    with pytest.raises(ValueError):
        shard_rows(2, 2, 128, 64)
