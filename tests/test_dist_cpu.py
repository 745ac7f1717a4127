"""World-size-2 gloo test of the multi-GPU host path (sharding + end-of-run
gathers); the decode hot path itself has no collective."""

import os
import socket

import pytest
import torch.multiprocessing as mp

from paper_2512_01278_b200.dist import shard_bounds, shard_ids


def test_shards_partition_requests():
    for n in (0, 1, 7, 128, 512):
        for world in (1, 2, 3, 4, 8):
            ids = [i for r in range(world) for i in shard_ids(n, r, world)]
            assert ids == list(range(n))
            sizes = [len(shard_ids(n, r, world)) for r in range(world)]
            assert max(sizes) - min(sizes) <= 1


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, q):
    import torch.distributed as dist

    from paper_2512_01278_b200.dist import gather_outputs, gather_throughput, shard_ids
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    ids = shard_ids(10, rank, world)
    outs = {i: [i, i + 1] for i in ids}          # stand-in for per-request token streams
    tok, sec = gather_throughput(len(ids) * 100.0, 1.0 + rank, device="cpu")
    merged = gather_outputs(outs)
    if rank == 0:
        q.put((tok, sec, sorted(merged)))
    dist.barrier()
    dist.destroy_process_group()


def test_gloo_world2_gather():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    tok, sec, ids = q.get(timeout=120)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    assert tok == 1000.0          # all requests counted once
    assert sec == 2.0             # max over ranks
    assert ids == list(range(10))
