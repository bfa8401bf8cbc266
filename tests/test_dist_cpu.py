"""Host-side data-parallel logic on CPU with gloo (world_size 2): scene
sharding, reverse-order gradient buckets and bucketed SUM all-reduce."""
import os
import socket

import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2311_12862_b200.dist import GradReducer, make_buckets, shard_scenes


def test_shard_scenes_balanced_and_complete():
    counts = [120_000, 90_000, 130_000, 60_000, 125_000, 110_000, 70_000, 100_000]
    for world in (1, 2, 4, 8):
        parts = [shard_scenes(counts, r, world) for r in range(world)]
        assert sorted(i for p in parts for i in p) == list(range(len(counts)))
        loads = [sum(counts[i] for i in p) for p in parts]
        assert max(loads) - min(loads) <= max(counts)
    assert shard_scenes(counts, 0, 8) != shard_scenes(counts, 1, 8)


def test_buckets_reverse_contiguous():
    sizes = [27 * 4 * 32, 27 * 32 * 32, 32 * 32, 27 * 32 * 64, 27 * 64 * 64, 64 * 64]
    offs = [0]
    for s in sizes:
        offs.append(offs[-1] + s)
    b = make_buckets(sizes, bucket_bytes=200_000)
    assert b[0].layer_hi == len(sizes) - 1 and b[-1].layer_lo == 0
    covered = []
    for x in b:
        assert x.off_lo == offs[x.layer_lo] and x.off_hi == offs[x.layer_hi + 1]
        covered += list(range(x.layer_lo, x.layer_hi + 1))
    assert sorted(covered) == list(range(len(sizes)))
    for a, c in zip(b, b[1:]):
        assert c.layer_hi == a.layer_lo - 1  # reverse order, no gaps
    assert len(make_buckets(sizes, bucket_bytes=1 << 30)) == 1


def _worker(rank, world, port, out):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    sizes = [10, 7, 13, 5]
    grad = torch.arange(sum(sizes), dtype=torch.float32) * (rank + 1)
    red = GradReducer(grad)
    for b in make_buckets(sizes, bucket_bytes=60):
        red.launch(b)
    red.wait(scale=1.0 / world)
    out[rank] = grad.tolist()
    dist.destroy_process_group()


def test_bucketed_allreduce_gloo_world2():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    mgr = mp.Manager()
    out = mgr.dict()
    mp.spawn(_worker, args=(2, port, out), nprocs=2, join=True)
    n = 35
    want = [float(i) * (1 + 2) / 2 for i in range(n)]
    assert out[0] == pytest.approx(want) and out[1] == pytest.approx(want)
