"""Scene-sharded data parallelism through the engine: two
ranks share the one metered B200 (gloo over CUDA tensors stands in for NCCL;
the bucket / broadcast / all-reduce calls are the same torch.distributed
calls the NCCL run makes) and run DataParallelTrainer.train_step end to end:
native forward, bucketed chained backward interleaved with async all-reduce,
SGD on fp32 master weights.

* 4 scenes over 2 ranks: both ranks' master weights are identical and equal
  a world-1 trainer that saw all 4 scenes (to 1e-5);
* 1 scene over 2 ranks: the idle rank still joins the rank-0 broadcast and
  every bucket all-reduce, and both ranks equal the world-1 trainer.
"""
import os
import socket

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _scenes(n_scenes):
    from paper_2311_12862_b200.synth import planar_patches, quantize
    out = []
    for i in range(n_scenes):
        c = quantize(planar_patches(4000 + 700 * i, 50 + i, 1.0), [0.05] * 3)
        rng = np.random.default_rng(100 + i)
        out.append((c, rng.standard_normal((len(c), 4)).astype(np.float16),
                    rng.standard_normal((len(c), 96)).astype(np.float16)))
    return out


def _worker(rank, world, port, n_scenes, steps, out):
    import torch
    import torch.distributed as dist
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    torch.cuda.set_device(0)
    if world > 1:
        dist.init_process_group("gloo", rank=rank, world_size=world)
    from paper_2311_12862_b200 import models as M, sparse as sk
    from paper_2311_12862_b200.dist import DataParallelTrainer, shard_scenes
    from paper_2311_12862_b200.network import NetworkRunner
    # ranks start from DIFFERENT weights: the trainer's rank-0 broadcast must
    # make them identical
    net = NetworkRunner(M.minkunet18(), dtype=torch.float16, weight_seed=3 + rank)
    net.set_all(sk.DataflowConfig(sk.IMPLICIT_GEMM, 1, sk.tile_large()))
    tr = DataParallelTrainer(net, lr=1e-2, momentum=0.9, bucket_bytes=4 << 20)
    assert len(tr.buckets) > 1  # several bucket collectives per step
    scenes = _scenes(n_scenes)
    mine = shard_scenes([len(c) for c, _, _ in scenes], rank, world)
    losses = []
    for _ in range(steps):
        batch = [(sk.CoordSet.create(scenes[i][0]), torch.from_numpy(scenes[i][1]).cuda(),
                  torch.from_numpy(scenes[i][2]).cuda()) for i in mine]
        losses.append(float(tr.train_step(batch, n_scenes)))
    torch.cuda.synchronize()
    out[rank] = (tr.master.cpu().numpy(), mine, losses)
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()


def _run(world, n_scenes, steps=2):
    import torch.multiprocessing as mp
    mgr = mp.Manager()
    out = mgr.dict()
    mp.spawn(_worker, args=(world, _free_port(), n_scenes, steps, out), nprocs=world, join=True)
    return dict(out)


def _rel(a, b):
    return float(np.max(np.abs(a - b)) / max(1.0, float(np.max(np.abs(b)))))


@pytest.mark.parametrize("n_scenes", [4, 1])
def test_two_ranks_match_single_rank(n_scenes):
    two = _run(2, n_scenes)
    one = _run(1, n_scenes)
    w0, mine0, l0 = two[0]
    w1, mine1, l1 = two[1]
    assert sorted(mine0 + mine1) == list(range(n_scenes))
    if n_scenes == 1:
        assert mine1 == [] or mine0 == []  # one idle rank
    assert np.array_equal(w0, w1)  # identical replicas after every step
    w_ref = one[0][0]
    assert _rel(w0, w_ref) <= 1e-5, _rel(w0, w_ref)
    assert np.isfinite(w0).all()
    # the losses the ranks report sum to the world-1 loss of the same step
    assert abs(sum(l0[:1]) + sum(l1[:1]) - one[0][2][0]) <= 1e-3 * max(1.0, abs(one[0][2][0]))
