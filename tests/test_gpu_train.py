"""Data-parallel trainer on one GPU (world 1): gradients equal the plain
chained backward summed over scans, and SGD steps reduce the loss."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def test_trainer_step(reference):
    import torch
    from paper_2311_12862_b200 import sparse as sk
    from paper_2311_12862_b200.dist import DataParallelTrainer
    from paper_2311_12862_b200.models import toy_unet
    from paper_2311_12862_b200.network import NetworkRunner
    from paper_2311_12862_b200.synth import planar_patches, quantize

    net = NetworkRunner(toy_unet(), dtype=torch.float16, weight_seed=5)
    net.set_all(sk.DataflowConfig(sk.IMPLICIT_GEMM, 1))
    scenes = []
    for s in range(3):
        c = quantize(planar_patches(3000, 10 + s, 1.0), [0.05] * 3)
        cs = sk.CoordSet.create(c)
        x = torch.randn(cs.n, 1, device="cuda").half()
        tgt = torch.randn(cs.n, 2, device="cuda").half()
        scenes.append((cs, x, tgt))
    # reference gradient: independent backward per scan, summed
    ref = torch.zeros(net.num_params, device="cuda")
    for cs, x, tgt in scenes:
        y, _ = net.forward(cs, x)
        d = y.float() - tgt.float()
        g = torch.zeros(net.num_params, device="cuda")
        net.backward((2.0 / (d.numel() * 3)) * d, g)
        ref += g
    tr = DataParallelTrainer(net, lr=0.0, momentum=0.0)
    tr.train_step(scenes, global_batch=3)
    torch.cuda.synchronize()
    assert torch.allclose(tr.grad, ref, rtol=1e-3, atol=1e-6)
    tr.lr = 0.05
    losses = [float(tr.train_step(scenes, global_batch=3)) for _ in range(6)]
    assert losses[-1] < losses[0]


@pytest.mark.parametrize("replicas", [2, 3])
def test_trainer_replicas_match_single(replicas):
    """replicas=W (W runners on W threads/streams, gradients folded before the
    last scene) computes the same gradient and update as one runner."""
    import torch
    from paper_2311_12862_b200 import sparse as sk
    from paper_2311_12862_b200.dist import DataParallelTrainer
    from paper_2311_12862_b200.models import toy_unet
    from paper_2311_12862_b200.network import NetworkRunner
    from paper_2311_12862_b200.synth import planar_patches, quantize

    def make():
        net = NetworkRunner(toy_unet(), dtype=torch.float16, weight_seed=5)
        net.set_all(sk.DataflowConfig(sk.IMPLICIT_GEMM, 1))
        return net
    g = torch.Generator().manual_seed(0)
    data = []
    for s in range(5):
        c = quantize(planar_patches(3000, 20 + s, 1.0), [0.05] * 3)
        x = torch.randn(len(c), 1, generator=g).half()
        tgt = torch.randn(len(c), 2, generator=g).half()
        data.append((c, x, tgt))

    def scenes():
        return [(sk.CoordSet.create(c), x.cuda(), t.cuda()) for c, x, t in data]
    one = DataParallelTrainer(make(), lr=0.05, momentum=0.9)
    many = DataParallelTrainer(make(), lr=0.05, momentum=0.9, replicas=replicas)
    for _ in range(2):
        l1 = float(one.train_step(scenes(), global_batch=5))
        lw = float(many.train_step(scenes(), global_batch=5))
        torch.cuda.synchronize()
        assert abs(l1 - lw) <= 1e-3 * abs(l1)
        assert torch.allclose(one.grad, many.grad, rtol=1e-3, atol=1e-6)
        assert torch.allclose(one.master, many.master, rtol=1e-4, atol=1e-6)
    for n in many.nets[1:]:  # every replica carries the updated weights
        for i in range(n.num_layers):
            assert torch.equal(n.weight(i), many.net.weight(i))
