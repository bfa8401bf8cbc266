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
