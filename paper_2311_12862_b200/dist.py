"""Scene-sharded data-parallel training (BASELINE configs[3]).

A global batch of scans is dealt to ranks scene by scene (no collective
inside a layer: a layer does not shard naturally). Each rank runs the native
forward + chained backward (sk_net_forward / sk_net_backward) for its scans
and accumulates fp32 weight gradients in one flat buffer. For its last scan
the backward runs bucket by bucket in reverse layer order, and each finished
bucket is all-reduced asynchronously (NCCL over NVLink via torch.distributed),
so communication overlaps the remaining dgrad/wgrad. fp32 master weights take
an SGD-momentum step and are written back to the runner's fp16 weights.

With replicas=W > 1 a rank also keeps W NetworkRunners on its GPU (same
weights and configs, pipeline.replicate), each on its own host thread and CUDA
stream with its own fp32 gradient buffer: the rank's scenes are dealt to them
round-robin, so one runner's host syncs (output-coordinate counts) are filled
by the others' kernels. Their gradients are summed into the main buffer before
the main runner's last scene, whose bucketed backward still overlaps NCCL.

The bucketing / sharding / reduction logic is device-agnostic so it is
covered on CPU with gloo (tests/test_dist_cpu.py).
"""
from __future__ import annotations

import math
import threading
from dataclasses import dataclass

import torch
import torch.distributed as dist


def shard_scenes(voxel_counts, rank: int, world: int):
    """Greedy longest-processing-time bin packing of scenes by voxel count
    (load balance across ranks); deterministic, so every rank
    computes the same assignment. Returns this rank's scene indices."""
    order = sorted(range(len(voxel_counts)), key=lambda i: (-voxel_counts[i], i))
    load = [0] * world
    owner = [0] * len(voxel_counts)
    for i in order:
        r = min(range(world), key=lambda k: (load[k], k))
        owner[i] = r
        load[r] += voxel_counts[i]
    return [i for i in range(len(voxel_counts)) if owner[i] == rank]


@dataclass
class Bucket:
    layer_hi: int
    layer_lo: int
    off_lo: int   # flat fp32 range [off_lo, off_hi)
    off_hi: int


def make_buckets(layer_sizes, bucket_bytes: int = 25 << 20):
    """Reverse-layer-order buckets of about `bucket_bytes` fp32 gradients.
    layer_sizes[i] = #params of layer i (flat layout in layer order)."""
    offs = [0]
    for n in layer_sizes:
        offs.append(offs[-1] + n)
    buckets = []
    hi = len(layer_sizes) - 1
    while hi >= 0:
        lo, size = hi, layer_sizes[hi] * 4
        while lo > 0 and size + layer_sizes[lo - 1] * 4 <= bucket_bytes:
            lo -= 1
            size += layer_sizes[lo] * 4
        buckets.append(Bucket(hi, lo, offs[lo], offs[hi + 1]))
        hi = lo - 1
    return buckets


class GradReducer:
    """Async SUM all-reduce of flat-gradient buckets, averaged at wait()."""

    def __init__(self, grad: torch.Tensor, group=None):
        self.grad = grad
        self.group = group
        self.handles = []
        self.world = dist.get_world_size(group) if dist.is_initialized() else 1

    def launch(self, b: Bucket):
        if self.world > 1:
            self.handles.append(dist.all_reduce(self.grad[b.off_lo:b.off_hi],
                                                op=dist.ReduceOp.SUM, group=self.group,
                                                async_op=True))

    def wait(self, scale: float = 1.0):
        for h in self.handles:
            h.wait()
        self.handles.clear()
        if scale != 1.0:
            self.grad.mul_(scale)


class DataParallelTrainer:
    """Mixed-precision data-parallel trainer over a native NetworkRunner:
    fp16 activations / weights on the device, fp32 accumulate, fp32 master
    weights and gradients, SGD with momentum."""

    def __init__(self, net, lr: float = 1e-2, momentum: float = 0.9,
                 bucket_bytes: int = 25 << 20, group=None, replicas: int = 1):
        self.net = net
        from .pipeline import replicate
        self.nets = replicate(net, max(1, replicas))
        self.lr, self.momentum = lr, momentum
        self.group = group
        self.world = dist.get_world_size(group) if dist.is_initialized() else 1
        sizes = [kd * ci * co for (kd, ci, co, _) in net.layer_shapes]
        self.buckets = make_buckets(sizes, bucket_bytes)
        self.offsets = [off for (_, _, _, off) in net.layer_shapes]
        self.master = torch.cat([net.weight(i).float().flatten()
                                 for i in range(net.num_layers)]).contiguous()
        if self.world > 1:  # identical replicas: rank 0's weights everywhere
            dist.broadcast(self.master, src=0, group=group)
            self._push_weights()
        self.grad = torch.zeros_like(self.master)
        self.rgrads = [torch.zeros_like(self.master) for _ in self.nets[1:]]
        self.rstreams = [torch.cuda.Stream() for _ in self.nets[1:]]
        self.mom = torch.zeros_like(self.master)
        self.reducer = GradReducer(self.grad, group)

    def _push_weights(self):
        for n in self.nets:
            for i, (kd, ci, co, off) in enumerate(n.layer_shapes):
                n.weight(i).copy_(self.master[off:off + kd * ci * co].view(kd, ci, co))
            n.weights_updated()

    @staticmethod
    def _scene_grad(net, cs, x, tgt, global_batch):
        y, _ = net.forward(cs, x)
        diff = y.float() - tgt.float()
        return (diff * diff).mean(), (2.0 / (diff.numel() * global_batch)) * diff

    def _replica_scenes(self, r, scenes, global_batch, start, out):
        """Replica r >= 1: its scenes on its own stream into rgrads[r-1]."""
        try:
            torch.cuda.set_device(self.grad.device)
            st = self.rstreams[r - 1]
            with torch.cuda.stream(st):
                st.wait_event(start)
                loss = torch.zeros((), device="cuda")
                for k, (cs, x, tgt) in enumerate(scenes):
                    l, g = self._scene_grad(self.nets[r], cs, x, tgt, global_batch)
                    loss += l
                    self.nets[r].backward(g, self.rgrads[r - 1], accumulate=k > 0)
                out[r] = loss
        except BaseException as e:
            out[r] = e

    def train_step(self, scenes, global_batch: int):
        """scenes: this rank's [(CoordSet, feats, target)]; loss = mean over the
        global batch of per-scan mean squared error. Returns the local loss sum."""
        loss_sum = torch.zeros((), device="cuda")
        W = len(self.nets)
        if W > 1 and len(scenes) > 1:
            return self._train_step_replicas(scenes, global_batch)
        for si, (cs, x, tgt) in enumerate(scenes):
            y, _ = self.net.forward(cs, x)
            diff = y.float() - tgt.float()
            loss_sum += (diff * diff).mean()
            g = (2.0 / (diff.numel() * global_batch)) * diff
            last = si == len(scenes) - 1
            if not last:
                self.net.backward(g, self.grad, accumulate=si > 0)
                continue
            for b in self.buckets:  # reverse layer order, overlap with NCCL
                self.net.backward(g, self.grad, b.layer_hi, b.layer_lo, accumulate=si > 0)
                self.reducer.launch(b)
        if not scenes:  # an idle rank still joins every collective
            self.grad.zero_()
            for b in self.buckets:
                self.reducer.launch(b)
        self.reducer.wait()
        # SGD with momentum on the fp32 master copy
        self.mom.mul_(self.momentum).add_(self.grad)
        self.master.add_(self.mom, alpha=-self.lr)
        self._push_weights()
        return loss_sum

    def _train_step_replicas(self, scenes, global_batch: int):
        W = min(len(self.nets), len(scenes))
        mine = scenes[0::W]
        cur = torch.cuda.current_stream()
        start = torch.cuda.Event()
        start.record(cur)
        out = [None] * W
        th = [threading.Thread(target=self._replica_scenes,
                               args=(r, scenes[r::W], global_batch, start, out))
              for r in range(1, W)]
        for t in th:
            t.start()
        loss_sum = torch.zeros((), device="cuda")
        for si, (cs, x, tgt) in enumerate(mine[:-1]):  # concurrently with the replicas
            l, g = self._scene_grad(self.net, cs, x, tgt, global_batch)
            loss_sum += l
            self.net.backward(g, self.grad, accumulate=si > 0)
        for t in th:
            t.join()
        for r in range(1, W):
            if isinstance(out[r], BaseException):
                raise out[r]
            cur.wait_stream(self.rstreams[r - 1])
            loss_sum += out[r]
        # fold the replicas' gradients in, then the main runner's last scene
        # runs bucket by bucket with each finished bucket all-reduced
        if len(mine) == 1:
            self.grad.zero_()
        for rg in self.rgrads[:W - 1]:
            self.grad.add_(rg)
        cs, x, tgt = mine[-1]
        l, g = self._scene_grad(self.net, cs, x, tgt, global_batch)
        loss_sum += l
        for b in self.buckets:
            self.net.backward(g, self.grad, b.layer_hi, b.layer_lo, accumulate=True)
            self.reducer.launch(b)
        self.reducer.wait()
        self.mom.mul_(self.momentum).add_(self.grad)
        self.master.add_(self.mom, alpha=-self.lr)
        self._push_weights()
        return loss_sum
