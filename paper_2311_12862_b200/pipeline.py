"""Scan serving pipeline: host scans in, host features out, with the PCIe
copies overlapped with the network and several scans in flight.

The reference serves a scan as copy-in -> NetworkRunner::forward -> copy-out
on one thread (its benches call forward on resident tensors).
On a B200 two things leave the GPU idle in that loop: the copy-out of
MinkUNet-18's 96-channel fp16 output (~25 MB per scan, ~0.5 ms at PCIe
rate), and the host syncs inside a forward (output-coordinate counts size the
next layer's buffers), during which the device drains and waits for the host.
So the pipeline runs W workers, each a host thread with its own
NetworkRunner (same weights and dataflow configs) and three CUDA streams:

  copy-in  stream: H2D of the worker's next scan into one of `depth` device
                   slots while its current scan computes
  compute  stream: CoordSet.create + forward (the host thread blocks here at
                   the forward's syncs; the other workers' kernels fill the gap)
  copy-out stream: D2H of the worker's previous scan into one of `depth`
                   pinned host slots while the current scan computes

Scan i goes to worker i % W. Events order the slots: a device input slot is
refilled only after the forward that read it finished, a host output slot is
overwritten only after its previous result was handed to the caller.
"""
from __future__ import annotations

import threading

import torch

from . import sparse as _sk


def replicate(net, count: int):
    """`count` runners: `net` plus copies with its weights and per-group,
    per-phase dataflow configs (so a tuned runner can serve as W workers).
    With count > 1 every runner's overlapped map build and programmatic
    dependent launch are switched off (early-resident CTAs would hold shared
    memory the other runners' kernels need: -7 % scans/s at 6 in flight); the
    other runners in flight fill the sync bubbles it hides, and its extra
    stream and helper thread cost more than they save (MinkUNet, 4 in flight:
    2.08 vs 1.88 ms/scan)."""
    from .network import NetworkRunner
    out = [net]
    if count > 1:
        net.set_overlap(False)
        net.set_pdl(False)
    for _ in range(count - 1):
        r = NetworkRunner(net.layers, dtype=net.dtype, dims=net.dims, ctx=net.ctx, weight_seed=None)
        for i in range(net.num_layers):
            r.set_weight(i, net.weight(i))
        for g in range(net.num_groups):
            for ph in ("forward", "dgrad", "wgrad"):
                r.set_config(g, net.config(g, ph), ph)
        r.set_overlap(False)
        r.set_pdl(False)
        out.append(r)
    return out


class _Worker:
    def __init__(self, net, max_voxels, c_in, depth, stream=None):
        self.net = net
        self.depth = depth
        dt = net.dtype
        c_out = net.layer_shapes[-1][2]
        self.s_cmp = stream if stream is not None else torch.cuda.Stream()
        self.s_in = torch.cuda.Stream()
        self.s_out = torch.cuda.Stream()
        self.d_c = [torch.empty((max_voxels, 4), dtype=torch.int32, device="cuda")
                    for _ in range(depth)]
        self.d_f = [torch.empty((max_voxels, c_in), dtype=dt, device="cuda") for _ in range(depth)]
        self.d_out = [torch.empty((max_voxels, c_out), dtype=dt, device="cuda")
                      for _ in range(depth)]
        self.h_out = [torch.empty((max_voxels, c_out), dtype=dt).pin_memory() for _ in range(depth)]
        self.ev_in = [torch.cuda.Event() for _ in range(depth)]
        self.cs = [None] * depth
        self.ev_used = [None] * depth
        self.ev_out = [torch.cuda.Event() for _ in range(depth)]
        self.d2h_bytes = 0
        self.h2d_bytes = 0
        self.error = None
        self.device = torch.cuda.current_device()

    def _stage_in(self, slot, coords, feats):
        if self.ev_used[slot] is not None:
            self.s_in.wait_event(self.ev_used[slot])
        n = coords.shape[0]
        with torch.cuda.stream(self.s_in):
            self.d_c[slot][:n].copy_(coords, non_blocking=True)
            self.d_f[slot][:n].copy_(feats, non_blocking=True)
            # the coordinate set (hash insert + its validation read-back) is
            # built on the copy-in stream: the read-back then waits for this
            # scan's H2D only, not for the previous forward on the compute stream
            self.cs[slot] = _sk.CoordSet.create(self.d_c[slot][:n])
        self.ev_in[slot].record(self.s_in)
        self.h2d_bytes += coords.numel() * coords.element_size() + feats.numel() * feats.element_size()

    def run(self, start_ev, jobs, on_result, before_scan):
        """jobs: list of (global index, (coords, feats))."""
        try:
            torch.cuda.set_device(self.device)  # worker threads start on device 0
            self.s_cmp.wait_event(start_ev)
            self.s_in.wait_event(start_ev)
            pending = []

            def deliver(upto):
                while pending and pending[0][0] <= upto:
                    k, j, sl, nj = pending.pop(0)
                    if on_result is not None:
                        self.ev_out[sl].synchronize()
                        on_result(j, self.h_out[sl][:nj])

            if jobs:
                self._stage_in(0, *jobs[0][1])
            with torch.cuda.stream(self.s_cmp):
                for k, (j, (coords, feats)) in enumerate(jobs):
                    slot = k % self.depth
                    if k + 1 < len(jobs):
                        self._stage_in((k + 1) % self.depth, *jobs[k + 1][1])
                    if before_scan is not None:
                        before_scan(j)
                    self.s_cmp.wait_event(self.ev_in[slot])
                    n = coords.shape[0]
                    cs, self.cs[slot] = self.cs[slot], None
                    # the device output slot is free once its previous D2H landed
                    self.s_cmp.wait_event(self.ev_out[slot])
                    y, _ = self.net.forward(cs, self.d_f[slot][:n], out=self.d_out[slot])
                    ev = torch.cuda.Event()
                    ev.record(self.s_cmp)
                    self.ev_used[slot] = ev
                    deliver(k - self.depth)  # host slot `slot` is free again
                    m = y.shape[0]  # output rows (a strided network returns fewer)
                    self.s_out.wait_event(ev)
                    with torch.cuda.stream(self.s_out):
                        self.h_out[slot][:m].copy_(y, non_blocking=True)
                    self.ev_out[slot].record(self.s_out)
                    self.d2h_bytes += y.numel() * y.element_size()
                    pending.append((k, j, slot, m))
            deliver(len(jobs))
        except BaseException as e:  # surfaced by ScanPipeline.run
            self.error = e


class ScanPipeline:
    def __init__(self, nets, max_voxels: int, c_in: int, depth: int = 2, streams=None):
        """nets: one NetworkRunner or a list (one worker thread per runner;
        see replicate()). streams: optional compute stream per runner (reusing
        the streams a runner already ran on reuses its cached device blocks)."""
        if depth < 2:
            # scan k+1 is staged while scan k's forward is still to be enqueued:
            # one slot would overwrite scan k's inputs
            raise _sk.ValidationError("ScanPipeline depth must be >= 2")
        if not isinstance(nets, (list, tuple)):
            nets = [nets]
        self.max_voxels = max_voxels
        streams = streams or [None] * len(nets)
        self.workers = [_Worker(n, max_voxels, c_in, depth, s) for n, s in zip(nets, streams)]

    @property
    def d2h_bytes(self) -> int:
        return sum(w.d2h_bytes for w in self.workers)

    @property
    def h2d_bytes(self) -> int:
        return sum(w.h2d_bytes for w in self.workers)

    def reset_counters(self) -> None:
        for w in self.workers:
            w.d2h_bytes = w.h2d_bytes = 0

    def run(self, scans, on_result=None, before_scan=None) -> None:
        """scans: sequence of (coords int32 [n, 4], feats [n, c_in] in the
        runners' dtype), pinned host tensors. on_result(i, host_view) gets scan
        i's [n, c_out] output once it is on the host (from the worker thread
        that ran it; the view is valid until the callback returns). before_scan(i)
        runs on the worker's compute stream ahead of scan i (benches flush L2
        there). Returns when every scan is enqueued; the caller's stream waits
        for all outputs."""
        for c, _ in scans:
            if c.shape[0] > self.max_voxels:
                raise _sk.ValidationError("scan larger than the pipeline's max_voxels")
        cur = torch.cuda.current_stream()
        start = torch.cuda.Event()
        start.record(cur)
        W = len(self.workers)
        jobs = [[(i, scans[i]) for i in range(w, len(scans), W)] for w in range(W)]
        if W == 1:
            self.workers[0].run(start, jobs[0], on_result, before_scan)
        else:
            th = [threading.Thread(target=wk.run, args=(start, jobs[w], on_result, before_scan))
                  for w, wk in enumerate(self.workers)]
            for t in th:
                t.start()
            for t in th:
                t.join()
        for wk in self.workers:
            if wk.error is not None:
                e, wk.error = wk.error, None
                raise e
            cur.wait_stream(wk.s_cmp)
            cur.wait_stream(wk.s_out)
