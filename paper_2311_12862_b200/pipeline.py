"""Scan serving pipeline: host scans in, host features out, with the PCIe
copies overlapped with the network on their own CUDA streams.

The reference serves a scan as copy-in -> NetworkRunner::forward -> copy-out
on one thread (its benches call forward on resident tensors).
On a B200 the copy-out of MinkUNet-18's 96-channel fp16 output (~25 MB per
scan) costs ~0.5 ms at PCIe rate, an eighth of the forward, so serving runs
three streams:

  copy-in  stream: H2D of scan i+1's coordinates and features into one of
                   `depth` device slots while scan i computes
  compute  stream: (the caller's current stream) CoordSet.create + forward
  copy-out stream: D2H of scan i's output into one of `depth` pinned host
                   slots while scan i+1 computes

Events order the slots: a device input slot is refilled only after the
forward that read it finished, a host output slot is overwritten only after
its previous result was handed to the caller.
"""
from __future__ import annotations

import torch

from . import sparse as _sk


class ScanPipeline:
    def __init__(self, net, max_voxels: int, c_in: int, depth: int = 2):
        self.net = net
        self.depth = depth
        self.max_voxels = max_voxels
        dt = net.dtype
        c_out = net.layer_shapes[-1][2]
        self.s_in = torch.cuda.Stream()
        self.s_out = torch.cuda.Stream()
        self.d_c = [torch.empty((max_voxels, 4), dtype=torch.int32, device="cuda")
                    for _ in range(depth)]
        self.d_f = [torch.empty((max_voxels, c_in), dtype=dt, device="cuda") for _ in range(depth)]
        self.h_out = [torch.empty((max_voxels, c_out), dtype=dt).pin_memory() for _ in range(depth)]
        self.ev_in = [torch.cuda.Event() for _ in range(depth)]
        self.ev_used = [None] * depth
        self.ev_out = [torch.cuda.Event() for _ in range(depth)]
        self.d2h_bytes = 0
        self.h2d_bytes = 0

    def _stage_in(self, slot: int, coords: torch.Tensor, feats: torch.Tensor) -> None:
        n = coords.shape[0]
        if n > self.max_voxels:
            raise _sk.ValidationError("scan larger than the pipeline's max_voxels")
        if self.ev_used[slot] is not None:
            self.s_in.wait_event(self.ev_used[slot])
        with torch.cuda.stream(self.s_in):
            self.d_c[slot][:n].copy_(coords, non_blocking=True)
            self.d_f[slot][:n].copy_(feats, non_blocking=True)
        self.ev_in[slot].record(self.s_in)
        self.h2d_bytes += coords.numel() * coords.element_size() + feats.numel() * feats.element_size()

    def run(self, scans, on_result=None, before_scan=None) -> None:
        """scans: sequence of (coords int32 [n, 4], feats [n, c_in] in the
        runner's dtype), pinned host tensors. on_result(i, host_view) gets scan
        i's [n, c_out] output once it is on the host (the view is valid until
        the callback returns). before_scan(i) runs on the compute stream ahead
        of scan i's work (benches flush L2 there). Returns after every output
        copy is enqueued; the caller's stream waits for them."""
        cur = torch.cuda.current_stream()
        self.s_in.wait_stream(cur)  # staging starts after the caller's prior work
        n_scans = len(scans)
        pending = []  # (i, slot, n) whose D2H is in flight

        def deliver(upto: int) -> None:
            while pending and pending[0][0] <= upto:
                j, sl, nj = pending.pop(0)
                if on_result is not None:
                    self.ev_out[sl].synchronize()
                    on_result(j, self.h_out[sl][:nj])

        if n_scans:
            self._stage_in(0, *scans[0])
        for i in range(n_scans):
            slot = i % self.depth
            if i + 1 < n_scans:
                self._stage_in((i + 1) % self.depth, *scans[i + 1])
            if before_scan is not None:
                before_scan(i)
            cur.wait_event(self.ev_in[slot])
            n = scans[i][0].shape[0]
            cs = _sk.CoordSet.create(self.d_c[slot][:n])
            y, _ = self.net.forward(cs, self.d_f[slot][:n])
            ev = torch.cuda.Event()
            ev.record(cur)
            self.ev_used[slot] = ev
            deliver(i - self.depth)  # host slot `slot` is free again
            self.s_out.wait_event(ev)
            with torch.cuda.stream(self.s_out):
                self.h_out[slot][:n].copy_(y, non_blocking=True)
            y.record_stream(self.s_out)
            self.ev_out[slot].record(self.s_out)
            self.d2h_bytes += y.numel() * y.element_size()
            pending.append((i, slot, n))
        deliver(n_scans)
        cur.wait_stream(self.s_out)
