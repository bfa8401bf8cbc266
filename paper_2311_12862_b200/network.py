"""NetworkRunner / tuner mirror (network.hpp:81-119, tuner.hpp:15-94) over the
native sk_net runtime in libsk200.so.

The per-layer dispatch loop, map caches, timing split, chained backward and
the greedy group tuner all run in C++ (csrc/network.cu); this class only owns
the handle and moves tensors.
"""
from __future__ import annotations

import ctypes as C
import math

import numpy as np
import torch

from . import _lib
from ._lib import DataflowCfg, ValidationError, check, lib
from .models import spec_text
from .sparse import (Context, CoordSet, DataflowConfig, TilePreset, _DTYPES, _ptr, _stream)

PHASES = {"forward": 0, "dgrad": 1, "wgrad": 2}


class _CudaArray:
    def __init__(self, ptr, shape, typestr):
        self.__cuda_array_interface__ = {"shape": tuple(shape), "typestr": typestr,
                                         "data": (int(ptr), False), "version": 3,
                                         "strides": None}


def device_view(ptr, shape, dtype) -> torch.Tensor:
    """Zero-copy torch tensor over library-owned device memory."""
    if int(np.prod(shape)) == 0:
        return torch.empty(shape, dtype=dtype, device="cuda")
    if dtype == torch.bfloat16:
        return torch.as_tensor(_CudaArray(ptr, shape, "<i2"), device="cuda").view(torch.bfloat16)
    ts = {torch.float16: "<f2", torch.float32: "<f4"}[dtype]
    return torch.as_tensor(_CudaArray(ptr, shape, ts), device="cuda")


def cfg_from_c(c: DataflowCfg) -> DataflowConfig:
    t = c.tile
    return DataflowConfig(c.kind, c.splits,
                          TilePreset(t.cta_m, t.cta_n, t.cta_k, t.warp_rows, t.load_width),
                          c.reorder)


def default_space():
    """default_space (tuner.cpp:9-26) as the C++ tuner enumerates it."""
    out = []
    for i in range(lib().sk_tune_space_size()):
        c = DataflowCfg()
        check(lib().sk_tune_space_entry(i, C.byref(c)))
        out.append(cfg_from_c(c))
    return out


class NetworkRunner:
    def __init__(self, layers, dims: int = 3, dtype=torch.float16, ctx: Context | None = None,
                 weight_seed: int | None = 3):
        self.ctx = ctx or Context.get()
        self.dims = dims
        self.dtype = dtype
        self.layers = list(layers)
        self.spec = spec_text(self.layers)
        p = C.c_void_p()
        check(lib().sk_net_create(self.ctx.ptr, dims, self.spec.encode(), _DTYPES[dtype],
                                  C.byref(p)))
        self.ptr = p
        self.num_layers = lib().sk_net_num_layers(p)
        self.num_groups = lib().sk_net_num_groups(p)
        self.layer_shapes = []
        for i in range(self.num_layers):
            kd, ci, co, off = C.c_int(), C.c_int(), C.c_int(), C.c_int64()
            check(lib().sk_net_layer_info(p, i, C.byref(kd), C.byref(ci), C.byref(co),
                                          C.byref(off)))
            self.layer_shapes.append((kd.value, ci.value, co.value, off.value))
        self.num_params = lib().sk_net_num_params(p)
        if weight_seed is not None:
            self.init_weights(weight_seed)

    def __del__(self):
        try:
            if self.ptr:
                lib().sk_net_destroy(self.ptr)
                self.ptr = None
        except Exception:
            pass

    # ---- structure ----
    def group_of_layer(self, i: int) -> int:
        return lib().sk_net_group_of_layer(self.ptr, i)

    def groups(self):
        g = [[] for _ in range(self.num_groups)]
        for i in range(self.num_layers):
            g[self.group_of_layer(i)].append(i)
        return g

    # ---- weights ----
    def weight(self, i: int) -> torch.Tensor:
        """Zero-copy torch view of layer i's device weights [K^D, c_in, c_out]."""
        kd, ci, co, _ = self.layer_shapes[i]
        p = C.c_void_p()
        check(lib().sk_net_weight_ptr(self.ptr, i, C.byref(p)))
        return device_view(p.value, (kd, ci, co), self.dtype)

    def set_weight(self, i: int, w: torch.Tensor) -> None:
        self.weight(i).copy_(w.to(device="cuda", dtype=self.dtype))

    def init_weights(self, seed: int = 3) -> None:
        """N(0, 1/sqrt(K^D c_in)) timing weights."""
        g = torch.Generator().manual_seed(seed)
        for i, (kd, ci, co, _) in enumerate(self.layer_shapes):
            self.set_weight(i, torch.randn(kd, ci, co, generator=g) / math.sqrt(kd * ci))

    # ---- configs ----
    def set_config(self, group: int, cfg: DataflowConfig, phase: str = "forward") -> None:
        check(lib().sk_net_set_config(self.ptr, group, PHASES[phase], C.byref(cfg.c())))

    def set_all(self, cfg: DataflowConfig, phases=("forward", "dgrad", "wgrad")) -> None:
        for g in range(self.num_groups):
            for ph in phases:
                self.set_config(g, cfg, ph)

    def config(self, group: int, phase: str = "forward") -> DataflowConfig:
        c = DataflowCfg()
        check(lib().sk_net_get_config(self.ptr, group, PHASES[phase], C.byref(c)))
        return cfg_from_c(c)

    # ---- execution ----
    def forward(self, coords: CoordSet, feats: torch.Tensor, stats: bool = False,
                out: torch.Tensor | None = None):
        """NetworkRunner::forward; returns (features [n_out, c_out] torch copy, stats).
        out: optional preallocated [>= n_out, c_out] device tensor the result is
        copied into (on the current stream) instead of a fresh allocation."""
        feats = feats.to(device="cuda", dtype=self.dtype).contiguous()
        out_p, n_out = C.c_void_p(), C.c_int()
        mp = np.zeros(self.num_groups) if stats else None
        kr = np.zeros(self.num_groups) if stats else None
        check(lib().sk_net_forward(self.ptr, coords.ptr, _ptr(feats), feats.shape[1], _stream(),
                                   C.byref(out_p), C.byref(n_out),
                                   mp.ctypes.data_as(C.c_void_p) if stats else None,
                                   kr.ctypes.data_as(C.c_void_p) if stats else None))
        self._last_in = feats
        co = self.layer_shapes[-1][2]
        if out is not None:
            if out.shape[0] < n_out.value or out.shape[1] != co or out.dtype != self.dtype:
                raise ValidationError("out must be [>= n_out, c_out] in the runner's dtype")
            y = out[:n_out.value]
            y.copy_(device_view(out_p.value, (n_out.value, co), self.dtype))
        else:
            y = self._wrap(out_p.value, n_out.value, co)
        return y, ({"mapping_ms": mp, "kernel_ms": kr} if stats else None)

    def _wrap(self, ptr, rows, cols):
        # copy out of the library-owned buffer (valid until the next forward)
        return device_view(ptr, (rows, cols), self.dtype).clone()

    def forward_profiled(self, coords: CoordSet, feats: torch.Tensor):
        """Per-layer GPU ms (CUDA events, no per-layer sync) and map-build ms."""
        feats = feats.to(device="cuda", dtype=self.dtype).contiguous()
        lm = np.zeros(self.num_layers)
        mp = C.c_double()
        check(lib().sk_net_forward_profiled(self.ptr, coords.ptr, _ptr(feats), feats.shape[1],
                                            _stream(), lm.ctypes.data_as(C.c_void_p),
                                            C.byref(mp)))
        return lm, mp.value

    def layer_output(self, i: int) -> torch.Tensor:
        p, rows = C.c_void_p(), C.c_int()
        check(lib().sk_net_layer_output(self.ptr, i, C.byref(p), C.byref(rows)))
        return self._wrap(p.value, rows.value, self.layer_shapes[i][2])

    def measure_ms(self, coords: CoordSet, feats: torch.Tensor, forward=True, dgrad=False,
                   wgrad=False) -> float:
        feats = feats.to(device="cuda", dtype=self.dtype).contiguous()
        ms = C.c_double()
        check(lib().sk_net_measure(self.ptr, coords.ptr, _ptr(feats), feats.shape[1],
                                   int(forward), int(dgrad), int(wgrad), _stream(), C.byref(ms)))
        return ms.value

    def set_overlap(self, on: bool) -> None:
        """Overlapped map build (sk_net_set_overlap; default on)."""
        check(lib().sk_net_set_overlap(self.ptr, int(bool(on))))

    def set_pdl(self, on: bool) -> None:
        """Programmatic dependent launch of the runner's kernels (sk_net_set_pdl; default on)."""
        check(lib().sk_net_set_pdl(self.ptr, int(bool(on))))

    def set_tune_cold(self, on: bool) -> None:
        """Tuner probes on fresh copies of the tuning set, so map preparation
        is timed with each candidate (sk_net_set_tune_cold; default off)."""
        check(lib().sk_net_set_tune_cold(self.ptr, int(bool(on))))

    def map_build_count(self) -> int:
        return lib().sk_net_map_builds(self.ptr)

    def modeled_group_traffic(self, group: int, cfg: DataflowConfig) -> float:
        b = C.c_double()
        check(lib().sk_net_group_traffic(self.ptr, group, C.byref(cfg.c()), _stream(),
                                         C.byref(b)))
        return b.value

    def backward(self, grad_out: torch.Tensor, wgrad: torch.Tensor, layer_hi: int | None = None,
                 layer_lo: int = 0, accumulate: bool = False) -> None:
        """Chained backward of the last forward into the flat fp32 `wgrad`
        (layers [layer_lo, layer_hi]; the first call must start at the last layer)."""
        hi = self.num_layers - 1 if layer_hi is None else layer_hi
        g = grad_out.to(device="cuda", dtype=self.dtype).contiguous()
        assert wgrad.dtype == torch.float32 and wgrad.numel() == self.num_params
        check(lib().sk_net_backward(self.ptr, _ptr(g), _ptr(wgrad), hi, layer_lo, int(accumulate),
                                    _stream()))
        self._grad_keep = g

    def weights_updated(self) -> None:
        """Mark the device weights as changed (e.g. written through weight(i))."""
        p = C.c_void_p()
        check(lib().sk_net_weight_ptr(self.ptr, 0, C.byref(p)))

    def weight_grad(self, wgrad: torch.Tensor, i: int) -> torch.Tensor:
        kd, ci, co, off = self.layer_shapes[i]
        return wgrad[off:off + kd * ci * co].view(kd, ci, co)

    def tune(self, coords: CoordSet, feats: torch.Tensor, training: int = 0, warmup: int = 2,
             runs: int = 5):
        """tune_inference (training=0) / tune_training (1 = workload_pattern,
        2 = sparse_mapping); leaves the winning configs installed."""
        feats = feats.to(device="cuda", dtype=self.dtype).contiguous()
        cap = 2 * self.num_groups * 32
        log = np.zeros((cap, 4), np.float64)
        lat, n = C.c_double(), C.c_int()
        check(lib().sk_net_tune(self.ptr, coords.ptr, _ptr(feats), feats.shape[1], training,
                                warmup, runs, _stream(), C.byref(lat),
                                log.ctypes.data_as(C.c_void_p), cap, C.byref(n)))
        return lat.value, log[: min(n.value, cap)]
