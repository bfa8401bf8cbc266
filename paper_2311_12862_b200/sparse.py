"""Host-side mirror of the sparsekit operator API over the sk200 C ABI.

Names follow the reference (namespace sparsekit, /root/reference/proj):

  CoordSet          coordinate half of SparseTensor (tensor.hpp:86-115) + its
                    CoordLookup hash (tensor.hpp:118-130), device resident
  build_out_coords  kmap.cpp:73-94
  build_kmap        build_kmap_os / build_kmap_ws (kmap.cpp:96-143)
  KernelMap         KernelMapOS / KernelMapWS views (kmap.hpp:40-93),
                    split_and_sort / pad_map via prepare() (kmap.cpp:211-288),
                    transpose_map (kmap.cpp:290-315)
  DataflowConfig    exec.hpp:65-73 (+ TilePreset, exec.hpp:46-54)
  conv_forward / conv_dgrad / conv_wgrad   exec.hpp:105-124

Tensors are torch CUDA tensors (PyTorch is the device-memory/stream plumbing);
every call is ordered on torch's current stream. Errors raise
ValidationError / ContractError like the reference.
"""
from __future__ import annotations

import ctypes as C
import dataclasses
import threading

import numpy as np
import torch

from . import _lib
from ._lib import (ContractError, DataflowCfg, KmapInfo, SkError, Tile, ValidationError, check,
                   i32x3, lib)

__all__ = ["Context", "CoordSet", "KernelMap", "DataflowConfig", "TilePreset", "tile_small",
           "tile_large", "quantize", "build_out_coords", "build_kmap", "kmap_from_edges", "conv_forward", "conv_dgrad",
           "conv_wgrad", "ValidationError", "ContractError", "SkError", "GATHER_GEMM_SCATTER",
           "FETCH_ON_DEMAND", "IMPLICIT_GEMM"]

GATHER_GEMM_SCATTER, FETCH_ON_DEMAND, IMPLICIT_GEMM = 0, 1, 2
_KIND_NAMES = {0: "gather_gemm_scatter", 1: "fetch_on_demand", 2: "implicit_gemm"}
_DTYPES = {torch.float32: _lib.SK_F32, torch.float16: _lib.SK_F16, torch.bfloat16: _lib.SK_BF16}


def _stream() -> C.c_void_p:
    return C.c_void_p(torch.cuda.current_stream().cuda_stream)


def _ptr(t: torch.Tensor) -> C.c_void_p:
    return C.c_void_p(t.data_ptr())


class Context:
    """sk_ctx: one per device (ExecContext + MapCache owner)."""

    _lock = threading.Lock()
    _by_device: dict = {}

    def __init__(self, device: int = 0):
        p = C.c_void_p()
        check(lib().sk_ctx_create(device, C.byref(p)))
        self.ptr, self.device = p, device
        self._deterministic = False

    @classmethod
    def get(cls, device=None) -> "Context":
        if device is None:
            device = torch.cuda.current_device()
        with cls._lock:
            if device not in cls._by_device:
                cls._by_device[device] = Context(device)
            return cls._by_device[device]

    @property
    def deterministic(self) -> bool:
        return self._deterministic

    @deterministic.setter
    def deterministic(self, on: bool) -> None:
        check(lib().sk_ctx_set_deterministic(self.ptr, int(bool(on))))
        self._deterministic = bool(on)

    def set_kmap_block_rows(self, min_rows: int) -> None:
        """Stride-1 3-D K=3/5 maps over input sets of >= min_rows voxels are
        queried through a 4x4x4 block index (default 1 << 16; identical
        results)."""
        check(lib().sk_ctx_set_kmap_block_rows(self.ptr, int(min_rows)))


class CoordSet:
    """Device coordinate set with a stable id (coord_set_id, tensor.cpp:26-29)."""

    def __init__(self, ptr, ctx: Context):
        self.ptr, self.ctx = ptr, ctx

    @classmethod
    def create(cls, coords, dims: int = 3, stride_tag=(1, 1, 1), ctx: Context | None = None):
        """coords: int32 [n, 4] (batch, x, y, z) as a CUDA tensor or host array."""
        ctx = ctx or Context.get()
        p = C.c_void_p()
        if isinstance(coords, torch.Tensor) and coords.is_cuda:
            c = coords.to(torch.int32).contiguous()
            check(lib().sk_coords_create(ctx.ptr, dims, c.shape[0], _ptr(c), i32x3(stride_tag),
                                         _stream(), C.byref(p)))
        else:
            c = np.ascontiguousarray(np.asarray(coords, dtype=np.int32).reshape(-1, 4))
            check(lib().sk_coords_create_host(ctx.ptr, dims, c.shape[0],
                                              c.ctypes.data_as(C.c_void_p), i32x3(stride_tag),
                                              _stream(), C.byref(p)))
        return cls(p, ctx)

    def __del__(self):
        try:
            if self.ptr:
                lib().sk_coords_release(self.ptr)
                self.ptr = None
        except Exception:
            pass

    @property
    def n(self) -> int:
        return lib().sk_coords_n(self.ptr)

    @property
    def dims(self) -> int:
        return lib().sk_coords_dims(self.ptr)

    @property
    def id(self) -> int:
        return lib().sk_coords_id(self.ptr)

    @property
    def stride_tag(self):
        out = (C.c_int32 * 3)()
        check(lib().sk_coords_stride_tag(self.ptr, out))
        return tuple(out)

    def numpy(self) -> np.ndarray:
        out = np.zeros((self.n, 4), np.int32)
        check(lib().sk_coords_export(self.ptr, out.ctypes.data_as(C.c_void_p), _stream()))
        return out

    def downsample(self, stride) -> "CoordSet":
        return build_out_coords(self, stride)

    def __eq__(self, other):
        return isinstance(other, CoordSet) and self.id == other.id

    def __hash__(self):
        return hash(self.id)


def _stride3(stride, dims=3):
    if isinstance(stride, int):
        s = [stride] * 3
    else:
        s = list(stride) + [1] * (3 - len(stride))
    if dims == 2:
        s[2] = 1
    return s


def quantize(raw, dims: int = 3, feats=None, voxel=(1.0, 1.0, 1.0), rule: str = "first",
             batch=None, dtype=torch.float32, ctx: Context | None = None):
    """quantize (tensor.cpp:87-142; DedupRule tensor.hpp:45) on the GPU:
    floor(raw / voxel) per axis, first-appearance dedup, features of the
    first point ("first") or the mean ("mean"); no features -> one occupancy
    channel of ones. raw: [m, dims] float64 (host or CUDA); batch: [m] int32
    or None; feats: [m, C] float64 or None. Returns (CoordSet, features [n,
    max(C, 1)] of `dtype` on the GPU)."""
    ctx = ctx or Context.get()
    if rule not in ("first", "mean"):
        raise ValidationError("unknown dedup rule")
    r = torch.as_tensor(raw, dtype=torch.float64).reshape(-1, dims).to("cuda").contiguous()
    m = r.shape[0]
    b = None if batch is None else torch.as_tensor(batch, dtype=torch.int32).to("cuda").contiguous()
    rows = torch.empty(max(m, 1), dtype=torch.int32, device="cuda")
    vox = (C.c_double * 3)(*[float(v) for v in (list(voxel) + [1.0] * 3)[:3]])
    p = C.c_void_p()
    check(lib().sk_quantize(ctx.ptr, dims, m, _ptr(r) if m else None,
                            _ptr(b) if b is not None and m else None, vox, _stream(), C.byref(p),
                            _ptr(rows)))
    cs = CoordSet(p, ctx)
    ch = 0 if feats is None else int(np.asarray(feats).shape[-1] if not torch.is_tensor(feats)
                                     else feats.shape[-1])
    out = torch.empty(cs.n, max(ch, 1), dtype=dtype, device="cuda")
    f = None
    if ch:
        f = torch.as_tensor(feats, dtype=torch.float64).reshape(m, ch).to("cuda").contiguous()
    check(lib().sk_quantize_features(ctx.ptr, m, ch, _ptr(f) if f is not None else None,
                                     _ptr(rows), cs.n, 0 if rule == "first" else 1,
                                     {**_DTYPES, torch.float64: 3}[dtype], _ptr(out), _stream()))
    return cs, out


def build_out_coords(coords: CoordSet, stride) -> CoordSet:
    """build_out_coords (kmap.cpp:73-94); cached per (set, stride)."""
    p = C.c_void_p()
    check(lib().sk_out_coords(coords.ctx.ptr, coords.ptr, i32x3(_stride3(stride, coords.dims)),
                              _stream(), C.byref(p)))
    return CoordSet(p, coords.ctx)


def build_kmap(inp: CoordSet, out: CoordSet, kernel_size, stride=1,
               transposed: bool = False, dilation=1) -> "KernelMap":
    """build_kmap_os / build_kmap_ws (kmap.cpp:96-143); cached per MapKey.
    kernel_size may be a per-axis triple (odd or even) and dilation an int or
    triple -- an extension beyond the reference (sk_kmap_build_ex)."""
    p = C.c_void_p()
    if isinstance(kernel_size, int) and dilation in (1, (1, 1, 1), [1, 1, 1]):
        check(lib().sk_kmap_build(inp.ctx.ptr, inp.ptr, out.ptr, kernel_size,
                                  i32x3(_stride3(stride, inp.dims)), int(transposed), _stream(),
                                  C.byref(p)))
    else:
        k = (kernel_size,) * 3 if isinstance(kernel_size, int) else tuple(kernel_size)
        d = (dilation,) * 3 if isinstance(dilation, int) else tuple(dilation)
        if inp.dims == 2:
            k, d = (k[0], k[1], 1), (d[0], d[1], 1)
        check(lib().sk_kmap_build_ex(inp.ctx.ptr, inp.ptr, out.ptr, i32x3(k),
                                     i32x3(_stride3(stride, inp.dims)), i32x3(d), int(transposed),
                                     _stream(), C.byref(p)))
    return KernelMap(p, inp.ctx)


def kmap_from_edges(edges, num_relations: int, n_in: int, n_out: int,
                    ctx: Context | None = None) -> "KernelMap":
    """kmap_from_edges (kmap.cpp:317-336): graph (R-GCN) map; edges [E, 3] =
    (src, dst, relation). Runs through GATHER_GEMM_SCATTER / FETCH_ON_DEMAND."""
    ctx = ctx or Context.get()
    e = torch.as_tensor(np.asarray(edges, dtype=np.int32).reshape(-1, 3)).cuda().contiguous()
    p = C.c_void_p()
    check(lib().sk_kmap_from_edges(ctx.ptr, _ptr(e) if e.numel() else None, e.shape[0],
                                   num_relations, n_in, n_out, _stream(), C.byref(p)))
    return KernelMap(p, ctx)


class KernelMap:
    def __init__(self, ptr, ctx: Context):
        self.ptr, self.ctx = ptr, ctx
        self._info = None

    def __del__(self):
        try:
            if self.ptr:
                lib().sk_kmap_release(self.ptr)
                self.ptr = None
        except Exception:
            pass

    def info(self) -> KmapInfo:
        if self._info is None:
            inf = KmapInfo()
            check(lib().sk_kmap_get_info(self.ptr, _stream(), C.byref(inf)))
            self._info = inf
        return self._info

    @property
    def n_in(self):
        return self.info().n_in

    @property
    def n_out(self):
        return self.info().n_out

    @property
    def num_offsets(self):
        return self.info().num_offsets

    def total_pairs(self) -> int:
        return int(self.info().total_pairs)

    def transpose(self) -> "KernelMap":
        p = C.c_void_p()
        check(lib().sk_kmap_transpose(self.ctx.ptr, self.ptr, _stream(), C.byref(p)))
        return KernelMap(p, self.ctx)

    def prepare(self, splits: int, pad_multiple: int = 128) -> None:
        check(lib().sk_kmap_prepare(self.ctx.ptr, self.ptr, splits, pad_multiple, _stream()))

    # ---- host exports (parity tests) ----
    def os(self):
        inf = self.info()
        words = (inf.num_offsets + 63) // 64
        ent = np.zeros((inf.n_out, inf.num_offsets), np.int32)
        m = np.zeros((max(inf.n_out, 1), words), np.uint64)
        check(lib().sk_kmap_export_os(self.ptr, ent.ctypes.data_as(C.c_void_p),
                                      m.ctypes.data_as(C.c_void_p), _stream()))
        return ent, m[: inf.n_out]

    def ws(self):
        kd = self.info().num_offsets
        ptr = np.zeros(kd + 1, np.int64)
        check(lib().sk_kmap_export_ws(self.ptr, ptr.ctypes.data_as(C.c_void_p), None, None,
                                      _stream()))
        n = int(ptr[-1])
        a = np.zeros(max(n, 1), np.int32)
        b = np.zeros(max(n, 1), np.int32)
        check(lib().sk_kmap_export_ws(self.ptr, ptr.ctypes.data_as(C.c_void_p),
                                      a.ctypes.data_as(C.c_void_p),
                                      b.ctypes.data_as(C.c_void_p), _stream()))
        return ptr, a[:n], b[:n]

    def split(self, splits: int, pad_multiple: int = 1):
        """[(begin, end, entries, out_row, masks)] like split_and_sort+pad_map."""
        out = []
        ns = max(splits, 1)
        for s in range(ns):
            b, e, n, w = C.c_int(), C.c_int(), C.c_int(), C.c_int()
            check(lib().sk_kmap_export_split(self.ptr, splits, pad_multiple, s, C.byref(b),
                                             C.byref(e), C.byref(n), C.byref(w), None, None,
                                             None, _stream()))
            ent = np.zeros((n.value, e.value - b.value), np.int32)
            orow = np.zeros(n.value, np.int32)
            m = np.zeros((max(n.value, 1), w.value), np.uint64)
            check(lib().sk_kmap_export_split(self.ptr, splits, pad_multiple, s, C.byref(b),
                                             C.byref(e), C.byref(n), C.byref(w),
                                             ent.ctypes.data_as(C.c_void_p),
                                             orow.ctypes.data_as(C.c_void_p),
                                             m.ctypes.data_as(C.c_void_p), _stream()))
            out.append((b.value, e.value, ent, orow, m[: n.value]))
        return out

    def count_macs(self, splits, pad_multiple, warp_rows, c_in, c_out):
        e, r = C.c_int64(), C.c_int64()
        check(lib().sk_kmap_count_macs(self.ptr, splits, pad_multiple, warp_rows, c_in, c_out,
                                       C.byref(e), C.byref(r), _stream()))
        return e.value, r.value


@dataclasses.dataclass(frozen=True)
class TilePreset:
    """TilePreset (exec.hpp:46-54) with tcgen05 meanings."""
    cta_m: int = 128
    cta_n: int = 0      # 0 = whole C_out (<= 256) per tile
    cta_k: int = 0      # 0 = auto (64/32/16 by C_in)
    warp_rows: int = 128
    load_width: int = 4


def tile_small() -> TilePreset:
    return TilePreset(128, 64, 0, 128, 4)


def tile_large() -> TilePreset:
    return TilePreset(128, 0, 0, 128, 4)


@dataclasses.dataclass(frozen=True)
class DataflowConfig:
    """DataflowConfig (exec.hpp:65-73)."""
    kind: int = GATHER_GEMM_SCATTER
    splits: int = 0
    tile: TilePreset = dataclasses.field(default_factory=tile_small)
    reorder: int = 0  # offline

    def name(self) -> str:  # DataflowConfig::name (exec.cpp:61-69)
        s = _KIND_NAMES[self.kind]
        if self.kind == IMPLICIT_GEMM:
            t = self.tile
            if t == tile_large():
                tn = "_large"
            elif t == tile_small():
                tn = "_small"
            else:  # B200 kernel variants (include/sk200.h sk_tile)
                tn = (f"_m{t.cta_m}" + (f"n{t.cta_n}" if t.cta_n else "") +
                      (f"k{t.cta_k}" if t.cta_k else "") + ("_tma" if t.load_width == 1 else ""))
            s += f"_s{self.splits}" + tn
            s += "_online" if self.reorder else "_offline"
        return s

    def c(self) -> DataflowCfg:
        t = self.tile
        return DataflowCfg(self.kind, self.splits,
                           Tile(t.cta_m, t.cta_n, t.cta_k, t.warp_rows, t.load_width),
                           self.reorder)


def _dtype(t: torch.Tensor) -> int:
    if t.dtype not in _DTYPES:
        raise ValidationError(f"unsupported dtype {t.dtype}")
    return _DTYPES[t.dtype]


def _check_feats(x: torch.Tensor, rows: int, name: str):
    if not x.is_cuda:
        raise ValidationError(f"{name} must be a CUDA tensor")
    if x.dim() != 2 or x.shape[0] != rows:
        raise ContractError(f"{name} row count does not match map")


def conv_forward(kmap: KernelMap, x: torch.Tensor, w: torch.Tensor,
                 cfg: DataflowConfig = DataflowConfig(), out: torch.Tensor | None = None):
    """conv_forward (exec.cpp:368-383). x [n_in, c_in], w [K^D, c_in, c_out]."""
    inf = kmap.info()
    _check_feats(x, inf.n_in, "x")
    if w.dim() != 3 or w.shape[0] != inf.num_offsets or w.shape[1] != x.shape[1]:
        raise ContractError("C_in mismatch")
    if w.dtype != x.dtype:
        raise ContractError("precision mismatch")
    x, w = x.contiguous(), w.contiguous()
    c_in, c_out = w.shape[1], w.shape[2]
    y = out if out is not None else torch.empty(inf.n_out, c_out, dtype=x.dtype, device=x.device)
    check(lib().sk_conv_forward(kmap.ctx.ptr, kmap.ptr, C.byref(cfg.c()), _dtype(x), c_in, c_out,
                                _ptr(x), _ptr(w), _ptr(y), _stream()))
    return y


def conv_dgrad(kmap: KernelMap, dy: torch.Tensor, w: torch.Tensor,
               cfg: DataflowConfig = DataflowConfig(), out: torch.Tensor | None = None):
    """conv_dgrad (exec.cpp:385-396): dx [n_in, c_in] from dy [n_out, c_out]."""
    inf = kmap.info()
    _check_feats(dy, inf.n_out, "dy")
    if w.dim() != 3 or w.shape[2] != dy.shape[1]:
        raise ContractError("C_out mismatch")
    dy, w = dy.contiguous(), w.contiguous()
    c_in, c_out = w.shape[1], w.shape[2]
    dx = out if out is not None else torch.empty(inf.n_in, c_in, dtype=dy.dtype, device=dy.device)
    check(lib().sk_conv_dgrad(kmap.ctx.ptr, kmap.ptr, C.byref(cfg.c()), _dtype(dy), c_in, c_out,
                              _ptr(dy), _ptr(w), _ptr(dx), _stream()))
    return dx


def conv_wgrad(kmap: KernelMap, x: torch.Tensor, dy: torch.Tensor,
               cfg: DataflowConfig = DataflowConfig(), out: torch.Tensor | None = None):
    """conv_wgrad (exec.cpp:398-414): fp32 dW [K^D, c_in, c_out]."""
    inf = kmap.info()
    _check_feats(x, inf.n_in, "x")
    _check_feats(dy, inf.n_out, "dy")
    if x.dtype != dy.dtype:
        raise ContractError("precision mismatch")
    x, dy = x.contiguous(), dy.contiguous()
    dw = out if out is not None else torch.empty(inf.num_offsets, x.shape[1], dy.shape[1],
                                                 dtype=torch.float32, device=x.device)
    check(lib().sk_conv_wgrad(kmap.ctx.ptr, kmap.ptr, C.byref(cfg.c()), _dtype(x), x.shape[1],
                              dy.shape[1], _ptr(x), _ptr(dy), _ptr(dw), _stream()))
    return dw
