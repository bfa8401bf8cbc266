"""TEST INFRASTRUCTURE — not product code.

ctypes/numpy front end for the two CPU checkers under oracle/:

* ``Restatement`` — the plain-C restatement (oracle/sk_oracle.c ->
  oracle/lib/libsk_oracle.so). Each wrapper names the reference function it
  restates.
* ``Reference`` — the unmodified reference library compiled from
  /root/reference/proj/src (oracle/_ref/libsparsekit_ref.so) behind the
  oracle/ref_capi.cpp shim.

Only tests/, ``__graft_entry__.smoke()`` and bench.py's cpu_baseline /
``--impl reference`` leg import this module. The product package
(paper_2311_12862_b200) never does.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
RESTATEMENT_SO = os.path.join(HERE, "lib", "libsk_oracle.so")
REFERENCE_SO = os.path.join(HERE, "_ref", "libsparsekit_ref.so")

_i32p = np.ctypeslib.ndpointer(np.int32, flags="C_CONTIGUOUS")
_i64p = np.ctypeslib.ndpointer(np.int64, flags="C_CONTIGUOUS")
_u64p = np.ctypeslib.ndpointer(np.uint64, flags="C_CONTIGUOUS")
_f64p = np.ctypeslib.ndpointer(np.float64, flags="C_CONTIGUOUS")


def build(reference: bool = True) -> None:
    """Compile the restatement (always) and the reference (when its sources
    are mounted, i.e. in the build container)."""
    targets = ["restatement"]
    if reference and os.path.isdir("/root/reference/proj/src"):
        targets.append("reference")
        # the INTEGRATION.md shim against the reference headers (needs the
        # product library, which build() compiles first)
        if os.path.exists(os.path.join(os.path.dirname(HERE), "paper_2311_12862_b200",
                                       "libsk200.so")):
            targets.append("shim")
    subprocess.run(["make", "-s", "-C", HERE, *targets], check=True)


def kd_of(dims: int, k: int) -> int:
    return k * k if dims == 2 else k * k * k


def _c(a, dt):
    return np.ascontiguousarray(a, dtype=dt)


class Restatement:
    """oracle/sk_oracle.c."""

    def __init__(self, path: str = RESTATEMENT_SO):
        if not os.path.exists(path):
            raise FileNotFoundError(f"{path} missing: run `make -C oracle restatement`")
        L = self.lib = C.CDLL(path)
        L.sko_offsets.argtypes = [C.c_int, C.c_int, _i32p]
        L.sko_out_coords.argtypes = [C.c_int, C.c_int, _i32p, _i32p, _i32p, C.POINTER(C.c_int)]
        L.sko_kmap_os_ex.argtypes = [C.c_int, _i32p, _i32p, C.c_int, _i32p, C.c_int, _i32p,
                                     _i32p, C.c_int, _i32p]
        L.sko_kmap_os.argtypes = [C.c_int, C.c_int, C.c_int, _i32p, C.c_int, _i32p, _i32p,
                                  C.c_int, _i32p]
        L.sko_masks.argtypes = [C.c_int, C.c_int, _i32p, _u64p]
        L.sko_masks.restype = None
        L.sko_split_bounds.argtypes = [C.c_int, C.c_int, _i32p]
        L.sko_split_sort.argtypes = [C.c_int, C.c_int, _i32p, C.c_int, C.c_int, _i32p, _i32p,
                                     _u64p]
        L.sko_transpose_os.argtypes = [C.c_int, C.c_int, C.c_int, _i32p, _i32p]
        L.sko_ws_from_os.argtypes = [C.c_int, C.c_int, _i32p, _i64p, C.c_void_p, C.c_void_p]
        L.sko_ws_from_os.restype = None
        L.sko_conv_f64.argtypes = [C.c_int, C.c_int, _i32p, C.c_int, C.c_int, _f64p, _f64p, _f64p]
        L.sko_conv_f64.restype = None
        L.sko_dgrad_f64.argtypes = [C.c_int, C.c_int, _i32p, C.c_int, C.c_int, _f64p, _f64p,
                                    _f64p]
        L.sko_dgrad_f64.restype = None
        L.sko_wgrad_f64.argtypes = [C.c_int, C.c_int, _i32p, C.c_int, C.c_int, _f64p, _f64p,
                                    _f64p]
        L.sko_wgrad_f64.restype = None
        L.sko_charged_macs.argtypes = [C.c_int, C.c_int, _i32p, C.c_int, C.c_int, C.c_int]
        L.sko_charged_macs.restype = C.c_int64

    # OffsetSet (kmap.cpp:58-71)
    def offsets(self, dims, k):
        out = np.zeros((kd_of(dims, k), 3), np.int32)
        if self.lib.sko_offsets(dims, k, out):
            raise ValueError("kernel size must be odd")
        return out

    # build_out_coords (kmap.cpp:73-94)
    def out_coords(self, dims, coords, stride):
        coords = _c(coords, np.int32).reshape(-1, 4)
        out = np.zeros_like(coords)
        n = C.c_int()
        rc = self.lib.sko_out_coords(dims, len(coords), coords, _c(stride, np.int32), out,
                                     C.byref(n))
        if rc:
            raise ValueError("bad stride")
        return out[: n.value].copy()

    # build_kmap_ws + ws_to_os (kmap.cpp:96-183)
    def kmap_os(self, dims, k, in_coords, out_coords, stride, transposed=False):
        in_coords = _c(in_coords, np.int32).reshape(-1, 4)
        out_coords = _c(out_coords, np.int32).reshape(-1, 4)
        kd = kd_of(dims, k)
        ent = np.zeros((len(out_coords), kd), np.int32)
        rc = self.lib.sko_kmap_os(dims, k, len(in_coords), in_coords, len(out_coords), out_coords,
                                  _c(stride, np.int32), int(transposed), ent)
        if rc:
            raise ValueError(f"kmap build failed rc={rc}")
        return ent

    # compute_masks (kmap.cpp:34-47)
    def kmap_os_ex(self, dims, kernel, dilation, in_coords, out_coords, stride,
                   transposed=False):
        """EXTENSION: per-axis / even kernel sizes and
        dilation; restated definition, not pinned by the reference."""
        in_coords = _c(in_coords, np.int32).reshape(-1, 4)
        out_coords = _c(out_coords, np.int32).reshape(-1, 4)
        kd = int(kernel[0] * kernel[1] * (kernel[2] if dims == 3 else 1))
        ent = np.zeros((len(out_coords), kd), np.int32)
        rc = self.lib.sko_kmap_os_ex(dims, _c(kernel, np.int32), _c(dilation, np.int32),
                                     len(in_coords), in_coords, len(out_coords), out_coords,
                                     _c(stride, np.int32), int(transposed), ent)
        if rc:
            raise ValueError(f"sko_kmap_os_ex failed ({rc})")
        return ent

    def masks(self, entries):
        entries = _c(entries, np.int32)
        n, w = entries.shape
        m = np.zeros((n, (w + 63) // 64), np.uint64)
        self.lib.sko_masks(n, w, entries, m)
        return m

    def split_bounds(self, kd, splits):
        b = np.zeros(max(splits, 1) + 1, np.int32)
        if self.lib.sko_split_bounds(kd, splits, b):
            raise ValueError("split count out of range")
        return b

    # split_and_sort + pad_map (kmap.cpp:211-288). Returns a list of splits,
    # each (begin, end, entries[rows_padded, w], out_row[rows_padded], masks).
    def split_sort(self, entries, splits, pad=1):
        entries = _c(entries, np.int32)
        n, kd = entries.shape
        b = self.split_bounds(kd, splits)
        ns = max(splits, 1)
        rp = (n + pad - 1) // pad * pad
        words = [(int(b[s + 1] - b[s]) + 63) // 64 for s in range(ns)]
        ent = np.zeros(rp * kd + 1, np.int32)
        orow = np.zeros(rp * ns + 1, np.int32)
        msk = np.zeros(rp * sum(words) + 1, np.uint64)
        if self.lib.sko_split_sort(n, kd, entries, splits, pad, ent, orow, msk):
            raise ValueError("split_sort failed")
        out, eo, mo = [], 0, 0
        for s in range(ns):
            w = int(b[s + 1] - b[s])
            out.append((int(b[s]), int(b[s + 1]), ent[eo:eo + rp * w].reshape(rp, w).copy(),
                        orow[s * rp:(s + 1) * rp].copy(),
                        msk[mo:mo + rp * words[s]].reshape(rp, words[s]).copy()))
            eo += rp * w
            mo += rp * words[s]
        return out

    # transpose_map (kmap.cpp:290-315)
    def transpose_os(self, entries, n_in):
        entries = _c(entries, np.int32)
        n_out, kd = entries.shape
        t = np.zeros((n_in, kd), np.int32)
        if self.lib.sko_transpose_os(n_out, n_in, kd, entries, t):
            raise ValueError("duplicate neighbour")
        return t

    # os_to_ws (kmap.cpp:185-209) -> CSR over offsets
    def ws(self, entries):
        entries = _c(entries, np.int32)
        n_out, kd = entries.shape
        ptr = np.zeros(kd + 1, np.int64)
        self.lib.sko_ws_from_os(n_out, kd, entries, ptr, None, None)
        inn = np.zeros(max(int(ptr[-1]), 1), np.int32)
        out = np.zeros_like(inn)
        self.lib.sko_ws_from_os(n_out, kd, entries, ptr, inn.ctypes.data, out.ctypes.data)
        return ptr, inn[: ptr[-1]], out[: ptr[-1]]

    # conv_ref (exec.cpp:101-115)
    def conv(self, entries, x, w):
        entries = _c(entries, np.int32)
        n_out, kd = entries.shape
        x = _c(x, np.float64)
        w = _c(w, np.float64).reshape(kd, x.shape[1], -1)
        y = np.zeros((n_out, w.shape[2]), np.float64)
        self.lib.sko_conv_f64(n_out, kd, entries, x.shape[1], w.shape[2], x, w, y)
        return y

    # conv_dgrad (exec.cpp:385-396); t_entries from transpose_os
    def dgrad(self, t_entries, dy, w):
        t_entries = _c(t_entries, np.int32)
        n_in, kd = t_entries.shape
        dy = _c(dy, np.float64)
        w = _c(w, np.float64).reshape(kd, -1, dy.shape[1])
        dx = np.zeros((n_in, w.shape[1]), np.float64)
        self.lib.sko_dgrad_f64(n_in, kd, t_entries, w.shape[1], w.shape[2], dy, w, dx)
        return dx

    # wgrad_impl (exec.cpp:259-279)
    def wgrad(self, entries, x, dy):
        entries = _c(entries, np.int32)
        n_out, kd = entries.shape
        x = _c(x, np.float64)
        dy = _c(dy, np.float64)
        dw = np.zeros((kd, x.shape[1], dy.shape[1]), np.float64)
        self.lib.sko_wgrad_f64(n_out, kd, entries, x.shape[1], dy.shape[1], x, dy, dw)
        return dw

    # count_macs (cost.cpp:7-30) over a prepared map (list from split_sort)
    def count_macs(self, splits, warp_rows, c_in, c_out):
        charged = 0
        eff = 0
        for (_, _, ent, _, _) in splits:
            charged += self.lib.sko_charged_macs(ent.shape[0], ent.shape[1], _c(ent, np.int32),
                                                 warp_rows, c_in, c_out)
            eff += int((ent != -1).sum()) * c_in * c_out
        return eff, charged - eff


class RefMap:
    def __init__(self, ref: "Reference", ptr):
        self.ref, self.ptr = ref, ptr

    def __del__(self):
        try:
            self.ref.lib.ref_map_free(self.ptr)
        except Exception:
            pass

    @property
    def kd(self):
        return self.ref.lib.ref_map_num_offsets(self.ptr)

    @property
    def n_in(self):
        return self.ref.lib.ref_map_n_in(self.ptr)

    @property
    def n_out(self):
        return self.ref.lib.ref_map_n_out(self.ptr)

    def pairs(self, k):
        n = self.ref.lib.ref_map_pairs(self.ptr, k, None, None)
        a = np.zeros(max(n, 1), np.int32)
        b = np.zeros(max(n, 1), np.int32)
        self.ref.lib.ref_map_pairs(self.ptr, k, a.ctypes.data, b.ctypes.data)
        return a[:n], b[:n]

    def os(self):
        kd = self.kd
        ent = np.zeros((self.n_out, kd), np.int32)
        words = (kd + 63) // 64
        m = np.zeros((max(self.n_out, 1), words), np.uint64)
        mw = C.c_int()
        self.ref._check(self.ref.lib.ref_map_os(self.ptr, ent, m, C.byref(mw)))
        return ent, m[: self.n_out]

    def prepare(self, splits, pad=1):
        L = self.ref.lib
        self.ref._check(L.ref_map_prepare(self.ptr, splits, pad))
        out = []
        for s in range(L.ref_prep_num_splits(self.ptr)):
            b, e, n, w = C.c_int(), C.c_int(), C.c_int(), C.c_int()
            self.ref._check(L.ref_prep_split_info(self.ptr, s, C.byref(b), C.byref(e), C.byref(n),
                                                  C.byref(w)))
            ent = np.zeros((n.value, e.value - b.value), np.int32)
            orow = np.zeros(n.value, np.int32)
            m = np.zeros((max(n.value, 1), w.value), np.uint64)
            self.ref._check(L.ref_prep_split_data(self.ptr, s, ent, orow, m))
            out.append((b.value, e.value, ent, orow, m[: n.value]))
        return out

    def count_macs(self, warp_rows, c_in, c_out):
        e, r = C.c_int64(), C.c_int64()
        self.ref._check(self.ref.lib.ref_prep_count_macs(self.ptr, warp_rows, c_in, c_out,
                                                         C.byref(e), C.byref(r)))
        return e.value, r.value

    def transpose(self):
        p = C.c_void_p()
        self.ref._check(self.ref.lib.ref_map_transpose(self.ptr, C.byref(p)))
        return RefMap(self.ref, p)


class Reference:
    """The compiled reference (oracle/_ref/libsparsekit_ref.so)."""

    def __init__(self, path: str = REFERENCE_SO):
        if not os.path.exists(path):
            raise FileNotFoundError(f"{path} missing: run `make -C oracle reference` "
                                    "in the build container")
        L = self.lib = C.CDLL(path)
        L.ref_last_error.restype = C.c_char_p
        L.ref_out_coords.argtypes = [C.c_int, C.c_int, _i32p, _i32p, _i32p, C.POINTER(C.c_int)]
        L.ref_map_build.argtypes = [C.c_int, C.c_int, C.c_int, _i32p, C.c_int, _i32p, _i32p,
                                    C.c_int, C.POINTER(C.c_void_p)]
        L.ref_map_transpose.argtypes = [C.c_void_p, C.POINTER(C.c_void_p)]
        L.ref_map_from_edges.argtypes = [C.c_int, _i32p, C.c_int, C.c_int, C.c_int,
                                         C.POINTER(C.c_void_p)]
        L.ref_map_free.argtypes = [C.c_void_p]
        L.ref_map_free.restype = None
        for f in ("ref_map_num_offsets", "ref_map_n_in", "ref_map_n_out", "ref_prep_num_splits"):
            getattr(L, f).argtypes = [C.c_void_p]
        L.ref_map_pairs.argtypes = [C.c_void_p, C.c_int, C.c_void_p, C.c_void_p]
        L.ref_map_pairs.restype = C.c_int64
        L.ref_map_os.argtypes = [C.c_void_p, _i32p, _u64p, C.POINTER(C.c_int)]
        L.ref_map_prepare.argtypes = [C.c_void_p, C.c_int, C.c_int]
        L.ref_prep_split_info.argtypes = [C.c_void_p, C.c_int] + [C.POINTER(C.c_int)] * 4
        L.ref_prep_split_data.argtypes = [C.c_void_p, C.c_int, _i32p, _i32p, _u64p]
        L.ref_prep_count_macs.argtypes = [C.c_void_p, C.c_int, C.c_int, C.c_int,
                                          C.POINTER(C.c_int64), C.POINTER(C.c_int64)]
        L.ref_conv_forward.argtypes = [C.c_void_p] + [C.c_int] * 9 + [_f64p, _f64p, _f64p]
        L.ref_conv_ref.argtypes = [C.c_void_p, C.c_int, C.c_int, C.c_int, _f64p, _f64p, _f64p]
        L.ref_conv_dgrad.argtypes = [C.c_void_p] + [C.c_int] * 8 + [_f64p, _f64p, _f64p]
        L.ref_conv_wgrad.argtypes = [C.c_void_p] + [C.c_int] * 4 + [_f64p, _f64p, _f64p]
        L.ref_gen_voxels.argtypes = [C.c_int, C.c_int, C.c_uint64, C.c_double, _f64p, C.c_int32,
                                     C.c_void_p, C.POINTER(C.c_int)]
        L.ref_gen_cloud.argtypes = [C.c_int, C.c_int, C.c_uint64, C.c_double, _f64p]
        L.ref_quantize.argtypes = [C.c_int, C.c_int, _f64p, C.c_int, C.c_void_p, _f64p, C.c_int,
                                   C.c_void_p, C.c_void_p, C.c_void_p, C.POINTER(C.c_int)]
        L.ref_net_create.argtypes = [C.c_int, C.c_char_p, C.c_int, C.c_int, C.c_uint64,
                                     C.c_void_p, C.POINTER(C.c_void_p)]
        L.ref_net_free.argtypes = [C.c_void_p]
        L.ref_net_free.restype = None
        L.ref_net_num_groups.argtypes = [C.c_void_p]
        L.ref_net_group_of_layer.argtypes = [C.c_void_p, C.c_int]
        L.ref_net_set_input.argtypes = [C.c_void_p, C.c_int, _i32p, C.c_int, _f64p, C.c_int]
        L.ref_net_forward.argtypes = [C.c_void_p] + [C.POINTER(C.c_double)] * 3
        L.ref_net_measure.argtypes = [C.c_void_p, C.c_int, C.c_int, C.c_int,
                                      C.POINTER(C.c_double)]
        L.ref_net_output.argtypes = [C.c_void_p, C.c_void_p, C.POINTER(C.c_int),
                                     C.POINTER(C.c_int)]
        L.ref_net_group_traffic.argtypes = [C.c_void_p, C.c_int, C.c_int, C.c_int, C.c_int,
                                            C.POINTER(C.c_double)]
        self.has_io = hasattr(L, "ref_tspw_write")  # io.cpp compiled in (json.hpp found)
        if self.has_io:
            L.ref_tspw_write.argtypes = [C.c_char_p, C.c_int, _i32p, _f64p]
            L.ref_tspw_read.argtypes = [C.c_char_p, C.POINTER(C.c_int), _i32p, C.c_int, C.c_void_p]
            L.ref_tune_roundtrip.argtypes = [C.c_char_p, C.c_char_p, C.c_int, C.POINTER(C.c_int)]
            L.ref_tune_sample.argtypes = [C.c_char_p, C.c_int, C.POINTER(C.c_int)]

    def _check(self, rc):
        if rc:
            msg = self.lib.ref_last_error().decode()
            if rc == 1:
                raise ValueError(msg)
            raise RuntimeError(f"reference error {rc}: {msg}")

    # ---- io.cpp: TSPW weights, TuneResult JSON (write_tspw / read_tspw,
    # tune_result_to_json / _from_json)
    def tspw_write(self, path, layers):
        shapes = _c(np.array([w.shape for w in layers], np.int32).reshape(-1), np.int32)
        vals = _c(np.concatenate([np.asarray(w, np.float64).ravel() for w in layers]), np.float64)
        self._check(self.lib.ref_tspw_write(path.encode(), len(layers), shapes, vals))

    def tspw_read(self, path):
        n = C.c_int()
        shapes = np.zeros(3 * 1024, np.int32)
        self._check(self.lib.ref_tspw_read(path.encode(), C.byref(n), shapes, 1024, None))
        sh = shapes[:3 * n.value].reshape(-1, 3)
        vals = np.zeros(int(np.prod(sh, axis=1).sum()), np.float64)
        self._check(self.lib.ref_tspw_read(path.encode(), C.byref(n), shapes, 1024,
                                           vals.ctypes.data))
        out, off = [], 0
        for kd, ci, co in sh:
            cnt = int(kd) * int(ci) * int(co)
            out.append(vals[off:off + cnt].reshape(kd, ci, co))
            off += cnt
        return out

    def _text(self, fn, *args):
        ln = C.c_int()
        self._check(fn(*args, None, 0, C.byref(ln)))
        buf = C.create_string_buffer(ln.value + 1)
        self._check(fn(*args, buf, ln.value + 1, C.byref(ln)))
        return buf.value.decode()

    def tune_roundtrip(self, text):
        return self._text(self.lib.ref_tune_roundtrip, text.encode())

    def tune_sample(self):
        return self._text(self.lib.ref_tune_sample)

    def out_coords(self, dims, coords, stride):
        coords = _c(coords, np.int32).reshape(-1, 4)
        out = np.zeros((max(len(coords), 1), 4), np.int32)
        n = C.c_int()
        self._check(self.lib.ref_out_coords(dims, len(coords), coords, _c(stride, np.int32), out,
                                            C.byref(n)))
        return out[: n.value].copy()

    def kmap(self, dims, k, in_coords, out_coords, stride, transposed=False) -> RefMap:
        in_coords = _c(in_coords, np.int32).reshape(-1, 4)
        out_coords = _c(out_coords, np.int32).reshape(-1, 4)
        p = C.c_void_p()
        self._check(self.lib.ref_map_build(dims, k, len(in_coords), in_coords, len(out_coords),
                                           out_coords, _c(stride, np.int32), int(transposed),
                                           C.byref(p)))
        return RefMap(self, p)

    def graph_map(self, edges, relations, n_in, n_out) -> RefMap:
        """kmap_from_edges (kmap.cpp:317-336)."""
        e = _c(np.asarray(edges, np.int32).reshape(-1, 3), np.int32)
        p = C.c_void_p()
        self._check(self.lib.ref_map_from_edges(len(e), e, relations, n_in, n_out, C.byref(p)))
        return RefMap(self, p)

    # kind: 0 gather_gemm_scatter, 1 fetch_on_demand, 2 implicit_gemm
    def conv_forward(self, m: RefMap, x, w, kind=0, splits=0, tile_large=False, online=False,
                     prec=1, deterministic=True, threads=1):
        x = _c(x, np.float64)
        w = _c(w, np.float64)
        c_in, c_out = x.shape[1], w.shape[-1]
        y = np.zeros((m.n_out, c_out), np.float64)
        self._check(self.lib.ref_conv_forward(m.ptr, kind, splits, int(tile_large), int(online),
                                              prec, int(deterministic), threads, c_in, c_out,
                                              x, w.reshape(-1), y))
        return y

    def conv_ref(self, m: RefMap, x, w, prec=1):
        x = _c(x, np.float64)
        w = _c(w, np.float64)
        y = np.zeros((m.n_out, w.shape[-1]), np.float64)
        self._check(self.lib.ref_conv_ref(m.ptr, prec, x.shape[1], w.shape[-1], x, w.reshape(-1),
                                          y))
        return y

    def conv_dgrad(self, m: RefMap, dy, w, kind=0, splits=0, tile_large=False, prec=1,
                   deterministic=True, threads=1):
        dy = _c(dy, np.float64)
        w = _c(w, np.float64)
        c_in, c_out = w.shape[-2], w.shape[-1]
        dx = np.zeros((m.n_in, c_in), np.float64)
        self._check(self.lib.ref_conv_dgrad(m.ptr, kind, splits, int(tile_large), prec,
                                            int(deterministic), threads, c_in, c_out, dy,
                                            w.reshape(-1), dx))
        return dx

    def conv_wgrad(self, m: RefMap, x, dy, prec=1, threads=1):
        x = _c(x, np.float64)
        dy = _c(dy, np.float64)
        dw = np.zeros((m.kd, x.shape[1], dy.shape[1]), np.float64)
        self._check(self.lib.ref_conv_wgrad(m.ptr, prec, threads, x.shape[1], dy.shape[1], x, dy,
                                            dw))
        return dw

    # gen_cloud + quantize(first), occupancy only (gen.cpp:32-85, tensor.cpp:87-142)
    def gen_voxels(self, kind, n, seed, extent, voxel, batch=0):
        vox = _c(voxel, np.float64)
        cnt = C.c_int()
        self._check(self.lib.ref_gen_voxels(kind, n, seed, extent, vox, batch, None,
                                            C.byref(cnt)))
        out = np.zeros((cnt.value, 4), np.int32)
        self._check(self.lib.ref_gen_voxels(kind, n, seed, extent, vox, batch,
                                            out.ctypes.data, C.byref(cnt)))
        return out

    def gen_cloud(self, kind, n, seed, extent):
        pts = np.zeros((n, 3), np.float64)
        self._check(self.lib.ref_gen_cloud(kind, n, seed, extent, pts))
        return pts

    def quantize(self, raw, dims, feats, voxel, rule=0, batch=None):
        raw = _c(raw, np.float64)
        m = raw.size // dims
        ch = 0 if feats is None else np.asarray(feats).shape[1]
        f = None if feats is None else _c(feats, np.float64)
        b = None if batch is None else _c(batch, np.int32)
        vox = _c(voxel, np.float64)
        cnt = C.c_int()
        args = (dims, m, raw, ch, None if f is None else f.ctypes.data, vox, rule,
                None if b is None else b.ctypes.data)
        self._check(self.lib.ref_quantize(*args, None, None, C.byref(cnt)))
        coords = np.zeros((cnt.value, 4), np.int32)
        of = np.zeros((cnt.value, max(ch, 1)), np.float64)
        self._check(self.lib.ref_quantize(*args, coords.ctypes.data, of.ctypes.data,
                                          C.byref(cnt)))
        return coords, of

    def network(self, dims, spec_text, prec=0, threads=0, weight_seed=3, weights=None):
        """NetworkRunner over `spec_text`; weights = list of [K^D, c_in, c_out]
        arrays (layer order) or None for seeded timing weights."""
        p = C.c_void_p()
        flat = None
        if weights is not None:
            flat = np.ascontiguousarray(np.concatenate([np.asarray(w, np.float64).ravel()
                                                        for w in weights]))
        self._check(self.lib.ref_net_create(dims, spec_text.encode(), prec, threads, weight_seed,
                                            None if flat is None else flat.ctypes.data,
                                            C.byref(p)))
        net = RefNet(self, p)
        net._weights_keep = flat
        return net


class RefNet:
    def __init__(self, ref: Reference, ptr):
        self.ref, self.ptr = ref, ptr

    def __del__(self):
        try:
            self.ref.lib.ref_net_free(self.ptr)
        except Exception:
            pass

    @property
    def num_groups(self):
        return self.ref.lib.ref_net_num_groups(self.ptr)

    def group_of_layer(self, i):
        return self.ref.lib.ref_net_group_of_layer(self.ptr, i)

    def set_input(self, coords, feats, prec=0):
        coords = _c(coords, np.int32)
        feats = _c(feats, np.float64)
        self.ref._check(self.ref.lib.ref_net_set_input(self.ptr, len(coords), coords,
                                                       feats.shape[1], feats, prec))

    def forward(self):
        t, mp, kr = C.c_double(), C.c_double(), C.c_double()
        self.ref._check(self.ref.lib.ref_net_forward(self.ptr, C.byref(t), C.byref(mp),
                                                     C.byref(kr)))
        return t.value, mp.value, kr.value

    def measure(self, fwd=True, dgrad=False, wgrad=False):
        t = C.c_double()
        self.ref._check(self.ref.lib.ref_net_measure(self.ptr, int(fwd), int(dgrad), int(wgrad),
                                                     C.byref(t)))
        return t.value

    def group_traffic(self, group, kind, splits=0, tile_large=False):
        """modeled_group_traffic (network.cpp:453-471) after forward()/output()."""
        b = C.c_double()
        self.ref._check(self.ref.lib.ref_net_group_traffic(self.ptr, group, kind, splits,
                                                           int(tile_large), C.byref(b)))
        return b.value

    def output(self):
        n, c = C.c_int(), C.c_int()
        self.ref._check(self.ref.lib.ref_net_output(self.ptr, None, C.byref(n), C.byref(c)))
        y = np.zeros((n.value, c.value), np.float64)
        self.ref._check(self.ref.lib.ref_net_output(self.ptr, y.ctypes.data, C.byref(n),
                                                    C.byref(c)))
        return y
