"""ctypes binding of libsk200.so (the C ABI in include/sk200.h).

The product path has no CPU fallback: if the library is missing or a GPU call
fails, this raises. Status codes map to the reference's exception taxonomy
(common.hpp:19-27): SK_ERR_VALIDATION -> ValidationError (a ValueError),
SK_ERR_CONTRACT -> ContractError, everything else -> SkError.
"""
from __future__ import annotations

import ctypes as C
import os

PKG = os.path.dirname(os.path.abspath(__file__))
# SK200_LIB: developer A/B runs against another build of the same ABI
LIB_PATH = os.environ.get("SK200_LIB") or os.path.join(PKG, "libsk200.so")

# exported symbols, in header order (include/sk200.h); tests check the .so
# exports exactly these
SYMBOLS = [
    "sk_last_error", "sk_version", "sk_kernel_launches", "sk_ctx_create", "sk_ctx_destroy", "sk_ctx_set_deterministic", "sk_ctx_set_kmap_block_rows",
    "sk_coords_create", "sk_coords_create_host", "sk_coords_retain", "sk_coords_release",
    "sk_quantize", "sk_quantize_features", "sk_kmap_from_edges", "sk_kmap_build_ex",
    "sk_coords_n", "sk_coords_dims", "sk_coords_id", "sk_coords_device_ptr",
    "sk_coords_stride_tag", "sk_coords_export", "sk_out_coords", "sk_kmap_build",
    "sk_kmap_transpose", "sk_kmap_prepare", "sk_kmap_retain", "sk_kmap_release",
    "sk_kmap_get_info", "sk_kmap_export_os", "sk_kmap_export_ws", "sk_kmap_export_split",
    "sk_conv_forward", "sk_conv_dgrad", "sk_conv_wgrad", "sk_kmap_count_macs",
    "sk_net_create", "sk_net_destroy", "sk_net_num_layers", "sk_net_num_groups",
    "sk_net_group_of_layer", "sk_net_layer_info", "sk_net_num_params", "sk_net_weight_ptr",
    "sk_net_set_config", "sk_net_get_config", "sk_net_forward", "sk_net_layer_output",
    "sk_net_forward_profiled",
    "sk_net_measure", "sk_net_map_builds", "sk_net_set_overlap", "sk_net_set_pdl", "sk_net_set_tune_cold", "sk_net_group_traffic", "sk_net_backward",
    "sk_net_tune", "sk_tune_space_size", "sk_tune_space_entry",
]

SK_F32, SK_F16, SK_BF16 = 0, 1, 2
GATHER_GEMM_SCATTER, FETCH_ON_DEMAND, IMPLICIT_GEMM = 0, 1, 2


class SkError(RuntimeError):
    pass


class ValidationError(ValueError):
    """sparsekit::ValidationError (common.hpp:19-22)."""


class ContractError(SkError):
    """sparsekit::ContractError (common.hpp:24-27)."""


class Tile(C.Structure):
    _fields_ = [("cta_m", C.c_int), ("cta_n", C.c_int), ("cta_k", C.c_int),
                ("warp_rows", C.c_int), ("load_width", C.c_int)]


class DataflowCfg(C.Structure):
    _fields_ = [("kind", C.c_int), ("splits", C.c_int), ("tile", Tile), ("reorder", C.c_int)]


class KmapInfo(C.Structure):
    _fields_ = [("dims", C.c_int), ("kernel_size", C.c_int), ("num_offsets", C.c_int),
                ("n_in", C.c_int), ("n_out", C.c_int), ("transposed", C.c_int),
                ("stride", C.c_int * 3), ("total_pairs", C.c_int64)]


_lib = None


def lib():
    """Load libsk200.so once; raise loudly when it is absent."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        raise SkError(f"{LIB_PATH} not built: run `python -m paper_2311_12862_b200.build` "
                      "(there is no CPU fallback)")
    L = C.CDLL(LIB_PATH)
    vp, i32p, i64p, u64p = C.c_void_p, C.POINTER(C.c_int32), C.POINTER(C.c_int64), C.POINTER(C.c_uint64)
    pp = C.POINTER(C.c_void_p)
    sig = {
        "sk_last_error": ([], C.c_char_p),
        "sk_version": ([], C.c_char_p),
        "sk_kernel_launches": ([], C.c_uint64),
        "sk_ctx_create": ([C.c_int, pp], C.c_int),
        "sk_ctx_destroy": ([vp], C.c_int),
        "sk_ctx_set_deterministic": ([vp, C.c_int], C.c_int),
        "sk_ctx_set_kmap_block_rows": ([vp, C.c_int], C.c_int),
        "sk_coords_create": ([vp, C.c_int, C.c_int, vp, i32p, vp, pp], C.c_int),
        "sk_coords_create_host": ([vp, C.c_int, C.c_int, vp, i32p, vp, pp], C.c_int),
        "sk_coords_retain": ([vp], C.c_int),
        "sk_coords_release": ([vp], C.c_int),
        "sk_coords_n": ([vp], C.c_int),
        "sk_coords_dims": ([vp], C.c_int),
        "sk_coords_id": ([vp], C.c_uint64),
        "sk_coords_device_ptr": ([vp], vp),
        "sk_coords_stride_tag": ([vp, i32p], C.c_int),
        "sk_coords_export": ([vp, vp, vp], C.c_int),
        "sk_out_coords": ([vp, vp, i32p, vp, pp], C.c_int),
        "sk_quantize": ([vp, C.c_int, C.c_int, vp, vp, C.POINTER(C.c_double), vp, pp, vp],
                        C.c_int),
        "sk_quantize_features": ([vp, C.c_int, C.c_int, vp, vp, C.c_int, C.c_int, C.c_int, vp,
                                  vp], C.c_int),
        "sk_kmap_build": ([vp, vp, vp, C.c_int, i32p, C.c_int, vp, pp], C.c_int),
        "sk_kmap_transpose": ([vp, vp, vp, pp], C.c_int),
        "sk_kmap_build_ex": ([vp, vp, vp, i32p, i32p, i32p, C.c_int, vp, pp], C.c_int),
        "sk_kmap_from_edges": ([vp, vp, C.c_int, C.c_int, C.c_int, C.c_int, vp, pp], C.c_int),
        "sk_kmap_prepare": ([vp, vp, C.c_int, C.c_int, vp], C.c_int),
        "sk_kmap_retain": ([vp], C.c_int),
        "sk_kmap_release": ([vp], C.c_int),
        "sk_kmap_get_info": ([vp, vp, C.POINTER(KmapInfo)], C.c_int),
        "sk_kmap_export_os": ([vp, vp, vp, vp], C.c_int),
        "sk_kmap_export_ws": ([vp, vp, vp, vp, vp], C.c_int),
        "sk_kmap_export_split": ([vp, C.c_int, C.c_int, C.c_int] + [C.POINTER(C.c_int)] * 4 +
                                 [vp, vp, vp, vp], C.c_int),
        "sk_conv_forward": ([vp, vp, C.POINTER(DataflowCfg), C.c_int, C.c_int, C.c_int, vp, vp,
                             vp, vp], C.c_int),
        "sk_conv_dgrad": ([vp, vp, C.POINTER(DataflowCfg), C.c_int, C.c_int, C.c_int, vp, vp,
                           vp, vp], C.c_int),
        "sk_conv_wgrad": ([vp, vp, C.POINTER(DataflowCfg), C.c_int, C.c_int, C.c_int, vp, vp,
                           vp, vp], C.c_int),
        "sk_kmap_count_macs": ([vp, C.c_int, C.c_int, C.c_int, C.c_int, C.c_int, i64p, i64p, vp],
                               C.c_int),
        "sk_net_create": ([vp, C.c_int, C.c_char_p, C.c_int, pp], C.c_int),
        "sk_net_destroy": ([vp], C.c_int),
        "sk_net_num_layers": ([vp], C.c_int),
        "sk_net_num_groups": ([vp], C.c_int),
        "sk_net_group_of_layer": ([vp, C.c_int], C.c_int),
        "sk_net_layer_info": ([vp, C.c_int, C.POINTER(C.c_int), C.POINTER(C.c_int),
                               C.POINTER(C.c_int), i64p], C.c_int),
        "sk_net_num_params": ([vp], C.c_int64),
        "sk_net_weight_ptr": ([vp, C.c_int, pp], C.c_int),
        "sk_net_set_config": ([vp, C.c_int, C.c_int, C.POINTER(DataflowCfg)], C.c_int),
        "sk_net_get_config": ([vp, C.c_int, C.c_int, C.POINTER(DataflowCfg)], C.c_int),
        "sk_net_forward": ([vp, vp, vp, C.c_int, vp, pp, C.POINTER(C.c_int), vp, vp], C.c_int),
        "sk_net_layer_output": ([vp, C.c_int, pp, C.POINTER(C.c_int)], C.c_int),
        "sk_net_forward_profiled": ([vp, vp, vp, C.c_int, vp, vp, C.POINTER(C.c_double)], C.c_int),
        "sk_net_measure": ([vp, vp, vp, C.c_int, C.c_int, C.c_int, C.c_int, vp,
                            C.POINTER(C.c_double)], C.c_int),
        "sk_net_map_builds": ([vp], C.c_int64),
        "sk_net_set_overlap": ([vp, C.c_int], C.c_int),
        "sk_net_set_pdl": ([vp, C.c_int], C.c_int),
        "sk_net_set_tune_cold": ([vp, C.c_int], C.c_int),
        "sk_net_group_traffic": ([vp, C.c_int, C.POINTER(DataflowCfg), vp,
                                  C.POINTER(C.c_double)], C.c_int),
        "sk_net_backward": ([vp, vp, vp, C.c_int, C.c_int, C.c_int, vp], C.c_int),
        "sk_net_tune": ([vp, vp, vp, C.c_int, C.c_int, C.c_int, C.c_int, vp,
                         C.POINTER(C.c_double), vp, C.c_int, C.POINTER(C.c_int)], C.c_int),
        "sk_tune_space_size": ([], C.c_int),
        "sk_tune_space_entry": ([C.c_int, C.POINTER(DataflowCfg)], C.c_int),
    }
    for name, (args, res) in sig.items():
        f = getattr(L, name)
        f.argtypes = args
        f.restype = res
    _lib = L
    return L


def check(rc: int) -> None:
    if rc == 0:
        return
    msg = lib().sk_last_error().decode()
    if rc == 1:
        raise ValidationError(msg)
    if rc == 2:
        raise ContractError(msg)
    raise SkError(f"sk200 error {rc}: {msg}")


def i32x3(v) -> "C.Array":
    a = (C.c_int32 * 3)(*[int(x) for x in v])
    return a
