"""File formats shared with the reference (io.cpp), so
weights and tuned dataflow assignments move between the CPU reference and
sk200 unchanged:

  TSPW weights   read_tspw / write_tspw (io.cpp:163-195): "TSPW", u32 version
                 1, u32 layer count, per layer u32 K^D, C_in, C_out and the
                 [K^D][C_in][C_out] values as little-endian f32
  DataflowConfig dataflow_config_to_json / _from_json (io.cpp:262-300)
  TuneResult     tune_result_to_json / _from_json (io.cpp:310-376), with
                 TuneResult.assignment() (tuner.hpp:74: dgrad / wgrad fall back
                 to the forward choice)

JSON text matches nlohmann::json::dump(2) (sorted keys, two-space indent),
so a file written here is byte-identical to the reference's for the same
content. TilePreset values are the reference's (exec.cpp:45-46); sk200 maps
the reference's small / large presets to its own tcgen05 presets
(sparse.tile_small / tile_large) by name.
"""
from __future__ import annotations

import dataclasses
import json
import struct

import numpy as np

from ._lib import ValidationError
from . import sparse as _sk

TSPW_VERSION = 1
_KINDS = ["gather_gemm_scatter", "fetch_on_demand", "implicit_gemm"]
# TilePreset values of the reference (exec.cpp:45-46) <-> sk200 presets
_REF_SMALL = {"cta_m": 32, "cta_n": 16, "cta_k": 16, "warp_rows": 8, "load_width": 4}
_REF_LARGE = {"cta_m": 64, "cta_n": 32, "cta_k": 32, "warp_rows": 8, "load_width": 8}


# ---- TSPW -------------------------------------------------------------------

def write_tspw(path: str, layers) -> None:
    """layers: sequence of [K^D, C_in, C_out] arrays (any float dtype)."""
    out = bytearray(b"TSPW")
    out += struct.pack("<II", TSPW_VERSION, len(layers))
    for w in layers:
        a = np.asarray(w, dtype=np.float64)
        if a.ndim != 3:
            raise ValidationError("weight tensor must be [K^D, C_in, C_out]")
        out += struct.pack("<III", *a.shape)
        out += a.astype("<f4").tobytes()
    with open(path, "wb") as f:
        f.write(bytes(out))


def read_tspw(path: str):
    """-> list of float32 [K^D, C_in, C_out] arrays; ValidationError on a bad file."""
    buf = open(path, "rb").read()
    pos = 0

    def take(n):
        nonlocal pos
        if pos + n > len(buf):
            raise ValidationError(f"{path}: truncated file")
        b = buf[pos:pos + n]
        pos += n
        return b

    if take(4) != b"TSPW":
        raise ValidationError(f"{path}: bad magic")
    version, n = struct.unpack("<II", take(8))
    if version != TSPW_VERSION:
        raise ValidationError(f"{path}: unsupported version")
    out = []
    for _ in range(n):
        kd, ci, co = struct.unpack("<III", take(12))
        if kd == 0 or ci == 0 or co == 0:
            raise ValidationError(f"{path}: zero-sized weight tensor")
        out.append(np.frombuffer(take(4 * kd * ci * co), dtype="<f4").astype(np.float32)
                   .reshape(kd, ci, co))
    if pos != len(buf):
        raise ValidationError(f"{path}: trailing bytes")
    return out


# ---- DataflowConfig / TuneResult JSON -----------------------------------------

def _cfg_to_obj(cfg: "_sk.DataflowConfig") -> dict:
    if cfg.tile == _sk.tile_large():
        tile = dict(_REF_LARGE)
    elif cfg.tile == _sk.tile_small():
        tile = dict(_REF_SMALL)
    else:
        tile = dataclasses.asdict(cfg.tile)
    return {"kind": _KINDS[cfg.kind], "splits": int(cfg.splits), "tile": tile,
            "reorder": "online" if cfg.reorder else "offline"}


def _cfg_from_obj(j: dict) -> "_sk.DataflowConfig":
    try:
        kind = _KINDS.index(j["kind"])
    except (KeyError, ValueError):
        raise ValidationError(f"unknown dataflow kind: {j.get('kind')}")
    t = dict(_REF_SMALL)
    t.update(j.get("tile", {}))
    if t == _REF_LARGE:
        tile = _sk.tile_large()
    elif t == _REF_SMALL:
        tile = _sk.tile_small()
    else:
        tile = _sk.TilePreset(**{k: int(v) for k, v in t.items()})
    reorder = j.get("reorder", "offline")
    if reorder not in ("offline", "online"):
        raise ValidationError(f"unknown reorder mode: {reorder}")
    splits = int(j.get("splits", 0))
    if splits < 0 or splits > 64:
        raise ValidationError("split count out of range")
    return _sk.DataflowConfig(kind, splits, tile, 1 if reorder == "online" else 0)


def _dump(obj) -> str:
    # nlohmann::json::dump(2): keys sorted (std::map), ", " -> ",\n", ": "
    return json.dumps(obj, indent=2, sort_keys=True, ensure_ascii=False) + "\n"


def dataflow_config_to_json(cfg) -> str:
    return _dump(_cfg_to_obj(cfg))


def dataflow_config_from_json(text: str):
    try:
        return _cfg_from_obj(json.loads(text))
    except json.JSONDecodeError as e:
        raise ValidationError(f"config parse error: {e}")


@dataclasses.dataclass
class GroupChoice:
    id: int
    forward: "_sk.DataflowConfig"
    layer_names: list = dataclasses.field(default_factory=list)
    dgrad: "_sk.DataflowConfig | None" = None
    wgrad: "_sk.DataflowConfig | None" = None


@dataclasses.dataclass
class TuneResult:
    groups: list = dataclasses.field(default_factory=list)
    latency_ms: float = 0.0
    tuning_wall_ms: float = 0.0
    seed: int = 0
    log: list = dataclasses.field(default_factory=list)  # (pass, group, cfg, ms)

    def assignment(self):
        """GroupAssignment (tuner.hpp:74): per group (forward, dgrad, wgrad)."""
        return [(g.forward, g.dgrad or g.forward, g.wgrad or g.forward) for g in self.groups]


def tune_result_to_json(res: TuneResult) -> str:
    groups = []
    for g in res.groups:
        jg = {"id": int(g.id), "layers": list(g.layer_names), "forward": _cfg_to_obj(g.forward)}
        if g.dgrad is not None:
            jg["dgrad"] = _cfg_to_obj(g.dgrad)
        if g.wgrad is not None:
            jg["wgrad"] = _cfg_to_obj(g.wgrad)
        groups.append(jg)
    log = [{"pass": int(p), "group": int(gr), "config": _cfg_to_obj(c), "ms": float(ms)}
           for p, gr, c, ms in res.log]
    return _dump({"groups": groups, "latency_ms": float(res.latency_ms),
                  "tuning_wall_ms": float(res.tuning_wall_ms), "seed": int(res.seed),
                  "log": log})


def tune_result_from_json(text: str) -> TuneResult:
    try:
        j = json.loads(text)
        res = TuneResult(latency_ms=float(j.get("latency_ms", 0.0)),
                         tuning_wall_ms=float(j.get("tuning_wall_ms", 0.0)),
                         seed=int(j.get("seed", 0)))
        for jg in j["groups"]:
            res.groups.append(GroupChoice(
                int(jg["id"]), _cfg_from_obj(jg["forward"]), list(jg.get("layers", [])),
                _cfg_from_obj(jg["dgrad"]) if "dgrad" in jg else None,
                _cfg_from_obj(jg["wgrad"]) if "wgrad" in jg else None))
        for jm in j.get("log", []):
            res.log.append((int(jm.get("pass", 0)), int(jm["group"]),
                            _cfg_from_obj(jm["config"]), float(jm["ms"])))
        return res
    except (json.JSONDecodeError, KeyError, TypeError) as e:
        raise ValidationError(f"tune result parse error: {e}")


def tune_result_of(net, latency_ms: float = 0.0, log=None, seed: int = 0) -> TuneResult:
    """Snapshot a NetworkRunner's installed per-group configs as a TuneResult."""
    res = TuneResult(latency_ms=latency_ms, seed=seed)
    groups = net.groups()
    for g in range(net.num_groups):
        res.groups.append(GroupChoice(g, net.config(g, "forward"),
                                      [net.layers[i].name for i in groups[g]],
                                      net.config(g, "dgrad"), net.config(g, "wgrad")))
    if log is not None:
        from .network import default_space
        space = default_space()
        for row in log:
            res.log.append((int(row[0]), int(row[1]), space[int(row[2])], float(row[3])))
    return res


def apply_tune_result(net, res: TuneResult) -> None:
    """Install a TuneResult's assignment on a NetworkRunner (group ids in order)."""
    if len(res.groups) != net.num_groups:
        raise ValidationError("tune result group count does not match the network")
    for g, (f, d, w) in enumerate(res.assignment()):
        net.set_config(g, f, "forward")
        net.set_config(g, d, "dgrad")
        net.set_config(g, w, "wgrad")
