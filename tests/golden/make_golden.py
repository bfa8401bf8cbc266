"""Regenerate tests/golden/*.json from the reference's frozen golden vectors.

Run in the build container (needs /root/reference):

    python tests/golden/make_golden.py

fig2.json   the paper's Fig. 2 toy instance, transcribed literally from
            /root/reference/proj/tests/golden.hpp:22-84 (regex extraction of
            the C++ initialiser lists, so the fixture cannot drift from the
            source it pins).
random.json small seeded instances (coords, out coords, OS maps, sorted
            splits, conv outputs) produced by the COMPILED reference
            (oracle/_ref/libsparsekit_ref.so), so GPU tests on a box without
            /root/reference still have reference-made answers.
"""
from __future__ import annotations

import json
import os
import re
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
GOLDEN_HPP = "/root/reference/proj/tests/golden.hpp"


def _body(src: str, fn: str) -> str:
    m = re.search(r"\b" + fn + r"\(\)\s*\{(.*?)\n\}", src, re.S)
    if not m:
        raise SystemExit(f"{fn} not found in golden.hpp")
    return m.group(1)


def _ints(s: str):
    return [int(v) for v in re.findall(r"-?\d+", s)]


def _nums(s: str):
    return [float(v) for v in re.findall(r"-?\d+(?:\.\d+)?", s)]


def fig2() -> dict:
    src = open(GOLDEN_HPP).read()
    # coords: {batch, {x, y, z}} -> 4 ints each
    in_c = _ints(_body(src, "fig_in_coords").split("return", 1)[1])
    out_c = _ints(_body(src, "fig_out_coords").split("return", 1)[1])
    ws_body = _body(src, "fig_ws_pairs").split("return", 1)[1]
    ws = []
    for line in ws_body.strip().splitlines():
        line = line.strip()
        if not line.startswith("{{"):
            continue
        v = _ints(line)
        ws.append([[v[i], v[i + 1]] for i in range(0, len(v), 2)])
    os_ = _ints(_body(src, "fig_os_matrix").split("return", 1)[1])
    masks = _ints(re.search(r"fig_masks\(\)\s*\{\s*return\s*\{(.*?)\};", src, re.S).group(1))
    s1 = _ints(re.search(r"fig_sorted_order_s1\(\)\s*\{\s*return\s*\{(.*?)\};", src,
                         re.S).group(1))
    s3 = _ints(_body(src, "fig_sorted_order_s3").split("return", 1)[1])
    consts = {k: int(v) for k, v in re.findall(r"constexpr int64_t (k\w+) = (\d+);", src)}
    c1 = _nums(re.search(r"fig_conv_c1\(\)\s*\{\s*return\s*\{(.*?)\};", src, re.S).group(1))
    c2 = _nums(_body(src, "fig_conv_c2").split("return", 1)[1])
    return {
        "source": "proj/tests/golden.hpp:22-84",
        "dims": 2, "kernel": 3,
        "in_coords": [in_c[i:i + 4] for i in range(0, len(in_c), 4)],
        "out_coords": [out_c[i:i + 4] for i in range(0, len(out_c), 4)],
        "ws_pairs": ws,
        "os_matrix": [os_[i:i + 9] for i in range(0, len(os_), 9)],
        "masks": masks,
        "sorted_order_s1": s1,
        "sorted_order_s3": [s3[i:i + 6] for i in range(0, len(s3), 6)],
        "effective_macs": consts["kFigEffectiveMacs"],
        "redundant_unsorted": consts["kFigRedundantUnsorted"],
        "redundant_s1": consts["kFigRedundantS1"],
        "redundant_s3": consts["kFigRedundantS3"],
        # conv with x_j = j+1, w_k = k+1 (C=1) and x_j=(j+1,2j), W_k=[[k+1,.5],[-1,k]] (C=2)
        "conv_c1": c1,
        "conv_c2": [c2[i:i + 2] for i in range(0, len(c2), 2)],
    }


def random_instances() -> dict:
    sys.path.insert(0, ROOT)
    from oracle.oracle import Reference

    ref = Reference()
    cases = []
    rng = np.random.default_rng(20231121)
    for i, (n, stride, k, cin, cout) in enumerate([(300, 1, 3, 4, 8), (400, 2, 3, 8, 4),
                                                    (250, 1, 5, 2, 3), (500, 3, 3, 3, 5)]):
        raw = rng.integers(-12, 13, size=(n, 3)).astype(np.int32)
        # first-appearance dedup, the make_random_instance recipe (golden.hpp:95-106)
        _, first = np.unique(raw, axis=0, return_index=True)
        raw = raw[np.sort(first)]
        coords = np.concatenate([np.zeros((len(raw), 1), np.int32), raw], 1)
        st = [stride] * 3
        out = ref.out_coords(3, coords, st)
        m = ref.kmap(3, k, coords, out, st)
        ent, masks = m.os()
        x = rng.standard_normal((len(coords), cin))
        w = rng.standard_normal((m.kd, cin, cout))
        y = ref.conv_ref(m, x, w)
        prep = m.prepare(2, 8)
        cases.append({
            "seed_index": i, "kernel": k, "stride": st,
            "in_coords": coords.tolist(), "out_coords": out.tolist(),
            "os": ent.tolist(), "masks": [[int(v) for v in r] for r in masks],
            "split2_pad8": [{"begin": b, "end": e, "out_row": orow.tolist(),
                             "entries": en.tolist()} for (b, e, en, orow, _) in prep],
            "x": x.tolist(), "w": w.tolist(), "y": y.tolist(),
        })
    return {"source": "oracle/_ref/libsparsekit_ref.so (compiled reference)", "cases": cases}


if __name__ == "__main__":
    with open(os.path.join(HERE, "fig2.json"), "w") as f:
        json.dump(fig2(), f, indent=1)
    with open(os.path.join(HERE, "random.json"), "w") as f:
        json.dump(random_instances(), f)
    print("wrote fig2.json, random.json")
