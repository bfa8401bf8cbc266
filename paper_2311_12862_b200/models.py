"""Network specs in the reference's NetworkSpec vocabulary (network.hpp:20-41).

The reference runner supports only conv / conv_transposed layers with <= 2
summed producers (no concat / BN / ReLU / bias), so the
benchmark networks are written exactly as SURVEY.md Appendix B gives them and
both bench arms (sk200 and the compiled reference) run the SAME spec text:

    name kind c_in c_out kernel stride inputs transpose_of
"""
from __future__ import annotations

from dataclasses import dataclass, field


@dataclass
class Layer:
    name: str
    kind: str
    c_in: int
    c_out: int
    kernel: int = 3
    stride: int = 1
    inputs: list = field(default_factory=list)
    transpose_of: str = ""

    def line(self) -> str:
        ins = ",".join(self.inputs) if self.inputs else "-"
        return (f"{self.name} {self.kind} {self.c_in} {self.c_out} {self.kernel} {self.stride} "
                f"{ins} {self.transpose_of or '-'}")


def spec_text(layers) -> str:
    return "\n".join(l.line() for l in layers) + "\n"


class _Builder:
    def __init__(self):
        self.layers = []
        self.ch = {}

    def conv(self, name, inputs, c_in, c_out, k=3, s=1, kind="conv", tof=""):
        self.layers.append(Layer(name, kind, c_in, c_out, k, s, list(inputs), tof))
        self.ch[name] = c_out
        return name

    def res(self, prefix, xs, co):
        """res(inputs x_0[, x_1] -> co) by linearity."""
        cs = [self.ch[x] if x else None for x in xs]
        a = [self.conv(f"{prefix}_a{i}", [x] if x else [], cs[i], co) for i, x in enumerate(xs)]
        b = self.conv(f"{prefix}_b", a, co, co)
        if len(xs) == 1 and cs[0] == co:
            short = xs[0]
        else:
            p = [self.conv(f"{prefix}_p{i}", [x], cs[i], co, k=1) for i, x in enumerate(xs)]
            short = p[0] if len(p) == 1 else self.conv(f"{prefix}_ps", p, co, co, k=1)
        return self.conv(f"{prefix}_y", [b, short], co, co, k=1)


def minkunet18(in_channels: int = 4, cs=(32, 32, 64, 128, 256, 256, 128, 96, 96)):
    """MinkUNet-18 skeleton: 77 layers, 14 map groups."""
    b = _Builder()
    b.ch[""] = in_channels
    b.conv("stem0", [], in_channels, cs[0])
    x = [b.conv("stem1", ["stem0"], cs[0], cs[0])]
    cur = x[0]
    for i in range(1, 5):
        c = b.ch[cur]
        d = b.conv(f"d{i}", [cur], c, c, 3, 2)
        r = b.res(f"e{i}r0", [d], cs[i])
        cur = b.res(f"e{i}r1", [r], cs[i])
        x.append(cur)
    for j in range(1, 5):
        c = b.ch[cur]
        # u_j: 256->256, 256->128, 128->96, 96->96
        u = b.conv(f"u{j}", [cur], c, cs[4] if j == 1 else cs[4 + j], 3, 2,
                   kind="conv_transposed", tof=f"d{5 - j}")
        r = b.res(f"u{j}r0", [u, x[4 - j]], cs[4 + j])
        cur = b.res(f"u{j}r1", [r], cs[4 + j])
    return b.layers


def second_encoder(in_channels: int = 4):
    """SECOND/CenterPoint sparse 3D encoder: subm 4->16,
    16->16; [s2 conv + 2 subm] at 32/64/64; s2 out 64->128; all K=3."""
    b = _Builder()
    b.conv("conv_in", [], in_channels, 16)
    cur = b.conv("subm0", ["conv_in"], 16, 16)
    for i, c in enumerate((32, 64, 64)):
        cin = b.ch[cur]
        cur = b.conv(f"down{i}", [cur], cin, c, 3, 2)
        cur = b.conv(f"subm{i}a", [cur], c, c)
        cur = b.conv(f"subm{i}b", [cur], c, c)
    b.conv("conv_out", [cur], 64, 128, 3, 2)
    return b.layers


def toy_unet():
    """The 6-layer network of test_net_io.cpp:22-34."""
    return [Layer("c1", "conv", 1, 4, 3, 1, []), Layer("c2", "conv", 4, 4, 3, 1, ["c1"]),
            Layer("down", "conv", 4, 8, 3, 2, ["c2"]), Layer("mid", "conv", 8, 8, 3, 1, ["down"]),
            Layer("up", "conv_transposed", 8, 4, 3, 2, ["mid"], "down"),
            Layer("head", "conv", 4, 2, 3, 1, ["up", "c2"])]
