"""C4 diagnostics: per-layer weight-gradient error of the fp16 / fp32 runners
vs fp64 autograd over the exported maps (dev tool)."""
import os, sys
import numpy as np
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2311_12862_b200 import models as M, network as N, sparse as sk, synth as S

def mre(a, b):
    return float(np.max(np.abs(a - b) / np.maximum(np.abs(b), 1.0)))

layers = M.minkunet18()
n_pts = int(sys.argv[1]) if len(sys.argv) > 1 else 200_000
coords = S.lidar_scan(n_points=n_pts, seed=2)
cs = sk.CoordSet.create(coords)
rng = np.random.default_rng(7)
probe = N.NetworkRunner(layers, dtype=torch.float32)
ws = [torch.from_numpy(rng.standard_normal((kd, ci, co)) / np.sqrt(kd * ci)).half()
      for (kd, ci, co, _) in probe.layer_shapes]
x = torch.from_numpy(np.random.default_rng(8).standard_normal((len(coords), 4))).half()
names = [l.name for l in layers]
sets, fwd, maps = {"": cs}, {}, []
for l in layers:
    src = l.inputs[0] if l.inputs else ""
    if l.kind == "conv":
        o = sk.build_out_coords(sets[src], l.stride)
        key = (src, l.kernel, l.stride)
        if key not in fwd:
            fwd[key] = sk.build_kmap(sets[src], o, l.kernel, l.stride)
        sets[l.name] = o
        maps.append(torch.from_numpy(fwd[key].os()[0]).long().cuda())
    else:
        j = layers[names.index(l.transpose_of)]
        jsrc = j.inputs[0] if j.inputs else ""
        maps.append(torch.from_numpy(fwd[(jsrc, j.kernel, j.stride)].transpose().os()[0]).long().cuda())
        sets[l.name] = sets[jsrc]
wr = [w.double().cuda().requires_grad_(True) for w in ws]
outs = {}
for i, l in enumerate(layers):
    xi = (x.double().cuda() if not l.inputs else outs[l.inputs[0]] if len(l.inputs) == 1
          else outs[l.inputs[0]] + outs[l.inputs[1]])
    ent = maps[i]
    y = torch.zeros(ent.shape[0], l.c_out, dtype=torch.float64, device="cuda")
    for k in range(ent.shape[1]):
        idx = ent[:, k]
        rows = torch.nonzero(idx >= 0).flatten()
        if rows.numel():
            y = y.index_add(0, rows, xi[idx[rows]] @ wr[i][k])
    outs[l.name] = y
    outs[l.name].retain_grad()
y_ref = outs[layers[-1].name]
r = torch.from_numpy(np.random.default_rng(9).standard_normal(tuple(y_ref.shape))).half()
(y_ref * r.double().cuda()).sum().backward()
res = {}
cfgs = {"igemm_s1": sk.DataflowConfig(sk.IMPLICIT_GEMM, 1, sk.tile_large()),
        "fod": sk.DataflowConfig(sk.FETCH_ON_DEMAND),
        "ggs": sk.DataflowConfig(sk.GATHER_GEMM_SCATTER)}
for dtype in ("float32", "float16"):
    for cname, cfg in cfgs.items():
        if dtype == "float32" and cname != "igemm_s1":
            continue
        dt = getattr(torch, dtype)
        net = N.NetworkRunner(layers, dtype=dt)
        for i, w in enumerate(ws):
            net.set_weight(i, w.to(dt).cuda())
        net.weights_updated()
        net.set_all(cfg)
        y, _ = net.forward(cs, x.to(dt).cuda())
        g = torch.zeros(net.num_params, device="cuda")
        net.backward(r.to(dt).cuda(), g)
        torch.cuda.synchronize()
        res[(dtype, cname)] = [net.weight_grad(g, i).double().cpu().numpy() for i in range(len(layers))]
        print(dtype, cname, "out err", mre(y.double().cpu().numpy(), y_ref.detach().cpu().numpy()))
print(f"{'layer':10s} {'K':>2s} {'s':>2s} {'cin':>4s} {'cout':>4s} {'max|dW|':>9s} " +
      " ".join(f"{k[0][-2:]}{k[1]:>9s}" for k in res) + "  16vs32")
for i, l in enumerate(layers):
    want = wr[i].grad.cpu().numpy()
    errs = [mre(v[i], want) for v in res.values()]
    e1632 = mre(res[("float16", "igemm_s1")][i], res[("float32", "igemm_s1")][i])
    print(f"{l.name:10s} {l.kernel:2d} {l.stride:2d} {l.c_in:4d} {l.c_out:4d} {np.abs(want).max():9.3g} " +
          " ".join(f"{e:11.3g}" for e in errs) + f" {e1632:9.3g}")
