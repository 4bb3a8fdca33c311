"""Debug: determinism of calib_loss on the ragged3 case, and per-set weight codes vs the oracle."""
import os, sys
import numpy as np
import torch
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import oracle as O
import synth
import paper_2603_04800_b200 as M

c = synth.config_inputs("c2", T=1000, d=208, n=288, r=48)
bf = lambda b: torch.from_numpy(np.ascontiguousarray(b).view(np.int16)).view(torch.bfloat16).cuda()
tt = lambda a: torch.from_numpy(np.ascontiguousarray(a)).cuda()
R, cnt = O.calibrate_stats(c["X"], c["ids"], 3)
so = O.init_factors(R, cnt, c["W"])
for k in range(3):
    qw, dw = M.quantize_weight(bf(c["W"]), tt(so[k]), 8)
    qo, do = O.quantize_weight(c["W"], so[k], 8)
    print("set", k, "codes equal", np.array_equal(qw.cpu().numpy(), qo), "dw equal", np.array_equal(dw.cpu().numpy(), do))
X, W = bf(c["X"]), bf(c["W"])
Yref = M.reference_output(X, W)
outs = []
for it in range(4):
    s, n_, l = M.calib_loss(X, tt(c["ids"]), tt(so), W, 8, 8, Yref)
    torch.cuda.synchronize()
    outs.append(s.cpu().numpy())
    print("run", it, s.cpu().numpy(), n_.cpu().numpy(), float(l.cpu()[0]))
so_, co_, lo = O.calib_loss(c["X"], c["ids"], so, c["W"], 8, 8)
print("oracle", so_, co_, lo)

# pieces through the public API
qx, dx, mask = M.quantize_activations(X, tt(c["ids"]), tt(so), 8)
qxo, dxo = O.quantize_activations(c["X"], c["ids"], so, 8)
print("qx equal", np.array_equal(qx.cpu().numpy(), qxo), "dx equal", np.array_equal(dx.cpu().numpy(), dxo))
Yr = Yref.cpu().numpy().astype(np.float64)
tot = []
for m in range(3):
    qw, dw = M.quantize_weight(W, tt(so[m]), 8)
    acc = M.linear_forward(X, tt(c["ids"]), tt(so), qw, dw, 8, 8, acc_debug=True).cpu().numpy().astype(np.float64)
    y = acc * dxo[:, None].astype(np.float64) * dw.cpu().numpy().astype(np.float64)[None, :]
    sel = c["ids"] == m
    tot.append(np.abs(y[sel] - Yr[sel]).sum())
print("python-composed sums", tot)
