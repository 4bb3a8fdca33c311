"""Inspect the loss workspace (perm, tile_mod, grouped qx/dx, partials) after masq_calib_loss."""
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
X, W = bf(c["X"]), bf(c["W"])
Yref = M.reference_output(X, W)
s, n_, l = M.calib_loss(X, tt(c["ids"]), tt(so), W, 8, 8, Yref)
torch.cuda.synchronize()
ws = M.masq.default_workspace()
base = ws.buf.data_ptr(); off0 = (-base) % 256
buf = ws.buf[off0:].cpu().numpy()
T, d, n, Mm = 1000, 208, 288, 3
a256 = lambda x: (x + 255) // 256 * 256
Tg = ((T + 127) // 128) * 128 + Mm * 128
o = 0; o += a256(256)
inv_o = o; o += a256(4 * Mm * d)
qx_o = o; o += a256(Tg * d)
dx_o = o; o += a256(4 * Tg)
perm_o = o; o += a256(4 * Tg)
tm_o = o; o += a256(4 * (Tg // 128))
qw_o = o; o += a256(Mm * n * d)
dw_o = o; o += a256(4 * Mm * n)
am_o = o; o += a256(4 * Mm * n)
pa_o = o
perm = buf[perm_o:perm_o + 4 * Tg].view(np.int32)
tm = buf[tm_o:tm_o + 4 * (Tg // 128)].view(np.uint32)
print("Tg", Tg, "tile_mod", tm)
print("perm head", perm[:8], "valid", (perm >= 0).sum())
ids = c["ids"]
for m in range(3):
    sel = np.nonzero(ids == m)[0]
    print("mod", m, "count", sel.size)
# expected perm: stable grouping
qx = buf[qx_o:qx_o + Tg * d].view(np.int8).reshape(Tg, d)
dx = buf[dx_o:dx_o + 4 * Tg].view(np.float32)
qxo, dxo = O.quantize_activations(c["X"], ids, so, 8)
ok = [np.array_equal(qx[p], qxo[perm[p]]) and dx[p] == dxo[perm[p]] for p in range(Tg) if perm[p] >= 0]
print("grouped qx rows correct:", sum(ok), "of", len(ok))
qw = buf[qw_o:qw_o + Mm * n * d].view(np.int8).reshape(Mm, n, d)
for m in range(3):
    qo, do = O.quantize_weight(c["W"], so[m], 8)
    print("qw set", m, np.array_equal(qw[m], qo))
num_n = (n + 255) // 256
pa = buf[pa_o:pa_o + 8 * (Tg // 128) * num_n * 8].view(np.float64).reshape(Tg // 128, num_n, 8)
print("partials per tile", pa.sum(axis=2))
print("sums", s.cpu().numpy())
dw = buf[dw_o:dw_o + 4 * Mm * n].view(np.float32).reshape(Mm, n)
for m in range(3):
    qo, do = O.quantize_weight(c["W"], so[m], 8)
    bad = np.nonzero(qw[m] != qo)
    print("set", m, "bad codes", bad[0].size, "rows(j) with bad:", np.unique(bad[0])[:10], "cols(i):", np.unique(bad[1])[:20])
    print("   dw equal", np.array_equal(dw[m], do), "first dw", dw[m][:3], do[:3])
    if bad[0].size:
        j, i = bad[0][0], bad[1][0]
        print("   sample", j, i, qw[m][j, i], qo[j, i])
