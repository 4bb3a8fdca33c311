"""One masq_linear_forward_w4g call at a c3 shape (measurement tool for ncu; not product)."""
import os
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import synth  # noqa: E402
import paper_2603_04800_b200 as M  # noqa: E402

T = int(sys.argv[1]) if len(sys.argv) > 1 else 16384
d, n = (int(x) for x in (sys.argv[2].split("x") if len(sys.argv) > 2 else ["3584", "37888"]))
dev = torch.device("cuda", 0)
ids = torch.from_numpy(synth.modality_ids(synth.CONFIGS["c3"]["pattern"], T=T)).to(dev)
X = (torch.randn(T, d, device=dev) * 2).to(torch.bfloat16)
W = (torch.randn(d, n, device=dev) / d ** 0.5).to(torch.bfloat16)
R, cnt = M.calibrate_stats(X, ids, 2)
s = M.init_factors(R, cnt, W)
pk, sc = M.quantize_weight_w4g(W, s[0])
Y = torch.empty(T, n, device=dev)
for _ in range(3):
    M.linear_forward_w4g(X, ids, s, pk, sc, 8, Y=Y)
torch.cuda.synchronize()
print("ok")
