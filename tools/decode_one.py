"""Run masq_linear_decode once at the c3 gate_up shape (for ncu captures; measurement tool)."""
import os
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_2603_04800_b200 as M  # noqa: E402

d, n, T = int(os.environ.get("D", 3584)), int(os.environ.get("N", 37888)), int(os.environ.get("T", 1))
dev = torch.device("cuda", 0)
W = (torch.randn(d, n, device=dev) / d ** 0.5).to(torch.bfloat16)
s = torch.rand(d, device=dev) + 0.5
packed, scales = M.quantize_weight_int4(W, s)
X = (torch.randn(T, d, device=dev) * 3).to(torch.bfloat16)
for _ in range(3):
    Y = M.linear_decode(X, s, packed, scales)
torch.cuda.synchronize()
print("ok", float(Y.abs().sum()))
