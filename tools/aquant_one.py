"""Run masq_quantize_activations at a c3 shape (for ncu captures; measurement tool)."""
import os
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import synth  # noqa: E402
import paper_2603_04800_b200 as M  # noqa: E402

d, T = int(os.environ.get("D", 3584)), int(os.environ.get("T", 16384))
dev = torch.device("cuda", 0)
ids = torch.from_numpy(synth.modality_ids(synth.CONFIGS["c3"]["pattern"], T=T)).to(dev)
X = (torch.randn(T, d, device=dev) * 3).to(torch.bfloat16)
s = torch.rand(2, d, device=dev) + 0.5
for _ in range(3):
    qx, dx, mask = M.quantize_activations(X, ids, s, 8)
torch.cuda.synchronize()
print("ok", int(qx.float().abs().sum()))
