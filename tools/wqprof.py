import os, sys, torch
sys.path.insert(0, "/root/repo")
import synth, paper_2603_04800_b200 as M
dev = torch.device("cuda", 0)
T = 2048
ids = torch.from_numpy(synth.modality_ids(synth.CONFIGS["c3"]["pattern"], T=T)).to(dev)
d, n = 3584, 37888
X = (torch.randn(T, d, device=dev) * 3).to(torch.bfloat16)
W = (torch.randn(d, n, device=dev) / d ** 0.5).to(torch.bfloat16)
R, cnt = M.calibrate_stats(X, ids, 2)
s = M.init_factors(R, cnt, W)
Yref = M.reference_output(X, W)
for _ in range(3):
    M.calib_loss(X, ids, s, W, 4, 8, Yref)
torch.cuda.synchronize()
