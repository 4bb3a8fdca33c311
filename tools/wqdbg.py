import os, subprocess, sys, json
import numpy as np
code = r'''
import os, sys, numpy as np, torch
sys.path.insert(0, "/root/repo")
import paper_2603_04800_b200 as M
d, n = int(sys.argv[1]), int(sys.argv[2])
g = torch.Generator(device="cuda"); g.manual_seed(5)
W = (torch.randn(d, n, generator=g, device="cuda") / d ** 0.5).to(torch.bfloat16)
s = (torch.rand(d, generator=g, device="cuda") + 0.5)
qw, dw = M.quantize_weight(W, s, 4)
torch.cuda.synchronize()
np.save(sys.argv[3], qw.cpu().numpy())
'''
open("/tmp/wqd.py", "w").write(code)
d, n = 3584, 4608
subprocess.run([sys.executable, "/tmp/wqd.py", str(d), str(n), "/tmp/a.npy"], env=dict(os.environ, MASQ_WQUANT_V1="1"), check=True)
subprocess.run([sys.executable, "/tmp/wqd.py", str(d), str(n), "/tmp/b.npy"], check=True)
a, b = np.load("/tmp/a.npy"), np.load("/tmp/b.npy")
bad = np.argwhere(a != b)
print("mismatches", len(bad), "of", a.size)
if len(bad):
    js, is_ = bad[:, 0], bad[:, 1]
    tj, ti = js // 128, is_ // 128
    tiles = sorted(set(zip(ti.tolist(), tj.tolist())))
    print("bad tiles (it, jt):", len(tiles), tiles[:20])
    tj_n = (n + 127) // 128
    ts = sorted(set(int(x) * tj_n + int(y) for x, y in tiles))
    print("tile ids:", ts[:40])
    print("iteration index k = t // 296:", sorted(set(t // 296 for t in ts)))
