import sys, ctypes
sys.path.insert(0, '/root/repo'); sys.path.insert(0, '/root/repo/tests')
import torch
import paper_2603_04800_b200 as M
from paper_2603_04800_b200._lib import lib
from test_gpu_parity import bf, case, oracle_state, tt
prof = int(sys.argv[1])
c = case("ragged3"); _, _, so, _, _ = oracle_state(c)
X, W, ids, s = bf(c["X"]), bf(c["W"]), tt(c["ids"]), tt(so)
ws = M.Workspace(torch.device("cuda", 0))
Y = torch.empty(X.shape[0], W.shape[1], device="cuda"); Yr = torch.empty_like(Y)
def step():
    R, cnt = M.calibrate_stats(X, ids, 3, ws=ws)
    M.calib_layer(X, ids, s, W, 8, 8, Y=Y, Yref=Yr, ws=ws)
step(); torch.cuda.synchronize()
if prof: lib().masq_profile_enable(1)
g = torch.cuda.CUDAGraph()
with torch.cuda.graph(g):
    step()
g.replay(); torch.cuda.synchronize()
print("replay ok", torch.cuda.synchronize())
if prof:
    cap = 64
    names = ctypes.create_string_buffer(32 * cap); tot = (ctypes.c_double * cap)(); cnt = (ctypes.c_int64 * cap)()
    nk = lib().masq_profile_collect(cap, names, tot, cnt); lib().masq_profile_enable(0)
    print("collect", nk)
step(); torch.cuda.synchronize(); print("eager after ok")
