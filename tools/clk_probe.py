"""SM clock (NVML) while the int8 forward GEMM runs back to back at the gate_up shape, with and
without its Y stores (MASQ_GEMM_EXP=2) — measurement tool: is the store cost a power/clock effect?"""
import os
import sys
import threading
import time

import pynvml
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_2603_04800_b200 as M  # noqa: E402

dev = torch.device("cuda", 0)
T, d, n = 16384, 3584, 37888
ids = torch.zeros(T, dtype=torch.uint8, device=dev)
X = (torch.randn(T, d, device=dev)).to(torch.bfloat16)
W = (torch.randn(d, n, device=dev) / 60).to(torch.bfloat16)
R, cnt = M.calibrate_stats(X, ids, 1)
s = M.init_factors(R, cnt, W)
qw, dw = M.quantize_weight(W, s[0], 4)
Y = torch.empty(T, n, device=dev)
for _ in range(3):
    M.linear_forward(X, ids, s, qw, dw, 4, 8, Y=Y)
torch.cuda.synchronize()
pynvml.nvmlInit()
h = pynvml.nvmlDeviceGetHandleByIndex(0)
clk, pw = [], []
stop = False


def sampler():
    while not stop:
        clk.append(pynvml.nvmlDeviceGetClockInfo(h, pynvml.NVML_CLOCK_SM))
        pw.append(pynvml.nvmlDeviceGetPowerUsage(h) / 1000.0)
        time.sleep(0.005)


th = threading.Thread(target=sampler)
th.start()
a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
a.record()
for _ in range(200):
    M.linear_forward(X, ids, s, qw, dw, 4, 8, Y=Y)
b.record()
torch.cuda.synchronize()
stop = True
th.join()
ms = a.elapsed_time(b) / 200
clk.sort()
pw.sort()
print(f"exp={os.environ.get('MASQ_GEMM_EXP', '0')} call_ms={ms:.3f} sm_mhz_median={clk[len(clk) // 2]} "
      f"power_w_median={pw[len(pw) // 2]:.0f} samples={len(clk)}")
