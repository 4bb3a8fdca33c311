"""N1 timing (measurement tool, not product): the S-optimisation step at the c3 linears.

Per linear of a c3 decoder layer (T = 16384 calibration tokens): the loss alone
(masq_calib_loss) vs the loss + straight-through gradient (masq_calib_loss_grad) + Adam,
split per kernel, with the gradient GEMM's tensor throughput on its algorithmic flops
(P = X_m^T G and Q' = D^T G: 2 x 2 T d n, which is also what it issues).
"""
import ctypes
import json
import os
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import synth  # noqa: E402
import paper_2603_04800_b200 as M  # noqa: E402
from paper_2603_04800_b200._lib import lib  # noqa: E402


def prof(fn, reps=5):
    fn()
    torch.cuda.synchronize()
    lib().masq_profile_enable(1)
    for _ in range(reps):
        fn()
    torch.cuda.synchronize()
    names = ctypes.create_string_buffer(32 * 64)
    tot = (ctypes.c_double * 64)()
    cnt = (ctypes.c_int64 * 64)()
    n = lib().masq_profile_collect(64, names, tot, cnt)
    lib().masq_profile_enable(0)
    return {names.raw[32 * i:32 * i + 32].split(b"\0", 1)[0].decode(): tot[i] / reps for i in range(n)}


def main():
    dev = torch.device("cuda", 0)
    T = 16384
    ids = torch.from_numpy(synth.modality_ids(synth.CONFIGS["c3"]["pattern"], T=T)).to(dev)
    out = {}
    for name, d, n in synth.LAYER_LINEARS["c3"]:
        X = (torch.randn(T, d, device=dev) * 3).to(torch.bfloat16)
        W = (torch.randn(d, n, device=dev) / d ** 0.5).to(torch.bfloat16)
        R, cnt = M.calibrate_stats(X, ids, 2)
        s = M.init_factors(R, cnt, W)
        Yref = M.reference_output(X, W)
        theta = torch.log(s.double())
        m1, m2 = torch.zeros_like(theta), torch.zeros_like(theta)
        grad = torch.empty_like(theta)
        tl = prof(lambda: M.calib_loss(X, ids, s, W, 4, 8, Yref))
        tg = prof(lambda: (M.calib_loss_grad(X, ids, s, W, 4, 8, Yref, grad=grad),
                           M.adam_step(theta, grad, m1, m2, 1, 1e-3)))
        gg = tg.get("gradgemm", 0.0)
        r = {"loss_ms": sum(tl.values()), "loss_grad_adam_ms": sum(tg.values()), "kernels_ms": tg,
             "gradgemm_tflops_alg": 4.0 * T * d * n / gg / 1e9}
        out[f"{name}_d{d}_n{n}"] = r
        print(name, json.dumps(r), flush=True)
    os.makedirs(os.path.join(ROOT, "gpurun_out"), exist_ok=True)
    with open(os.path.join(ROOT, "gpurun_out", "n1_bench.json"), "w") as f:
        json.dump(out, f, indent=1)


if __name__ == "__main__":
    main()
