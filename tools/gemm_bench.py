"""Micro-benchmark of the forward GEMM variants at one linear shape (measurement tool, not product).

Times (CUDA events, kernel-level via the library profiler): gemm_fwd with r=0 / r=64, the
acc debug tap, the bf16 X.W GEMM, and cuBLAS int8 (torch._int_mm) on the same shape as an anchor.
"""
import argparse
import ctypes
import json
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import synth  # noqa: E402
import paper_2603_04800_b200 as M  # noqa: E402
from paper_2603_04800_b200._lib import lib  # noqa: E402


def prof(fn, reps=10):
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
    out = {}
    for i in range(n):
        nm = names.raw[32 * i:32 * i + 32].split(b"\0", 1)[0].decode()
        out[nm] = tot[i] / reps
    return out


def evt(fn, reps=10):
    fn()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(reps):
        fn()
    b.record()
    torch.cuda.synchronize()
    return a.elapsed_time(b) / reps


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--T", type=int, default=16384)
    ap.add_argument("--d", type=int, default=3584)
    ap.add_argument("--n", type=int, default=18944)
    args = ap.parse_args()
    T, d, n = args.T, args.d, args.n
    dev = torch.device("cuda", 0)
    ids = synth.modality_ids(synth.CONFIGS["c3"]["pattern"], T=T)
    X = torch.from_numpy(synth.activations(ids, d, 2, 1).view(np.int16)).view(torch.bfloat16).to(dev)
    W = (torch.randn(d, n, device=dev) / d ** 0.5).to(torch.bfloat16)
    L1 = (torch.randn(1, d, 64, device=dev) / d ** 0.5).to(torch.bfloat16)
    L2 = (torch.randn(1, 64, n, device=dev) / 8).to(torch.bfloat16)
    idt = torch.from_numpy(ids).to(dev)
    R, cnt = M.calibrate_stats(X, idt, 2)
    s = M.init_factors(R, cnt, W)
    qw, dw = M.quantize_weight(W, s[0], 4)
    Y = torch.empty(T, n, device=dev)
    ops = 2.0 * T * d * n
    res = {"shape": [T, d, n]}
    res["fwd_r0"] = prof(lambda: M.linear_forward(X, idt, s, qw, dw, 4, 8, Y=Y))
    res["fwd_r64"] = prof(lambda: M.linear_forward(X, idt, s, qw, dw, 4, 8, L1, L2, Y=Y))
    res["acc"] = prof(lambda: M.linear_forward(X, idt, s, qw, dw, 4, 8, acc_debug=True))
    res["ref"] = prof(lambda: M.reference_output(X, W, Yref=Y))
    qx, dx, _ = M.quantize_activations(X, idt, s, 8)
    qwt = qw.t()
    try:
        res["cublas_int_mm_ms"] = evt(lambda: torch._int_mm(qx, qwt))
    except Exception as e:  # noqa: BLE001
        res["cublas_int_mm_ms"] = repr(e)
    Xt = X
    Wc = W.contiguous()
    res["cublas_bf16_ms"] = evt(lambda: torch.matmul(Xt, Wc))
    a = torch.randint(-128, 127, (8192, 8192), dtype=torch.int8, device=dev)
    b = torch.randint(-128, 127, (8192, 8192), dtype=torch.int8, device=dev).t()
    res["cublas_int_mm_8192_ms"] = evt(lambda: torch._int_mm(a, b))
    res["cublas_int_mm_8192_tops"] = 2 * 8192 ** 3 / (res["cublas_int_mm_8192_ms"] / 1e3) / 1e12
    for k in ("fwd_r0", "fwd_r64", "acc"):
        g = res[k].get("gemm_fwd", res[k].get("gemm_acc"))
        res[k + "_gemm_tops"] = ops / (g / 1e3) / 1e12
    res["ref_tflops"] = ops / (res["ref"]["gemm_ref"] / 1e3) / 1e12
    if isinstance(res["cublas_int_mm_ms"], float):
        res["cublas_int_mm_tops"] = ops / (res["cublas_int_mm_ms"] / 1e3) / 1e12
    res["cublas_bf16_tflops"] = ops / (res["cublas_bf16_ms"] / 1e3) / 1e12
    print(json.dumps(res))


if __name__ == "__main__":
    main()
