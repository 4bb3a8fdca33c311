"""N3 prefill timing (measurement tool, not product): masq_linear_forward_w4g (packed int4, 128-channel
group scales, tcgen05) against masq_linear_forward (W4 codes in int8 containers, per-channel scales)
on the c3 linears at T tokens (default 16384; CMC rank 64 for the image tokens), CUDA events,
per-kernel times from the library profiler.  Writes gpurun_out/w4g_bench.json."""
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


def timed(fn, reps=10):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    lib().masq_profile_enable(1)
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(reps):
        fn()
    b.record()
    torch.cuda.synchronize()
    nm = ctypes.create_string_buffer(32 * 64)
    tot = (ctypes.c_double * 64)()
    cn = (ctypes.c_int64 * 64)()
    k = lib().masq_profile_collect(64, nm, tot, cn)
    lib().masq_profile_enable(0)
    ker = {nm.raw[32 * i:32 * i + 32].split(b"\0", 1)[0].decode(): tot[i] / reps for i in range(k)}
    return a.elapsed_time(b) / reps, ker


def main():
    dev = torch.device("cuda", 0)
    tokens = [int(x) for x in (sys.argv[1].split(",") if len(sys.argv) > 1 else ["16384", "4096", "1024"])]
    r = 64
    out = {}
    for T in tokens:
        ids = torch.from_numpy(synth.modality_ids(synth.CONFIGS["c3"]["pattern"], T=T)).to(dev)
        for name, d, n in synth.LAYER_LINEARS["c3"]:
            X = (torch.randn(T, d, device=dev) * 2).to(torch.bfloat16)
            W = (torch.randn(d, n, device=dev) / d ** 0.5).to(torch.bfloat16)
            L1 = (torch.randn(1, d, r, device=dev) / d ** 0.5).to(torch.bfloat16)
            L2 = (torch.randn(1, r, n, device=dev) * 0.5).to(torch.bfloat16)
            R, cnt = M.calibrate_stats(X, ids, 2)
            s = M.init_factors(R, cnt, W)
            qw, dw = M.quantize_weight(W, s[0], 4)
            pk, sc = M.quantize_weight_w4g(W, s[0])
            Y = torch.empty(T, n, device=dev)
            ms8, k8 = timed(lambda: M.linear_forward(X, ids, s, qw, dw, 4, 8, L1, L2, Y=Y))
            ms4, k4 = timed(lambda: M.linear_forward_w4g(X, ids, s, pk, sc, 8, L1, L2, Y=Y))
            ops = 2.0 * T * d * n
            g8, g4 = k8.get("gemm_fwd", 0.0), k4.get("gemm_w4g", 0.0)
            rec = {"T": T, "d": d, "n": n,
                   "int8_container": {"call_ms": ms8, "gemm_ms": g8, "weight_bytes": n * d + 4 * n,
                                      "call_tops": ops / (ms8 * 1e-3) / 1e12,
                                      "gemm_tops": ops / (g8 * 1e-3) / 1e12 if g8 else None, "kernels_ms": k8},
                   "w4g_packed": {"call_ms": ms4, "gemm_ms": g4, "weight_bytes": n * d // 2 + 4 * n * (d // 128),
                                  "call_tops": ops / (ms4 * 1e-3) / 1e12,
                                  "gemm_tops": ops / (g4 * 1e-3) / 1e12 if g4 else None, "kernels_ms": k4}}
            out[f"{name}_T{T}"] = rec
            print(name, T, json.dumps({k: (v if not isinstance(v, dict) else {kk: vv for kk, vv in v.items()
                                                                           if kk != "kernels_ms"})
                                       for k, v in rec.items()}), flush=True)
            del X, W, qw, pk, Y
            torch.cuda.empty_cache()
    os.makedirs(os.path.join(ROOT, "gpurun_out"), exist_ok=True)
    json.dump(out, open(os.path.join(ROOT, "gpurun_out", "w4g_bench.json"), "w"), indent=1)


if __name__ == "__main__":
    main()
