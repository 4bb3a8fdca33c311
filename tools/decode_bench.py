"""N3 timing (measurement tool, not product): masq_linear_decode on the c3 linears for T in
{1, 4, 16} decode tokens.  Reports the decode kernel's time (profiler events) and the whole call
captured in a CUDA graph (launch overhead amortised), with achieved GB/s on the algorithmic bytes
(packed codes n*d/2 + scales 4*n*d/128 + X 2*T*d + Y 4*T*n)."""
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


def kernel_ms(fn, name, reps=50):
    fn()
    torch.cuda.synchronize()
    lib().masq_profile_enable(1)
    for _ in range(reps):
        fn()
    torch.cuda.synchronize()
    nm = ctypes.create_string_buffer(32 * 64)
    tot = (ctypes.c_double * 64)()
    cn = (ctypes.c_int64 * 64)()
    k = lib().masq_profile_collect(64, nm, tot, cn)
    lib().masq_profile_enable(0)
    ker = {nm.raw[32 * i:32 * i + 32].split(b"\0", 1)[0].decode(): tot[i] / reps for i in range(k)}
    return ker.get(name, 0.0), ker


def graph_ms(fn, reps=200):
    s = torch.cuda.Stream()
    s.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(s):
        fn()
    torch.cuda.current_stream().wait_stream(s)
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g):
        fn()
    g.replay()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(reps):
        g.replay()
    b.record()
    torch.cuda.synchronize()
    return a.elapsed_time(b) / reps


def main():
    dev = torch.device("cuda", 0)
    peak = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))["hbm_gbs"] if os.path.exists(
        os.path.join(ROOT, "MEASURED_PEAKS.json")) else 6650.0
    out = {"hbm_peak_gbs": peak}
    for name, d, n in synth.LAYER_LINEARS["c3"]:
        W = (torch.randn(d, n, device=dev) / d ** 0.5).to(torch.bfloat16)
        s = torch.rand(d, device=dev) + 0.5
        packed, scales = M.quantize_weight_int4(W, s)
        ws = M.Workspace(dev)
        for T in (1, 4, 16):
            X = (torch.randn(T, d, device=dev) * 3).to(torch.bfloat16)
            Y = torch.empty(T, n, device=dev)
            fn = lambda: M.linear_decode(X, s, packed, scales, Y=Y, ws=ws)   # noqa: E731
            km, ker = kernel_ms(fn, "decode_w4a8")
            gm = graph_ms(fn)
            by = n * d / 2 + 4 * n * d / 128 + 2 * T * d + 4 * T * n
            rec = {"kernel_ms": km, "graph_call_ms": gm, "bytes": by, "kernel_gbs": by / km / 1e6,
                   "kernel_frac_hbm": by / km / 1e6 / peak, "call_gbs": by / gm / 1e6,
                   "bf16_weight_bytes_ratio": (n * d * 2) / by, "kernels": ker}
            out[f"{name}_T{T}"] = rec
            print(name, T, json.dumps({k: v for k, v in rec.items() if k != "kernels"}), flush=True)
    os.makedirs(os.path.join(ROOT, "gpurun_out"), exist_ok=True)
    with open(os.path.join(ROOT, "gpurun_out", "decode_bench.json"), "w") as f:
        json.dump(out, f, indent=1)


if __name__ == "__main__":
    main()
