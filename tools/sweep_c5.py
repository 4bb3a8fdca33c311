"""c5 token-count sweep (BASELINE.json configs[4]): T = 1k .. 256k mixed-modality tokens through
masq_linear_forward at d = 3584 -> n in {3584, 18944}, W4A8, CMC rank r in {0, 64}, 1 GPU.

Inputs are generated on the device with the synth/ recipe's distribution (x = gamma_m c^m_i z,
1% outlier channels, text 1 / image 20, c3 span layout) from a seeded torch generator, because
host generation of 256k x 3584 activations would dominate the run; parity at these sizes is
covered by tests/test_gpu_parity.py (sampled rows).  Reports, per point: whole-call time and
TOP/s (2*T*d*n / call time), the GEMM kernel time and TOP/s, both as fractions of the INT8
peak derived from MEASURED_PEAKS.json (2 x bf16 sustained) and of the 4.5 POP/s spec.
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


def device_inputs(T, d, n, r, seed, dev):
    g = torch.Generator(device=dev)
    g.manual_seed(seed)
    ids_h = synth.modality_ids(synth.CONFIGS["c3"]["pattern"], T=T)
    ids = torch.from_numpy(ids_h).to(dev)
    chan = torch.exp(torch.randn(2, d, generator=g, device=dev))
    out = torch.randperm(d, generator=g, device=dev)[: max(1, d // 100)]
    chan[:, out] *= 10.0
    gam = torch.tensor([1.0, 20.0], device=dev)
    scale = gam[:, None] * chan
    X = torch.randn(T, d, generator=g, device=dev)
    X.mul_(scale[ids.long()])
    X = X.to(torch.bfloat16)
    W = (torch.randn(d, n, generator=g, device=dev) / d ** 0.5).to(torch.bfloat16)
    L1 = (torch.randn(1, d, r, generator=g, device=dev) / d ** 0.5).to(torch.bfloat16) if r else None
    L2 = (torch.randn(1, r, n, generator=g, device=dev) * (4.0 / r ** 0.5)).to(torch.bfloat16) if r else None
    return X, ids, W, L1, L2


def collect():
    names = ctypes.create_string_buffer(32 * 64)
    tot = (ctypes.c_double * 64)()
    cnt = (ctypes.c_int64 * 64)()
    k = lib().masq_profile_collect(64, names, tot, cnt)
    return {names.raw[32 * i:32 * i + 32].split(b"\0", 1)[0].decode(): (tot[i], cnt[i]) for i in range(k)}


def main():
    dev = torch.device("cuda", 0)
    pk = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))
    int8_peak = 2.0 * float(pk["bf16_tflops_sustained"])
    d = 3584
    rows = []
    for n in (3584, 18944):
        for r in (0, 64):
            for k in range(int(os.environ.get("C5_KMAX", "9"))):
                T = 1024 * 2 ** k
                X, ids, W, L1, L2 = device_inputs(T, d, n, r, 260304800 + 4000 + k, dev)
                R, cnt = M.calibrate_stats(X, ids, 2)
                s = M.init_factors(R, cnt, W)
                qw, dw = M.quantize_weight(W, s[0], 4)
                Y = torch.empty(T, n, device=dev)
                fn = lambda: M.linear_forward(X, ids, s, qw, dw, 4, 8, L1, L2, Y=Y)  # noqa: E731
                for _ in range(3):
                    fn()
                torch.cuda.synchronize()
                reps = max(3, min(50, int(2e11 / (2.0 * T * d * n)) + 3))
                # whole-call time with the profiler off (its event pairs would add to small calls),
                # then the per-kernel split with it on
                a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                a.record()
                for _ in range(reps):
                    fn()
                b.record()
                torch.cuda.synchronize()
                call_ms = a.elapsed_time(b) / reps
                lib().masq_profile_enable(1)
                for _ in range(reps):
                    fn()
                torch.cuda.synchronize()
                kern = collect()
                lib().masq_profile_enable(0)
                gemm_ms = kern["gemm_fwd"][0] / reps
                ops = 2.0 * T * d * n
                rows.append(dict(T=T, d=d, n=n, r=r, call_ms=call_ms, gemm_ms=gemm_ms,
                                 call_tops=ops / call_ms / 1e9, gemm_tops=ops / gemm_ms / 1e9,
                                 call_frac_measured=ops / call_ms / 1e9 / int8_peak,
                                 gemm_frac_measured=ops / gemm_ms / 1e9 / int8_peak,
                                 call_frac_spec=ops / call_ms / 1e9 / 4500.0,
                                 kernels_ms={k2: v[0] / reps for k2, v in kern.items()}))
                print(json.dumps(rows[-1]), flush=True)
                del X, W, L1, L2, Y, qw
                torch.cuda.empty_cache()
    print(json.dumps({"c5_sweep": rows, "int8_peak_tops": int8_peak}))


if __name__ == "__main__":
    main()
