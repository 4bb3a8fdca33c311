"""A3 weight quantization alone (measurement tool): masq_quantize_weight with one factor set (the public
call) at the four c3 linears, per-kernel ms from the library profiler and the algorithmic
rate (one bf16 W read + one int8 code set per weight).  Run once per kernel variant (env knobs)."""
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


def main():
    dev = torch.device("cuda", 0)
    out = {"env": {k: v for k, v in os.environ.items() if k.startswith("MASQ_")}}
    for name, d, n in synth.LAYER_LINEARS["c3"]:
        W = (torch.randn(d, n, device=dev) / d ** 0.5).to(torch.bfloat16)
        s = torch.exp(torch.randn(d, device=dev) * 0.5).contiguous()
        for _ in range(2):
            M.quantize_weight(W, s, 4)
        torch.cuda.synchronize()
        reps = 10
        lib().masq_profile_enable(1)
        for _ in range(reps):
            M.quantize_weight(W, s, 4)
        torch.cuda.synchronize()
        nm = ctypes.create_string_buffer(32 * 64)
        tot = (ctypes.c_double * 64)()
        cn = (ctypes.c_int64 * 64)()
        k = lib().masq_profile_collect(64, nm, tot, cn)
        lib().masq_profile_enable(0)
        ker = {nm.raw[32 * i:32 * i + 32].split(b"\0", 1)[0].decode(): tot[i] / reps for i in range(k)}
        ms = sum(ker.values())
        out[name] = {"d": d, "n": n, "kernels_ms": ker, "ms": ms, "GBps": 3.0 * d * n / ms / 1e6}
        print(name, json.dumps(out[name]), flush=True)
        del W
    print(json.dumps(out))


if __name__ == "__main__":
    main()
