"""Per-kernel timings of the HBM-bound kernels at the c3 shapes (measurement tool, not product).

Reports ms per call and achieved GB/s of algorithmic bytes for stats, activation quantization,
weight quantization (1 and 2 sets) and init, at d = 3584 and d = 18944.
"""
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
    return {names.raw[32 * i:32 * i + 32].split(b"\0", 1)[0].decode(): tot[i] / reps for i in range(n)}


def main():
    dev = torch.device("cuda", 0)
    T = 16384
    ids_h = synth.modality_ids(synth.CONFIGS["c3"]["pattern"], T=T)
    ids = torch.from_numpy(ids_h).to(dev)
    out = {}
    for d, n in ((3584, 18944), (18944, 3584)):
        X = (torch.randn(T, d, device=dev) * 3).to(torch.bfloat16)
        W = (torch.randn(d, n, device=dev) / d ** 0.5).to(torch.bfloat16)
        R, cnt = M.calibrate_stats(X, ids, 2)
        s = M.init_factors(R, cnt, W)
        r = {}
        t = prof(lambda: M.calibrate_stats(X, ids, 2, R=R, count=cnt))
        r["stats_ms"] = t["stats"]
        r["stats_gbs"] = (2 * T * d + T) / t["stats"] / 1e6
        t = prof(lambda: M.quantize_activations(X, ids, s, 8))
        r["aquant_ms"] = t["aquant"]
        r["aquant_gbs"] = (3 * T * d + 4 * T) / t["aquant"] / 1e6
        wkeys = ("wq_strip", "wcolmax", "wscale", "wquant")
        t = prof(lambda: M.quantize_weight(W, s[0], 4))
        r["wq1"] = t
        wt = sum(t.get(k, 0.0) for k in wkeys)
        r["wq1_ms"] = wt
        r["wq1_gbs_1read"] = (2 * d * n + d * n) / wt / 1e6          # algorithmic: W once + codes
        Yref = M.reference_output(X[:2048], W)
        t2 = prof(lambda: M.calib_loss(X[:2048], ids[:2048], s, W, 4, 8, Yref))
        wt2 = sum(t2.get(k, 0.0) for k in wkeys)
        r["wq2_ms"] = wt2
        r["wq2_gbs_1read"] = (2 * d * n + 2 * d * n) / wt2 / 1e6
        t = prof(lambda: M.init_factors(R, cnt, W))
        r["init_ms"] = t["init"]
        r["init_gbs"] = 2 * d * n / t["init"] / 1e6
        out[f"d{d}_n{n}"] = r
    print(json.dumps(out))


if __name__ == "__main__":
    main()
