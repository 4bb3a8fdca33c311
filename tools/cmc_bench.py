"""N2 timing (measurement tool, not product): masq_cmc_factors at the c3 linears (T = 16384
calibration tokens, r = 64), per stage: the tensor-core Gram (split-bf16, 4 products) with its
executed bf16 rate, and the f64 library stages (Cholesky / small-side GEMMs, eigensolve)."""
import ctypes
import json
import os
import sys
import time

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import synth  # noqa: E402
import paper_2603_04800_b200 as M  # noqa: E402
from paper_2603_04800_b200._lib import lib  # noqa: E402


def main():
    dev = torch.device("cuda", 0)
    T, r = 16384, 64
    ids = torch.from_numpy(synth.modality_ids(synth.CONFIGS["c3"]["pattern"], T=T)).to(dev)
    names = sys.argv[1].split(",") if len(sys.argv) > 1 else ["qkv", "o", "gate_up", "down"]
    out = {}
    for name, d, n in synth.LAYER_LINEARS["c3"]:
        if name not in names:
            continue
        X = (torch.randn(T, d, device=dev) * 3).to(torch.bfloat16)
        W = (torch.randn(d, n, device=dev) / d ** 0.5).to(torch.bfloat16)
        R, cnt = M.calibrate_stats(X, ids, 2)
        s = M.init_factors(R, cnt, W)
        qw, dw = M.quantize_weight(W, s[0], 4)
        M.cmc_factors(X, ids, s, W, qw, dw, r)              # warm (handles, lwork)
        torch.cuda.synchronize()
        lib().masq_profile_enable(1)
        t0 = time.time()
        L1, L2, resid = M.cmc_factors(X, ids, s, W, qw, dw, r)
        torch.cuda.synchronize()
        wall = time.time() - t0
        nm = ctypes.create_string_buffer(32 * 64)
        tot = (ctypes.c_double * 64)()
        cn = (ctypes.c_int64 * 64)()
        k = lib().masq_profile_collect(64, nm, tot, cn)
        lib().masq_profile_enable(0)
        ker = {nm.raw[32 * i:32 * i + 32].split(b"\0", 1)[0].decode(): tot[i] for i in range(k)}
        t_nt = int((ids != 0).sum())
        nti, ntj = -(-d // 128), -(-d // 256)
        tiles = sum(min(nti, 2 * jt + 2) for jt in range(ntj))
        executed = 4 * 2.0 * t_nt * tiles * 128 * 256          # 4 split-bf16 products over the computed tiles
        gms = ker.get("cmc_gram", 0.0)
        total_ms = sum(ker.values())
        eig_ms = sum(v for k_, v in ker.items() if k_.startswith("cmc_eig"))
        rec = {"wall_s": wall, "kernels_ms": ker, "resid": resid.cpu().tolist(), "tokens_non_text": t_nt,
               "gram_ms": gms, "gram_algorithmic_tflop": t_nt * d * d / 1e12,
               "gram_executed_bf16_tflops": executed / (gms / 1e3) / 1e12 if gms else None,
               "eig_ms": eig_ms, "eig_share": eig_ms / total_ms if total_ms else None,
               "route": "small-side n x n" if n < d else "Cholesky + eig(M M^T)"}
        out[f"{name}_d{d}_n{n}"] = rec
        print(name, json.dumps(rec), flush=True)
    os.makedirs(os.path.join(ROOT, "gpurun_out"), exist_ok=True)
    with open(os.path.join(ROOT, "gpurun_out", "cmc_bench.json"), "w") as f:
        json.dump(out, f, indent=1)


if __name__ == "__main__":
    main()
