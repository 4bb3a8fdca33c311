"""c5 small-T study (measurement tool, not product): masq_linear_forward at d = 3584 -> n, W4A8, CMC r = 64,
timed (a) eagerly back to back from Python and (b) as one captured CUDA graph replayed back to back,
with the per-kernel breakdown of (b) from the library profiler (events captured into the graph)."""
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
    n = int(os.environ.get("C5_N", 3584))
    r = int(os.environ.get("C5_R", 64))
    out = {}
    for T in [int(x) for x in os.environ.get("C5_T", "1024,2048,4096,8192,16384").split(",")]:
        ids = torch.from_numpy(synth.modality_ids(synth.CONFIGS["c3"]["pattern"], T=T)).to(dev)
        X = (torch.randn(T, 3584, device=dev) * 2).to(torch.bfloat16)
        W = (torch.randn(3584, n, device=dev) / 60).to(torch.bfloat16)
        L1 = (torch.randn(1, 3584, r, device=dev) / 60).to(torch.bfloat16) if r else None
        L2 = (torch.randn(1, r, n, device=dev) * 0.5).to(torch.bfloat16) if r else None
        R, cnt = M.calibrate_stats(X, ids, 2)
        s = M.init_factors(R, cnt, W)
        qw, dw = M.quantize_weight(W, s[0], 4)
        Y = torch.empty(T, n, device=dev)
        ws = M.Workspace(dev)

        def fwd():
            M.linear_forward(X, ids, s, qw, dw, 4, 8, L1, L2, Y=Y, ws=ws)

        for _ in range(5):
            fwd()
        torch.cuda.synchronize()
        reps = 50
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        for _ in range(reps):
            fwd()
        b.record()
        torch.cuda.synchronize()
        eager = a.elapsed_time(b) / reps
        g = torch.cuda.CUDAGraph()
        side = torch.cuda.Stream()
        with torch.cuda.stream(side):
            fwd()
            torch.cuda.synchronize()
            with torch.cuda.graph(g, stream=side):
                fwd()
        torch.cuda.synchronize()
        for _ in range(5):
            g.replay()
        torch.cuda.synchronize()
        a.record()
        for _ in range(reps):
            g.replay()
        b.record()
        torch.cuda.synchronize()
        graph = a.elapsed_time(b) / reps
        lib().masq_profile_enable(1)
        fwd()
        torch.cuda.synchronize()
        nm = ctypes.create_string_buffer(32 * 64)
        tot = (ctypes.c_double * 64)()
        cn = (ctypes.c_int64 * 64)()
        k = lib().masq_profile_collect(64, nm, tot, cn)
        lib().masq_profile_enable(0)
        ker = {nm.raw[32 * i:32 * i + 32].split(b"\0", 1)[0].decode(): round(tot[i] * 1e3, 1) for i in range(k)}
        ops = 2.0 * T * 3584 * n
        rec = {"T": T, "n": n, "r": r, "eager_ms": eager, "graph_ms": graph,
               "eager_tops": ops / (eager * 1e-3) / 1e12, "graph_tops": ops / (graph * 1e-3) / 1e12,
               "kernels_us_single_call": ker}
        out[f"T{T}"] = rec
        print(json.dumps(rec), flush=True)
    os.makedirs(os.path.join(ROOT, "gpurun_out"), exist_ok=True)
    json.dump(out, open(os.path.join(ROOT, "gpurun_out", f"c5_graph_n{n}.json"), "w"), indent=1)


if __name__ == "__main__":
    main()
