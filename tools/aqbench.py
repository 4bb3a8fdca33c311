"""Back-to-back timing of masq_quantize_activations (A4) at the c3 shapes (measurement tool).

Times 50 consecutive calls between two CUDA events (so launch gaps are hidden the way they are
inside a step) and reports ms per call and GB/s of algorithmic bytes (2 B read + 1 B code per
activation + 4 B scale per token).  MASQ_AQUANT_V1=1 selects the previous kernel."""
import json
import os
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import synth  # noqa: E402
import paper_2603_04800_b200 as M  # noqa: E402
from paper_2603_04800_b200 import masq as MM  # noqa: E402
from paper_2603_04800_b200._lib import lib  # noqa: E402


def main():
    dev = torch.device("cuda", 0)
    T = int(os.environ.get("AQ_T", 16384))
    ids_h = synth.modality_ids(synth.CONFIGS["c3"]["pattern"], T=T)
    ids = torch.from_numpy(ids_h).to(dev)
    out = {}
    for d in [int(x) for x in os.environ.get("AQ_D", "2048,3584,11008,18944").split(",")]:
        X = (torch.randn(T, d, device=dev) * 3).to(torch.bfloat16)
        s = torch.rand(2, d, device=dev) + 0.5
        qx = torch.empty(T, d, dtype=torch.int8, device=dev)
        dx = torch.empty(T, dtype=torch.float32, device=dev)
        mask = torch.empty((T + 127) // 128, dtype=torch.int32, device=dev)
        ws = MM.default_workspace(dev)
        p, n = ws.ptr_size(MM.workspace_size(MM.OP_QACT, T, d, 0, 2))
        st = torch.cuda.current_stream().cuda_stream

        def call():
            rc = lib().masq_quantize_activations(X.data_ptr(), 1, X.stride(0), ids.data_ptr(), T, d, 2,
                                                 s.data_ptr(), 8, qx.data_ptr(), dx.data_ptr(),
                                                 mask.data_ptr(), p, n, st)
            assert rc == 0, rc
        for _ in range(5):
            call()
        torch.cuda.synchronize()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        reps = 50
        a.record()
        for _ in range(reps):
            call()
        b.record()
        torch.cuda.synchronize()
        ms = a.elapsed_time(b) / reps
        out[f"d{d}"] = dict(ms=ms, gbs=(3 * T * d + 4 * T) / ms / 1e6)
    print(json.dumps(dict(v1=bool(os.environ.get("MASQ_AQUANT_V1")), T=T, res=out)))


if __name__ == "__main__":
    main()
