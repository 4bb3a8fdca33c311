"""X.W reference GEMM (A8's target, kModeRef) alone at one shape (measurement tool): for ncu DRAM
traffic / raster experiments.  usage: python tools/refgemm.py [d] [n] [T] [reps]"""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2603_04800_b200 as M  # noqa: E402


def main():
    d = int(sys.argv[1]) if len(sys.argv) > 1 else 3584
    n = int(sys.argv[2]) if len(sys.argv) > 2 else 37888
    T = int(sys.argv[3]) if len(sys.argv) > 3 else 16384
    reps = int(sys.argv[4]) if len(sys.argv) > 4 else 3
    dev = torch.device("cuda", 0)
    X = (torch.randn(T, d, device=dev)).to(torch.bfloat16)
    W = (torch.randn(d, n, device=dev) / d ** 0.5).to(torch.bfloat16)
    Y = torch.empty(T, n, device=dev)
    for _ in range(2):
        M.reference_output(X, W, Yref=Y)
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(reps):
        M.reference_output(X, W, Yref=Y)
    b.record()
    torch.cuda.synchronize()
    ms = a.elapsed_time(b) / reps
    print(f"group={os.environ.get('MASQ_RASTER_GROUP', 'default')} d={d} n={n} T={T} ms={ms:.4f} "
          f"tflops={2 * T * d * n / ms / 1e9:.1f}")


if __name__ == "__main__":
    main()
