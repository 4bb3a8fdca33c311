"""Programmatic dependent launch (csrc/internal.h launch_k, MASQ_PDL, default on): every library
kernel may become resident while its predecessor on the stream drains and must execute
griddepcontrol.wait before its first global access.  A kernel that read or wrote global memory
before that wait would read stale codes / masks / Z rows of the previous call, or overwrite a
workspace buffer its predecessor still reads.  Checked here:
  * chains of calls on ONE stream sharing ONE workspace, issued back to back with no host
    synchronisation, alternating shapes (so each call's workspace buffers hold the other call's
    data until overwritten), give bytes identical to the same calls each followed by a device
    synchronisation: the forward with CMC at small T (split-K first factor + combine kernel, the
    cluster-pair first factor), the fused calibration layer (3 modalities, W8A8), the deep-K
    forward (stream-K GEMM);
  * the same calls in a process with MASQ_PDL=0 (plain stream serialisation) give identical
    bytes (sha256 of every output)."""
import hashlib
import os
import subprocess
import sys

import numpy as np
import pytest
import torch

import synth

pytestmark = pytest.mark.gpu

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)


def _bf(bits):
    return torch.from_numpy(np.ascontiguousarray(bits).view(np.int16)).view(torch.bfloat16).cuda()


def _problems():
    """(kind, inputs on the device) — factors, weights and CMC factors made by the library itself."""
    import paper_2603_04800_b200 as m
    out = []
    for kind, cfg, d, n, T in [("fwd", "c3", 3584, 3584, 1024), ("fwd", "c3", 3584, 3584, 3000),
                               ("fwd", "c3", 3584, 4608, 777), ("layer", "c2", 2048, 2048, 1500),
                               ("layer", "c2", 2048, 2560, 4096), ("fwd", "c3", 9216, 1024, 2500)]:
        c = synth.config_inputs(cfg, d=d, n=n, T=T, layer=3, r=64 if cfg == "c3" else 0)
        X, ids, W = _bf(c["X"]), torch.from_numpy(c["ids"]).cuda(), _bf(c["W"])
        R, cnt = m.calibrate_stats(X, ids, c["n_mod"])
        s = m.init_factors(R, cnt, W)
        qw, dw = m.quantize_weight(W, s[0], c["wbits"])
        L1 = _bf(c["L1"]) if c["r"] else None
        L2 = _bf(c["L2"]) if c["r"] else None
        out.append(dict(kind=kind, X=X, ids=ids, W=W, s=s, qw=qw, dw=dw, L1=L1, L2=L2,
                        wb=c["wbits"], ab=c["abits"]))
    torch.cuda.synchronize()
    return out


def _call(m, p, ws):
    if p["kind"] == "fwd":
        return (m.linear_forward(p["X"], p["ids"], p["s"], p["qw"], p["dw"], p["wb"], p["ab"], p["L1"], p["L2"],
                                 ws=ws),)
    Y, Yref, sums, counts, loss = m.calib_layer(p["X"], p["ids"], p["s"], p["W"], p["wb"], p["ab"], ws=ws)
    return Y, Yref, sums, counts, loss


def _digest(outs):
    h = hashlib.sha256()
    for o in outs:
        h.update(o.detach().cpu().contiguous().view(torch.uint8).numpy().tobytes())
    return h.hexdigest()


def chain_digests():
    """One digest per call of the back-to-back chain (problems in order, then reversed, twice)."""
    import paper_2603_04800_b200 as m
    probs = _problems()
    ws = m.Workspace(probs[0]["X"].device)
    for p in probs:                                 # size the shared workspace once
        _call(m, p, ws)
    torch.cuda.synchronize()
    order = list(range(len(probs))) + list(reversed(range(len(probs)))) + list(range(len(probs)))
    outs = [_call(m, probs[i], ws) for i in order]  # no synchronisation in between
    torch.cuda.synchronize()
    m.check(ws)
    return order, [_digest(o) for o in outs], probs, ws


def test_back_to_back_chain_matches_synchronised_calls():
    import paper_2603_04800_b200 as m
    order, got, probs, ws = chain_digests()
    want = {}
    for i in set(order):
        torch.cuda.synchronize()
        want[i] = _digest(_call(m, probs[i], ws))
        torch.cuda.synchronize()
    for k, i in enumerate(order):
        assert got[k] == want[i], (k, i, probs[i]["kind"], tuple(probs[i]["X"].shape))


SCRIPT = r"""
import sys
sys.path.insert(0, {here!r}); sys.path.insert(0, {root!r})
import test_gpu_pdl as t
order, digests, _, _ = t.chain_digests()
print("DIGESTS", " ".join(digests))
"""


def test_without_pdl_identical_bytes():
    order, got, _, _ = chain_digests()
    env = dict(os.environ)
    env["MASQ_PDL"] = "0"
    p = subprocess.run([sys.executable, "-c", SCRIPT.format(here=HERE, root=ROOT)], env=env, capture_output=True,
                       text=True, timeout=900)
    assert p.returncode == 0, p.stdout[-2000:] + p.stderr[-4000:]
    line = [x for x in p.stdout.splitlines() if x.startswith("DIGESTS ")][-1]
    assert line.split()[1:] == got
