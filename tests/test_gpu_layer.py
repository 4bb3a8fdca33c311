"""GPU: the fused per-linear calibration call (masq_calib_layer) equals the separate calls
(quantize_weight(s[0]) + linear_forward + reference_output + calib_loss): weight codes, Y, Yref
and counts bit for bit; the loss sums to 1e-12 relative (the text rows' |y - yref| is summed in
the forward's epilogue, in token order, instead of in the loss GEMM's grouped order)."""
import numpy as np
import pytest
import torch

import oracle as O
from test_gpu_parity import M, bf, case, oracle_state, tt

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("name,use_cmc", [("c1", True), ("ragged3", True), ("c3_qkv", True), ("c2_qkv", False)])
def test_calib_layer_equals_separate_calls(name, use_cmc):
    m = M()
    c = case(name)
    _, _, so, _, _ = oracle_state(c)
    X, W, ids, s = bf(c["X"]), bf(c["W"]), tt(c["ids"]), tt(so)
    L1 = L2 = None
    if use_cmc and c["r"] > 0:
        L1, L2 = bf(c["L1"]), bf(c["L2"])
    d, n = W.shape
    qt = torch.empty(n, d, dtype=torch.int8, device="cuda")
    dt = torch.empty(n, dtype=torch.float32, device="cuda")
    Y, Yref, sums, counts, loss = m.calib_layer(X, ids, s, W, c["wbits"], c["abits"], L1, L2, qw_text=qt, dw_text=dt)
    m.check()
    qw, dw = m.quantize_weight(W, s[0], c["wbits"])
    Y2 = m.linear_forward(X, ids, s, qw, dw, c["wbits"], c["abits"], L1, L2)
    Yr2 = m.reference_output(X, W)
    s2, c2, l2 = m.calib_loss(X, ids, s, W, c["wbits"], c["abits"], Yr2)
    assert torch.equal(qt, qw) and torch.equal(dt, dw)
    assert torch.equal(Y, Y2) and torch.equal(Yref, Yr2)
    assert torch.equal(counts, c2)
    assert torch.allclose(sums, s2, rtol=1e-12, atol=0) and torch.allclose(loss, l2, rtol=1e-12, atol=0)
    _, _, lo = O.calib_loss(c["X"], c["ids"], so, c["W"], c["wbits"], c["abits"])
    assert abs(float(loss.cpu()[0]) - lo) <= 1e-3 * abs(lo)


@pytest.mark.parametrize("profile", [False, True])
def test_calib_layer_cuda_graph_replay(profile):
    """The library is stream-ordered and allocation-free, so a calibration step can be captured
    as a CUDA graph (also with the opt-in profiler on) and replayed: results equal the eager run."""
    import ctypes
    from paper_2603_04800_b200._lib import lib
    m = M()
    c = case("ragged3")
    _, _, so, _, _ = oracle_state(c)
    X, W, ids, s = bf(c["X"]), bf(c["W"]), tt(c["ids"]), tt(so)
    L1, L2 = bf(c["L1"]), bf(c["L2"])
    ws = m.Workspace(torch.device("cuda", 0))
    n = W.shape[1]
    outs = [torch.empty(X.shape[0], n, device="cuda") for _ in range(2)]
    sums = torch.empty(3, dtype=torch.float64, device="cuda")
    counts = torch.empty(3, dtype=torch.int64, device="cuda")
    loss = torch.empty(1, dtype=torch.float64, device="cuda")
    R = torch.empty(3, X.shape[1], device="cuda")
    cnt = torch.empty(3, dtype=torch.int64, device="cuda")

    def step():
        m.calibrate_stats(X, ids, 3, R=R, count=cnt, ws=ws)
        m.calib_layer(X, ids, s, W, 8, 8, L1, L2, Y=outs[0], Yref=outs[1], sums=sums, counts=counts, loss=loss,
                      ws=ws)

    step()
    torch.cuda.synchronize()
    ref = [t.clone() for t in (outs[0], outs[1], sums, counts, loss, R)]
    if profile:
        lib().masq_profile_enable(1)
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g):
        step()
    for t in (outs[0], outs[1], sums, loss, R):
        t.zero_()
    g.replay()
    g.replay()
    torch.cuda.synchronize()
    if profile:
        names = ctypes.create_string_buffer(32 * 64)
        tot = (ctypes.c_double * 64)()
        cn = (ctypes.c_int64 * 64)()
        assert lib().masq_profile_collect(64, names, tot, cn) > 0
        lib().masq_profile_enable(0)
    for a, b in zip((outs[0], outs[1], sums, counts, loss, R), ref):
        assert torch.equal(a, b)
    m.check(ws)
    step()                                              # eager again after the graph
    torch.cuda.synchronize()
