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
