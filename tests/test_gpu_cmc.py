"""GPU parity for N2: CMC factor construction (masq_cmc_factors) against
oracle.cmc_layer_factors (Theorem 2).

L1 and L2 are unique only up to the sign of each singular pair, so the product L1 L2 is
compared in the norm Theorem 2 is stated in: ||A (P_gpu - P_oracle)||_F <= 1e-6 ||A dW||_F
(f32 outputs), and the optional residual against the oracle's reconstruction loss.
"""
import numpy as np
import pytest
import torch

import oracle as O
import synth
from test_gpu_parity import M, bf, tt

pytestmark = pytest.mark.gpu


def _case(T=2048, d=128, n=192, shuffle=False):
    return synth.config_inputs("c2", T=T, d=d, n=n, r=0, shuffle=shuffle)


@pytest.mark.parametrize("kw,r,eps", [(dict(), 16, 1e-8), (dict(d=96, n=160, shuffle=True), 8, 0.0),
                                      (dict(T=1536, d=208, n=96), 32, 1e-8)])
def test_cmc_factors_parity(kw, r, eps):
    m = M()
    c = _case(**kw)
    n_mod = c["n_mod"]
    R, cnt = O.calibrate_stats(c["X"], c["ids"], n_mod)
    s = O.init_factors(R, cnt, c["W"])
    X, W, ids = bf(c["X"]), bf(c["W"]), tt(c["ids"])
    qw, dw = m.quantize_weight(W, tt(s[0]), c["wbits"])
    L1, L2, resid = m.cmc_factors(X, ids, tt(s), W, qw, dw, r, eps_rel=eps, dtype=torch.float32)
    m.check()
    L1o, L2o, lo = O.cmc_layer_factors(c["X"], c["ids"], s, c["W"], c["wbits"], r, eps)
    xs = O.smooth_activations(O.decode(c["X"]), c["ids"], s)
    qwo, dwo = O.quantize_weight(c["W"], s[0], c["wbits"])
    for k in range(n_mod - 1):
        A = xs[c["ids"] == k + 1].astype(np.float64)
        dW = O.weight_residual(c["W"], s[k + 1], qwo, dwo)
        Pg = L1[k].double().cpu().numpy() @ L2[k].double().cpu().numpy()
        Po = L1o[k] @ L2o[k]
        base = np.linalg.norm(A @ dW)
        assert np.linalg.norm(A @ (Pg - Po)) <= 1e-6 * base
        assert abs(float(resid[k]) - lo[k]) <= 1e-6 * base ** 2
        n1, n2 = O.naive_svd_factors(dW, r)
        assert float(resid[k]) <= O.reconstruction_loss(A, dW, n1, n2)
    # bf16 outputs are the f32 ones rounded to nearest even
    B1, B2, _ = m.cmc_factors(X, ids, tt(s), W, qw, dw, r, eps_rel=eps, dtype=torch.bfloat16, with_resid=False)
    assert torch.equal(B1, L1.to(torch.bfloat16)) and torch.equal(B2, L2.to(torch.bfloat16))


def test_cmc_factors_feed_the_forward():
    """The constructed bf16 factors plug into masq_linear_forward, and CMC reduces the non-text
    output error against the modality's own ideal X_m S_m^-1 . S_m W."""
    m = M()
    c = _case()
    n_mod = c["n_mod"]
    R, cnt = O.calibrate_stats(c["X"], c["ids"], n_mod)
    s = O.init_factors(R, cnt, c["W"])
    X, W, ids = bf(c["X"]), bf(c["W"]), tt(c["ids"])
    qw, dw = m.quantize_weight(W, tt(s[0]), 8)
    L1, L2, _ = m.cmc_factors(X, ids, tt(s), W, qw, dw, 32)
    Y0 = m.linear_forward(X, ids, tt(s), qw, dw, 8, 8).cpu().numpy()
    Y1 = m.linear_forward(X, ids, tt(s), qw, dw, 8, 8, L1, L2).cpu().numpy()
    Yref = O.decode(c["X"]).astype(np.float64) @ O.decode(c["W"]).astype(np.float64)
    nt = c["ids"] != 0
    e0 = np.linalg.norm(Y0[nt] - Yref[nt])
    e1 = np.linalg.norm(Y1[nt] - Yref[nt])
    assert e1 < e0
    assert np.array_equal(Y0[~nt], Y1[~nt])                       # text rows untouched


def test_cmc_factors_errors():
    m = M()
    c = _case(T=512, d=64, n=96)
    X, W, ids = bf(c["X"]), bf(c["W"]), tt(c["ids"])
    s = torch.ones(3, 64, device="cuda")
    qw, dw = m.quantize_weight(W, s[0], 8)
    with pytest.raises(m.MasqError) as e:
        m.cmc_factors(X, ids, s, W, qw, dw, 65)
    assert e.value.status == 2


def test_cmc_two_phase_sharded_equals_one_call():
    """Token-sharded N2: the Grams of two halves accumulated (the single-GPU stand-in for the SUM
    all-reduce) then masq_cmc_factors_from_gram equal the one-call factors (A-weighted norm)
    and the oracle's Gram-route factors."""
    m = M()
    c = _case()
    n_mod = c["n_mod"]
    R, cnt = O.calibrate_stats(c["X"], c["ids"], n_mod)
    s = O.init_factors(R, cnt, c["W"])
    X, W, ids = bf(c["X"]), bf(c["W"]), tt(c["ids"])
    qw, dw = m.quantize_weight(W, tt(s[0]), c["wbits"])
    L1, L2, res1 = m.cmc_factors(X, ids, tt(s), W, qw, dw, 16, dtype=torch.float32)
    h = c["T"] // 2
    G = m.cmc_gram(X[:h], ids[:h], tt(s))
    G = m.cmc_gram(X[h:], ids[h:], tt(s), G=G, accumulate=True)
    P1, P2, res2 = m.cmc_factors_from_gram(G, tt(s), W, qw, dw, 16, dtype=torch.float32)
    m.check()
    xs = O.smooth_activations(O.decode(c["X"]), c["ids"], s)
    qwo, dwo = O.quantize_weight(c["W"], s[0], c["wbits"])
    for k in range(n_mod - 1):
        A = xs[c["ids"] == k + 1].astype(np.float64)
        dW = O.weight_residual(c["W"], s[k + 1], qwo, dwo)
        base = np.linalg.norm(A @ dW)
        a = L1[k].double().cpu().numpy() @ L2[k].double().cpu().numpy()
        b = P1[k].double().cpu().numpy() @ P2[k].double().cpu().numpy()
        assert np.linalg.norm(A @ (a - b)) <= 1e-6 * base
        Gk = np.triu(G[k].cpu().numpy())                         # column-major lower = row-major upper
        Gk = Gk + np.triu(Gk, 1).T
        Go = A.T @ A
        assert np.abs(Gk - Go).max() <= 1e-10 * np.abs(Go).max()
        assert abs(float(res2[k]) - float(res1[k])) <= 1e-6 * base ** 2
