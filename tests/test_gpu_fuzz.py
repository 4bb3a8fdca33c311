"""GPU: seeded randomized shapes against the oracle — every §8(a) row through the ABI on small
random problems (d multiple of 16, n multiple of 32, ragged T, 1-4 modalities in random runs,
random bit widths, CMC ranks 0/16/32, f32 and bf16 X), to cover tile and tail boundaries the
fixed configs miss.  Same bars as tests/test_gpu_parity.py."""
import numpy as np
import pytest
import torch

import oracle as O
import synth
from test_gpu_parity import M, TOL_L, TOL_Y, bf, max_abs_norm, max_abs_norm_per_modality, tt

pytestmark = pytest.mark.gpu


def _problem(seed):
    g = np.random.Generator(np.random.PCG64(1000 + seed))
    n_mod = int(g.integers(1, 5))
    d = 16 * int(g.integers(1, 40))
    n = 32 * int(g.integers(1, 20))
    T = max(int(g.integers(1, 1400)), n_mod)           # room for every modality (the oracle rejects empty ones)
    runs, ids = [], []
    while sum(len(x) for x in ids) < T:
        m = int(g.integers(0, n_mod))
        ids.append(np.full(int(g.integers(1, 300)), m, np.uint8))
    ids = np.concatenate(ids)[:T]
    ids[: n_mod] = np.arange(n_mod, dtype=np.uint8)[: min(n_mod, T)]      # every modality present
    gamma = {m: float(np.exp(g.normal(0, 1.5))) for m in range(n_mod)}
    X = synth.activations(ids, d, n_mod, 2000 + seed, gamma=gamma)
    W = synth.weight(d, n, 3000 + seed)
    r = int(g.choice([0, 16, 32])) if n_mod > 1 else 0
    L1, L2 = synth.lowrank(d, n, r, n_mod, 4000 + seed) if r > 0 else (None, None)
    wbits, abits = int(g.integers(2, 9)), int(g.integers(2, 9))
    f32x = bool(g.integers(0, 2)) and r == 0
    return dict(ids=ids, X=X, W=W, L1=L1, L2=L2, n_mod=n_mod, d=d, n=n, T=T, r=r, wbits=wbits, abits=abits,
                f32x=f32x)


def _seeds():
    # MASQ_FUZZ_SEEDS="a:b" widens the sweep for an extended run (default: seeds 0..39)
    import os
    a, b = (int(x) for x in os.environ.get("MASQ_FUZZ_SEEDS", "0:40").split(":"))
    return range(a, b)


@pytest.mark.parametrize("seed", _seeds())
def test_random_problem_parity(seed):
    m = M()
    c = _problem(seed)
    n_mod, wbits, abits = c["n_mod"], c["wbits"], c["abits"]
    Xo = O.decode(c["X"]).astype(np.float32) if c["f32x"] else c["X"]
    Xg = tt(Xo) if c["f32x"] else bf(c["X"])
    ids = tt(c["ids"])
    R, cnt = O.calibrate_stats(Xo, c["ids"], n_mod)
    s = O.init_factors(R, cnt, c["W"])
    Rg, cg = m.calibrate_stats(Xg, ids, n_mod)
    sg = m.init_factors(Rg, cg, bf(c["W"]))
    m.check()
    assert np.array_equal(Rg.cpu().numpy(), R) and np.array_equal(cg.cpu().numpy(), cnt)
    assert np.array_equal(sg.cpu().numpy(), s)
    qw, dw = O.quantize_weight(c["W"], s[0], wbits)
    qwg, dwg = m.quantize_weight(bf(c["W"]), sg[0], wbits)
    assert np.array_equal(qwg.cpu().numpy(), qw) and np.array_equal(dwg.cpu().numpy(), dw)
    qx, dx = O.quantize_activations(Xo, c["ids"], s, abits)
    qxg, dxg, _ = m.quantize_activations(Xg, ids, sg, abits)
    assert np.array_equal(qxg.cpu().numpy(), qx) and np.array_equal(dxg.cpu().numpy(), dx)
    L1 = bf(c["L1"]) if c["r"] else None
    L2 = bf(c["L2"]) if c["r"] else None
    Y = m.linear_forward(Xg, ids, sg, qwg, dwg, wbits, abits, L1, L2).cpu().numpy()
    Yo = O.linear_forward(Xo, c["ids"], s, qw, dw, abits, list(c["L1"]) if c["r"] else None,
                          list(c["L2"]) if c["r"] else None)
    assert max_abs_norm_per_modality(Y, Yo, c["ids"]) <= TOL_Y
    if not c["f32x"]:
        Yref = m.reference_output(Xg, bf(c["W"]))
        sums, counts, loss = m.calib_loss(Xg, ids, sg, bf(c["W"]), wbits, abits, Yref)
        so, co, lo = O.calib_loss(Xo, c["ids"], s, c["W"], wbits, abits)
        assert np.array_equal(counts.cpu().numpy(), co)
        assert abs(float(loss.cpu()[0]) - lo) <= TOL_L * abs(lo) + 1e-300
        Yl, Yr2, s2, c2, l2 = m.calib_layer(Xg, ids, sg, bf(c["W"]), wbits, abits, L1, L2)
        assert torch.equal(Yr2, Yref) and torch.equal(c2, counts)
        assert abs(float(l2.cpu()[0]) - lo) <= TOL_L * abs(lo) + 1e-300


@pytest.mark.parametrize("seed", range(8))
def test_random_gradient_parity(seed):
    """N1 on random shapes: loss and straight-through gradient (with the scale terms)."""
    from test_gpu_grad import TOL_G, _grad_err
    m = M()
    c = _problem(100 + seed)
    if c["f32x"] or c["T"] < 8:
        pytest.skip("bf16 X and a few tokens per modality needed")
    n_mod, wbits, abits = c["n_mod"], c["wbits"], c["abits"]
    R, cnt = O.calibrate_stats(c["X"], c["ids"], n_mod)
    s = O.init_factors(R, cnt, c["W"])
    X, W = bf(c["X"]), bf(c["W"])
    Yref = m.reference_output(X, W)
    _, _, loss, grad = m.calib_loss_grad(X, tt(c["ids"]), tt(s), W, wbits, abits, Yref)
    lo, go = O.calib_loss_grad(c["X"], c["ids"], s, c["W"], wbits, abits)
    assert abs(float(loss.cpu()[0]) - lo) <= TOL_L * abs(lo) + 1e-300
    assert _grad_err(grad.cpu().numpy(), go) <= TOL_G


@pytest.mark.parametrize("seed", range(8))
def test_random_decode_parity(seed):
    """N3 on random shapes: grouped int4 codes bit-exact, decode output vs the oracle."""
    m = M()
    g = np.random.Generator(np.random.PCG64(7000 + seed))
    d, n, T = 128 * int(g.integers(1, 40)), 8 * int(g.integers(1, 200)), int(g.integers(1, 17))
    ids = np.zeros(T, np.uint8)
    X = synth.activations(ids, d, 1, 7100 + seed)
    W = synth.weight(d, n, 7200 + seed)
    s = np.exp(g.normal(0, 0.5, d)).astype(np.float32)
    packed, scales = m.quantize_weight_int4(bf(W), tt(s))
    q, dl = O.quantize_weight_grouped(W, s, 4, 128)
    assert np.array_equal(m.unpack_int4(packed, d, n).cpu().numpy(), q)
    Y = m.linear_decode(bf(X), tt(s), packed, scales).cpu().numpy()
    Yo = O.linear_decode(X, s, q, dl, 8, 128)
    assert max_abs_norm(Y, Yo) <= TOL_Y
