"""GPU parity for N4: the baseline factor methods — beta closed forms
(SmoothQuant / unified / AWQ), the mean-abs statistic, range ratio / unified range / dominance
counts, and the AWQ beta grid scored by the calibration loss — against the oracle.

Bar: integer and comparison outputs (counts, alpha, unified range, dominance) bit-exact; the
f64-pow factors within 1 ulp of f32; the mean-abs sums within 1e-5 relative (f32 partials over
64-token slabs); grid losses within 1e-3.
"""
import numpy as np
import pytest
import torch

import oracle as O
from test_gpu_parity import M, bf, case, tt

pytestmark = pytest.mark.gpu


def _ulps(a, b):
    return np.abs(a.view(np.int32).astype(np.int64) - b.view(np.int32).astype(np.int64))


@pytest.mark.parametrize("beta", [0.0, 0.3, 0.5, 0.85, 1.0])
def test_smooth_factors(beta):
    m = M()
    g = np.random.Generator(np.random.PCG64(21))
    R = np.exp(g.normal(0, 2, (3, 4096))).astype(np.float32)
    R[0, :7] = 0.0                                              # floored numerators
    wm = np.exp(g.normal(-2, 1, 4096)).astype(np.float32)
    s = m.smooth_factors(tt(R), beta, den=tt(wm)).cpu().numpy()
    assert _ulps(s, O.smooth_factors(R, wm, beta)).max() <= 1
    s2 = m.smooth_factors(tt(R), beta).cpu().numpy()
    assert _ulps(s2, O.smooth_factors(R, None, beta)).max() <= 1


@pytest.mark.parametrize("name", ["c1", "ragged3", "c2_qkv"])
def test_meanabs_and_range_stats(name):
    m = M()
    c = case(name)
    n_mod = c["n_mod"]
    S, cnt, mean, uni = m.calibrate_meanabs(bf(c["X"]), tt(c["ids"]), n_mod)
    m.check()
    So, co = O.meanabs_stats(c["X"], c["ids"], n_mod)
    assert np.array_equal(cnt.cpu().numpy(), co)
    assert np.allclose(S.cpu().numpy(), So, rtol=1e-5, atol=0)
    mo = (So / co[:, None]).astype(np.float32)
    assert np.allclose(mean.cpu().numpy(), mo, rtol=1e-5)
    assert np.allclose(uni.cpu().numpy(), (So.sum(0) / co.sum()).astype(np.float32), rtol=1e-5)
    # accumulation over two batches == one pass
    h = (c["T"] // 2) // 64 * 64
    X, ids = bf(c["X"]), tt(c["ids"])
    S2, c2, _, _ = m.calibrate_meanabs(X[:h], ids[:h], n_mod)
    S2, c2, _, _ = m.calibrate_meanabs(X[h:], ids[h:], n_mod, sumabs=S2, count=c2, reset=False)
    assert torch.equal(c2, cnt) and np.allclose(S2.cpu().numpy(), So, rtol=1e-5)
    # range statistics from the A1 ranges
    R, _ = O.calibrate_stats(c["X"], c["ids"], n_mod)
    alpha, runi, dom = m.range_stats(tt(R), 1, 0)
    assert np.array_equal(alpha.cpu().numpy(), O.range_ratio(R, 1, 0))
    assert np.array_equal(runi.cpu().numpy(), O.unified_stats(R))
    assert np.array_equal(dom.cpu().numpy(), O.dominance_stats(R))


def test_range_stats_ties_and_spec_examples():
    m = M()
    d = 512
    base = np.exp(np.random.Generator(np.random.PCG64(3)).normal(0, 1, d)).astype(np.float32)
    R = np.stack([base * np.float32(10), base])
    alpha, _, dom = m.range_stats(tt(R), 0, 1)
    assert np.array_equal(alpha.cpu().numpy(), O.range_ratio(R, 0, 1)) and dom.cpu().tolist() == [d, 0, 0]
    T3 = np.stack([base, base, base * np.float32(0.5)])
    _, _, dom = m.range_stats(tt(T3), 0, 1)
    assert dom.cpu().tolist() == [d, 0, 0, d]                   # all tied between 0 and 1 -> first + tied


def test_unified_factors_and_awq_grid():
    from paper_2603_04800_b200 import baselines as B
    m = M()
    c = case("ragged3")
    n_mod = c["n_mod"]
    X, W, ids = bf(c["X"]), bf(c["W"]), tt(c["ids"])
    R, cnt = m.calibrate_stats(X, ids, n_mod)
    _, wmax = m.init_factors(R, cnt, W, return_wmax=True)
    su = B.unified_factors(R, wmax, 0.5).cpu().numpy()
    Ro, _ = O.calibrate_stats(c["X"], c["ids"], n_mod)
    suo = O.smooth_factors(O.unified_stats(Ro), O.weight_absmax(c["W"]), 0.5)
    assert _ulps(su, np.repeat(suo[None], n_mod, 0)).max() <= 1
    betas = [0.0, 0.25, 0.5, 0.75]
    b, losses, _ = B.awq_grid_search(X, ids, W, 4, 8, betas, n_mod)
    bo, lo = O.awq_grid_search(c["X"], c["ids"], c["W"], 4, 8, betas, n_mod)
    assert np.allclose(losses, lo, rtol=1e-3)
    assert b == bo


def test_count_modalities():
    m = M()
    c = case("ragged3")
    cnt = m.count_modalities(tt(c["ids"]), 3)
    assert cnt.cpu().tolist() == np.bincount(c["ids"], minlength=3).tolist()
    cnt = m.count_modalities(tt(c["ids"][:100]), 3, count=cnt, reset=False)
    assert cnt.cpu().tolist() == (np.bincount(c["ids"], minlength=3) + np.bincount(c["ids"][:100], minlength=3)).tolist()
