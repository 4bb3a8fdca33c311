"""Pins of the CPU oracle against what the paper and the mathematics fix (no GPU).

Each test names the passage / identity it checks.  None of them re-types the
oracle's own formula: they use brute force, closed forms, special cases,
invariants or hand-worked values (tests/golden/).
"""
import itertools
import json
import os

import numpy as np
import pytest

import oracle as O
import synth

GOLD = os.path.join(os.path.dirname(__file__), "golden")
F32 = np.float32


def rng(seed=0):
    return np.random.Generator(np.random.PCG64(seed))


# ----------------------------------------------------------------------------- O1 stats
def test_stats_brute_force_loop():
    """O1 vs a naive per-element loop."""
    g = rng(1)
    T, d, M = 37, 11, 3
    X = g.standard_normal((T, d)).astype(F32) * 5
    ids = g.integers(0, M, T).astype(np.uint8)
    R, cnt = O.calibrate_stats(X, ids, M)
    for m in range(M):
        for i in range(d):
            best = 0.0
            for t in range(T):
                if ids[t] == m:
                    best = max(best, abs(float(X[t, i])))
            assert R[m, i] == F32(best)
        assert cnt[m] == int(sum(1 for t in range(T) if ids[t] == m))


def test_stats_identity_and_single_token():
    """X = I -> all ones; single token -> |x|."""
    R, cnt = O.calibrate_stats(np.eye(8, dtype=F32), np.zeros(8, np.uint8), 1)
    assert np.all(R == 1) and cnt[0] == 8
    x = np.array([[-3.5, 0.25, 0.0, 7.0]], F32)
    R, _ = O.calibrate_stats(x, np.array([1], np.uint8), 2)
    assert np.array_equal(R[1], np.abs(x[0])) and np.all(R[0] == 0)


def test_stats_unified_reduction():
    """max_m R^m == unified stats of the untagged X (PAPER.md:37 s^uni uses max over m,t)."""
    c = synth.config_inputs("c1")
    R, _ = O.calibrate_stats(c["X"], c["ids"], 2)
    Ru, _ = O.calibrate_stats(c["X"], np.zeros_like(c["ids"]), 1)
    assert np.array_equal(R.max(axis=0), Ru[0])


def test_stats_batch_coherence():
    """Running max over batches == one pass."""
    c = synth.config_inputs("c1")
    R1, n1 = O.calibrate_stats(c["X"], c["ids"], 2)
    R, n = None, None
    for a, b in [(0, 50), (50, 51), (51, 256)]:
        R, n = O.calibrate_stats(c["X"][a:b], c["ids"][a:b], 2, R, n)
    assert np.array_equal(R, R1) and np.array_equal(n, n1)


def test_stats_rejects_unknown_modality():
    with pytest.raises(ValueError):
        O.calibrate_stats(np.ones((2, 2), F32), np.array([0, 3], np.uint8), 2)


# ----------------------------------------------------------------------------- O2 init
def test_init_spec_examples():
    g = json.load(open(os.path.join(GOLD, "spec_examples.json")))
    for ex in g["init_factors"]:
        W = np.array([[ex["wmax"], -ex["wmax"] / 2]], F32)          # row absmax = wmax
        s = O.init_factors(np.array([[ex["R"]]], F32), np.array([1]), W)
        assert s[0, 0] == F32(ex["s"]), ex["citation"]


def test_init_equals_smoothquant_beta_half():
    """s^m = sqrt(R/wmax) equals SmoothQuant beta=0.5, R^0.5 / wmax^0.5 (PAPER.md:22 vs 57)."""
    c = synth.config_inputs("c1")
    R, cnt = O.calibrate_stats(c["X"], c["ids"], 2)
    s = O.init_factors(R, cnt, c["W"])
    wmax = np.abs(O.decode(c["W"]).astype(np.float64)).max(axis=1)
    sq = np.power(R.astype(np.float64), 0.5) / np.power(wmax, 0.5)[None, :]
    rel = np.abs(s.astype(np.float64) - sq) / sq
    assert rel.max() <= 2.0 ** -23        # within one f32 ulp


def test_init_rejects_empty_modality():
    with pytest.raises(ValueError):
        O.init_factors(np.ones((2, 3), F32), np.array([5, 0]), np.ones((3, 4), F32))


def test_init_floor_zero_range():
    """Zero range / zero weight row are floored at 1e-12."""
    s = O.init_factors(np.zeros((1, 2), F32), np.array([1]), np.array([[0.0, 0.0], [1.0, 1.0]], F32))
    assert s[0, 0] == F32(1.0) and s[0, 1] == np.sqrt(F32(1e-12), dtype=F32)


# ----------------------------------------------------------------------------- quantizer
def test_rha_edges():
    v = np.array([0.49999997, 0.5, -0.5, 1.5, 2.5, -2.5, -0.49999997, 3.0, -7.5], F32)
    assert rha_list(v) == [0, 1, -1, 2, 3, -3, 0, 3, -8]


def rha_list(v):
    return [int(x) for x in O.rha(v)]


@pytest.mark.parametrize("bits", [2, 3, 4, 6, 8])
def test_quantizer_brute_force_nearest_code(bits):
    """Code == nearest of all 2^b grid points to x/Delta, ties -> larger magnitude."""
    g = rng(bits)
    A = (g.standard_normal((40, 25)) * np.exp(g.standard_normal((40, 1)))).astype(F32)
    A[0, :5] = [0.5, -0.5, 1.5, 2.5, -3.5]                 # exact half-grid points on row 0
    codes, delta = O.quantize_rows(A, bits)
    grid = np.arange(-(2 ** (bits - 1)), 2 ** (bits - 1))
    for r in range(A.shape[0]):
        v = np.divide(A[r], delta[r], dtype=F32).astype(np.float64)
        for i, vi in enumerate(v):
            dist = np.abs(grid - vi)
            best = grid[dist == dist.min()]
            want = best[np.argmax(np.abs(best))]
            assert codes[r, i] == want, (r, i, vi)


def test_quantizer_spec_examples():
    g = json.load(open(os.path.join(GOLD, "spec_examples.json")))
    for ex in g["quantizer"]:
        codes, delta = O.quantize_rows(np.array([ex["x"]], F32), ex["bits"])
        want_delta = F32(1.0) / F32(127.0) if ex["delta"] == "1/127" else F32(1e-12)
        assert delta[0] == want_delta, ex["citation"]
        assert list(codes[0]) == ex["codes_by_hand"], ex["citation"]


@pytest.mark.parametrize("bits", [4, 8])
def test_quantizer_properties(bits):
    """Saturation, error bound |Q(x)-x| <= Delta/2, idempotence, power-of-two scale covariance
    (PAPER.md:76)."""
    g = rng(10 + bits)
    A = (g.standard_normal((64, 100)) * 3).astype(F32)
    qmax = 2 ** (bits - 1) - 1
    codes, delta = O.quantize_rows(A, bits)
    assert np.all(np.abs(codes).max(axis=1) == qmax)                      # saturation
    err = np.abs(O.dequantize_rows(codes, delta) - A.astype(np.float64))
    assert np.all(err <= delta[:, None].astype(np.float64) * (0.5 + 1e-6))  # rounding bound
    deq = np.multiply(codes.astype(F32), delta[:, None], dtype=F32)
    again = np.clip(O.rha(np.divide(deq, delta[:, None], dtype=F32)), -qmax - 1, qmax)
    assert np.array_equal(again.astype(np.int8), codes)                   # idempotence
    for k in (-3, 5):
        c2, d2 = O.quantize_rows(A * F32(2.0 ** k), bits)
        assert np.array_equal(c2, codes) and np.array_equal(d2, delta * F32(2.0 ** k))


def test_quantizer_zero_row():
    codes, delta = O.quantize_rows(np.zeros((2, 8), F32), 8)
    assert np.all(codes == 0) and np.all(delta == F32(1e-12))


# ----------------------------------------------------------------------------- O5
def test_int_gemm_vs_triple_loop():
    g = rng(5)
    qx = g.integers(-128, 128, (5, 33)).astype(np.int8)
    qw = g.integers(-128, 128, (7, 33)).astype(np.int8)
    acc = O.int_gemm(qx, qw)
    for t, j in itertools.product(range(5), range(7)):
        assert acc[t, j] == sum(int(qx[t, i]) * int(qw[j, i]) for i in range(33))


def test_int_gemm_extreme_magnitude_exact():
    """|acc| <= 127*127*d; at d = 18944 (c3 down) the f64 path is still exact (< 2^53)."""
    d = 18944
    qx = np.full((2, d), 127, np.int8)
    qx[1, ::2] = -128
    qw = np.full((2, d), -128, np.int8)
    acc = O.int_gemm(qx, qw)
    assert acc[0, 0] == 127 * -128 * d
    assert acc[1, 1] == (d // 2) * (-128 * -128) + (d // 2) * (127 * -128)


# ----------------------------------------------------------------------------- invariance
def test_invariance_before_quantization():
    """(X S^-1)(S W) = X W: exact for power-of-two s, <= 1e-6 rel for any s
    (the only rounding is the f32 smoothing of X, reading Q6)."""
    g = rng(7)
    for seed in range(20):
        g = rng(100 + seed)
        d = int(g.integers(2, 64))
        X = g.standard_normal((9, d)).astype(F32)
        W = g.standard_normal((d, 5)).astype(F32)
        ids = np.zeros(9, np.uint8)
        s2 = (2.0 ** g.integers(-6, 7, d)).astype(F32)
        xs = O.smooth_activations(X, ids, s2[None, :]).astype(np.float64)
        sw = (s2[:, None].astype(np.float64) * W)
        assert np.array_equal(xs @ sw, X.astype(np.float64) @ W.astype(np.float64)) or \
            np.allclose(xs @ sw, X.astype(np.float64) @ W, rtol=1e-12, atol=1e-12)
        s = np.exp(g.standard_normal(d)).astype(F32)
        xs = O.smooth_activations(X, ids, s[None, :]).astype(np.float64)
        ref = X.astype(np.float64) @ W
        rel = np.linalg.norm(xs @ (s[:, None].astype(np.float64) * W) - ref) / np.linalg.norm(ref)
        assert rel <= 1e-6


def _grid_aligned_case(seed=3, T=6, d=8, n=5, abits=8, wbits=4):
    """Inputs on which every quantization is lossless: power-of-two s and Deltas,
    integer codes with one saturated code per row / column."""
    g = rng(seed)
    qa, qw_ = 2 ** (abits - 1) - 1, 2 ** (wbits - 1) - 1
    s0 = (2.0 ** g.integers(-3, 4, d)).astype(F32)
    s = np.stack([s0, s0 * F32(4.0)])                     # S_1 = 4 S_0 keeps S_1 W lossless
    ids = np.array([0, 1, 0, 1, 1, 0][:T], np.uint8)
    cx = g.integers(-qa, qa + 1, (T, d)).astype(np.float64)
    cx[:, 0] = qa
    dx = 2.0 ** g.integers(-4, 3, T)
    xs = cx * dx[:, None]
    X = (xs * s[ids].astype(np.float64)).astype(F32)      # X = xs S  (exact: powers of two)
    cw = g.integers(-qw_, qw_ + 1, (d, n)).astype(np.float64)
    cw[0, :] = qw_
    dw = 2.0 ** g.integers(-5, 0, n)
    W = ((cw * dw[None, :]) / s0[:, None].astype(np.float64)).astype(F32)   # S_0 W on the grid
    return X, ids, s, W


def test_grid_aligned_lossless_forward_and_loss():
    """On grid-aligned inputs Q is the identity, so:
    text rows Y = X W exactly; image rows without CMC Y = (X S_v^-1)(S_t W) = X W / 4 exactly
    (S_v = 4 S_t: the cross-modal invariance break of PAPER.md:126-132); with the exact
    full-rank correction L1 = I, L2 = S_v W - Q(S_t W) = 3 S_t W, Y = X W exactly; L = 0."""
    X, ids, s, W = _grid_aligned_case()
    qw, dw = O.quantize_weight(W, s[0], 4)
    Y = O.linear_forward(X, ids, s, qw, dw, 8)
    XW = O.reference_output(X, W)
    text = ids == 0
    assert np.array_equal(Y[text], XW[text])
    assert np.array_equal(Y[~text], XW[~text] / 4)
    d = W.shape[0]
    dW = 3.0 * s[0].astype(np.float64)[:, None] * W.astype(np.float64)
    Yc = O.linear_forward(X, ids, s, qw, dw, 8, L1=[np.eye(d)], L2=[dW])
    assert np.array_equal(Yc, XW)
    sums, counts, loss = O.calib_loss(X, ids, s, W, 4, 8)
    assert loss == 0.0 and np.all(sums == 0) and list(counts) == [3, 3]


# ----------------------------------------------------------------------------- O7 CMC
def test_cmc_full_rank_identity():
    """With L1 L2 = Delta W = S_m W - deqQ(S_t W) exactly (L1 = I),
    Y_m - xs S_m W = (deqQ(xs) - xs) . deqQ(S_t W)  (PAPER.md:131 + 183)."""
    c = synth.config_inputs("c1")
    R, cnt = O.calibrate_stats(c["X"], c["ids"], 2)
    s = O.init_factors(R, cnt, c["W"])
    qw, dw = O.quantize_weight(c["W"], s[0], 8)
    base = (qw.astype(np.float64) * dw[:, None].astype(np.float64)).T          # deqQ(S_t W) [d x n]
    Wf = O.decode(c["W"]).astype(np.float64)
    dW = s[1].astype(np.float64)[:, None] * Wf - base
    d = Wf.shape[0]
    Y = O.linear_forward(c["X"], c["ids"], s, qw, dw, 8, L1=[np.eye(d)], L2=[dW])
    img = np.nonzero(c["ids"] == 1)[0]
    xs = O.smooth_activations(c["X"], c["ids"], s)[img].astype(np.float64)
    qx, dx = O.quantize_rows(xs.astype(F32), 8)
    lhs = Y[img] - xs @ (s[1].astype(np.float64)[:, None] * Wf)
    rhs = (O.dequantize_rows(qx, dx) - xs) @ base
    assert np.abs(lhs - rhs).max() <= 1e-9 * np.abs(Y[img]).max()


def test_cmc_rank0_all_text_and_routing():
    """rank 0 == base formula; all-text input ignores L; an image token's output does not
    depend on other modalities' factors."""
    c = synth.config_inputs("c2", d=64, n=48, T=1024, r=16)
    R, cnt = O.calibrate_stats(c["X"], c["ids"], 3)
    s = O.init_factors(R, cnt, c["W"])
    qw, dw = O.quantize_weight(c["W"], s[0], 8)
    L1 = [c["L1"][0], c["L1"][1]]
    L2 = [c["L2"][0], c["L2"][1]]
    Y0 = O.linear_forward(c["X"], c["ids"], s, qw, dw, 8)
    Y = O.linear_forward(c["X"], c["ids"], s, qw, dw, 8, L1, L2)
    text = c["ids"] == 0
    assert np.array_equal(Y[text], Y0[text]) and not np.array_equal(Y[~text], Y0[~text])
    ids_t = np.zeros_like(c["ids"])
    assert np.array_equal(O.linear_forward(c["X"], ids_t, s, qw, dw, 8, L1, L2),
                          O.linear_forward(c["X"], ids_t, s, qw, dw, 8))
    s_alt = s.copy()
    s_alt[2] *= F32(3.0)
    Ya = O.linear_forward(c["X"], c["ids"], s_alt, qw, dw, 8, L1, L2)
    img = c["ids"] == 1
    assert np.array_equal(Ya[img], Y[img])


def test_forward_order_equivariance_and_partition():
    """Permuting tokens permutes rows; per-modality sub-batches recombine."""
    c = synth.config_inputs("c1")
    R, cnt = O.calibrate_stats(c["X"], c["ids"], 2)
    s = O.init_factors(R, cnt, c["W"])
    qw, dw = O.quantize_weight(c["W"], s[0], 8)
    L1, L2 = [c["L1"][0]], [c["L2"][0]]
    Y = O.linear_forward(c["X"], c["ids"], s, qw, dw, 8, L1, L2)
    p = rng(9).permutation(c["T"])
    Yp = O.linear_forward(c["X"][p], c["ids"][p], s, qw, dw, 8, L1, L2)
    assert np.array_equal(Yp, Y[p])
    for m in (0, 1):
        sel = np.nonzero(c["ids"] == m)[0]
        Ym = O.linear_forward(c["X"][sel], c["ids"][sel], s, qw, dw, 8, L1, L2)
        assert np.array_equal(Ym, Y[sel])
    rows = np.array([3, 100, 255, 41])
    assert np.array_equal(O.linear_forward(c["X"], c["ids"], s, qw, dw, 8, L1, L2, rows=rows), Y[rows])


# ----------------------------------------------------------------------------- O8 loss
def test_loss_separability():
    """Mixed-batch per-modality sums == sums on each modality's sub-batch."""
    c = synth.config_inputs("c2", d=64, n=40, T=1024)
    R, cnt = O.calibrate_stats(c["X"], c["ids"], 3)
    s = O.init_factors(R, cnt, c["W"])
    sums, counts, loss = O.calib_loss(c["X"], c["ids"], s, c["W"], 4, 8)
    tot = 0.0
    for m in range(3):
        sel = np.nonzero(c["ids"] == m)[0]
        sm, cm, lm = O.calib_loss(c["X"][sel], c["ids"][sel], s, c["W"], 4, 8)
        assert np.isclose(sm[m], sums[m], rtol=1e-12) and cm[m] == counts[m]
        tot += lm
    assert np.isclose(tot, loss, rtol=1e-12)


# ----------------------------------------------------------------------------- golden
def test_hand_worked_example():
    g = json.load(open(os.path.join(GOLD, "hand_worked_w4a8.json")))
    i, e = g["inputs"], g["expected"]
    X = np.array(i["X"], F32)
    ids = np.array(i["ids"], np.uint8)
    s = np.array(i["s"], F32)
    W = np.array(i["W"], F32)
    qx, dx = O.quantize_activations(X, ids, s, i["abits"])
    assert qx.tolist() == e["qx"]
    qw, dw = O.quantize_weight(W, s[0], i["wbits"])
    assert qw.tolist() == e["qw_text_kmajor"]
    assert O.int_gemm(qx, qw).tolist() == e["acc"]
    Y0 = O.linear_forward(X, ids, s, qw, dw, i["abits"])
    assert np.allclose(Y0, e["Y_rank0"], rtol=1e-6, atol=1e-6)
    L1 = [np.array(i["L1_image"])]
    L2 = [np.array(i["L2_image"])]
    Y = O.linear_forward(X, ids, s, qw, dw, i["abits"], L1, L2)
    assert np.allclose(Y, e["Y_cmc"], rtol=1e-6, atol=1e-6)
    assert np.array_equal(O.reference_output(X, W), np.array(e["XW"]))
    sums, counts, loss = O.calib_loss(X, ids, s, W, i["wbits"], i["abits"])
    # the hand values use exact rationals; the oracle's Deltas are f32 (reading Q6), and the
    # loss is a difference of O(15)-sized outputs, so compare at 1e-6 of the output scale.
    assert np.allclose(sums, e["loss_sums"], rtol=0, atol=2e-5)
    assert counts.tolist() == e["loss_counts"]
    assert np.isclose(loss, e["loss"], rtol=0, atol=2e-5)


# ----------------------------------------------------------------------------- N1 gradient
def _autograd_ste_loss_grad(X, ids, s, W, wbits, abits):
    """Independent implementation of the straight-through graph with torch.autograd (f64):
    Delta = max(amax|u| / q_max, 1e-12) differentiable (through the arg-max element);
    Q(u) = Delta * (v + (round_half_away(v) - v).detach()), v = u / Delta — only round() is
    straight-through (reading Q24)."""
    import torch
    Xt = torch.from_numpy(O.decode(X).astype(np.float64))
    Wt = torch.from_numpy(O.decode(W).astype(np.float64))
    theta = torch.tensor(np.log(s.astype(np.float64)), requires_grad=True)

    def q_rows(u, bits):
        qmax = 2 ** (bits - 1) - 1
        delta = (u.abs().amax(dim=1, keepdim=True) / qmax).clamp_min(1e-12)
        v = u / delta
        vd = v.detach()
        r = torch.trunc(vd) + torch.sign(vd) * (torch.abs(vd - torch.trunc(vd)) >= 0.5)
        return delta * (v + (r.clamp(-qmax - 1, qmax) - vd))

    loss = 0.0
    n = Wt.shape[1]
    for m in range(s.shape[0]):
        sel = torch.from_numpy(np.nonzero(ids == m)[0])
        A = Xt[sel] * torch.exp(-theta[m])[None, :]
        B = torch.exp(theta[m])[:, None] * Wt
        Ah = q_rows(A, abits)
        Bh = q_rows(B.T, wbits).T                                   # per output channel
        E = Ah @ Bh - Xt[sel] @ Wt
        loss = loss + E.abs().sum() / (sel.numel() * n)
    loss.backward()
    return float(loss.detach()), theta.grad.numpy()


def test_loss_grad_matches_autograd_ste():
    """N1 pin: the closed-form straight-through gradient (incl. the arg-max scale terms) equals
    torch.autograd on the STE graph (up to the f32 smoothing / quantization of the oracle;
    codes are identical on these inputs, and no |.|-maximum is tied)."""
    c = synth.config_inputs("c2", T=1024, d=32, n=48)
    R, cnt = O.calibrate_stats(c["X"], c["ids"], 3)
    s = O.init_factors(R, cnt, c["W"])
    loss, grad = O.calib_loss_grad(c["X"], c["ids"], s, c["W"], 4, 8)
    _, _, loss_o8 = O.calib_loss(c["X"], c["ids"], s, c["W"], 4, 8)
    assert np.isclose(loss, loss_o8, rtol=1e-12)
    la, ga = _autograd_ste_loss_grad(c["X"], c["ids"], s, c["W"], 4, 8)
    assert np.isclose(la, loss, rtol=1e-5)
    assert np.abs(grad - ga).max() <= 1e-4 * np.abs(ga).max()


def test_loss_grad_uniform_rescale_is_a_null_direction():
    """s^m -> c s^m leaves every code and the loss unchanged (absmax scales rescale with it), and
    the straight-through gradient with the scale terms sees that: sum_i grad_i = 0 per modality
    (up to rounding), while dropping the scale terms (Delta held constant) would not."""
    c = synth.config_inputs("c1")
    R, cnt = O.calibrate_stats(c["X"], c["ids"], 2)
    s = O.init_factors(R, cnt, c["W"])
    loss, grad = O.calib_loss_grad(c["X"], c["ids"], s, c["W"], 4, 8)
    _, _, l2 = O.calib_loss(c["X"], c["ids"], s * np.float32(2.0), c["W"], 4, 8)
    assert abs(l2 - loss) <= 1e-12 * loss                         # exact invariance (power of 2)
    assert np.all(np.abs(grad.sum(axis=1)) <= 1e-9 * np.abs(grad).sum(axis=1))


def test_loss_grad_descent_direction_and_adam():
    """A small step against the gradient does not increase the (piecewise) loss; Adam's first
    step moves every coordinate by ~lr against the gradient sign (closed form at step 1)."""
    c = synth.config_inputs("c1")
    R, cnt = O.calibrate_stats(c["X"], c["ids"], 2)
    s = O.init_factors(R, cnt, c["W"])
    loss0, grad = O.calib_loss_grad(c["X"], c["ids"], s, c["W"], 4, 8)
    theta = np.log(s.astype(np.float64))
    th1, m1, m2 = O.adam_step(theta, grad, np.zeros_like(theta), np.zeros_like(theta), 1, 1e-3)
    nz = grad != 0
    step = (th1 - theta)[nz]
    assert np.all(np.sign(step) == -np.sign(grad[nz])) and np.all(np.abs(step) <= 1e-3 * (1 + 1e-12))
    assert np.all(np.abs(step) >= 1e-3 * (1 - 1e-8 / np.abs(grad[nz])) * (1 - 1e-9))
    assert np.all(th1[~nz] == theta[~nz])
    _, _, loss1 = O.calib_loss(c["X"], c["ids"], np.exp(th1).astype(np.float32), c["W"], 4, 8)
    assert loss1 <= loss0 * (1 + 1e-3)


def test_optimize_factors_contract():
    """SPEC.md:307-316 optimize_factors: epochs = 0 returns the init unchanged; the result is
    the best-so-far iterate (objective never above the init's, and equal to the objective
    recomputed at the returned factors); positivity is preserved."""
    c = synth.config_inputs("c1")
    R, cnt = O.calibrate_stats(c["X"], c["ids"], 2)
    s0 = O.init_factors(R, cnt, c["W"])
    L0 = O.calib_loss(c["X"], c["ids"], s0, c["W"], 4, 8)[2]
    s, best, hist = O.optimize_factors(c["X"], c["ids"], s0, c["W"], 4, 8, epochs=0)
    assert np.array_equal(s, s0) and best == L0 and hist == []
    s, best, hist = O.optimize_factors(c["X"], c["ids"], s0, c["W"], 4, 8, epochs=2, batch_tokens=64, lr=3e-2)
    assert len(hist) == 2 and best <= L0 and np.all(s > 0)
    assert best == O.calib_loss(c["X"], c["ids"], s, c["W"], 4, 8)[2]
    assert best == min([L0] + hist)


def test_optimize_factors_beats_unified_smoothing():
    """SPEC.md:315 example: a two-modality layer with a 30x range gap, W4A8, 2 epochs — the
    weighted loss ends strictly below the unified-smoothing closed form (one s from the range
    over all tokens, PAPER.md:19-23 / 36-39) on the same data."""
    g = np.random.Generator(np.random.PCG64(11))
    T, d, n = 512, 64, 96
    ids = np.repeat(np.array([0, 1, 0, 1], np.uint8), T // 4)
    ch = np.exp(g.normal(0, 0.5, d))
    X = g.normal(0, 1, (T, d)) * ch * np.where(ids == 1, 30.0, 1.0)[:, None]
    X = synth.f32_to_bf16_bits(X.astype(np.float32))
    W = synth.f32_to_bf16_bits((g.normal(0, 1, (d, n)) / np.sqrt(d)).astype(np.float32))
    R, cnt = O.calibrate_stats(X, ids, 2)
    Ru = np.repeat(R.max(axis=0, keepdims=True), 2, axis=0)
    su = O.init_factors(Ru, cnt, W)                      # unified: the same s for both modalities
    Lu = O.calib_loss(X, ids, su, W, 4, 8)[2]
    s0 = O.init_factors(R, cnt, W)
    s, best, _ = O.optimize_factors(X, ids, s0, W, 4, 8, epochs=2, batch_tokens=128)
    assert best < Lu


# ----------------------------------------------------------------------------- N4 baselines
def test_smooth_factors_closed_forms():
    """beta = 1 returns R exactly; beta = 0 returns 1/wmax (correctly rounded); beta = 0.5
    agrees with the A2 init sequence sqrt(R / wmax) within 1 ulp; log s = beta log(R wmax) -
    log wmax is increasing in beta exactly where R wmax > 1."""
    g = np.random.Generator(np.random.PCG64(5))
    R = np.exp(g.normal(0, 2, (2, 300))).astype(np.float32)
    wm = np.exp(g.normal(-2, 1, 300)).astype(np.float32)
    assert np.array_equal(O.smooth_factors(R, wm, 1.0), R)
    assert np.array_equal(O.smooth_factors(R, wm, 0.0)[0], (1.0 / wm.astype(np.float64)).astype(np.float32))
    s5 = O.smooth_factors(R, wm, 0.5)
    ref = np.sqrt(np.divide(R, wm[None, :], dtype=np.float32), dtype=np.float32)
    assert np.all(np.abs(s5.view(np.int32) - ref.view(np.int32)) <= 1)
    assert np.array_equal(O.smooth_factors(R, None, 1.0), R)
    hi = R.astype(np.float64) * wm[None, :] > 1.0
    assert np.all(O.smooth_factors(R, wm, 0.7)[hi] >= O.smooth_factors(R, wm, 0.6)[hi])
    assert np.all(O.smooth_factors(R, wm, 0.7)[~hi] <= O.smooth_factors(R, wm, 0.6)[~hi])


def test_range_ratio_and_dominance_spec_examples():
    """SPEC.md:317-326 / 484-490 examples, plus a loop oracle on random profiles."""
    g = np.random.Generator(np.random.PCG64(6))
    R = np.exp(g.normal(0, 1, (3, 64))).astype(np.float32)
    assert np.array_equal(O.range_ratio(R[[0, 0]], 0, 1), np.ones(64, np.float32))     # identical
    R10 = np.stack([R[0] * np.float32(10), R[0]])
    assert np.allclose(O.range_ratio(R10, 0, 1), 10.0, rtol=1e-6)                       # 10x everywhere
    dom = O.dominance_stats(R10)
    assert dom.tolist() == [64, 0, 0]                                                   # fraction 1.0
    half = np.stack([np.where(np.arange(64) < 32, 2.0, 1.0), np.where(np.arange(64) < 32, 1.0, 2.0)])
    assert O.dominance_stats(half.astype(np.float32)).tolist() == [32, 32, 0]           # 0.5 / 0.5
    tie = np.ones((2, 8), np.float32)
    assert O.dominance_stats(tie).tolist() == [8, 0, 8]                                 # ties: first + tied
    d = O.dominance_stats(R)
    assert d[:3].sum() == 64 and all(d[m] == int(np.sum(np.argmax(R, axis=0) == m)) for m in range(3))
    zero = np.zeros((2, 4), np.float32)
    assert np.all(O.range_ratio(zero, 0, 1) == 0.0)                                     # floored denominator


def test_meanabs_and_awq_grid():
    """Mean-abs statistic against a brute-force loop; the AWQ grid's beta = 0 point is s = 1
    (no smoothing) and its loss equals calib_loss with unit factors."""
    c = synth.config_inputs("c1")
    S, cnt = O.meanabs_stats(c["X"], c["ids"], 2)
    Xf = O.decode(c["X"]).astype(np.float64)
    for m in range(2):
        acc = np.zeros(Xf.shape[1])
        for t in range(Xf.shape[0]):
            if c["ids"][t] == m:
                acc += np.abs(Xf[t])
        assert np.allclose(S[m], acc, rtol=1e-12) and cnt[m] == int((c["ids"] == m).sum())
    betas = [0.0, 0.25, 0.5]
    b, losses = O.awq_grid_search(c["X"], c["ids"], c["W"], 4, 8, betas, 2)
    l1 = O.calib_loss(c["X"], c["ids"], np.ones((2, Xf.shape[1]), np.float32), c["W"], 4, 8)[2]
    assert losses[0] == l1 and b == betas[int(np.argmin(losses))]


# ----------------------------------------------------------------------------- N2 CMC factors
def _aniso(g, T, d, cond=1e3):
    """Activations with an anisotropic covariance (condition number ~cond^2)."""
    Q, _ = np.linalg.qr(g.normal(size=(d, d)))
    return g.normal(size=(T, d)) @ (np.logspace(0, np.log10(cond), d)[:, None] * Q.T)


def test_weight_residual_spec_examples():
    """s_m == s_t with a lossless Q -> 0; s_m = 2 s_t -> diag(s_t) W; a random
    case equals direct recomputation."""
    g = np.random.Generator(np.random.PCG64(31))
    d, n = 16, 32
    codes = g.integers(-7, 8, (d, n))
    codes[0] = 7                                               # every column's max |code| = 7
    W = synth.f32_to_bf16_bits((codes * np.float32(0.125)).astype(np.float32))   # exact grid values
    st = np.ones(d, np.float32)
    qw, dw = O.quantize_weight(W, st, 4)
    assert np.array_equal(O.weight_residual(W, st, qw, dw), np.zeros((d, n)))
    assert np.array_equal(O.weight_residual(W, 2 * st, qw, dw), O.decode(W).astype(np.float64))
    s = np.exp(g.normal(0, 0.5, d)).astype(np.float32)
    Wr = synth.f32_to_bf16_bits(g.normal(0, 1, (d, n)).astype(np.float32))
    qw, dw = O.quantize_weight(Wr, st * np.float32(1.5), 4)
    ref = np.array([[float(s[i]) * float(O.decode(Wr)[i, j]) - float(dw[j]) * int(qw[j, i]) for j in range(n)]
                    for i in range(d)])
    assert np.array_equal(O.weight_residual(Wr, s, qw, dw), ref)


def test_whitening_transform():
    """Gram = I -> T orthogonal; scaled orthonormal rows -> whitened Gram = I;
    random full rank (eps = 0): ||(A T^-1)^T (A T^-1) - I||_max <= 1e-8; T T^-1 = I."""
    g = np.random.Generator(np.random.PCG64(32))
    Q, _ = np.linalg.qr(g.normal(size=(40, 12)))
    T, Ti, _ = O.whitening_transform(Q, 0.0)
    assert np.abs(T.T @ T - np.eye(12)).max() <= 1e-10
    T, Ti, _ = O.whitening_transform(3.0 * Q, 0.0)
    assert np.abs((3 * Q @ Ti).T @ (3 * Q @ Ti) - np.eye(12)).max() <= 1e-8
    A = _aniso(g, 200, 24)
    T, Ti, _ = O.whitening_transform(A, 0.0)
    assert np.abs((A @ Ti).T @ (A @ Ti) - np.eye(24)).max() <= 1e-8
    assert np.abs(T @ Ti - np.eye(24)).max() <= 1e-8


def test_cmc_factors_theorem2():
    """Theorem 2: loss(L1 L2) = tail energy sum_{i>r}
    sigma_i^2 of SVD(A dW) (eps = 0); <= the naive SVD's loss and every perturbed / random rank-r
    candidate; full rank recovers dW; dW = 0 -> 0; monotone in r; and an independent whitening
    route (Cholesky factor instead of the eigendecomposition) gives the same L1 L2."""
    g = np.random.Generator(np.random.PCG64(33))
    T_, d, n, r = 300, 20, 28, 4
    A = _aniso(g, T_, d)
    dW = g.normal(size=(d, n))
    L1, L2 = O.cmc_factors(A, dW, r, 0.0)
    loss = O.reconstruction_loss(A, dW, L1, L2)
    tail = np.sum(np.linalg.svd(A @ dW, compute_uv=False)[r:] ** 2)
    assert abs(loss - tail) <= 1e-8 * tail
    n1, n2 = O.naive_svd_factors(dW, r)
    assert loss <= O.reconstruction_loss(A, dW, n1, n2)
    for k in range(200):
        e1, e2 = g.normal(size=L1.shape), g.normal(size=L2.shape)
        sc = 1e-3 if k < 100 else 1.0
        c1 = L1 + sc * e1 * np.abs(L1).max() if k < 100 else e1
        c2 = L2 + sc * e2 * np.abs(L2).max() if k < 100 else e2
        assert loss <= O.reconstruction_loss(A, dW, c1, c2)
    F1, F2 = O.cmc_factors(A, dW, d, 0.0)
    assert np.abs(F1 @ F2 - dW).max() <= 1e-8 * np.abs(dW).max()
    Z1, Z2 = O.cmc_factors(A, np.zeros((d, n)), r, 0.0)
    assert np.abs(Z1 @ Z2).max() == 0.0
    losses = [O.reconstruction_loss(A, dW, *O.cmc_factors(A, dW, k, 0.0)) for k in range(0, d + 1, 4)]
    assert all(a >= b * (1 - 1e-12) for a, b in zip(losses, losses[1:]))
    Lc = np.linalg.cholesky(A.T @ A)                   # A^T A = Lc Lc^T -> T' = Lc^T
    U, sig, Vt = np.linalg.svd(Lc.T @ dW, full_matrices=False)
    Lstar = np.linalg.solve(Lc.T, U[:, :r]) @ (sig[:r, None] * Vt[:r])
    assert np.abs(Lstar - L1 @ L2).max() <= 1e-8 * np.abs(Lstar).max()


@pytest.mark.parametrize("T_,d,n,r,eps", [(300, 40, 24, 6, 1e-8), (300, 40, 24, 6, 0.0), (60, 48, 20, 5, 1e-8),
                                           (200, 20, 28, 4, 1e-8)])
def test_cmc_small_side_equals_paper_route(T_, d, n, r, eps):
    """The n x n evaluation of eq:l1l2 (oracle.cmc_factors_small_side, used where the paper's d x d
    eigensolve is out of reach: d = 18944) gives the paper route's L1 L2 and loss — for d > n,
    d < n, a rank-deficient Gram (T < d, regularised) and eps = 0."""
    g = np.random.Generator(np.random.PCG64(91 + T_ + d))
    A = _aniso(g, T_, d)
    dW = g.normal(size=(d, n))
    L1, L2 = O.cmc_factors(A, dW, r, eps)
    S1, S2 = O.cmc_factors_small_side(A, dW, r, eps)
    base = np.linalg.norm(A @ dW)
    assert np.linalg.norm(A @ (L1 @ L2 - S1 @ S2)) <= 1e-9 * base
    assert abs(O.reconstruction_loss(A, dW, L1, L2) - O.reconstruction_loss(A, dW, S1, S2)) <= 1e-10 * base ** 2
    assert np.allclose(np.abs(L2), np.abs(S2), rtol=1e-6, atol=1e-9 * np.abs(L2).max())   # Sigma_r V_r^T up to sign


def test_cmc_isotropic_and_effective_rank():
    """isotropic activations -> whitened and naive losses agree; fig:effective_rank
    (SPEC.md:418): on anisotropic activations T dW has a lower effective rank than dW in >= 9 of
    10 seeded trials (dW = a residual with correlated structure)."""
    g = np.random.Generator(np.random.PCG64(34))
    Q, _ = np.linalg.qr(g.normal(size=(64, 16)))
    A = 2.0 * Q
    dW = g.normal(size=(16, 20))
    a = O.reconstruction_loss(A, dW, *O.cmc_factors(A, dW, 3, 0.0))
    b = O.reconstruction_loss(A, dW, *O.naive_svd_factors(dW, 3))
    assert abs(a - b) <= 1e-6 * b
    wins = 0
    for t in range(10):
        gg = np.random.Generator(np.random.PCG64(100 + t))
        A = _aniso(gg, 200, 24, cond=1e2)
        dW = gg.normal(size=(24, 32))
        T, _, _ = O.whitening_transform(A, 0.0)
        wins += O.effective_rank(T @ dW) <= O.effective_rank(dW)
    assert wins >= 9


# ----------------------------------------------------------------------------- N3 int4 groups
def test_grouped_weight_quantizer_pins():
    """group = d reduces to the per-output-channel O3 quantizer bit for bit; every code is the
    nearest grid point of its group's scale (ties away); pack/unpack round trip with the
    documented nibble order."""
    c = synth.config_inputs("c1")
    R, cnt = O.calibrate_stats(c["X"], c["ids"], 2)
    s = O.init_factors(R, cnt, c["W"])
    d = c["d"]
    q1, d1 = O.quantize_weight_grouped(c["W"], s[0], 4, d)
    q0, d0 = O.quantize_weight(c["W"], s[0], 4)
    assert np.array_equal(q1, q0) and np.array_equal(d1[:, 0], d0)
    q, dl = O.quantize_weight_grouped(c["W"], s[0], 4, 16)
    ws = np.multiply(s[0][:, None], O.decode(c["W"]), dtype=np.float32).T.astype(np.float64)
    grid = np.arange(-8, 8, dtype=np.float64)
    scale = np.repeat(dl.astype(np.float64), 16, axis=1)
    v = ws / scale
    best = grid[np.argmin(np.abs(v[..., None] - grid) - 1e-9 * np.abs(grid), axis=-1)]   # ties -> away
    assert np.array_equal(q.astype(np.float64), best)
    packed = O.pack_int4(q)
    assert packed.shape == (q.shape[0], d // 2)
    assert np.array_equal(O.unpack_int4(packed), q)
    assert O.pack_int4(np.array([[1, -1, -8, 7]], np.int8)).tolist() == [[0xF1, 0x78]]


def test_linear_decode_brute_force():
    """Y = Q(X S^-1) Q_g(S W) against a per-element loop over groups with integer partial sums
    (the decode kernel's arithmetic order) on a tiny case."""
    c = synth.config_inputs("c1")
    R, cnt = O.calibrate_stats(c["X"], c["ids"], 2)
    s = O.init_factors(R, cnt, c["W"])
    c = dict(c, X=c["X"][:8])
    g = 16
    q, dl = O.quantize_weight_grouped(c["W"], s[0], 4, g)
    Y = O.linear_decode(c["X"], s[0], q, dl, 8, g)
    inv = np.divide(np.float32(1), s[0], dtype=np.float32)
    qa, da = O.quantize_rows(np.multiply(O.decode(c["X"]), inv, dtype=np.float32), 8)
    T, d = qa.shape
    n = q.shape[0]
    ref = np.zeros((T, n))
    for t in range(T):
        for j in range(n):
            acc = 0.0
            for gg in range(d // g):
                sl = slice(gg * g, (gg + 1) * g)
                acc += float(dl[j, gg]) * int(np.dot(qa[t, sl].astype(np.int64), q[j, sl].astype(np.int64)))
            ref[t, j] = float(da[t]) * acc
    assert np.allclose(Y, ref, rtol=1e-12, atol=1e-12 * np.abs(ref).max())


def test_linear_forward_grouped_pins():
    """N3 prefill oracle: (1) group = d reduces to O3/O6 — the grouped codes / scales equal
    quantize_weight's bit for bit and the output equals linear_forward's (with CMC) to f64 rounding;
    (2) all-text tokens without CMC equal linear_decode; (3) a per-element loop over groups with
    integer partial sums on a tiny 3-modality case (CMC included as its own term)."""
    c = synth.config_inputs("c2", T=1024, d=256, n=96, r=16)
    R, cnt = O.calibrate_stats(c["X"], c["ids"], 3)
    s = O.init_factors(R, cnt, c["W"])
    qd, dd = O.quantize_weight_grouped(c["W"], s[0], 4, 256)
    qw, dw = O.quantize_weight(c["W"], s[0], 4)
    assert np.array_equal(qd, qw) and np.array_equal(dd[:, 0], dw)
    L1, L2 = list(c["L1"]), list(c["L2"])
    Yg = O.linear_forward_grouped(c["X"], c["ids"], s, qd, dd, 8, 256, L1, L2)
    Yf = O.linear_forward(c["X"], c["ids"], s, qw, dw, 8, L1, L2)
    assert np.allclose(Yg, Yf, rtol=1e-12, atol=1e-12 * np.abs(Yf).max())
    q, dl = O.quantize_weight_grouped(c["W"], s[0], 4, 128)
    ids0 = np.zeros_like(c["ids"])
    Yt = O.linear_forward_grouped(c["X"][:5], ids0[:5], s, q, dl, 8, 128)
    Yd = O.linear_decode(c["X"][:5], s[0], q, dl, 8, 128)
    assert np.array_equal(Yt, Yd)
    rows = np.array([0, 70, 600, 1000])                     # text, image, audio, text
    Yr = O.linear_forward_grouped(c["X"], c["ids"], s, q, dl, 8, 128, L1, L2, rows=rows)
    xs = O.smooth_activations(O.decode(c["X"])[rows], c["ids"][rows], s)
    qa, da = O.quantize_rows(xs, 8)
    for a, t in enumerate(rows):
        m = int(c["ids"][t])
        for j in range(0, 96, 7):
            acc = 0.0
            for gg in range(2):
                sl = slice(gg * 128, (gg + 1) * 128)
                acc += float(dl[j, gg]) * int(np.dot(qa[a, sl].astype(np.int64), q[j, sl].astype(np.int64)))
            ref = float(da[a]) * acc
            if m:
                l1 = O.decode(c["L1"][m - 1]).astype(np.float64)
                l2 = O.decode(c["L2"][m - 1]).astype(np.float64)
                ref += float(xs[a].astype(np.float64) @ l1 @ l2[:, j])
            assert abs(Yr[a, j] - ref) <= 1e-12 * max(abs(ref), 1.0)


def test_cmc_from_gram_equals_from_activations():
    """The Gram route (what token-sharded runs use after a SUM of the shards' Grams) gives the
    same factors and the same Theorem-2 loss; the shards' Grams add up to the batch Gram."""
    g = np.random.Generator(np.random.PCG64(35))
    A = _aniso(g, 240, 20)
    dW = g.normal(size=(20, 30))
    L1, L2 = O.cmc_factors(A, dW, 5)
    G = A[:100].T @ A[:100] + A[100:].T @ A[100:]
    M1, M2 = O.cmc_factors_from_gram(G, dW, 5)
    assert np.abs(M1 @ M2 - L1 @ L2).max() <= 1e-9 * np.abs(L1 @ L2).max()
    l_a = O.reconstruction_loss(A, dW, L1, L2)
    assert abs(O.reconstruction_loss_from_gram(G, dW, L1, L2) - l_a) <= 1e-9 * l_a
