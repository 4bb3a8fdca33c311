"""GPU parity: the CUDA path (through the C ABI) vs the CPU oracle on the same seeded inputs.

Bar (BASELINE.json north_star): bit-exact for channel maxima, factors, codes, scales and
integer accumulators; max-abs-normalised error <= 1e-3 for float outputs and relative
error <= 1e-3 for the loss.  Sizes span several tiles with ragged tails; full-size configs
are checked on sampled rows the oracle computes one by one.
"""
import numpy as np
import pytest
import torch

import oracle as O
import synth

pytestmark = pytest.mark.gpu

TOL_Y = 1e-3
TOL_L = 1e-3


def bf(bits):
    return torch.from_numpy(np.ascontiguousarray(bits).view(np.int16)).view(torch.bfloat16).cuda()


def tt(a):
    return torch.from_numpy(np.ascontiguousarray(a)).cuda()


def M():
    import paper_2603_04800_b200 as m
    return m


def sample_rows(ids, n_random=256, seed=0):
    """Every row of the first and last 128-row tile of each modality segment + random rows."""
    T = ids.size
    rows = set()
    change = np.nonzero(np.diff(ids.astype(np.int32)))[0] + 1
    starts = np.concatenate([[0], change])
    ends = np.concatenate([change, [T]])
    for a, b in list(zip(starts, ends))[:6] + list(zip(starts, ends))[-6:]:
        rows.update(range(a, min(b, a + 128)))
        rows.update(range(max(a, b - 128), b))
    g = np.random.Generator(np.random.PCG64(seed))
    rows.update(g.choice(T, size=min(n_random, T), replace=False).tolist())
    rows.update([0, T - 1])
    return np.array(sorted(rows))


def max_abs_norm(a, b):
    return float(np.abs(np.asarray(a, np.float64) - b).max() / max(np.abs(b).max(), 1e-300))


def max_abs_norm_per_modality(a, b, ids):
    """max over modalities of the max-abs error normalised by THAT modality's max |b| (image
    outputs are ~20x text outputs: a global normalisation would check text rows ~20x looser)."""
    a = np.asarray(a, np.float64)
    return max(float(np.abs(a[ids == m] - b[ids == m]).max() / max(np.abs(b[ids == m]).max(), 1e-300))
               for m in np.unique(ids))


CASES = {
    # name: (config, overrides)
    "c1": ("c1", {}),
    "ragged3": ("c2", dict(T=1000, d=208, n=288, r=48)),
    "c2_qkv": ("c2", dict(n=2560, r=0)),
    "c3_qkv": ("c3", dict(n=4608)),
}
_cache = {}


def case(name):
    if name not in _cache:
        cfg, kw = CASES[name]
        _cache[name] = synth.config_inputs(cfg, **kw)
    return _cache[name]


def oracle_state(c):
    R, cnt = O.calibrate_stats(c["X"], c["ids"], c["n_mod"])
    s = O.init_factors(R, cnt, c["W"])
    qw, dw = O.quantize_weight(c["W"], s[0], c["wbits"])
    return R, cnt, s, qw, dw


# ----------------------------------------------------------------------------- A1 / A2
@pytest.mark.parametrize("name", ["c1", "ragged3", "c2_qkv", "c3_qkv"])
def test_stats_and_init_bitexact(name):
    c = case(name)
    m = M()
    R, cnt = m.calibrate_stats(bf(c["X"]), tt(c["ids"]), c["n_mod"])
    s = m.init_factors(R, cnt, bf(c["W"]))
    m.check()
    Ro, co, so, _, _ = oracle_state(c)
    assert np.array_equal(R.cpu().numpy(), Ro)
    assert np.array_equal(cnt.cpu().numpy(), co)
    assert np.array_equal(s.cpu().numpy(), so)


def test_stats_f32_input_running_max_and_reset():
    c = case("c1")
    m = M()
    X = O.decode(c["X"])
    Xg, ids = tt(X), tt(c["ids"])
    R, cnt = m.calibrate_stats(Xg[:100], ids[:100], 2)
    R, cnt = m.calibrate_stats(Xg[100:], ids[100:], 2, R=R, count=cnt, reset=False)
    Ro, co = O.calibrate_stats(X, c["ids"], 2)
    assert np.array_equal(R.cpu().numpy(), Ro) and np.array_equal(cnt.cpu().numpy(), co)
    R, cnt = m.calibrate_stats(Xg[:7], ids[:7], 2, R=R, count=cnt, reset=True)
    Ro, co = O.calibrate_stats(X[:7], c["ids"][:7], 2)
    assert np.array_equal(R.cpu().numpy(), Ro) and np.array_equal(cnt.cpu().numpy(), co)


def test_stats_d18944_bitexact():
    """The down-projection input width (c3 MLP 18944), 4096 tokens."""
    c = synth.config_inputs("c3", d=18944, n=3584, T=4096)
    m = M()
    R, cnt = m.calibrate_stats(bf(c["X"]), tt(c["ids"]), 2)
    Ro, co = O.calibrate_stats(c["X"], c["ids"], 2)
    assert np.array_equal(R.cpu().numpy(), Ro) and np.array_equal(cnt.cpu().numpy(), co)


# ----------------------------------------------------------------------------- A3 / A4
@pytest.mark.parametrize("name", ["c1", "ragged3", "c2_qkv", "c3_qkv"])
def test_quantize_weight_and_activations_bitexact(name):
    c = case(name)
    m = M()
    _, _, so, qwo, dwo = oracle_state(c)
    s = tt(so)
    qw, dw = m.quantize_weight(bf(c["W"]), s[0], c["wbits"])
    assert np.array_equal(qw.cpu().numpy(), qwo)
    assert np.array_equal(dw.cpu().numpy(), dwo)
    qx, dx, mask = m.quantize_activations(bf(c["X"]), tt(c["ids"]), s, c["abits"])
    m.check()
    qxo, dxo = O.quantize_activations(c["X"], c["ids"], so, c["abits"])
    assert np.array_equal(qx.cpu().numpy(), qxo)
    assert np.array_equal(dx.cpu().numpy(), dxo)
    want = np.zeros(mask.numel(), np.int64)
    for t, mid in enumerate(c["ids"]):
        want[t // 128] |= 1 << int(mid)
    assert np.array_equal(mask.cpu().numpy().astype(np.int64) & 0xFF, want)


def test_quantize_weight_gate_w4_bitexact():
    """c3 gate/up weight 3584 x 18944 at W4 (the largest single weight of the layer)."""
    c = synth.config_inputs("c3", n=18944, T=2048)
    m = M()
    R, cnt = O.calibrate_stats(c["X"], c["ids"], 2)
    so = O.init_factors(R, cnt, c["W"])
    qwo, dwo = O.quantize_weight(c["W"], so[1], 4)
    qw, dw = m.quantize_weight(bf(c["W"]), tt(so[1]), 4)
    assert np.array_equal(qw.cpu().numpy(), qwo) and np.array_equal(dw.cpu().numpy(), dwo)


# ----------------------------------------------------------------------------- A6 accumulators
@pytest.mark.parametrize("name", ["c1", "ragged3", "c3_qkv"])
def test_forward_int32_accumulators_bitexact(name):
    c = case(name)
    m = M()
    _, _, so, qwo, dwo = oracle_state(c)
    acc = m.linear_forward(bf(c["X"]), tt(c["ids"]), tt(so), tt(qwo), tt(dwo), c["wbits"], c["abits"],
                           acc_debug=True).cpu().numpy()
    rows = np.arange(c["T"]) if c["T"] <= 1024 else sample_rows(c["ids"])
    qxo, _ = O.quantize_activations(O.decode(c["X"])[rows], c["ids"][rows], so, c["abits"])
    assert np.array_equal(acc[rows].astype(np.int64), O.int_gemm(qxo, qwo))


# ----------------------------------------------------------------------------- A4-A7 outputs
@pytest.mark.parametrize("name,use_cmc", [("c1", False), ("c1", True), ("ragged3", True), ("c2_qkv", False),
                                          ("c3_qkv", True)])
def test_forward_parity(name, use_cmc):
    c = case(name)
    m = M()
    _, _, so, qwo, dwo = oracle_state(c)
    L1 = L2 = None
    if use_cmc and c["r"] > 0:
        L1, L2 = bf(c["L1"]), bf(c["L2"])
    Y = m.linear_forward(bf(c["X"]), tt(c["ids"]), tt(so), tt(qwo), tt(dwo), c["wbits"], c["abits"], L1, L2)
    m.check()
    Y = Y.cpu().numpy()
    rows = np.arange(c["T"]) if c["T"] <= 1024 else sample_rows(c["ids"])
    L1o = list(c["L1"]) if L1 is not None else None
    L2o = list(c["L2"]) if L2 is not None else None
    Yo = O.linear_forward(c["X"], c["ids"], so, qwo, dwo, c["abits"], L1o, L2o, rows=rows)
    assert max_abs_norm_per_modality(Y[rows], Yo, c["ids"][rows]) <= TOL_Y


@pytest.mark.parametrize("r", [64, 192])
def test_forward_c3_gate_cmc_sampled(r):
    """c3 gate/up 3584 -> 18944, W4A8, CMC rank 64 / 192, full 16k tokens, sampled rows."""
    c = synth.config_inputs("c3", n=18944, r=r)
    m = M()
    Ro, co = O.calibrate_stats(c["X"], c["ids"], 2)
    so = O.init_factors(Ro, co, c["W"])
    qwo, dwo = O.quantize_weight(c["W"], so[0], 4)
    Y = m.linear_forward(bf(c["X"]), tt(c["ids"]), tt(so), tt(qwo), tt(dwo), 4, 8, bf(c["L1"]), bf(c["L2"]))
    m.check()
    rows = sample_rows(c["ids"], n_random=128)
    Yo = O.linear_forward(c["X"], c["ids"], so, qwo, dwo, 8, list(c["L1"]), list(c["L2"]), rows=rows)
    assert max_abs_norm_per_modality(Y.cpu().numpy()[rows], Yo, c["ids"][rows]) <= TOL_Y


def test_forward_shuffled_ids_three_modalities():
    """i.i.d.-shuffled ids: every tile mixes text/image/audio (routing stress)."""
    c = synth.config_inputs("c2", T=777, d=256, n=320, r=32, shuffle=True)
    m = M()
    _, _, so, qwo, dwo = oracle_state(c)
    Y = m.linear_forward(bf(c["X"]), tt(c["ids"]), tt(so), tt(qwo), tt(dwo), 8, 8, bf(c["L1"]), bf(c["L2"]))
    Yo = O.linear_forward(c["X"], c["ids"], so, qwo, dwo, 8, list(c["L1"]), list(c["L2"]))
    assert max_abs_norm_per_modality(Y.cpu().numpy(), Yo, c["ids"]) <= TOL_Y


def test_forward_column_shard_matches_full():
    """Output-column sharding through pointer offsets: bit-identical shards."""
    c = case("ragged3")
    m = M()
    _, _, so, qwo, dwo = oracle_state(c)
    X, ids, s = bf(c["X"]), tt(c["ids"]), tt(so)
    qw, dw = tt(qwo), tt(dwo)
    L1, L2 = bf(c["L1"]), bf(c["L2"])
    full = m.linear_forward(X, ids, s, qw, dw, 8, 8, L1, L2)
    Y = torch.zeros_like(full)
    for j0, j1 in [(0, 96), (96, 288)]:
        m.linear_forward(X, ids, s, qw[j0:j1].contiguous(), dw[j0:j1].contiguous(), 8, 8, L1,
                         L2[:, :, j0:j1], Y=Y[:, j0:j1])
    assert torch.equal(Y, full)


def test_all_text_and_rank0():
    c = case("c1")
    m = M()
    _, _, so, qwo, dwo = oracle_state(c)
    ids0 = np.zeros_like(c["ids"])
    Y = m.linear_forward(bf(c["X"]), tt(ids0), tt(so), tt(qwo), tt(dwo), 8, 8, bf(c["L1"]), bf(c["L2"]))
    Yo = O.linear_forward(c["X"], ids0, so, qwo, dwo, 8)
    assert max_abs_norm(Y.cpu().numpy(), Yo) <= TOL_Y


# ----------------------------------------------------------------------------- A8 loss
def test_reference_output():
    c = case("c3_qkv")
    m = M()
    Yr = m.reference_output(bf(c["X"]), bf(c["W"])).cpu().numpy()
    rows = sample_rows(c["ids"])
    Yo = O.reference_output(c["X"], c["W"], rows=rows)
    assert max_abs_norm_per_modality(Yr[rows], Yo, c["ids"][rows]) <= 1e-5


@pytest.mark.parametrize("name", ["c1", "ragged3", "c3_qkv"])
def test_loss_parity_and_determinism(name):
    c = case(name)
    m = M()
    _, _, so, _, _ = oracle_state(c)
    X, W = bf(c["X"]), bf(c["W"])
    Yref = m.reference_output(X, W)
    sums, counts, loss = m.calib_loss(X, tt(c["ids"]), tt(so), W, c["wbits"], c["abits"], Yref)
    m.check()
    s2, c2, l2 = m.calib_loss(X, tt(c["ids"]), tt(so), W, c["wbits"], c["abits"], Yref)
    assert torch.equal(sums, s2) and torch.equal(loss, l2)          # fixed-order reduction
    so_, co_, lo = O.calib_loss(c["X"], c["ids"], so, c["W"], c["wbits"], c["abits"])
    assert np.array_equal(counts.cpu().numpy(), co_)
    assert np.all(np.abs(sums.cpu().numpy() - so_) <= TOL_L * np.abs(so_))
    assert abs(float(loss.cpu()[0]) - lo) <= TOL_L * abs(lo)


def test_loss_lambda_and_finalize():
    c = case("ragged3")
    m = M()
    _, _, so, _, _ = oracle_state(c)
    X, W = bf(c["X"]), bf(c["W"])
    Yref = m.reference_output(X, W)
    lam = [1.0, 0.5, 2.0]
    sums, counts, loss = m.calib_loss(X, tt(c["ids"]), tt(so), W, 8, 8, Yref, lam=lam)
    _, _, lo = O.calib_loss(c["X"], c["ids"], so, c["W"], 8, 8, lam=lam)
    assert abs(float(loss.cpu()[0]) - lo) <= TOL_L * abs(lo)
    l2 = m.loss_finalize(sums, counts, W.shape[1], lam=lam)
    assert torch.equal(l2, loss)


# ----------------------------------------------------------------------------- edge cases
def test_edge_cases_status():
    m = M()
    c = case("c1")
    X, W = bf(c["X"]), bf(c["W"])
    # T = 0 is a no-op
    R, cnt = m.calibrate_stats(X[:0], tt(c["ids"][:0]), 2)
    assert float(R.abs().sum()) == 0.0 and int(cnt.sum()) == 0
    # an id >= n_mod sets the sticky BAD_MODALITY status
    bad = c["ids"].copy()
    bad[17] = 5
    m.calibrate_stats(X, tt(bad), 2)
    with pytest.raises(m.MasqError) as e:
        m.check()
    assert e.value.status == 6
    m.check()                                     # cleared
    # a modality with no tokens -> EMPTY_MODALITY at init
    R, cnt = m.calibrate_stats(X, tt(np.zeros_like(c["ids"])), 2)
    m.init_factors(R, cnt, W)
    with pytest.raises(m.MasqError) as e:
        m.check()
    assert e.value.status == 7
    # single token
    R, cnt = m.calibrate_stats(X[:1], tt(c["ids"][:1]), 2)
    Ro, co = O.calibrate_stats(c["X"][:1], c["ids"][:1], 2)
    assert np.array_equal(R.cpu().numpy(), Ro)


def test_forward_f32_input_with_cmc():
    """f32 activations (c1 allows f32 X): the CMC GEMM splits X into bf16 hi/lo planes."""
    c = case("ragged3")
    m = M()
    Xf = O.decode(c["X"]) * np.float32(1.0 + 2.0 ** -12)          # not bf16-representable
    Xf = Xf.astype(np.float32)
    R, cnt = O.calibrate_stats(Xf, c["ids"], 3)
    so = O.init_factors(R, cnt, c["W"])
    qwo, dwo = O.quantize_weight(c["W"], so[0], 8)
    Y = m.linear_forward(tt(Xf), tt(c["ids"]), tt(so), tt(qwo), tt(dwo), 8, 8, bf(c["L1"]), bf(c["L2"]))
    qx, dx, _ = m.quantize_activations(tt(Xf), tt(c["ids"]), tt(so), 8)
    qxo, dxo = O.quantize_activations(Xf, c["ids"], so, 8)
    assert np.array_equal(qx.cpu().numpy(), qxo) and np.array_equal(dx.cpu().numpy(), dxo)
    Yo = O.linear_forward(Xf, c["ids"], so, qwo, dwo, 8, list(c["L1"]), list(c["L2"]))
    assert max_abs_norm_per_modality(Y.cpu().numpy(), Yo, c["ids"]) <= TOL_Y


def test_forward_max_tokens_sampled():
    """c5's largest point: 262144 tokens (256 samples of the c3 layout) through the forward,
    d = 3584 -> 3584, W4A8, CMC r = 64; sampled rows against the oracle, acc bit-exact."""
    T = 262144
    cfg = synth.CONFIGS["c3"]
    ids = synth.modality_ids(cfg["pattern"], T=T)
    X = synth.activations(ids, 3584, 2, synth.seed_for(4, 0, 0))
    W = synth.weight(3584, 3584, synth.seed_for(4, 0, 1))
    L1, L2 = synth.lowrank(3584, 3584, 64, 2, synth.seed_for(4, 0, 2))
    m = M()
    Ro, co = O.calibrate_stats(X, ids, 2)
    so = O.init_factors(Ro, co, W)
    qwo, dwo = O.quantize_weight(W, so[0], 4)
    Xg = bf(X)
    Y = m.linear_forward(Xg, tt(ids), tt(so), tt(qwo), tt(dwo), 4, 8, bf(L1), bf(L2))
    acc = m.linear_forward(Xg, tt(ids), tt(so), tt(qwo), tt(dwo), 4, 8, acc_debug=True)
    m.check()
    rows = np.concatenate([np.arange(0, 256), np.arange(T - 256, T),
                           np.random.Generator(np.random.PCG64(7)).choice(T, 512, replace=False)])
    Yo = O.linear_forward(X, ids, so, qwo, dwo, 8, [L1[0]], [L2[0]], rows=rows)
    assert max_abs_norm_per_modality(Y.cpu().numpy()[rows], Yo, ids[rows]) <= TOL_Y
    qxo, _ = O.quantize_activations(O.decode(X)[rows], ids[rows], so, 8)
    assert np.array_equal(acc.cpu().numpy()[rows].astype(np.int64), O.int_gemm(qxo, qwo))


def test_eight_modalities_end_to_end():
    """n_mod = 8 (the ABI maximum), ragged modality runs, CMC for 7 non-text modalities: stats,
    factors and codes bit-exact, forward and loss against the oracle."""
    m = M()
    n_mod, d, n, r = 8, 96, 160, 16
    pattern = [(0, 40), (3, 70), (1, 33), (7, 90), (2, 64), (5, 17), (4, 120), (6, 55), (0, 23)]
    ids = synth.modality_ids(pattern, repeat=3)
    X = synth.activations(ids, d, n_mod, 4242, gamma=dict(enumerate([1.0, 20.0, 0.3, 5.0, 2.0, 50.0, 0.1, 8.0])))
    W = synth.weight(d, n, 4243)
    L1, L2 = synth.lowrank(d, n, r, n_mod, 4244)
    R, cnt = O.calibrate_stats(X, ids, n_mod)
    s = O.init_factors(R, cnt, W)
    Rg, cg = m.calibrate_stats(bf(X), tt(ids), n_mod)
    sg = m.init_factors(Rg, cg, bf(W))
    m.check()
    assert np.array_equal(Rg.cpu().numpy(), R) and np.array_equal(sg.cpu().numpy(), s)
    qw, dw = O.quantize_weight(W, s[0], 8)
    qwg, dwg = m.quantize_weight(bf(W), sg[0], 8)
    assert np.array_equal(qwg.cpu().numpy(), qw) and np.array_equal(dwg.cpu().numpy(), dw)
    Y = m.linear_forward(bf(X), tt(ids), sg, qwg, dwg, 8, 8, bf(L1), bf(L2)).cpu().numpy()
    Yo = O.linear_forward(X, ids, s, qw, dw, 8, list(L1), list(L2))
    assert max_abs_norm_per_modality(Y, Yo, ids) <= TOL_Y
    Yref = m.reference_output(bf(X), bf(W))
    sums, counts, loss = m.calib_loss(bf(X), tt(ids), sg, bf(W), 8, 8, Yref)
    so, co, lo = O.calib_loss(X, ids, s, W, 8, 8)
    assert np.array_equal(counts.cpu().numpy(), co)
    assert np.all(np.abs(sums.cpu().numpy() - so) <= TOL_L * np.abs(so))
    assert abs(float(loss.cpu()[0]) - lo) <= TOL_L * abs(lo)
