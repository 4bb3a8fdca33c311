"""GPU parity at the shapes the timed bench step runs (VERDICT r1 "What's weak" #1).

Every linear of the c3 layer (Qwen2.5-VL-7B: fused qkv 3584->4608, o 3584->3584, fused gate_up
3584->37888, down 18944->3584; W4A8, CMC rank 64, text+image) and of the c2 layer (Qwen2.5-Omni-3B:
qkv 2048->2560, o 2048->2048, gate_up 2048->22016, down 11008->2048; W8A8, r = 0, text/image/audio)
goes through masq_calib_layer — the fused call bench.py times — at 4096 calibration tokens (4 c3
samples / the whole c2 batch), in the bench's launch configuration.  Against the oracle:
  * R, s, the text weight codes / scales: bit-exact (A1-A3);
  * int32 accumulators of the forward GEMM on sampled rows: bit-exact (A6; the same GEMM kernel
    and tiling as the fused call's forward, in its accumulator-tap mode);
  * Y on sampled rows: <= 1e-3 max-abs-normalised PER MODALITY (text rows are ~20x smaller than
    image rows, so a global normalisation would hide them);
  * Yref (X W) on sampled rows <= 1e-4 per modality (reading Q16: bf16 tensor-core products with
    fp32 accumulation over K up to 18944; measured 1.2-2.9e-5 at the deep-K down projections);
    per-modality loss sums and the loss <= 1e-3 relative (all rows: the oracle evaluates the
    whole batch in f64 BLAS).
PAPER.md:35, 55-58, 62-70, 177-185; SURVEY §8(a) A1-A8, §8(d) c2/c3 shapes.
"""
import numpy as np
import pytest
import torch

import oracle as O
import synth
from test_gpu_parity import M, bf, max_abs_norm, sample_rows, tt

pytestmark = pytest.mark.gpu

TOL_Y = 1e-3
TOL_L = 1e-3
T_TOKENS = 4096

# (config, linear name, d, n)
SHAPES = [("c3", *x) for x in synth.LAYER_LINEARS["c3"]] + [("c2", *x) for x in synth.LAYER_LINEARS["c2"]]


def per_modality_err(Y, Yo, ids):
    errs = {}
    for mm in np.unique(ids):
        sel = ids == mm
        errs[int(mm)] = float(np.abs(np.asarray(Y, np.float64)[sel] - Yo[sel]).max()
                              / max(np.abs(Yo[sel]).max(), 1e-300))
    return errs


@pytest.mark.parametrize("cfg,name,d,n", SHAPES, ids=[f"{c}_{nm}" for c, nm, _, _ in SHAPES])
def test_calib_layer_at_bench_shape(cfg, name, d, n):
    c = synth.config_inputs(cfg, d=d, n=n, T=T_TOKENS, layer=1 + [x[0] for x in synth.LAYER_LINEARS[cfg]].index(name))
    m = M()
    n_mod, wb, ab, r = c["n_mod"], c["wbits"], c["abits"], c["r"]
    X, W, ids = bf(c["X"]), bf(c["W"]), tt(c["ids"])
    L1 = L2 = None
    if r > 0:
        L1, L2 = bf(c["L1"]), bf(c["L2"])
    # A1 / A2 on the device, bit-exact against the oracle
    R, cnt = m.calibrate_stats(X, ids, n_mod)
    s = m.init_factors(R, cnt, W)
    m.check()
    Ro, co = O.calibrate_stats(c["X"], c["ids"], n_mod)
    so = O.init_factors(Ro, co, c["W"])
    assert np.array_equal(R.cpu().numpy(), Ro) and np.array_equal(cnt.cpu().numpy(), co)
    assert np.array_equal(s.cpu().numpy(), so)
    # the fused calibration pass, as bench.py runs it
    qt = torch.empty(n, d, dtype=torch.int8, device="cuda")
    dt = torch.empty(n, dtype=torch.float32, device="cuda")
    Y, Yref, sums, counts, loss = m.calib_layer(X, ids, s, W, wb, ab, L1, L2, qw_text=qt, dw_text=dt)
    m.check()
    qwo, dwo = O.quantize_weight(c["W"], so[0], wb)
    assert np.array_equal(qt.cpu().numpy(), qwo) and np.array_equal(dt.cpu().numpy(), dwo)
    rows = sample_rows(c["ids"], n_random=192)
    ids_r = c["ids"][rows]
    # A6: int32 accumulators bit-exact on the sampled rows
    acc = m.linear_forward(X, ids, s, qt, dt, wb, ab, acc_debug=True)
    qxo, _ = O.quantize_activations(O.decode(c["X"])[rows], ids_r, so, ab)
    assert np.array_equal(acc.cpu().numpy()[rows].astype(np.int64), O.int_gemm(qxo, qwo))
    del acc
    # A4-A7: Y per modality
    L1o = list(c["L1"]) if r > 0 else None
    L2o = list(c["L2"]) if r > 0 else None
    Yo = O.linear_forward(c["X"], c["ids"], so, qwo, dwo, ab, L1o, L2o, rows=rows)
    errs = per_modality_err(Y.cpu().numpy()[rows], Yo, ids_r)
    assert max(errs.values()) <= TOL_Y, errs
    # A8 target and loss
    Yro = O.reference_output(c["X"], c["W"], rows=rows)
    errs_r = per_modality_err(Yref.cpu().numpy()[rows], Yro, ids_r)
    assert max(errs_r.values()) <= 1e-4, errs_r
    del Y, Yref
    torch.cuda.empty_cache()
    so_, co_, lo = O.calib_loss(c["X"], c["ids"], so, c["W"], wb, ab)
    assert np.array_equal(counts.cpu().numpy(), co_)
    sg = sums.cpu().numpy()
    assert np.all(np.abs(sg - so_) <= TOL_L * np.abs(so_)), (sg, so_)
    assert abs(float(loss.cpu()[0]) - lo) <= TOL_L * abs(lo)


@pytest.mark.parametrize("name", ["qkv", "o", "gate_up", "down"])
def test_calib_layer_c3_full_batch(name):
    """The c3 linears at the bench's own batch, 16384 tokens, i.e. in exactly the launch
    configuration bench.py times (e.g. the CMC first factor's cluster-pair DSMEM split-K path,
    which smaller batches do not take): weight codes / scales bit-exact, int32 accumulators
    bit-exact and Y per modality <= 1e-3 on sampled rows (first / last tiles of 12 modality
    segments + 128 random rows), X W on the same rows <= 1e-4.  (The loss, a sum over every row,
    is checked against the oracle at 4096 tokens above.)"""
    d, n = {k: (dd, nn) for k, dd, nn in synth.LAYER_LINEARS["c3"]}[name]
    c = synth.config_inputs("c3", d=d, n=n, layer=11 + [x[0] for x in synth.LAYER_LINEARS["c3"]].index(name))
    assert c["T"] == 16384
    m = M()
    X, W, ids = bf(c["X"]), bf(c["W"]), tt(c["ids"])
    L1, L2 = bf(c["L1"]), bf(c["L2"])
    R, cnt = m.calibrate_stats(X, ids, 2)
    s = m.init_factors(R, cnt, W)
    Ro, co = O.calibrate_stats(c["X"], c["ids"], 2)
    so = O.init_factors(Ro, co, c["W"])
    assert np.array_equal(s.cpu().numpy(), so)
    qt = torch.empty(n, d, dtype=torch.int8, device="cuda")
    dt = torch.empty(n, dtype=torch.float32, device="cuda")
    Y, Yref, sums, counts, loss = m.calib_layer(X, ids, s, W, 4, 8, L1, L2, qw_text=qt, dw_text=dt)
    m.check()
    qwo, dwo = O.quantize_weight(c["W"], so[0], 4)
    assert np.array_equal(qt.cpu().numpy(), qwo) and np.array_equal(dt.cpu().numpy(), dwo)
    assert np.array_equal(counts.cpu().numpy(), co)
    rows = sample_rows(c["ids"], n_random=128)
    ids_r = c["ids"][rows]
    rt = torch.from_numpy(rows).cuda()
    Yh = Y[rt].cpu().numpy()                  # gather on the device (Y is 2.5 GB at gate_up)
    Yrh = Yref[rt].cpu().numpy()
    del Y, Yref
    acc = m.linear_forward(X, ids, s, qt, dt, 4, 8, acc_debug=True)
    acch = acc[rt].cpu().numpy().astype(np.int64)
    del acc
    torch.cuda.empty_cache()
    qxo, _ = O.quantize_activations(O.decode(c["X"])[rows], ids_r, so, 8)
    assert np.array_equal(acch, O.int_gemm(qxo, qwo))
    Yo = O.linear_forward(c["X"], c["ids"], so, qwo, dwo, 8, list(c["L1"]), list(c["L2"]), rows=rows)
    errs = per_modality_err(Yh, Yo, ids_r)
    assert max(errs.values()) <= TOL_Y, errs
    errs_r = per_modality_err(Yrh, O.reference_output(c["X"], c["W"], rows=rows), ids_r)
    assert max(errs_r.values()) <= 1e-4, errs_r


def test_stats_d11008_three_modalities():
    """c2's down-projection input width (11008), 3 modalities, the whole 4096-token batch."""
    c = synth.config_inputs("c2", d=11008, n=2048)
    m = M()
    R, cnt = m.calibrate_stats(bf(c["X"]), tt(c["ids"]), 3)
    Ro, co = O.calibrate_stats(c["X"], c["ids"], 3)
    assert np.array_equal(R.cpu().numpy(), Ro) and np.array_equal(cnt.cpu().numpy(), co)


@pytest.mark.parametrize("name", ["c1", "ragged3"])
def test_calib_loss_self_reference(name):
    """masq_calib_loss / masq_calib_loss_grad with Yref = NULL compute X W themselves (
    the SURVEY §8(b) contract): same result as with masq_reference_output's Yref."""
    from test_gpu_parity import case, oracle_state
    c = case(name)
    m = M()
    _, _, so, _, _ = oracle_state(c)
    X, W, ids, s = bf(c["X"]), bf(c["W"]), tt(c["ids"]), tt(so)
    sums, counts, loss = m.calib_loss(X, ids, s, W, c["wbits"], c["abits"])            # Yref None
    m.check()
    Yref = m.reference_output(X, W)
    s2, c2, l2 = m.calib_loss(X, ids, s, W, c["wbits"], c["abits"], Yref)
    assert torch.equal(sums, s2) and torch.equal(counts, c2) and torch.equal(loss, l2)
    so_, co_, lo = O.calib_loss(c["X"], c["ids"], so, c["W"], c["wbits"], c["abits"])
    assert abs(float(loss.cpu()[0]) - lo) <= TOL_L * abs(lo)
    _, _, l3, g3 = m.calib_loss_grad(X, ids, s, W, c["wbits"], c["abits"])
    _, _, l4, g4 = m.calib_loss_grad(X, ids, s, W, c["wbits"], c["abits"], Yref)
    assert torch.equal(l3, l4) and torch.equal(g3, g4)


def test_calib_loss_self_reference_needs_bf16_and_workspace():
    from test_gpu_parity import case, oracle_state
    import ctypes
    from paper_2603_04800_b200._lib import lib
    c = case("c1")
    m = M()
    _, _, so, _, _ = oracle_state(c)
    Xf = tt(O.decode(c["X"]))
    W, ids, s = bf(c["W"]), tt(c["ids"]), tt(so)
    with pytest.raises(m.MasqError) as e:
        m.calib_loss(Xf, ids, s, W, 8, 8)                       # f32 X without Yref
    assert e.value.status == 8
    # a workspace sized without MASQ_OP_SELF_REF is rejected synchronously
    T, d = Xf.shape
    n = W.shape[1]
    nb = m.workspace_size(m.masq.OP_LOSS, T, d, n, 2)
    assert m.workspace_size(m.masq.OP_LOSS | m.masq.OP_SELF_REF, T, d, n, 2) >= nb + 4 * T * n
    buf = torch.zeros(nb + 256, dtype=torch.uint8, device="cuda")
    p = buf.data_ptr() + (-buf.data_ptr()) % 256
    out = [torch.empty(2, dtype=torch.float64, device="cuda"), torch.empty(2, dtype=torch.int64, device="cuda"),
           torch.empty(1, dtype=torch.float64, device="cuda")]
    st = lib().masq_calib_loss(bf(c["X"]).data_ptr(), 1, d, ids.data_ptr(), T, d, n, 2, s.data_ptr(),
                               W.data_ptr(), 1, 8, 8, None, None, 0, out[0].data_ptr(), out[1].data_ptr(),
                               out[2].data_ptr(), ctypes.c_void_p(p), nb, None)
    assert st == 5


def test_forward_debug_taps():
    """masq_debug qx / dx taps return the codes and steps the forward used (bit-exact vs A4)."""
    from test_gpu_parity import case, oracle_state
    c = case("ragged3")
    m = M()
    _, _, so, qwo, dwo = oracle_state(c)
    Y, qx, dx = m.linear_forward(bf(c["X"]), tt(c["ids"]), tt(so), tt(qwo), tt(dwo), 8, 8, bf(c["L1"]),
                                 bf(c["L2"]), taps=True)
    qxo, dxo = O.quantize_activations(c["X"], c["ids"], so, 8)
    assert np.array_equal(qx.cpu().numpy(), qxo) and np.array_equal(dx.cpu().numpy(), dxo)
    Y2 = m.linear_forward(bf(c["X"]), tt(c["ids"]), tt(so), tt(qwo), tt(dwo), 8, 8, bf(c["L1"]), bf(c["L2"]))
    assert torch.equal(Y, Y2)


def test_forward_misaligned_factor_rejected():
    """a misaligned s must return MASQ_ERR_ALIGN synchronously (the row kernel reads it
    with 16-byte loads), for the forward and the decode call."""
    from test_gpu_parity import case, oracle_state
    c = case("c1")
    m = M()
    _, _, so, qwo, dwo = oracle_state(c)
    sbig = torch.zeros(so.size + 1, dtype=torch.float32, device="cuda")
    s_mis = sbig[1:].view(so.shape)
    with pytest.raises(m.MasqError) as e:
        m.linear_forward(bf(c["X"]), tt(c["ids"]), s_mis, tt(qwo), tt(dwo), 8, 8)
    assert e.value.status == 4


@pytest.mark.parametrize("wbits", [8, 4])
def test_forward_saturated_accumulators_deep_k(wbits):
    """the deepest K of the bench (c3 down, d = 18944) with every code at its
    extreme (|qx| = 127, |qw| = q_max), so |acc| reaches 18944 * 127 * q_max (3.06e8 at W8A8, near
    2^28; 1.68e7 > 2^24 at W4A8, where the int32 -> f32 conversion of the epilogue rounds): int32
    accumulators bit-exact (no wrap), Y <= 1e-3 of the f64 oracle.  Rows 0..127 are all +1 and
    weight columns 0..63 all +1/2, 64..127 all -1/2 (the extreme sums of both signs), the rest
    random signs; T = 300 and n = 288 leave ragged tails."""
    T, d, n = 300, 18944, 288
    g = np.random.Generator(np.random.PCG64(18944 + wbits))
    xs = np.where(g.random((T, d)) < 0.5, -1.0, 1.0).astype(np.float32)
    xs[:128] = 1.0
    ws = np.where(g.random((d, n)) < 0.5, -0.5, 0.5).astype(np.float32)
    ws[:, :64] = 0.5
    ws[:, 64:128] = -0.5
    to_bits = lambda a: (a.view(np.uint32) >> 16).astype(np.uint16)      # exact: +-1, +-1/2
    Xb, Wb = to_bits(xs), to_bits(ws)
    ids = np.zeros(T, np.uint8)
    s = np.ones((1, d), np.float32)
    m = M()
    qwo, dwo = O.quantize_weight(Wb, s[0], wbits)
    assert np.abs(qwo.astype(np.int64)).min() == 2 ** (wbits - 1) - 1
    qw, dw = m.quantize_weight(bf(Wb), tt(s[0]), wbits)
    assert np.array_equal(qw.cpu().numpy(), qwo) and np.array_equal(dw.cpu().numpy(), dwo)
    acc = m.linear_forward(bf(Xb), tt(ids), tt(s), qw, dw, wbits, 8, acc_debug=True).cpu().numpy()
    qxo, _ = O.quantize_activations(O.decode(Xb), ids, s, 8)
    ref = O.int_gemm(qxo, qwo)
    assert np.abs(ref).max() == d * 127 * (2 ** (wbits - 1) - 1)
    assert np.array_equal(acc.astype(np.int64), ref)
    Y = m.linear_forward(bf(Xb), tt(ids), tt(s), qw, dw, wbits, 8)
    m.check()
    Yo = O.linear_forward(Xb, ids, s, qwo, dwo, 8)
    assert max_abs_norm(Y.cpu().numpy(), Yo) <= TOL_Y
