"""GPU parity for the N3 prefill path: packed int4 weights with 128-channel group
scales in the CTA-pair tcgen05 GEMM (masq_quantize_weight_w4g + masq_linear_forward_w4g) against
oracle.quantize_weight_grouped / oracle.linear_forward_grouped (
reading Q28).

Bars: codes, scales and the packed bytes bit-exact (the byte layout rebuilt here from the oracle's
codes); the int32 sums of the group accumulators bit-exact against the oracle's integer GEMM
(every group is one kind::i8 k-block; their unscaled sum is the full K dot product); Y <= 1e-3
max-abs-normalised PER MODALITY (north_star's float bar)."""
import numpy as np
import pytest
import torch

import oracle as O
import synth
from test_gpu_parity import M, bf, sample_rows, tt

pytestmark = pytest.mark.gpu

TOL_Y = 1e-3


def pack_w4g(codes):
    """The prefill layout of include/masq.h from integer codes [n x d]: [d/128][n][64] with byte
    16c + i of (group g, channel j) = code[j][128g + 32c + i] & 0xF | (code[j][128g + 32c + 16 + i]
    & 0xF) << 4."""
    c = np.asarray(codes, np.int16) & 0xF
    n, d = c.shape
    c = c.reshape(n, d // 128, 4, 2, 16)                      # [n][group][32-code chunk][lo/hi][16]
    b = (c[:, :, :, 0, :] | (c[:, :, :, 1, :] << 4)).astype(np.uint8).reshape(n, d // 128, 64)
    return np.ascontiguousarray(b.transpose(1, 0, 2))


def per_modality_err(Y, Yo, ids):
    out = {}
    for mm in np.unique(ids):
        sel = ids == mm
        out[int(mm)] = float(np.abs(np.asarray(Y, np.float64)[sel] - Yo[sel]).max()
                             / max(np.abs(Yo[sel]).max(), 1e-300))
    return out


def _run(c, rows=None, use_cmc=True, abits=8):
    m = M()
    n_mod = c["n_mod"]
    R, cnt = O.calibrate_stats(c["X"], c["ids"], n_mod)
    s = O.init_factors(R, cnt, c["W"])
    q, dl = O.quantize_weight_grouped(c["W"], s[0], 4, 128)
    packed, scales = m.quantize_weight_w4g(bf(c["W"]), tt(s[0]))
    assert np.array_equal(scales.cpu().numpy(), dl)
    assert np.array_equal(packed.cpu().numpy(), pack_w4g(q))
    X, ids, sg = bf(c["X"]), tt(c["ids"]), tt(s)
    L1 = L2 = None
    if use_cmc and c["r"] > 0:
        L1, L2 = bf(c["L1"]), bf(c["L2"])
    Y = m.linear_forward_w4g(X, ids, sg, packed, scales, abits, L1, L2)
    acc = m.linear_forward_w4g(X, ids, sg, packed, scales, abits, acc_debug=True)
    m.check()
    rows = np.arange(c["T"]) if rows is None else rows
    qx, _ = O.quantize_activations(O.decode(c["X"])[rows], c["ids"][rows], s, abits)
    assert np.array_equal(acc.cpu().numpy()[rows].astype(np.int64), O.int_gemm(qx, q))
    L1o = list(c["L1"]) if L1 is not None else None
    L2o = list(c["L2"]) if L2 is not None else None
    Yo = O.linear_forward_grouped(c["X"], c["ids"], s, q, dl, abits, 128, L1o, L2o, rows=rows)
    errs = per_modality_err(Y.cpu().numpy()[rows], Yo, c["ids"][rows])
    assert max(errs.values()) <= TOL_Y, errs
    return errs


@pytest.mark.parametrize("kw", [dict(T=1000, d=256, n=288, r=32), dict(T=777, d=384, n=320, r=16, shuffle=True),
                                dict(T=700, d=128, n=96, r=0), dict(T=2048, d=640, n=544, r=48)])
def test_w4g_small_ragged(kw):
    """Ragged T / n tails, one to several groups, 3 modalities (contiguous and i.i.d.-shuffled)."""
    _run(synth.config_inputs("c2", **kw))


def test_w4g_decode_sized_text_equals_decode_path():
    """For a handful of text tokens the prefill GEMM and the decode kernel compute the same
    function of the same codes and scales (two layouts): both against the oracle."""
    m = M()
    ids0 = np.zeros(16, np.uint8)
    X = synth.activations(ids0, 3584, 1, 991)
    W = synth.weight(3584, 512, 992)
    s = np.exp(np.random.Generator(np.random.PCG64(993)).normal(0, 0.5, 3584)).astype(np.float32)
    q, dl = O.quantize_weight_grouped(W, s, 4, 128)
    pk, sc = m.quantize_weight_w4g(bf(W), tt(s))
    Y = m.linear_forward_w4g(bf(X), tt(ids0), tt(s[None, :]), pk, sc).cpu().numpy()
    pd, sd = m.quantize_weight_int4(bf(W), tt(s))
    Yd = m.linear_decode(bf(X), tt(s), pd, sd).cpu().numpy()
    Yo = O.linear_decode(X, s, q, dl, 8, 128)
    scale = np.abs(Yo).max()
    assert np.abs(Y - Yo).max() <= TOL_Y * scale and np.abs(Yd - Yo).max() <= TOL_Y * scale


@pytest.mark.parametrize("name,d,n", [("qkv", 3584, 4608), ("down", 18944, 3584)])
def test_w4g_c3_shapes(name, d, n):
    """c3 linears (W4 g128 A8, CMC rank 64 for image tokens) at 4096 tokens, sampled rows."""
    c = synth.config_inputs("c3", d=d, n=n, T=4096, layer=3)
    _run(c, rows=sample_rows(c["ids"], n_random=128))


def test_w4g_limits():
    m = M()
    c = synth.config_inputs("c1")
    X, ids = bf(c["X"]), tt(c["ids"])
    s = torch.ones(2, 192, device="cuda")
    W = bf(synth.weight(192, 128, 5))
    with pytest.raises(m.MasqError) as e:                     # d % 128 != 0
        m.quantize_weight_w4g(W, s[0])
    assert e.value.status == 2
