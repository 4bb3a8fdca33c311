"""GPU parity of A4 (routed smoothing + per-token quantization) at every
launch shape of the bf16 activation quantizer, and on rows built to land on the rounding ties,
where the packed fast path must hand over to the exact IEEE-quotient + round-half-away path
(reading Q5/Q6).  Bit-exact against the oracle."""
import numpy as np
import pytest
import torch

import oracle as O
import synth

pytestmark = pytest.mark.gpu


def bf(bits):
    return torch.from_numpy(np.ascontiguousarray(bits).view(np.int16)).view(torch.bfloat16).cuda()


def tt(a):
    return torch.from_numpy(np.ascontiguousarray(a)).cuda()


def to_bf16_bits(x):
    """Exact for values representable in bf16 (the test only builds such values)."""
    b = np.asarray(x, np.float32).view(np.uint32)
    assert np.all(b & 0xFFFF == 0)
    return (b >> 16).astype(np.uint16)


# d spans every (chunks per thread, factors-in-registers) variant of the launcher and the
# generic fallback (d > 32768), each with a ragged row count and three modalities
@pytest.mark.parametrize("d", [64, 2048, 3584, 11008, 16384, 18944, 28672, 40960])
@pytest.mark.parametrize("abits", [8, 4])
def test_aquant_widths_bitexact(d, abits):
    import paper_2603_04800_b200 as m
    T = 389
    ids = np.repeat(np.array([0, 1, 2, 0, 1], np.uint8), [40, 150, 77, 1, 121])
    X = synth.activations(ids, d, 3, synth.seed_for(1, 0, 0))
    W = synth.weight(d, 16, synth.seed_for(1, 0, 1))
    R, cnt = O.calibrate_stats(X, ids, 3)
    so = O.init_factors(R, cnt, W)
    qx, dx, mask = m.quantize_activations(bf(X), tt(ids), tt(so), abits)
    m.check()
    qxo, dxo = O.quantize_activations(X, ids, so, abits)
    assert np.array_equal(dx.cpu().numpy(), dxo)
    assert np.array_equal(qx.cpu().numpy(), qxo)


@pytest.mark.parametrize("abits", [8, 4, 2])
def test_aquant_ties_round_half_away(abits):
    """Rows whose scaled values sit exactly on half-integers of the grid: rint (ties to even)
    would be wrong on half of them; the kernel must produce round-half-away codes."""
    import paper_2603_04800_b200 as m
    q = 2 ** (abits - 1) - 1
    d, T = 3584, 260
    g = np.random.Generator(np.random.PCG64(7))
    halves = (g.integers(-q, q, size=(T, d)) + 0.5).astype(np.float32)     # k + 1/2, |.| < q
    halves[:, 0] = q                                                        # absmax q -> Delta = 1
    halves[::3, 1] = -q
    X = to_bf16_bits(halves * 0.25)        # s = 1/4 (power of two): xs = halves exactly
    ids = (np.arange(T) % 3 == 1).astype(np.uint8)
    s = np.full((2, d), 0.25, np.float32)
    qx, dx, _ = m.quantize_activations(bf(X), tt(ids), tt(s), abits)
    m.check()
    qxo, dxo = O.quantize_activations(X, ids, s, abits)
    assert np.all(dxo == 1.0)
    assert np.array_equal(dx.cpu().numpy(), dxo)
    assert np.array_equal(qx.cpu().numpy(), qxo)
    # and the oracle itself rounds those ties away from zero
    v = halves[:, 2:].astype(np.float64)
    assert np.array_equal(qxo[:, 2:].astype(np.float64), np.sign(v) * np.floor(np.abs(v) + 0.5))


def test_aquant_edge_rows():
    """All-zero rows (Delta floored at 1e-12, codes 0), a single token, the smallest width (d = 16),
    a strided X view (ld_x > d) and an id >= n_mod (zero codes, Delta 0, sticky BAD_MODALITY)."""
    import paper_2603_04800_b200 as m
    g = np.random.Generator(np.random.PCG64(11))
    for d in (16, 3584):
        T = 37
        ids = g.integers(0, 2, T).astype(np.uint8)
        X = synth.activations(ids, d, 2, 5)
        X[3] = 0                                            # bf16 +0 row
        s = (g.random((2, d)) + 0.5).astype(np.float32)
        qx, dx, _ = m.quantize_activations(bf(X), tt(ids), tt(s), 8)
        m.check()
        qxo, dxo = O.quantize_activations(X, ids, s, 8)
        assert dxo[3] == np.float32(1e-12) and not qxo[3].any()
        assert np.array_equal(dx.cpu().numpy(), dxo) and np.array_equal(qx.cpu().numpy(), qxo)
        # single token
        qx1, dx1, _ = m.quantize_activations(bf(X[5:6]), tt(ids[5:6]), tt(s), 8)
        assert np.array_equal(qx1.cpu().numpy(), qxo[5:6]) and np.array_equal(dx1.cpu().numpy(), dxo[5:6])
        # strided rows: a column window of a wider activation matrix
        Xw = np.zeros((T, d + 64), np.uint16)
        Xw[:, 32:32 + d] = X
        Xv = bf(Xw)[:, 32:32 + d]
        assert Xv.stride(0) == d + 64
        qx2, dx2, _ = m.quantize_activations(Xv, tt(ids), tt(s), 8)
        assert np.array_equal(qx2.cpu().numpy(), qxo) and np.array_equal(dx2.cpu().numpy(), dxo)
    # bad modality id: zero codes, Delta 0, sticky status 6
    bad = ids.copy()
    bad[9] = 7
    qx3, dx3, _ = m.quantize_activations(bf(X), tt(bad), tt(s), 8)
    with pytest.raises(m.MasqError) as e:
        m.check()
    assert e.value.status == 6
    m.check()
    assert not qx3.cpu().numpy()[9].any() and float(dx3[9]) == 0.0
    keep = np.arange(T) != 9
    assert np.array_equal(qx3.cpu().numpy()[keep], qxo[keep])
