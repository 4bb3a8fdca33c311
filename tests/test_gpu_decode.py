"""GPU parity for N3: packed int4 weights with 128-channel groups and the
decode-shaped W4A8 forward, against oracle.quantize_weight_grouped / linear_decode.

Bar: codes, scales and the packed bytes bit-exact (the layout is rebuilt here from the oracle's
codes following include/masq.h / csrc/decode.cu's documented order); Y within 1e-3
max-abs-normalised (group sums are exact integers, f32 accumulation over groups).
"""
import numpy as np
import pytest
import torch

import oracle as O
import synth
from test_gpu_parity import M, bf, tt

pytestmark = pytest.mark.gpu


def _inputs(d, n, T=16, seed=0):
    c = synth.config_inputs("c3", T=1024, d=d, n=n, r=0)
    R, cnt = O.calibrate_stats(c["X"], c["ids"], 2)
    s = O.init_factors(R, cnt, c["W"])
    return c, s


def _expected_packed(codes):
    """Documented order: tile (jt, g) of 512 B; lane L = 4 gid + tig; word ks; byte e holds
    code[8 jt + gid][128 g + 32 ks + 4 tig + e] + 8 (low nibble) and code[..][.. + 16] + 8 (high)."""
    n, d = codes.shape
    c = (codes.astype(np.int16) + 8).astype(np.uint8).reshape(n // 8, 8, d // 128, 4, 2, 4, 4)
    # axes: jt, gid, g, ks, half(16), tig, e  -> bytes [jt][g][gid][tig][ks][e]
    lo = c[:, :, :, :, 0]
    hi = c[:, :, :, :, 1]
    b = lo | (hi << 4)                                   # jt, gid, g, ks, tig, e
    return np.ascontiguousarray(b.transpose(0, 2, 1, 4, 3, 5)).reshape(-1)


@pytest.mark.parametrize("d,n", [(256, 96), (3584, 4608), (18944, 512)])
def test_int4_weight_quantizer_bitexact(d, n):
    m = M()
    c, s = _inputs(d, n)
    packed, scales = m.quantize_weight_int4(bf(c["W"]), tt(s[0]))
    q, dl = O.quantize_weight_grouped(c["W"], s[0], 4, 128)
    assert np.array_equal(scales.cpu().numpy(), dl.reshape(n // 8, 8, d // 128).transpose(0, 2, 1))
    assert np.array_equal(m.unpack_int4(packed, d, n).cpu().numpy(), q)
    assert np.array_equal(packed.cpu().numpy(), _expected_packed(q))


@pytest.mark.parametrize("d,n,T", [(256, 96, 1), (256, 96, 16), (3584, 4608, 3), (3584, 4608, 16),
                                   (18944, 512, 8), (2176, 200, 5)])
def test_linear_decode_parity(d, n, T):
    m = M()
    c, s = _inputs(d, n)
    W = bf(c["W"])
    packed, scales = m.quantize_weight_int4(W, tt(s[0]))
    rows = np.arange(T) * 37 % c["T"]
    Xh = c["X"][rows]
    Y = m.linear_decode(bf(Xh), tt(s[0]), packed, scales).cpu().numpy()
    m.check()
    q, dl = O.quantize_weight_grouped(c["W"], s[0], 4, 128)
    Yo = O.linear_decode(Xh, s[0], q, dl, 8, 128)
    err = np.abs(Y - Yo).max() / np.abs(Yo).max()
    assert err <= 1e-3, err
    # deterministic and strided output
    Y2 = torch.zeros(T, n + 8, device="cuda")
    m.linear_decode(bf(Xh), tt(s[0]), packed, scales, Y=Y2[:, :n])
    assert np.array_equal(Y2[:, :n].cpu().numpy(), Y) and float(Y2[:, n:].abs().sum()) == 0.0


def test_linear_decode_limits():
    m = M()
    c, s = _inputs(256, 96)
    packed, scales = m.quantize_weight_int4(bf(c["W"]), tt(s[0]))
    with pytest.raises(m.MasqError) as e:
        m.linear_decode(bf(c["X"][:17]), tt(s[0]), packed, scales)
    assert e.value.status == 2


def test_linear_decode_quantizer_paths_agree():
    """The decode call's one-launch bf16 quantizer (1/s formed in the kernel, no ids buffer) and
    the fallback path taken for f32 X (inverse-factor kernel + row kernel) see the same values
    (bf16 -> f32 is exact), so they must give bit-identical Y; a strided bf16 X view too."""
    m = M()
    d, n, T = 3584, 4608, 7
    c, s = _inputs(d, n)
    packed, scales = m.quantize_weight_int4(bf(c["W"]), tt(s[0]))
    Xh = c["X"][np.arange(T) * 53 % c["T"]]
    Yb = m.linear_decode(bf(Xh), tt(s[0]), packed, scales).cpu().numpy()
    Yf = m.linear_decode(tt(O.decode(Xh)), tt(s[0]), packed, scales).cpu().numpy()
    Xw = np.zeros((T, d + 128), np.uint16)
    Xw[:, 64:64 + d] = Xh
    Yv = m.linear_decode(bf(Xw)[:, 64:64 + d], tt(s[0]), packed, scales).cpu().numpy()
    m.check()
    assert np.array_equal(Yb, Yf) and np.array_equal(Yb, Yv)
    q, dl = O.quantize_weight_grouped(c["W"], s[0], 4, 128)
    Yo = O.linear_decode(Xh, s[0], q, dl, 8, 128)
    assert np.abs(Yb - Yo).max() / np.abs(Yo).max() <= 1e-3
