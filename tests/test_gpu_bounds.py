"""Out-of-bounds write checks (compute-sanitizer is closed on this pool): every output is placed
inside a larger buffer pre-filled with a sentinel; after the call the sentinel must survive
everywhere outside the logical output (extra rows, the padding of a leading dimension, guard
words after vectors).  Ragged shapes exercise every tile / box boundary."""
import numpy as np
import pytest
import torch

import oracle as O
import synth

pytestmark = pytest.mark.gpu

SENT_F = -12345.678


def bf(bits):
    return torch.from_numpy(np.ascontiguousarray(bits).view(np.int16)).view(torch.bfloat16).cuda()


def tt(a):
    return torch.from_numpy(np.ascontiguousarray(a)).cuda()


def M():
    import paper_2603_04800_b200 as m
    return m


@pytest.mark.parametrize("T,d,n,r", [(1000, 208, 288, 48), (1153, 64, 32, 16), (1300, 96, 544, 0), (4096 + 77, 256, 96, 32)])
def test_forward_writes_stay_in_bounds(T, d, n, r):
    c = synth.config_inputs("c2", T=T, d=d, n=n, r=r if r else 16)
    m = M()
    R, cnt = O.calibrate_stats(c["X"], c["ids"], 3)
    so = O.init_factors(R, cnt, c["W"])
    qwo, dwo = O.quantize_weight(c["W"], so[0], 8)
    ld = n + 40                                             # padded leading dimension
    big = torch.full((T + 70, ld), SENT_F, dtype=torch.float32, device="cuda")
    Y = big[:T, :n]
    L1 = bf(c["L1"]) if r else None
    L2 = bf(c["L2"]) if r else None
    m.linear_forward(bf(c["X"]), tt(c["ids"]), tt(so), tt(qwo), tt(dwo), 8, 8, L1, L2, Y=Y)
    m.check()
    b = big.cpu().numpy()
    assert np.all(b[T:] == np.float32(SENT_F)), "rows beyond T written"
    assert np.all(b[:T, n:] == np.float32(SENT_F)), "columns beyond d_out written"
    assert np.all(np.isfinite(b[:T, :n]))


@pytest.mark.parametrize("d,n,bits", [(208, 288, 8), (64, 32, 4), (4096 + 16, 96, 2)])
def test_weight_quantizer_writes_stay_in_bounds(d, n, bits):
    rng = np.random.Generator(np.random.PCG64(d + n))
    W = synth.f32_to_bf16_bits(rng.standard_normal((d, n)).astype(np.float32))
    s = np.exp(rng.standard_normal(d)).astype(np.float32)
    m = M()
    qbig = torch.full((n * d + 4096,), 77, dtype=torch.int8, device="cuda")
    dbig = torch.full((n + 64,), SENT_F, dtype=torch.float32, device="cuda")
    import ctypes
    from paper_2603_04800_b200._lib import lib
    ws = m.Workspace()
    p, nb = ws.ptr_size(m.workspace_size(2, 0, d, n, 1))
    Wg, sg = bf(W), tt(s)
    st = lib().masq_quantize_weight(ctypes.c_void_p(Wg.data_ptr()), 1, ctypes.c_void_p(sg.data_ptr()), d, n, bits,
                                    ctypes.c_void_p(qbig.data_ptr()), ctypes.c_void_p(dbig.data_ptr()), p, nb,
                                    ctypes.c_void_p(torch.cuda.current_stream().cuda_stream))
    assert st == 0
    torch.cuda.synchronize()
    q = qbig.cpu().numpy()
    dd = dbig.cpu().numpy()
    qo, do = O.quantize_weight(W, s, bits)
    assert np.array_equal(q[: n * d].reshape(n, d), qo)
    assert np.all(q[n * d:] == 77)
    assert np.array_equal(dd[:n], do) and np.all(dd[n:] == np.float32(SENT_F))


def test_activation_quantizer_and_loss_writes_stay_in_bounds():
    T, d, n = 777, 96, 160
    c = synth.config_inputs("c2", T=T, d=d, n=n, shuffle=True)
    m = M()
    R, cnt = O.calibrate_stats(c["X"], c["ids"], 3)
    so = O.init_factors(R, cnt, c["W"])
    X, W, ids = bf(c["X"]), bf(c["W"]), tt(c["ids"])
    Ybig = torch.full((T + 5, n + 8), SENT_F, dtype=torch.float32, device="cuda")
    Yref = m.reference_output(X, W, Yref=Ybig[:T, :n])
    yb = Ybig.cpu().numpy()
    assert np.all(yb[T:] == np.float32(SENT_F)) and np.all(yb[:T, n:] == np.float32(SENT_F))
    sums = torch.full((3 + 4,), SENT_F, dtype=torch.float64, device="cuda")
    counts = torch.full((3 + 4,), -7, dtype=torch.int64, device="cuda")
    loss = torch.full((1 + 4,), SENT_F, dtype=torch.float64, device="cuda")
    m.calib_loss(X, ids, tt(so), W, 8, 8, Yref, sums=sums[:3], counts=counts[:3], loss=loss[:1])
    m.check()
    assert np.all(sums.cpu().numpy()[3:] == SENT_F) and np.all(counts.cpu().numpy()[3:] == -7)
    assert np.all(loss.cpu().numpy()[1:] == SENT_F)
    _, _, lo = O.calib_loss(c["X"], c["ids"], so, c["W"], 8, 8)
    assert abs(float(loss[0]) - lo) <= 1e-3 * abs(lo)


def test_stats_and_init_writes_stay_in_bounds():
    T, d, n = 1333, 48, 64                                    # >= one full c2 sample: all 3 modalities
    c = synth.config_inputs("c2", T=T, d=d, n=n)
    m = M()
    Rbig = torch.full((3 * d + 32,), SENT_F, dtype=torch.float32, device="cuda")
    cbig = torch.full((3 + 5,), -9, dtype=torch.int64, device="cuda")
    R, cnt = m.calibrate_stats(bf(c["X"]), tt(c["ids"]), 3, R=Rbig[:3 * d].view(3, d), count=cbig[:3])
    sbig = torch.full((3 * d + 32,), SENT_F, dtype=torch.float32, device="cuda")
    import ctypes
    from paper_2603_04800_b200._lib import lib
    ws = m.Workspace()
    p, nb = ws.ptr_size(m.workspace_size(1, 0, d, n, 3))
    Wg = bf(c["W"])
    st = lib().masq_init_factors(ctypes.c_void_p(R.data_ptr()), ctypes.c_void_p(cnt.data_ptr()),
                                 ctypes.c_void_p(Wg.data_ptr()), 1, d, n, 3, ctypes.c_void_p(sbig.data_ptr()), None,
                                 p, nb, ctypes.c_void_p(torch.cuda.current_stream().cuda_stream))
    assert st == 0
    torch.cuda.synchronize()
    assert np.all(Rbig.cpu().numpy()[3 * d:] == np.float32(SENT_F))
    assert np.all(cbig.cpu().numpy()[3:] == -9)
    assert np.all(sbig.cpu().numpy()[3 * d:] == np.float32(SENT_F))
    Ro, co = O.calibrate_stats(c["X"], c["ids"], 3)
    assert np.array_equal(sbig.cpu().numpy()[:3 * d].reshape(3, d), O.init_factors(Ro, co, c["W"]))
