"""GPU parity of the GEMM's stream-K remainder (gemm.cu: the 256 x 256 units past the last full
wave of CTA pairs are split along K over the pairs; the unit's owner adds the other segments'
partial accumulators — int32 exactly, f32 in a fixed order — before its epilogue).  Deep-K shapes
only take that path (>= 64 k-blocks per unit).  The checked rows include every row of the
remainder units (the last m-units of the raster), so each split unit is compared in full:
  * int32 accumulators bit-exact against the oracle's integer GEMM (A6);
  * Y <= 1e-3 max-abs-normalised per modality (CMC included);
  * X W (masq_reference_output) <= 1e-4 per modality against f64 (reading Q16).
Cases: c3 down 18944 -> 3584 at 4096 tokens (2 remainder units of 4 segments), c2 down
11008 -> 2048 at 4096 tokens (54 remainder units, segments crossing unit boundaries), and two
ragged deep-K shapes (T and n not multiples of the 256 x 256 unit)."""
import numpy as np
import pytest

import oracle as O
import synth
from test_gpu_parity import M, bf, sample_rows, tt
from test_gpu_shapes import per_modality_err

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("cfg,d,n,T,tail_rows", [("c3", 18944, 3584, 4096, 256), ("c2", 11008, 2048, 4096, 1792),
                                                ("c3", 16384, 2080, 3000, 952), ("c2", 8192, 1120, 2777, 800)])
def test_streamk_remainder_units(cfg, d, n, T, tail_rows):
    """(the last two: ragged T and n — partial m-units and a partial last n-tile inside split units)"""
    c = synth.config_inputs(cfg, d=d, n=n, T=T, layer=4)
    m = M()
    T, n_mod, wb, ab, r = c["T"], c["n_mod"], c["wbits"], c["abits"], c["r"]
    Ro, co = O.calibrate_stats(c["X"], c["ids"], n_mod)
    so = O.init_factors(Ro, co, c["W"])
    qwo, dwo = O.quantize_weight(c["W"], so[0], wb)
    X, ids = bf(c["X"]), tt(c["ids"])
    rows = np.union1d(sample_rows(c["ids"], n_random=64), np.arange(T - tail_rows, T))
    acc = m.linear_forward(X, ids, tt(so), tt(qwo), tt(dwo), wb, ab, acc_debug=True).cpu().numpy()
    qxo, _ = O.quantize_activations(O.decode(c["X"])[rows], c["ids"][rows], so, ab)
    assert np.array_equal(acc[rows].astype(np.int64), O.int_gemm(qxo, qwo))
    L1 = bf(c["L1"]) if r else None
    L2 = bf(c["L2"]) if r else None
    Y = m.linear_forward(X, ids, tt(so), tt(qwo), tt(dwo), wb, ab, L1, L2).cpu().numpy()
    m.check()
    Yo = O.linear_forward(c["X"], c["ids"], so, qwo, dwo, ab, list(c["L1"]) if r else None,
                          list(c["L2"]) if r else None, rows=rows)
    assert max(per_modality_err(Y[rows], Yo, c["ids"][rows]).values()) <= 1e-3
    Yr = m.reference_output(X, bf(c["W"])).cpu().numpy()
    Yro = O.decode(c["X"])[rows].astype(np.float64) @ O.decode(c["W"]).astype(np.float64)
    assert max(per_modality_err(Yr[rows], Yro, c["ids"][rows]).values()) <= 1e-4


def test_streamk_concurrent_streams():
    """Two deep-K stream-K GEMM calls on two CUDA streams at once (separate workspaces), repeated:
    their clusters compete for SMs, so each kernel may be only partly resident while its owners
    wait for partials; the waits go only to lower, earlier-dispatched clusters, so both complete.
    Results equal the same calls run alone (int32 accumulators: bit-identical)."""
    import torch
    m = M()
    c = synth.config_inputs("c3", d=18944, n=3584, T=4096, layer=5)
    Ro, co = O.calibrate_stats(c["X"], c["ids"], 2)
    so = O.init_factors(Ro, co, c["W"])
    qwo, dwo = O.quantize_weight(c["W"], so[0], 4)
    X, ids, s, qw, dw = bf(c["X"]), tt(c["ids"]), tt(so), tt(qwo), tt(dwo)
    want = m.linear_forward(X, ids, s, qw, dw, 4, 8, acc_debug=True)
    wref = m.reference_output(X, bf(c["W"]))
    torch.cuda.synchronize()
    streams = [torch.cuda.Stream(), torch.cuda.Stream()]
    wss = [m.Workspace(X.device), m.Workspace(X.device)]
    outs = []
    for it in range(4):
        for k in range(2):
            with torch.cuda.stream(streams[k]):
                if (it + k) % 2 == 0:
                    outs.append(("acc", m.linear_forward(X, ids, s, qw, dw, 4, 8, acc_debug=True, ws=wss[k])))
                else:
                    outs.append(("ref", m.reference_output(X, bf(c["W"]), ws=wss[k])))
    torch.cuda.synchronize()
    m.check()
    for kind, o in outs:
        assert torch.equal(o, want if kind == "acc" else wref), kind


@pytest.mark.parametrize("seed", range(5))
def test_streamk_random_deep_k(seed):
    """Seeded random deep-K problems (d >= 8192: the int8 GEMM's stream-K path; ragged T and n,
    2-3 modalities, CMC rank 0 / 32 / 64): int32 accumulators of every row of the last 8 m-units
    plus sampled rows bit-exact, Y <= 1e-3 per modality, X W <= 1e-4 per modality."""
    g = np.random.Generator(np.random.PCG64(7000 + seed))
    d = int(g.choice([8192, 12288, 16384]))
    n = 32 * int(g.integers(8, 100))
    T = int(g.integers(600, 5000))
    cfg = "c2" if g.integers(0, 2) else "c3"
    r = int(g.choice([0, 32, 64])) if cfg == "c3" else 0
    c = synth.config_inputs(cfg, d=d, n=n, T=T, layer=10 + seed, r=r)
    m = M()
    T, n_mod, wb, ab = c["T"], c["n_mod"], c["wbits"], c["abits"]
    Ro, co = O.calibrate_stats(c["X"], c["ids"], n_mod)
    if np.any(co == 0):
        pytest.skip("a modality without tokens at this T")
    so = O.init_factors(Ro, co, c["W"])
    qwo, dwo = O.quantize_weight(c["W"], so[0], wb)
    X, ids = bf(c["X"]), tt(c["ids"])
    rows = np.union1d(sample_rows(c["ids"], n_random=48), np.arange(max(0, T - 8 * 256), T, 3))
    acc = m.linear_forward(X, ids, tt(so), tt(qwo), tt(dwo), wb, ab, acc_debug=True).cpu().numpy()
    qxo, _ = O.quantize_activations(O.decode(c["X"])[rows], c["ids"][rows], so, ab)
    assert np.array_equal(acc[rows].astype(np.int64), O.int_gemm(qxo, qwo)), (seed, d, n, T)
    L1 = bf(c["L1"]) if r else None
    L2 = bf(c["L2"]) if r else None
    Y = m.linear_forward(X, ids, tt(so), tt(qwo), tt(dwo), wb, ab, L1, L2).cpu().numpy()
    m.check()
    Yo = O.linear_forward(c["X"], c["ids"], so, qwo, dwo, ab, list(c["L1"]) if r else None,
                          list(c["L2"]) if r else None, rows=rows)
    assert max(per_modality_err(Y[rows], Yo, c["ids"][rows]).values()) <= 1e-3
    Yr = m.reference_output(X, bf(c["W"])).cpu().numpy()
    Yro = O.decode(c["X"])[rows].astype(np.float64) @ O.decode(c["W"]).astype(np.float64)
    assert max(per_modality_err(Yr[rows], Yro, c["ids"][rows]).values()) <= 1e-4
