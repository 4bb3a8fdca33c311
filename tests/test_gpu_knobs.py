"""GPU parity of the GEMM's measurement-knob variants, each in a fresh process (the library reads
its knobs once per process):
  * MASQ_GEMM_CL=4 — 4-CTA clusters, two CTA pairs on adjacent n-tiles sharing the A tile by TMA
    multicast (gemm.cu); an odd number of n-tiles exercises the partner-only tile past the edge;
  * MASQ_STREAMK=0 — whole units only (the deep-K remainder split off).
Int32 accumulators bit-exact against the oracle's integer GEMM (A6), Y <= 1e-3
per modality with CMC (A7), X W <= 1e-4 per modality (reading Q16), the fused layer call's loss
sums <= 1e-3 (A8)."""
import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)

SCRIPT = r"""
import sys
import numpy as np
sys.path.insert(0, {here!r}); sys.path.insert(0, {root!r})
import oracle as O
import synth
from test_gpu_parity import M, bf, sample_rows, tt
from test_gpu_shapes import per_modality_err

m = M()
for cfg, d, n, T in {cases!r}:
    c = synth.config_inputs(cfg, d=d, n=n, T=T, layer=7)
    n_mod, wb, ab, r = c["n_mod"], c["wbits"], c["abits"], c["r"]
    Ro, co = O.calibrate_stats(c["X"], c["ids"], n_mod)
    so = O.init_factors(Ro, co, c["W"])
    qwo, dwo = O.quantize_weight(c["W"], so[0], wb)
    X, ids = bf(c["X"]), tt(c["ids"])
    rows = np.union1d(sample_rows(c["ids"], n_random=64), np.arange(max(0, T - 256), T))
    acc = m.linear_forward(X, ids, tt(so), tt(qwo), tt(dwo), wb, ab, acc_debug=True).cpu().numpy()
    qxo, _ = O.quantize_activations(O.decode(c["X"])[rows], c["ids"][rows], so, ab)
    assert np.array_equal(acc[rows].astype(np.int64), O.int_gemm(qxo, qwo)), (cfg, d, n, T)
    L1 = bf(c["L1"]) if r else None
    L2 = bf(c["L2"]) if r else None
    Y = m.linear_forward(X, ids, tt(so), tt(qwo), tt(dwo), wb, ab, L1, L2).cpu().numpy()
    Yo = O.linear_forward(c["X"], c["ids"], so, qwo, dwo, ab, list(c["L1"]) if r else None,
                          list(c["L2"]) if r else None, rows=rows)
    e = max(per_modality_err(Y[rows], Yo, c["ids"][rows]).values())
    assert e <= 1e-3, (cfg, d, n, T, e)
    Yr = m.reference_output(X, bf(c["W"])).cpu().numpy()
    Yro = O.decode(c["X"])[rows].astype(np.float64) @ O.decode(c["W"]).astype(np.float64)
    e = max(per_modality_err(Yr[rows], Yro, c["ids"][rows]).values())
    assert e <= 1e-4, (cfg, d, n, T, e)
    sums, counts, loss = m.calib_loss(X, ids, tt(so), bf(c["W"]), wb, ab, m.reference_output(X, bf(c["W"])))
    so_, co_, lo_ = O.calib_loss(c["X"], c["ids"], so, c["W"], wb, ab)
    s_ = sums.cpu().numpy()
    assert np.all(np.abs(s_ - so_) <= 1e-3 * np.abs(so_)), (cfg, s_, so_)
m.check()
print("ok")
"""


def _run(env_extra, cases):
    env = dict(os.environ)
    env.update(env_extra)
    code = SCRIPT.format(here=HERE, root=ROOT, cases=cases)
    p = subprocess.run([sys.executable, "-c", code], env=env, capture_output=True, text=True, timeout=900)
    assert p.returncode == 0 and p.stdout.strip().endswith("ok"), p.stdout[-2000:] + p.stderr[-4000:]


def test_gemm_four_cta_clusters_multicast():
    # c3 qkv: 18 n-tiles (even); c1-sized 3-modality case with n = 288 (2 n-tiles, the second
    # partial) and n = 800 (4 n-tiles -> 2 pairs) ; c2 o 2048 -> 2048 (8 n-tiles), 3 modalities
    _run({"MASQ_GEMM_CL": "4"}, [("c3", 3584, 4608, 2048), ("c2", 2048, 2048, 1500), ("c2", 1024, 800, 777),
                                 ("c3", 512, 288, 1000)])


def test_gemm_without_streamk():
    _run({"MASQ_STREAMK": "0"}, [("c3", 18944, 3584, 4096)])
