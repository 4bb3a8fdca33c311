"""world_size-2 gloo tests (CPU) of the multi-GPU host logic in paper_2603_04800_b200/parallel.py.

Each rank computes its token shard with the CPU oracle (standing in for the per-GPU kernels,
which need a B200), then the real reduction code runs over gloo:
  * R after the MAX all-reduce is bit-identical to the single-process R; counts add up;
  * the loss from SUM-reduced per-modality sums/counts equals the single-process loss;
  * output-column shards of the forward concatenate to the full forward;
  * N1 gradients of the token shards (global-count normalised) SUM to the full gradient;
  * N2: the shards' Gram matrices SUM to the batch Gram, and the CMC factors from it equal the
    single-process factors;
  * N4: the shards' mean-abs sums and counts SUM to the batch statistic.
"""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import oracle as O
import synth
from paper_2603_04800_b200 import parallel as P


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world_size, port, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world_size)
    try:
        c = synth.config_inputs("c2", T=4096, d=96, n=160, r=16)
        a, b = P.token_shard(c["T"], rank, world_size)
        # A1 on this rank's tokens, then the real exchange code
        R, cnt = O.calibrate_stats(c["X"][a:b], c["ids"][a:b], 3)
        Rt, ct = torch.from_numpy(R.copy()), torch.from_numpy(cnt.copy())
        P.reduce_stats([Rt], ct)
        # A8 partial sums with the factors of the full batch
        Rf, cf = O.calibrate_stats(c["X"], c["ids"], 3)
        s = O.init_factors(Rf, cf, c["W"])
        sums, counts, _ = O.calib_loss(c["X"][a:b], c["ids"][a:b], s, c["W"], 8, 8)
        st, nt = torch.from_numpy(sums.copy()), torch.from_numpy(counts.copy())
        P.reduce_loss(st, nt)
        # N1 gradient on this rank's tokens, normalised by the global counts, then SUM
        _, g = O.calib_loss_grad(c["X"][a:b], c["ids"][a:b], s, c["W"], 8, 8, count_norm=cf)
        gt = torch.from_numpy(g.copy())
        P.reduce_grad(gt)
        # N2: this rank's Gram of the smoothed image tokens, SUM-reduced -> the batch Gram
        xs = O.smooth_activations(O.decode(c["X"][a:b]), c["ids"][a:b], s)
        A = xs[c["ids"][a:b] == 1].astype(np.float64)
        Gt = torch.from_numpy(A.T @ A)
        P.reduce_gram(Gt)
        # N4: AWQ's mean-abs statistic, SUM of the shards' sums and counts
        Sa, ca = O.meanabs_stats(c["X"][a:b], c["ids"][a:b], 3)
        Sat, cat = torch.from_numpy(Sa.copy()), torch.from_numpy(ca.copy())
        P.reduce_loss(Sat, cat)
        # forward column shard
        qw, dw = O.quantize_weight(c["W"], s[0], 8)
        j0, j1 = P.column_shards(c["n"], world_size)[rank]
        Ys = O.linear_forward(c["X"], c["ids"], s, qw[j0:j1], dw[j0:j1], 8,
                              [c["L1"][0], c["L1"][1]], [c["L2"][0][:, j0:j1], c["L2"][1][:, j0:j1]])
        parts = [None] * world_size
        dist.all_gather_object(parts, (j0, j1, Ys))
        q.put((rank, Rt.numpy(), ct.numpy(), st.numpy(), nt.numpy(), parts, gt.numpy(), Gt.numpy(), Sat.numpy(),
               cat.numpy()))
    finally:
        dist.destroy_process_group()


@pytest.mark.timeout(300)
def test_two_rank_exchange_matches_single_process():
    world_size = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world_size, port, q)) for r in range(world_size)]
    for p in procs:
        p.start()
    res = [q.get(timeout=240) for _ in range(world_size)]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    c = synth.config_inputs("c2", T=4096, d=96, n=160, r=16)
    R1, c1 = O.calibrate_stats(c["X"], c["ids"], 3)
    s = O.init_factors(R1, c1, c["W"])
    sums1, counts1, loss1 = O.calib_loss(c["X"], c["ids"], s, c["W"], 8, 8)
    qw, dw = O.quantize_weight(c["W"], s[0], 8)
    Y1 = O.linear_forward(c["X"], c["ids"], s, qw, dw, 8, [c["L1"][0], c["L1"][1]], [c["L2"][0], c["L2"][1]])
    _, g1 = O.calib_loss_grad(c["X"], c["ids"], s, c["W"], 8, 8)
    xs1 = O.smooth_activations(O.decode(c["X"]), c["ids"], s)
    A1 = xs1[c["ids"] == 1].astype(np.float64)
    qw0, dw0 = O.quantize_weight(c["W"], s[0], 8)
    dW = O.weight_residual(c["W"], s[1], qw0, dw0)
    F1, F2 = O.cmc_factors(A1, dW, 8)
    Sf, cf_ = O.meanabs_stats(c["X"], c["ids"], 3)
    for rank, R, cnt, sums, counts, parts, g, G, Sa, ca in res:
        assert np.allclose(Sa, Sf, rtol=1e-12) and np.array_equal(ca, cf_)
        assert np.allclose(g, g1, rtol=1e-9, atol=1e-12 * np.abs(g1).max())
        H1, H2 = O.cmc_factors_from_gram(G, dW, 8)               # CMC factors from the reduced Gram
        assert np.linalg.norm(A1 @ (H1 @ H2 - F1 @ F2)) <= 1e-9 * np.linalg.norm(A1 @ dW)
        assert np.array_equal(R, R1), "MAX all-reduce of R must be bit-identical to one process"
        assert np.array_equal(cnt, c1)
        assert np.array_equal(counts, counts1)
        assert np.allclose(sums, sums1, rtol=1e-12)
        loss = O.loss_finalize(sums, counts, np.ones(3), c["n"])
        assert abs(loss - loss1) <= 1e-12 * abs(loss1)
        Y = np.concatenate([p[2] for p in sorted(parts, key=lambda t: t[0])], axis=1)
        assert np.array_equal(Y, Y1)


def test_shard_helpers():
    assert P.token_shard(16384, 0, 8) == (0, 2048)
    assert P.token_shard(16384, 7, 8) == (14336, 16384)
    assert P.token_shard(1000, 1, 2) == (1000, 1000)          # aligned to whole 1024-token samples
    sh = P.column_shards(18944, 8)
    assert sh[0] == (0, 2368) and sh[-1][1] == 18944 and all((b - a) % 32 == 0 for a, b in sh)
    sh = P.column_shards(288, 2)
    assert sh == [(0, 160), (160, 288)]
