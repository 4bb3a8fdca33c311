"""N1 driver: the S-optimisation loop (SPEC.md:307-316 optimize_factors) over the C ABI.

Host logic only — every numeric step runs in libmasq.so: masq_calib_loss_grad per batch,
masq_adam_step, masq_calib_loss for the per-epoch objective and masq_keep_best for the
best-so-far iterate.  The host reads one f64 per batch step (the finite-loss check of
SPEC.md:312) and one per epoch (the objective history).  Mirrors oracle.optimize_factors
step for step.
"""
from __future__ import annotations

import math

import torch

from . import masq as _m


def optimize_factors(X, mod_id, s0, W, wbits: int, abits: int, epochs: int = 2, batch_tokens: int = 1024,
                     lr: float = 1e-2, lam=None, Yref=None, max_rejections: int = 10, ws=None, stream=None,
                     group=None):
    """Returns (s_best f32 [M x d] device, best objective f64 [1] device, per-epoch objectives).

    Token-sharded (torch.distributed initialised, world > 1, every rank holding the same number of
    batches of its own tokens): each batch's gradient is normalised by the batch's GLOBAL token
    counts (one SUM of M counts per batch, once, before the loop) and SUM-reduced, the batch loss
    and the epoch objective are SUM-reduced (sums, counts) before the finite check / best-so-far,
    so every rank takes the same decisions and ends with the same factors."""
    T = X.shape[0]
    dev = X.device
    ws = ws or _m.default_workspace(dev)
    from . import parallel as _par
    _, world = _par.world()
    sharded = world > 1
    if Yref is None:
        Yref = _m.reference_output(X, W, ws=ws, stream=stream)
    s = s0.contiguous().clone()
    s_best = s.clone()
    best = torch.full((1,), float("nan"), dtype=torch.float64, device=dev)
    theta, m1, m2 = _m.adam_init(s, stream=stream)
    grad = torch.empty_like(theta)
    n_mod = s.shape[0]
    sums = torch.empty(n_mod, dtype=torch.float64, device=dev)
    counts = torch.empty(n_mod, dtype=torch.int64, device=dev)
    loss = torch.empty(1, dtype=torch.float64, device=dev)
    d_out = W.shape[1]
    batches = [(a, min(T, a + batch_tokens)) for a in range(0, T, batch_tokens)]
    norms = [None] * len(batches)
    if sharded:                                           # global counts of every batch, once
        norms = [_m.count_modalities(mod_id[a:b], n_mod, ws=ws, stream=stream) for a, b in batches]
        for c in norms:
            _par.reduce_loss(torch.zeros(1, dtype=torch.float64, device=dev), c, group=group)

    def finalize():
        if sharded:
            _par.reduce_loss(sums, counts, group=group)
            _m.loss_finalize(sums, counts, d_out, lam=lam, loss=loss, stream=stream)

    def objective():
        _m.calib_loss(X, mod_id, s, W, wbits, abits, Yref, lam=lam, sums=sums, counts=counts, loss=loss, ws=ws,
                      stream=stream)
        finalize()
        _m.keep_best(loss, best, s, s_best, stream=stream)

    objective()
    history = []
    t, rejections = 0, 0
    for _ in range(epochs):
        for bi, (a, b) in enumerate(batches):
            _m.calib_loss_grad(X[a:b], mod_id[a:b], s, W, wbits, abits, Yref[a:b], lam=lam, grad=grad, sums=sums,
                               counts=counts, loss=loss, count_norm=norms[bi], ws=ws, stream=stream)
            if sharded:
                _par.reduce_grad(grad, group=group)
                finalize()
            if not math.isfinite(float(loss.item())):
                lr, rejections = lr * 0.5, rejections + 1
                if rejections >= max_rejections:
                    return s_best, best, history
                continue
            rejections, t = 0, t + 1
            _m.adam_step(theta, grad, m1, m2, t, lr, s_out=s, stream=stream)
        objective()
        history.append(float(loss.item()))
    return s_best, best, history
