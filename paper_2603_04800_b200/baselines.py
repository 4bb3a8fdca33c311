"""N4 drivers: the baseline factor methods of PAPER.md:19-39 on the same device data.

Host logic only (loops over the beta grid); every numeric step runs in libmasq.so:
masq_range_stats (unified ranges), masq_smooth_factors (closed forms), masq_calibrate_meanabs
(AWQ statistic) and masq_calib_loss (the score).  Mirrors oracle.awq_grid_search.
"""
from __future__ import annotations

from . import masq as _m


def unified_factors(R, wmax, beta: float = 0.5, stream=None):
    """SmoothQuant with one factor for every modality: s = (max_m R^m)^beta /
    wmax^(1-beta), broadcast to [M x d]."""
    _, runi, _ = _m.range_stats(R, stream=stream)
    s = _m.smooth_factors(runi, beta, den=wmax, stream=stream)
    return s.expand(R.shape[0], -1).contiguous()


def awq_grid_search(X, mod_id, W, wbits: int, abits: int, betas, n_mod: int, lam=None, Yref=None, ws=None,
                    stream=None):
    """AWQ: unified s(beta) = mean_t|x_t,i|^beta over all tokens, scored by the
    calibration loss; returns (beta*, [loss(beta)] as floats, s(beta*) [M x d])."""
    ws = ws or _m.default_workspace(X.device)
    if Yref is None:
        Yref = _m.reference_output(X, W, ws=ws, stream=stream)
    _, _, _, uni = _m.calibrate_meanabs(X, mod_id, n_mod, ws=ws, stream=stream)
    losses, best, s_best = [], None, None
    for b in betas:
        s = _m.smooth_factors(uni, b, stream=stream).expand(n_mod, -1).contiguous()
        _, _, loss = _m.calib_loss(X, mod_id, s, W, wbits, abits, Yref, lam=lam, ws=ws, stream=stream)
        v = float(loss.item())
        losses.append(v)
        if best is None or v < best:
            best, s_best = v, s
    return float(betas[losses.index(best)]), losses, s_best
