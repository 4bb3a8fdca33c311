"""Thin PyTorch binding over the C ABI (include/masq.h): argument marshalling only.

Every step of the hot path runs in libmasq.so's sm_100a kernels; torch supplies device
memory (tensors), the current CUDA stream and nothing else.  Names follow the ABI.
"""
from __future__ import annotations

import ctypes

import torch

from ._lib import MasqDebug, lib

MASQ_F32, MASQ_BF16 = 0, 1
(OP_STATS, OP_INIT, OP_QWEIGHT, OP_QACT, OP_FORWARD, OP_LOSS, OP_REFERENCE, OP_LOSS_GRAD, OP_MEANABS,
 OP_CMC, OP_DECODE, OP_LAYER, OP_CMC_GRAM, OP_CMC_FACTORS) = range(14)
OP_SELF_REF = 0x100


class MasqError(RuntimeError):
    def __init__(self, status: int, where: str):
        msg = lib().masq_status_string(status).decode()
        super().__init__(f"{where}: status {status} ({msg})")
        self.status = status


def _ck(status: int, where: str):
    if status != 0:
        raise MasqError(status, where)


def _p(t):
    return None if t is None else ctypes.c_void_p(t.data_ptr())


def _stream(stream=None):
    s = torch.cuda.current_stream() if stream is None else stream
    return ctypes.c_void_p(s.cuda_stream)


def _dt(t: torch.Tensor) -> int:
    if t.dtype == torch.bfloat16:
        return MASQ_BF16
    if t.dtype == torch.float32:
        return MASQ_F32
    raise TypeError(f"unsupported dtype {t.dtype} (bf16 or f32)")


def _cuda(t: torch.Tensor, name: str):
    if not t.is_cuda:
        raise ValueError(f"{name} must be a CUDA tensor")
    return t


class Workspace:
    """Caller-owned scratch for the ABI (grown on demand; first bytes hold the sticky status)."""

    def __init__(self, device=None):
        self.device = torch.device("cuda", torch.cuda.current_device()) if device is None else torch.device(device)
        self.buf = None

    def get(self, nbytes: int) -> torch.Tensor:
        nbytes = max(int(nbytes), 256)
        if self.buf is None or self.buf.numel() < nbytes:
            new = torch.zeros(nbytes + 256, dtype=torch.uint8, device=self.device)
            if self.buf is not None:
                # kernels queued on any stream may still use the old block and its sticky status
                # word: wait for them, then carry the status (at the 256-aligned base) across
                torch.cuda.synchronize(self.device)
                o_old, o_new = (-self.buf.data_ptr()) % 256, (-new.data_ptr()) % 256
                new[o_new:o_new + 16].copy_(self.buf[o_old:o_old + 16])
            self.buf = new
        return self.buf

    def ptr_size(self, nbytes: int):
        b = self.get(nbytes)
        base = b.data_ptr()
        off = (-base) % 256
        return ctypes.c_void_p(base + off), b.numel() - off


_WS = {}


def default_workspace(device=None) -> Workspace:
    dev = torch.cuda.current_device() if device is None else torch.device(device).index
    if dev not in _WS:
        _WS[dev] = Workspace(torch.device("cuda", dev))
    return _WS[dev]


def workspace_size(op: int, T: int, d: int, d_out: int, n_mod: int, r: int = 0) -> int:
    return int(lib().masq_workspace_size(op, T, d, d_out, n_mod, r))


def check(ws: Workspace | None = None, stream=None):
    """Synchronize and raise if a device-side data error (bad id / empty modality) was flagged."""
    ws = ws or default_workspace()
    p, _ = ws.ptr_size(256)
    _ck(lib().masq_check(p, _stream(stream)), "masq_check")


# ----------------------------------------------------------------------------- A1
def calibrate_stats(X, mod_id, n_mod: int, R=None, count=None, reset: bool = True, ws=None, stream=None):
    _cuda(X, "X")
    T, d = X.shape
    if R is None:
        R = torch.zeros(n_mod, d, dtype=torch.float32, device=X.device)
    if count is None:
        count = torch.zeros(n_mod, dtype=torch.int64, device=X.device)
    ws = ws or default_workspace(X.device)
    p, n = ws.ptr_size(workspace_size(OP_STATS, T, d, 0, n_mod))
    _ck(lib().masq_calibrate_stats(_p(X), _dt(X), X.stride(0), _p(mod_id), T, d, n_mod, _p(R), _p(count),
                                   1 if reset else 0, p, n, _stream(stream)), "masq_calibrate_stats")
    return R, count


# ----------------------------------------------------------------------------- A2
def init_factors(R, count, W, ws=None, stream=None, return_wmax: bool = False):
    n_mod, d = R.shape
    d_out = W.shape[1]
    s = torch.empty(n_mod, d, dtype=torch.float32, device=R.device)
    wmax = torch.empty(d, dtype=torch.float32, device=R.device) if return_wmax else None
    ws = ws or default_workspace(R.device)
    p, n = ws.ptr_size(workspace_size(OP_INIT, 0, d, d_out, n_mod))
    _ck(lib().masq_init_factors(_p(R), _p(count), _p(W.contiguous()), _dt(W), d, d_out, n_mod, _p(s), _p(wmax),
                                p, n, _stream(stream)), "masq_init_factors")
    return (s, wmax) if return_wmax else s


# ----------------------------------------------------------------------------- A3
def quantize_weight(W, s_vec, wbits: int, ws=None, stream=None):
    d, d_out = W.shape
    qw = torch.empty(d_out, d, dtype=torch.int8, device=W.device)
    dw = torch.empty(d_out, dtype=torch.float32, device=W.device)
    ws = ws or default_workspace(W.device)
    p, n = ws.ptr_size(workspace_size(OP_QWEIGHT, 0, d, d_out, 1))
    _ck(lib().masq_quantize_weight(_p(W.contiguous()), _dt(W), _p(s_vec.contiguous()), d, d_out, wbits, _p(qw),
                                   _p(dw), p, n, _stream(stream)), "masq_quantize_weight")
    return qw, dw


# ----------------------------------------------------------------------------- A4
def quantize_activations(X, mod_id, s, abits: int, ws=None, stream=None):
    T, d = X.shape
    n_mod = s.shape[0]
    qx = torch.empty(T, d, dtype=torch.int8, device=X.device)
    dx = torch.empty(T, dtype=torch.float32, device=X.device)
    mask = torch.empty((T + 127) // 128, dtype=torch.int32, device=X.device)
    ws = ws or default_workspace(X.device)
    p, n = ws.ptr_size(workspace_size(OP_QACT, T, d, 0, n_mod))
    _ck(lib().masq_quantize_activations(_p(X), _dt(X), X.stride(0), _p(mod_id), T, d, n_mod, _p(s.contiguous()),
                                        abits, _p(qx), _p(dx), _p(mask), p, n, _stream(stream)),
        "masq_quantize_activations")
    return qx, dx, mask


# ----------------------------------------------------------------------------- A4-A7
def linear_forward(X, mod_id, s, qw, dw, wbits: int, abits: int, L1=None, L2=None, Y=None,
                   acc_debug: bool = False, taps: bool = False, ws=None, stream=None):
    """Y = Q(X_m S_m^-1) Q(S_t W) [+ X_m S_m^-1 L1^m L2^m for m != text].

    L1: bf16 [n_mod-1, d, r]; L2: bf16 [n_mod-1, r, d_out] (or a column view with a row stride).
    acc_debug=True returns the raw int32 accumulators instead (CMC skipped).
    taps=True returns (out, qx, dx): the activation codes / steps the call used (debug taps).
    """
    T, d = X.shape
    d_out = qw.shape[0]
    n_mod = s.shape[0]
    r = 0 if L1 is None else int(L1.shape[-1])
    ld_l2 = 0 if L2 is None else int(L2.stride(-2))
    dbg = None
    qx = dx = None
    if taps:
        qx = torch.empty(T, d, dtype=torch.int8, device=X.device)
        dx = torch.empty(T, dtype=torch.float32, device=X.device)
    if acc_debug:
        out = torch.empty(T, d_out, dtype=torch.int32, device=X.device)
        dbg = MasqDebug(out.data_ptr(), out.stride(0), None if qx is None else qx.data_ptr(),
                        None if dx is None else dx.data_ptr())
        Yp, ldy = None, d_out
    else:
        out = torch.empty(T, d_out, dtype=torch.float32, device=X.device) if Y is None else Y
        Yp, ldy = _p(out), out.stride(0)
        if taps:
            dbg = MasqDebug(None, 0, qx.data_ptr(), dx.data_ptr())
    ws = ws or default_workspace(X.device)
    p, n = ws.ptr_size(workspace_size(OP_FORWARD, T, d, d_out, n_mod, r if not acc_debug else 0))
    _ck(lib().masq_linear_forward(_p(X), _dt(X), X.stride(0), _p(mod_id), T, d, d_out, n_mod,
                                  _p(s.contiguous()), _p(qw), _p(dw), wbits, abits, _p(L1), _p(L2), ld_l2, r,
                                  Yp, ldy, p, n, ctypes.byref(dbg) if dbg is not None else None,
                                  _stream(stream)), "masq_linear_forward")
    return (out, qx, dx) if taps else out


# ----------------------------------------------------------------------------- A8
def reference_output(X, W, Yref=None, ws=None, stream=None):
    T, d = X.shape
    d_out = W.shape[1]
    out = torch.empty(T, d_out, dtype=torch.float32, device=X.device) if Yref is None else Yref
    ws = ws or default_workspace(X.device)
    p, n = ws.ptr_size(workspace_size(OP_REFERENCE, T, d, d_out, 1))
    _ck(lib().masq_reference_output(_p(X), X.stride(0), _p(W.contiguous()), T, d, d_out, _p(out), out.stride(0),
                                    p, n, _stream(stream)), "masq_reference_output")
    return out


def _lambda_arr(lam, n_mod):
    if lam is None:
        return None
    arr = (ctypes.c_float * n_mod)(*[float(v) for v in lam])
    return arr


def calib_loss(X, mod_id, s, W, wbits: int, abits: int, Yref=None, lam=None, sums=None, counts=None, loss=None,
               ws=None, stream=None):
    """Per-modality sums of |Q(X_m S_m^-1) Q(S_m W) - X_m W|, counts and the weighted MAE loss
    (PAPER.md:62-70).  Returns device tensors (sums f64 [M], counts i64 [M], loss f64 [1]).
    Yref None: the library computes the target X W itself (workspace OP_LOSS | OP_SELF_REF)."""
    T, d = X.shape
    d_out = W.shape[1]
    n_mod = s.shape[0]
    dev = X.device
    sums = torch.empty(n_mod, dtype=torch.float64, device=dev) if sums is None else sums
    counts = torch.empty(n_mod, dtype=torch.int64, device=dev) if counts is None else counts
    loss = torch.empty(1, dtype=torch.float64, device=dev) if loss is None else loss
    ws = ws or default_workspace(dev)
    p, n = ws.ptr_size(workspace_size(OP_LOSS | (OP_SELF_REF if Yref is None else 0), T, d, d_out, n_mod))
    lam_arr = _lambda_arr(lam, n_mod)
    _ck(lib().masq_calib_loss(_p(X), _dt(X), X.stride(0), _p(mod_id), T, d, d_out, n_mod, _p(s.contiguous()),
                              _p(W.contiguous()), _dt(W), wbits, abits,
                              ctypes.cast(lam_arr, ctypes.c_void_p) if lam_arr is not None else None,
                              _p(Yref), 0 if Yref is None else Yref.stride(0), _p(sums), _p(counts), _p(loss), p, n, _stream(stream)),
        "masq_calib_loss")
    return sums, counts, loss


def calib_layer(X, mod_id, s, W, wbits: int, abits: int, L1=None, L2=None, lam=None, Y=None, Yref=None,
                qw_text=None, dw_text=None, sums=None, counts=None, loss=None, ws=None, stream=None):
    """One fused calibration pass of a linear: (Y, Yref, sums, counts, loss); bit-identical to
    quantize_weight(s[0]) + linear_forward + reference_output + calib_loss."""
    T, d = X.shape
    n = W.shape[1]
    n_mod = s.shape[0]
    dev = X.device
    r = 0 if L1 is None else int(L1.shape[-1])
    ld_l2 = 0 if L2 is None else int(L2.stride(-2))
    Y = torch.empty(T, n, dtype=torch.float32, device=dev) if Y is None else Y
    Yref = torch.empty(T, n, dtype=torch.float32, device=dev) if Yref is None else Yref
    sums = torch.empty(n_mod, dtype=torch.float64, device=dev) if sums is None else sums
    counts = torch.empty(n_mod, dtype=torch.int64, device=dev) if counts is None else counts
    loss = torch.empty(1, dtype=torch.float64, device=dev) if loss is None else loss
    ws = ws or default_workspace(dev)
    p, nb = ws.ptr_size(workspace_size(OP_LAYER, T, d, n, n_mod, r))
    lam_arr = _lambda_arr(lam, n_mod)
    _ck(lib().masq_calib_layer(_p(X), X.stride(0), _p(mod_id), T, d, n, n_mod, _p(s.contiguous()), _p(W.contiguous()),
                               wbits, abits, _p(L1), _p(L2), ld_l2, r,
                               ctypes.cast(lam_arr, ctypes.c_void_p) if lam_arr is not None else None,
                               _p(Y), Y.stride(0), _p(Yref), Yref.stride(0), _p(qw_text), _p(dw_text), _p(sums),
                               _p(counts), _p(loss), p, nb, _stream(stream)), "masq_calib_layer")
    return Y, Yref, sums, counts, loss


def calib_loss_grad(X, mod_id, s, W, wbits: int, abits: int, Yref=None, lam=None, grad=None, sums=None, counts=None,
                    loss=None, count_norm=None, ws=None, stream=None):
    """N1: (sums, counts, loss, grad) with grad = dL/d ln s (straight-through), f64 [M x d].

    count_norm: optional device i64 [M] token counts for the gradient's 1/N_m (the global
    counts when the tokens are sharded over ranks; then SUM-all-reduce grad)."""
    T, d = X.shape
    d_out = W.shape[1]
    n_mod = s.shape[0]
    dev = X.device
    sums = torch.empty(n_mod, dtype=torch.float64, device=dev) if sums is None else sums
    counts = torch.empty(n_mod, dtype=torch.int64, device=dev) if counts is None else counts
    loss = torch.empty(1, dtype=torch.float64, device=dev) if loss is None else loss
    grad = torch.empty(n_mod, d, dtype=torch.float64, device=dev) if grad is None else grad
    ws = ws or default_workspace(dev)
    p, n = ws.ptr_size(workspace_size(OP_LOSS_GRAD | (OP_SELF_REF if Yref is None else 0), T, d, d_out, n_mod))
    lam_arr = _lambda_arr(lam, n_mod)
    _ck(lib().masq_calib_loss_grad(_p(X), _dt(X), X.stride(0), _p(mod_id), T, d, d_out, n_mod, _p(s.contiguous()),
                                   _p(W.contiguous()), _dt(W), wbits, abits,
                                   ctypes.cast(lam_arr, ctypes.c_void_p) if lam_arr is not None else None,
                                   _p(Yref), 0 if Yref is None else Yref.stride(0), _p(sums), _p(counts),
                                   _p(loss), _p(grad),
                                   _p(count_norm), p, n, _stream(stream)), "masq_calib_loss_grad")
    return sums, counts, loss, grad


def adam_step(theta, grad, m1, m2, step: int, lr: float, beta1: float = 0.9, beta2: float = 0.999,
              eps: float = 1e-8, s_out=None, stream=None):
    """Log-space Adam on device (f64 state); writes s_out = exp(theta) (f32) when given."""
    _ck(lib().masq_adam_step(_p(theta), _p(grad), _p(m1), _p(m2), theta.numel(), step, lr, beta1, beta2, eps,
                             _p(s_out), _stream(stream)), "masq_adam_step")
    return theta


def adam_init(s, theta=None, m1=None, m2=None, stream=None):
    """(theta, m1, m2) = (ln s, 0, 0) as f64 device tensors shaped like s."""
    theta = torch.empty(s.shape, dtype=torch.float64, device=s.device) if theta is None else theta
    m1 = torch.empty_like(theta) if m1 is None else m1
    m2 = torch.empty_like(theta) if m2 is None else m2
    _ck(lib().masq_adam_init(_p(s.contiguous()), _p(theta), _p(m1), _p(m2), s.numel(), _stream(stream)),
        "masq_adam_init")
    return theta, m1, m2


def keep_best(loss, best_loss, s, s_best, improved=None, stream=None):
    """Best-so-far on the device: s_best <- s and best_loss <- loss when loss < best_loss."""
    _ck(lib().masq_keep_best(_p(loss), _p(best_loss), _p(s), _p(s_best), s.numel(), _p(improved),
                             _stream(stream)), "masq_keep_best")


# ----------------------------------------------------------------------------- N2
def cmc_factors(X, mod_id, s, W, qw_text, dw_text, r: int, eps_rel: float = 1e-8, dtype=torch.bfloat16,
                with_resid: bool = True, ws=None, stream=None):
    """(L1 [M-1, d, r], L2 [M-1, r, n], resid f64 [M-1] or None): whitened truncated-SVD CMC
    factors for every non-text modality."""
    T, d = X.shape
    n = W.shape[1]
    n_mod = s.shape[0]
    dev = X.device
    L1 = torch.empty(n_mod - 1, d, r, dtype=dtype, device=dev)
    L2 = torch.empty(n_mod - 1, r, n, dtype=dtype, device=dev)
    resid = torch.empty(n_mod - 1, dtype=torch.float64, device=dev) if with_resid else None
    ws = ws or default_workspace(dev)
    p, nb = ws.ptr_size(workspace_size(OP_CMC, T, d, n, n_mod, r))
    _ck(lib().masq_cmc_factors(_p(X), _dt(X), X.stride(0), _p(mod_id), T, d, n, n_mod, _p(s.contiguous()),
                               _p(W.contiguous()), _dt(W), _p(qw_text), _p(dw_text), r, float(eps_rel), _p(L1), _p(L2),
                               _dt(L1), _p(resid), p, nb, _stream(stream)), "masq_cmc_factors")
    return L1, L2, resid


# ----------------------------------------------------------------------------- N3
def quantize_weight_int4(W, s_vec, group: int = 128, stream=None):
    """(packed uint8 [n*d/2] in the decode kernel's order, scales f32 [n/8, d/group, 8])."""
    d, n = W.shape
    packed = torch.empty(n * d // 2, dtype=torch.uint8, device=W.device)
    scales = torch.empty(n // 8, d // group, 8, dtype=torch.float32, device=W.device)
    _ck(lib().masq_quantize_weight_int4(_p(W.contiguous()), _dt(W), _p(s_vec.contiguous()), d, n, group, _p(packed),
                                        _p(scales), _stream(stream)), "masq_quantize_weight_int4")
    return packed, scales


def unpack_int4(packed, d: int, n: int, group: int = 128, stream=None):
    codes = torch.empty(n, d, dtype=torch.int8, device=packed.device)
    _ck(lib().masq_unpack_int4(_p(packed), d, n, group, _p(codes), _stream(stream)), "masq_unpack_int4")
    return codes


def linear_decode(X, s_t, packed, scales, abits: int = 8, group: int = 128, Y=None, ws=None, stream=None):
    """Decode-shaped W4A8 forward of 1..16 text tokens: f32 [T x n]."""
    T, d = X.shape
    n = scales.shape[0] * 8
    Y = torch.empty(T, n, dtype=torch.float32, device=X.device) if Y is None else Y
    ws = ws or default_workspace(X.device)
    p, nb = ws.ptr_size(workspace_size(OP_DECODE, T, d, n, 1))
    _ck(lib().masq_linear_decode(_p(X), _dt(X), X.stride(0), T, d, n, _p(s_t.contiguous()), _p(packed), _p(scales),
                                 group, abits, _p(Y), Y.stride(0), p, nb, _stream(stream)), "masq_linear_decode")
    return Y


def quantize_weight_w4g(W, s_vec, group: int = 128, stream=None):
    """(packed uint8 [d/group, n, 64] in the prefill GEMM's group-major nibble order, scales f32
    [n, d/group])."""
    d, n = W.shape
    packed = torch.empty(d // group, n, 64, dtype=torch.uint8, device=W.device)
    scales = torch.empty(n, d // group, dtype=torch.float32, device=W.device)
    _ck(lib().masq_quantize_weight_w4g(_p(W.contiguous()), _dt(W), _p(s_vec.contiguous()), d, n, group, _p(packed),
                                       _p(scales), _stream(stream)), "masq_quantize_weight_w4g")
    return packed, scales


def linear_forward_w4g(X, mod_id, s, packed, scales, abits: int = 8, L1=None, L2=None, Y=None, group: int = 128,
                       acc_debug: bool = False, ws=None, stream=None):
    """Prefill W4A8 forward with packed int4 group-scaled weights (+ CMC): f32 [T x n]
    (acc_debug: the int32 sum over groups of the unscaled accumulators)."""
    T, d = X.shape
    n = scales.shape[0]
    n_mod = s.shape[0]
    r = 0 if L1 is None else int(L1.shape[-1])
    ld_l2 = 0 if L2 is None else int(L2.stride(-2))
    dbg = None
    if acc_debug:
        out = torch.empty(T, n, dtype=torch.int32, device=X.device)
        dbg = MasqDebug(out.data_ptr(), out.stride(0), None, None)
        Yp, ldy = None, n
    else:
        out = torch.empty(T, n, dtype=torch.float32, device=X.device) if Y is None else Y
        Yp, ldy = _p(out), out.stride(0)
    ws = ws or default_workspace(X.device)
    p, nb = ws.ptr_size(workspace_size(OP_FORWARD, T, d, n, n_mod, r if not acc_debug else 0))
    _ck(lib().masq_linear_forward_w4g(_p(X), _dt(X), X.stride(0), _p(mod_id), T, d, n, n_mod, _p(s.contiguous()),
                                      _p(packed), _p(scales), group, abits, _p(L1), _p(L2), ld_l2, r, Yp, ldy, p, nb,
                                      ctypes.byref(dbg) if dbg is not None else None, _stream(stream)),
        "masq_linear_forward_w4g")
    return out


def cmc_gram(X, mod_id, s, G=None, accumulate: bool = False, ws=None, stream=None):
    """G f64 [M-1, d, d] (lower triangle) += / = A_m^T A_m for the non-text modalities."""
    T, d = X.shape
    n_mod = s.shape[0]
    G = torch.zeros(n_mod - 1, d, d, dtype=torch.float64, device=X.device) if G is None else G
    ws = ws or default_workspace(X.device)
    p, nb = ws.ptr_size(workspace_size(OP_CMC_GRAM, T, d, 0, n_mod))
    _ck(lib().masq_cmc_gram(_p(X), _dt(X), X.stride(0), _p(mod_id), T, d, n_mod, _p(s.contiguous()), _p(G),
                            1 if accumulate else 0, p, nb, _stream(stream)), "masq_cmc_gram")
    return G


def cmc_factors_from_gram(G, s, W, qw_text, dw_text, r: int, eps_rel: float = 1e-8, dtype=torch.bfloat16,
                          with_resid: bool = True, ws=None, stream=None):
    """(L1, L2, resid) from the (all-reduced) Gram matrices."""
    d, n = W.shape
    n_mod = s.shape[0]
    dev = W.device
    L1 = torch.empty(n_mod - 1, d, r, dtype=dtype, device=dev)
    L2 = torch.empty(n_mod - 1, r, n, dtype=dtype, device=dev)
    resid = torch.empty(n_mod - 1, dtype=torch.float64, device=dev) if with_resid else None
    ws = ws or default_workspace(dev)
    p, nb = ws.ptr_size(workspace_size(OP_CMC_FACTORS, 0, d, n, n_mod, r))
    _ck(lib().masq_cmc_factors_from_gram(_p(G), d, n, n_mod, _p(s.contiguous()), _p(W.contiguous()), _dt(W),
                                         _p(qw_text), _p(dw_text), r, float(eps_rel), _p(L1), _p(L2), _dt(L1),
                                         _p(resid), p, nb, _stream(stream)), "masq_cmc_factors_from_gram")
    return L1, L2, resid


# ----------------------------------------------------------------------------- N4
def smooth_factors(num, beta: float, den=None, s=None, stream=None):
    """s = num^beta / den^(1-beta) (f64 pow, one f32 rounding); den None = AWQ form."""
    num = num.contiguous()
    d = num.shape[-1]
    rows = num.numel() // d if d else 0
    s = torch.empty_like(num) if s is None else s
    _ck(lib().masq_smooth_factors(_p(num), rows, d, _p(den.contiguous()) if den is not None else None, float(beta),
                                  _p(s), _stream(stream)), "masq_smooth_factors")
    return s


def calibrate_meanabs(X, mod_id, n_mod: int, sumabs=None, count=None, reset: bool = True, ws=None, stream=None):
    """(sumabs f64 [M x d], count i64 [M], mean f32 [M x d], mean_unified f32 [d])."""
    T, d = X.shape
    dev = X.device
    sumabs = torch.zeros(n_mod, d, dtype=torch.float64, device=dev) if sumabs is None else sumabs
    count = torch.zeros(n_mod, dtype=torch.int64, device=dev) if count is None else count
    mean = torch.empty(n_mod, d, dtype=torch.float32, device=dev)
    uni = torch.empty(d, dtype=torch.float32, device=dev)
    ws = ws or default_workspace(dev)
    p, n = ws.ptr_size(workspace_size(OP_MEANABS, T, d, 0, n_mod))
    _ck(lib().masq_calibrate_meanabs(_p(X), _dt(X), X.stride(0), _p(mod_id), T, d, n_mod, _p(sumabs), _p(count),
                                     _p(mean), _p(uni), 1 if reset else 0, p, n, _stream(stream)),
        "masq_calibrate_meanabs")
    return sumabs, count, mean, uni


def count_modalities(mod_id, n_mod: int, count=None, reset: bool = True, ws=None, stream=None):
    """i64 [M] token counts per modality (device)."""
    T = mod_id.shape[0]
    count = torch.zeros(n_mod, dtype=torch.int64, device=mod_id.device) if count is None else count
    ws = ws or default_workspace(mod_id.device)
    p, nb = ws.ptr_size(workspace_size(OP_STATS, T, 16, 0, n_mod))
    _ck(lib().masq_count_modalities(_p(mod_id), T, n_mod, _p(count), 1 if reset else 0, p, nb, _stream(stream)),
        "masq_count_modalities")
    return count


def range_stats(R, dominant: int = 0, other: int = 1, stream=None):
    """(alpha f32 [d] or None, r_unified f32 [d], dom_counts i64 [M + 1])."""
    n_mod, d = R.shape
    alpha = torch.empty(d, dtype=torch.float32, device=R.device) if n_mod > 1 else None
    runi = torch.empty(d, dtype=torch.float32, device=R.device)
    dom = torch.empty(n_mod + 1, dtype=torch.int64, device=R.device)
    _ck(lib().masq_range_stats(_p(R.contiguous()), n_mod, d, dominant, other, _p(alpha), _p(runi), _p(dom),
                               _stream(stream)), "masq_range_stats")
    return alpha, runi, dom


def loss_finalize(sums, counts, d_out: int, lam=None, loss=None, stream=None):
    n_mod = sums.shape[0]
    loss = torch.empty(1, dtype=torch.float64, device=sums.device) if loss is None else loss
    lam_arr = _lambda_arr(lam, n_mod)
    _ck(lib().masq_loss_finalize(_p(sums), _p(counts), ctypes.cast(lam_arr, ctypes.c_void_p) if lam_arr else None,
                                 n_mod, d_out, _p(loss), _stream(stream)), "masq_loss_finalize")
    return loss


def version() -> str:
    return lib().masq_version().decode()
