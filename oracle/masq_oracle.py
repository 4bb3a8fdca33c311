"""MASQuant hot-path ORACLE — plain, slow, obviously-correct CPU reference.

TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and bench.py's
cpu_baseline / `--impl reference` leg may import or execute anything under
oracle/.  The product path (paper_2603_04800_b200/) never imports it and shares
no code with it (no kernels, helpers, tables or constants).

Precision contract:
  * Integer-valued parts (ranges R, factors s, codes, scales Delta, integer
    accumulators) follow a FIXED float32 operation sequence (IEEE mul / div /
    sqrt, no fused multiply-add), so the GPU path must match them bit-exactly.
  * Float parts (dequantized outputs, the CMC term, the loss) are evaluated in
    float64 from the exact f32 / bf16 input values.

Every function cites the passage it follows.  Pins: tests/test_oracle_pins.py.
Parity pinned for every function below (no "parity unpinned" entries): the
closed forms, brute-force, invariance and identity checks listed in
DESIGN.md §"Oracle pins".
"""
from __future__ import annotations

import numpy as np

F32 = np.float32
F64 = np.float64
FLOOR = np.float32(1e-12)          # SPEC.md:131, 164, 292 (Delta and s floors), reading Q7


# --------------------------------------------------------------------------- inputs
def decode(a: np.ndarray) -> np.ndarray:
    """bf16 bit patterns (uint16) -> exact float32; float32 passes through."""
    a = np.asarray(a)
    if a.dtype == np.uint16:
        return (a.astype(np.uint32) << 16).view(np.float32)
    return a.astype(np.float32, copy=False)


def _check_ids(ids: np.ndarray, n_mod: int) -> np.ndarray:
    ids = np.asarray(ids).astype(np.int64)
    if ids.size and (ids.min() < 0 or ids.max() >= n_mod):
        raise ValueError("token tagged with unknown modality")
    return ids


# --------------------------------------------------------------------------- O1
def calibrate_stats(X, ids, n_mod: int, R=None, count=None):
    """O1 — per-modality per-channel range R^m_i = max_t |x^m_{t,i}| and token counts.

    PAPER.md:35 (§4.1 "we measure the activation range per channel"),
    SPEC.md:196-204, 274-277 (running max over stored batches).
    R / count, when given, are the running state (batch coherence).
    """
    X = decode(X)
    ids = _check_ids(ids, n_mod)
    T, d = X.shape
    R = np.zeros((n_mod, d), F32) if R is None else np.array(R, F32, copy=True)
    count = np.zeros(n_mod, np.int64) if count is None else np.array(count, np.int64, copy=True)
    for m in range(n_mod):
        rows = X[ids == m]
        if rows.shape[0]:
            R[m] = np.maximum(R[m], np.abs(rows).max(axis=0))
        count[m] += rows.shape[0]
    return R, count


# --------------------------------------------------------------------------- O2
def weight_absmax(W) -> np.ndarray:
    """max_j |w_{j,i}| for every input channel i (reading Q8: W is
    D_in x D_out, so this is the max over row i of W)."""
    return np.abs(decode(W)).max(axis=1).astype(F32)


def init_factors(R, count, W) -> np.ndarray:
    """O2 — s^m_i = sqrt( max_t|x^m_{t,i}| / max_j|w_{j,i}| )   (§4.2).

    f32 sequence: sqrt( div( max(R,1e-12f), max(wmax,1e-12f) ) ) (Q6/Q7).
    A modality with zero calibration tokens is rejected.
    """
    R = np.asarray(R, F32)
    if (np.asarray(count) == 0).any():
        raise ValueError("modality with zero calibration tokens")
    wmax = weight_absmax(W)
    num = np.maximum(R, FLOOR)
    den = np.maximum(wmax, FLOOR)[None, :]
    return np.sqrt(np.divide(num, den, dtype=F32), dtype=F32)


# --------------------------------------------------------------------------- Q
def rha(v: np.ndarray) -> np.ndarray:
    """Round half away from zero (reading Q5; "rounding-to-nearest").
    trunc(v) + sign(v)*[|v - trunc(v)| >= 0.5]; v - trunc(v) is exact in f32."""
    v = np.asarray(v, F32)
    t = np.trunc(v)
    frac = np.abs(v - t)
    return (t + np.where(frac >= F32(0.5), np.sign(v), F32(0))).astype(F32)


def quantize_rows(A, bits: int):
    """Symmetric per-row uniform quantizer, z = 0 (PAPER.md:241-245 Eq. PTQ; Q3, Q4).

    Delta = max( div(max_i |a_i|, q_max), 1e-12f ),  q = clamp(rha(div(a, Delta)), -2^{b-1}, 2^{b-1}-1)
    Returns (codes int8 [rows x cols], Delta f32 [rows]).
    """
    if not (2 <= bits <= 8):
        raise ValueError("bits must be in [2, 8] on this path")
    A = np.asarray(A, F32)
    qmax = F32(2 ** (bits - 1) - 1)
    qmin = F32(-(2 ** (bits - 1)))
    amax = np.abs(A).max(axis=1) if A.shape[1] else np.zeros(A.shape[0], F32)
    delta = np.maximum(np.divide(amax, qmax, dtype=F32), FLOOR)
    v = np.divide(A, delta[:, None], dtype=F32)
    codes = np.clip(rha(v), qmin, qmax).astype(np.int8)
    return codes, delta.astype(F32)


def dequantize_rows(codes, delta) -> np.ndarray:
    """Q(x) = code * Delta (PAPER.md:244 with z = 0), in f64."""
    return np.asarray(codes, F64) * np.asarray(delta, F64)[:, None]


# --------------------------------------------------------------------------- O3
def quantize_weight(W, s, wbits: int):
    """O3 — Q(S W) per OUTPUT channel (reading Q1), stored K-major: qw [n x d].

    ws[i,j] = f32 mul(s_i, W[i,j])  (S W, PAPER.md:129 / 180-183 with S_t; PAPER.md:69 with S_m)
    Delta_w[j] = max(div(max_i |ws[i,j]|, q_w), 1e-12f); codes = clamp(rha(div(ws, Delta_w[j]))).
    """
    Wf = decode(W)
    s = np.asarray(s, F32)
    ws = np.multiply(s[:, None], Wf, dtype=F32)          # [d x n]
    return quantize_rows(np.ascontiguousarray(ws.T), wbits)   # rows = output channels


# --------------------------------------------------------------------------- O4
def smooth_activations(X, ids, s) -> np.ndarray:
    """X_m S_m^{-1} row by row: xs[t,i] = f32 mul(x[t,i], f32 div(1, s[m_t, i]))
    (reading Q6: S^{-1} applied as multiplication by the f32 reciprocal)."""
    Xf = decode(X)
    s = np.asarray(s, F32)
    ids = _check_ids(ids, s.shape[0])
    inv = np.divide(F32(1.0), s, dtype=F32)
    return np.multiply(Xf, inv[ids], dtype=F32)


def quantize_activations(X, ids, s, abits: int):
    """O4 — Q(X_m S_m^{-1}) per token, dynamic symmetric (PAPER.md:76 per-token Delta_t; Q2).
    Returns (qx int8 [T x d], Delta_x f32 [T])."""
    return quantize_rows(smooth_activations(X, ids, s), abits)


# --------------------------------------------------------------------------- O5 / O6
def int_gemm(qx, qw) -> np.ndarray:
    """O5 — acc[t,j] = sum_i qx[t,i] * qw[j,i], exact (every partial sum < 2^53, so f64 BLAS
    on integer-valued matrices is exact; pinned against an int64 triple loop)."""
    acc = np.asarray(qx, F64) @ np.asarray(qw, F64).T
    return acc.astype(np.int64)


def dequant_output(acc, dx, dw) -> np.ndarray:
    """O6 — Q(X S^-1) . Q(S W) = acc * Delta_x[t] * Delta_w[j], in f64."""
    return np.asarray(acc, F64) * np.asarray(dx, F64)[:, None] * np.asarray(dw, F64)[None, :]


# --------------------------------------------------------------------------- O7
def _values_f64(a) -> np.ndarray:
    """bf16 bits -> exact values; any float array kept at its own precision (as f64)."""
    a = np.asarray(a)
    return np.asarray(decode(a) if a.dtype == np.uint16 else a, F64)


def cmc_term(xs_rows, L1m, L2m) -> np.ndarray:
    """X_m S_m^{-1} . L1^m L2^m in f64 (full precision)."""
    return (np.asarray(xs_rows, F64) @ _values_f64(L1m)) @ _values_f64(L2m)


def linear_forward(X, ids, s, qw, dw, abits: int, L1=None, L2=None, rows=None) -> np.ndarray:
    """O4-O7 — the routed inference equation:

        Y_t = Q(x_t S_{m}^{-1}) . Q(S_t W)                              m = text (id 0)
        Y_t = Q(x_t S_{m}^{-1}) . Q(S_t W) + x_t S_m^{-1} . L1^m L2^m    m != text

    qw/dw are Q(S_text W) (output of quantize_weight with s[0]).  L1[m-1], L2[m-1] are the
    correction factors of modality m (bf16 bits or any float array); None => rank 0.
    rows: optional subset of token indices (per-token quantization is row-local).
    Output f64 [len(rows) x n] in the given token order.
    """
    Xf = decode(X)
    ids = _check_ids(ids, np.asarray(s).shape[0])
    if rows is not None:
        rows = np.asarray(rows, np.int64)
        Xf, ids = Xf[rows], ids[rows]
    xs = smooth_activations(Xf, ids, s)
    qx, dx = quantize_rows(xs, abits)
    Y = dequant_output(int_gemm(qx, qw), dx, dw)
    if L1 is not None and L2 is not None:
        for m in range(1, np.asarray(s).shape[0]):
            sel = np.nonzero(ids == m)[0]
            if sel.size:
                Y[sel] += cmc_term(xs[sel], L1[m - 1], L2[m - 1])
    return Y


# --------------------------------------------------------------------------- O8
def reference_output(X, W, rows=None) -> np.ndarray:
    """X W in f64 from the exact inputs ("X_m W"; reading Q16)."""
    Xf = decode(X)
    if rows is not None:
        Xf = Xf[np.asarray(rows, np.int64)]
    return np.asarray(Xf, F64) @ np.asarray(decode(W), F64)


def calib_loss(X, ids, s, W, wbits: int, abits: int, lam=None, rows=None, Yref=None):
    """O8 — per-modality sums of |Q(X_m S_m^-1) . Q(S_m W) - X_m W| (Eq. mas_quant),
    counts, and L = sum_m lambda_m * MAE_m with MAE_m = sum_m / (count_m * n) (reading Q9;
    lambda default 1.0).  Each modality uses its OWN weight Q(S_m W) (Q12).
    Modalities with zero tokens contribute 0.  Returns (sums f64 [M], counts i64 [M], loss f64).
    """
    s = np.asarray(s, F32)
    n_mod = s.shape[0]
    Xf = decode(X)
    ids = _check_ids(ids, n_mod)
    if rows is not None:
        rows = np.asarray(rows, np.int64)
        Xf, ids = Xf[rows], ids[rows]
    lam = np.ones(n_mod) if lam is None else np.asarray(lam, F64)
    Yr = reference_output(Xf, W) if Yref is None else np.asarray(Yref, F64)
    n = Yr.shape[1]
    qx, dx = quantize_activations(Xf, ids, s, abits)
    sums = np.zeros(n_mod, F64)
    counts = np.zeros(n_mod, np.int64)
    for m in range(n_mod):
        sel = np.nonzero(ids == m)[0]
        counts[m] = sel.size
        if not sel.size:
            continue
        qw, dw = quantize_weight(W, s[m], wbits)
        yq = dequant_output(int_gemm(qx[sel], qw), dx[sel], dw)
        sums[m] = np.abs(yq - Yr[sel]).sum()
    loss = loss_finalize(sums, counts, lam, n)
    return sums, counts, loss


def loss_finalize(sums, counts, lam, n: int) -> float:
    """L = sum_m lambda_m * sums_m / (counts_m * n) over modalities with tokens."""
    loss = 0.0
    for m in range(len(sums)):
        if counts[m] > 0:
            loss += float(lam[m]) * float(sums[m]) / (float(counts[m]) * n)
    return loss


# --------------------------------------------------------------------------- N1 (next row)
def _first_argmax_abs(A, axis: int):
    """Index of the first maximum of |A| along axis (np.argmax returns the first occurrence)."""
    return np.argmax(np.abs(A), axis=axis)


def calib_loss_grad(X, ids, s, W, wbits: int, abits: int, lam=None, count_norm=None):
    """N1 — gradient of L = sum_m lambda_m MAE_m (O8) w.r.t. theta^m = ln s^m (SPEC.md:307-316:
    log-space parameters; "gradient of the rounding operator treated as identity inside the
    clamp range and zero outside" — reading Q24: ONLY round() is straight-through; the dynamic
    scales Delta = max|.|/q_max stay functions of their inputs, so they are differentiated
    through their (first) arg-max element; the clamp is never active for absmax scales, and a
    floored Delta (1e-12f) has zero derivative).

    Per modality, with A = X_m S_m^-1 (xs), B = S_m W, Ahat = Q(A) = A + D, Bhat = Q(B),
    E = Ahat Bhat - X_m W and G = lambda_m / (N_m n) sign(E):
      Ahat_ti = Delta_t code_ti  with  d Ahat = dA + (code - A/Delta) dDelta_t  (round: identity)
      dA_ti/dtheta_l = -A_ti [i = l];  dDelta_t/dtheta_l = -Delta_t [l = k_t],  k_t = argmax_i |A_ti|
      dB_ij/dtheta_l =  B_ij [i = l];  dDelta_j/dtheta_l =  Delta_j [l = k_j],  k_j = argmax_i |B_ij|
    hence
      grad_l = sum_j (Ahat^T G)_lj B_lj - sum_j (A^T G)_lj Bhat_lj
             + sum_{j: k_j = l} beta_j - sum_{t: k_t = l} alpha_t,
      beta_j  = sum_i (Ahat^T G)_ij (Bhat - B)_ij,   alpha_t = sum_i (G Bhat^T)_ti (Ahat - A)_ti.
    count_norm: the N_m of the gradient's scale (default: this call's token counts) — a token
    shard passes the whole batch's counts, and the shards' gradients then add up to the batch
    gradient.  The returned loss always uses this call's own counts.
    Returns (loss f64, grad f64 [M x d]).
    """
    s = np.asarray(s, F32)
    n_mod = s.shape[0]
    Xf = decode(X)
    Wf = decode(W)
    ids = _check_ids(ids, n_mod)
    lam = np.ones(n_mod) if lam is None else np.asarray(lam, F64)
    n = Wf.shape[1]
    qa, qw_max = F32(2 ** (abits - 1) - 1), F32(2 ** (wbits - 1) - 1)
    xs_all = smooth_activations(Xf, ids, s)
    grad = np.zeros((n_mod, Wf.shape[0]), F64)
    loss = 0.0
    for m in range(n_mod):
        sel = np.nonzero(ids == m)[0]
        if not sel.size:
            continue
        xs = xs_all[sel]
        qx, dx = quantize_rows(xs, abits)
        Ahat = dequantize_rows(qx, dx)                                   # [T_m x d]
        qw, dw = quantize_weight(W, s[m], wbits)
        Bhat = dequantize_rows(qw, dw).T                                 # [d x n]
        Bs32 = np.multiply(s[m][:, None], Wf, dtype=F32)                 # S_m W as quantized (f32)
        Bs, A = Bs32.astype(F64), np.asarray(xs, F64)
        E = Ahat @ Bhat - np.asarray(Xf[sel], F64) @ np.asarray(Wf, F64)
        loss += float(lam[m]) / (sel.size * n) * np.abs(E).sum()
        G = float(lam[m]) / ((sel.size if count_norm is None else int(count_norm[m])) * n) * np.sign(E)
        GB = Ahat.T @ G                                                  # dL/dBhat  [d x n]
        g = (GB * Bs).sum(axis=1) - ((A.T @ G) * Bhat).sum(axis=1)
        # scale terms: weight columns (Delta_j not floored) and token rows (Delta_t not floored)
        beta = (GB * (Bhat - Bs)).sum(axis=0)                            # [n]
        live_j = np.divide(np.abs(Bs32).max(axis=0), qw_max, dtype=F32) >= FLOOR
        np.add.at(g, _first_argmax_abs(Bs32, 0)[live_j], beta[live_j])
        alpha = ((G @ Bhat.T) * (Ahat - A)).sum(axis=1)                  # [T_m]
        live_t = np.divide(np.abs(xs).max(axis=1), qa, dtype=F32) >= FLOOR
        np.add.at(g, _first_argmax_abs(xs, 1)[live_t], -alpha[live_t])
        grad[m] = g
    return loss, grad


def optimize_factors(X, ids, s0, W, wbits: int, abits: int, epochs: int = 2, batch_tokens: int = 1024,
                     lr: float = 1e-2, lam=None, max_rejections: int = 10):
    """N1 driver — SPEC.md:307-316 optimize_factors, step by step: theta = ln s0; per epoch one
    pass over the calibration batches (contiguous slices of batch_tokens tokens), each an Adam
    step (step 1e-2) on that batch's straight-through gradient; a non-finite loss
    or gradient rejects the step and halves the step size, 10 consecutive rejections end the
    run; after each epoch the objective over the whole set is evaluated and the best-so-far
    iterate kept (so the result never has a higher objective than s0).  Batch slices are views
    of the calibration set in token order (reading Q25: a batch is batch_tokens consecutive
    tokens; the default 1024 is one synthetic sample).
    Returns (s_best f32 [M x d], best objective, [objective after each epoch]).
    """
    s0 = np.asarray(s0, F32)
    T = np.asarray(ids).shape[0]
    objective = lambda s: calib_loss(X, ids, s, W, wbits, abits, lam=lam)[2]
    best, s_best = objective(s0), s0.copy()
    theta, m1, m2 = np.log(s0.astype(F64)), np.zeros(s0.shape), np.zeros(s0.shape)
    s, t, rejections, history = s0.copy(), 0, 0, []
    for _ in range(epochs):
        for a in range(0, T, batch_tokens):
            b = min(T, a + batch_tokens)
            loss, g = calib_loss_grad(X[a:b], ids[a:b], s, W, wbits, abits, lam=lam)
            if not np.isfinite(loss):                 # non-finite loss -> reject
                lr, rejections = lr * 0.5, rejections + 1
                if rejections >= max_rejections:
                    return s_best, best, history
                continue
            rejections, t = 0, t + 1
            theta, m1, m2 = adam_step(theta, g, m1, m2, t, lr)
            s = np.exp(theta).astype(F32)
        L = objective(s)
        history.append(L)
        if np.isfinite(L) and L < best:
            best, s_best = L, s.copy()
    return s_best, best, history


def adam_step(theta, grad, m1, m2, step: int, lr: float, b1: float = 0.9, b2: float = 0.999, eps: float = 1e-8):
    """Adam in log space (SPEC.md:334 adaptive-moment choice), f64: returns (theta, m1, m2);
    s = exp(theta).  step counts from 1."""
    m1 = b1 * np.asarray(m1, F64) + (1 - b1) * grad
    m2 = b2 * np.asarray(m2, F64) + (1 - b2) * grad * grad
    mh = m1 / (1 - b1 ** step)
    vh = m2 / (1 - b2 ** step)
    return np.asarray(theta, F64) - lr * mh / (np.sqrt(vh) + eps), m1, m2


# --------------------------------------------------------------------------- N4 baselines
def smooth_factors(num, den, beta: float) -> np.ndarray:
    """N4 — the beta-parameterised closed forms the paper compares against (PAPER.md:19-23
    SmoothQuant s_i = R_i^beta / wmax_i^(1-beta); PAPER.md:24-28 AWQ s_i = mean_i^beta with
    den = None; PAPER.md:36-39 unified factors = num taken over all modalities).  num, den are
    floored at 1e-12 (Q7); evaluated in f64 and rounded once to f32 (reading Q26).
    num: [.. x d]; den: [d] or None.  Returns f32 like num."""
    n = np.maximum(np.asarray(num, F32), FLOOR).astype(F64)
    r = n ** F64(beta)
    if den is not None:
        dd = np.maximum(np.asarray(den, F32), FLOOR).astype(F64)
        r = r / dd ** (F64(1.0) - F64(beta))
    return r.astype(F32)


def unified_stats(R) -> np.ndarray:
    """max_m R^m_i — the range a single unified factor is computed from."""
    return np.asarray(R, F32).max(axis=0)


def meanabs_stats(X, ids, n_mod: int):
    """AWQ's activation statistic per modality: sum_t |x^m_t,i| (f64, exact
    summation order irrelevant at f64 for the tested sizes) and token counts."""
    Xf = np.abs(decode(X).astype(F64))
    ids = _check_ids(ids, n_mod)
    S = np.zeros((n_mod, Xf.shape[1]), F64)
    cnt = np.zeros(n_mod, np.int64)
    for m in range(n_mod):
        sel = ids == m
        S[m] = Xf[sel].sum(axis=0)
        cnt[m] = int(sel.sum())
    return S, cnt


def range_ratio(R, dominant: int, other: int) -> np.ndarray:
    """alpha^{m,m'}_i = R^m_i / R^{m'}_i, R^{m'} floored at 1e-12 (Theorem 1;
    SPEC.md:317-320), f32 division."""
    R = np.asarray(R, F32)
    return np.divide(R[dominant], np.maximum(R[other], FLOOR), dtype=F32)


def dominance_stats(R):
    """Per modality, the number of channels whose max_m R^m_i it attains (PAPER.md:410,
    fig:modality_dominance): ties go to the first such modality and are also
    counted in a separate bucket.  Returns int64 [M + 1] (last entry = tied channels)."""
    R = np.asarray(R, F32)
    M, d = R.shape
    out = np.zeros(M + 1, np.int64)
    for i in range(d):
        col = R[:, i]
        top = col.max()
        winners = [m for m in range(M) if col[m] == top]
        out[winners[0]] += 1
        if len(winners) > 1:
            out[M] += 1
    return out


def awq_grid_search(X, ids, W, wbits: int, abits: int, betas, n_mod: int, lam=None):
    """AWQ-style search: unified s(beta) = (mean_t |x_t,i|)^beta over all
    tokens, beta* = argmin_beta of the loss (O8) — each point scored by calib_loss with the same
    s for every modality.  Returns (beta*, [loss(beta)])."""
    S, cnt = meanabs_stats(X, ids, n_mod)
    mean = (S.sum(axis=0) / cnt.sum()).astype(F32)
    losses = []
    for b in betas:
        s = smooth_factors(mean, None, b)
        losses.append(calib_loss(X, ids, np.repeat(s[None, :], n_mod, axis=0), W, wbits, abits, lam=lam)[2])
    return float(betas[int(np.argmin(losses))]), losses


# --------------------------------------------------------------------------- N2 CMC factors
def weight_residual(W, s_m, qw_t, dw_t) -> np.ndarray:
    """Delta W = S_m W - Q(S_t W), f64 of the exact values:
    s_m (f32) x w (bf16) is exact in f64, Q(S_t W) = dw_j * code_ji (qw_t is K-major [n x d])."""
    Wf = decode(W).astype(F64)
    return np.asarray(s_m, F32).astype(F64)[:, None] * Wf - dequantize_rows(qw_t, dw_t).T


def whitening_transform(A, eps_rel: float = 1e-8):
    """SVD(A^T A) = P Lambda P^T, T = (P Lambda^1/2)^T, with Lambda + eps I
    before the square roots, eps = eps_rel * lambda_max (reading Q27).
    A = X_m S_m^-1 (f64 of the f32 smoothed activations).  Returns (T, T^-1, lambda)."""
    A = np.asarray(A, F64)
    return whitening_from_gram(A.T @ A, eps_rel)


def whitening_from_gram(G, eps_rel: float = 1e-8):
    """The same transform from the Gram matrix G = A^T A (token-sharded runs SUM their shards'
    Grams)."""
    lam, P = np.linalg.eigh(np.asarray(G, F64))
    lam = np.maximum(lam, 0.0)
    lam_r = lam + eps_rel * lam.max()
    T = (P * np.sqrt(lam_r)[None, :]).T
    T_inv = P / np.sqrt(lam_r)[None, :]
    return T, T_inv, lam


def cmc_factors(A, dW, r: int, eps_rel: float = 1e-8):
    """PAPER.md:143-149 (eq:l1l2): SVD(T dW) = U Sigma V^T ~ U_r Sigma_r V_r^T,
    L1 = T^-1 U_r [d x r], L2 = Sigma_r V_r^T [r x n]; r = 0 -> empty factors."""
    A = np.asarray(A, F64)
    return cmc_factors_from_gram(A.T @ A, dW, r, eps_rel)


def cmc_factors_from_gram(G, dW, r: int, eps_rel: float = 1e-8):
    """cmc_factors with the activations entering only through G = A^T A."""
    T, T_inv, _ = whitening_from_gram(G, eps_rel)
    d, n = dW.shape
    if r == 0:
        return np.zeros((d, 0)), np.zeros((0, n))
    U, sig, Vt = np.linalg.svd(T @ dW, full_matrices=False)
    return T_inv @ U[:, :r], sig[:r, None] * Vt[:r]


def cmc_factors_small_side(A, dW, r: int, eps_rel: float = 1e-8):
    """The eq:l1l2 optimum evaluated from the n x n side, for d > n (the c3 down
    projection, d = 18944: the paper's d x d eigensolve is out of reach for a CPU oracle there).
    With T^T T = A^T A + eps lambda_max I (PAPER.md:139-142 and reading Q27), the squared singular
    values and right singular vectors of M = T dW are the eigenpairs of
        M^T M = dW^T T^T T dW = (A dW)^T (A dW) + eps lambda_max dW^T dW        (n x n),
    and L2 = Sigma_r V_r^T, L1 = T^-1 U_r = T^-1 M V_r Sigma_r^-1 = dW V_r Sigma_r^-1.
    lambda_max = the largest eigenvalue of A^T A (= that of A A^T, the smaller Gram is used).
    Pinned against cmc_factors (the paper's route) in tests/test_oracle_pins.py."""
    A = np.asarray(A, F64)
    dW = np.asarray(dW, F64)
    n = dW.shape[1]
    if r == 0:
        return np.zeros((dW.shape[0], 0)), np.zeros((0, n))
    small = A @ A.T if A.shape[0] < A.shape[1] else A.T @ A
    lam_max = max(float(np.linalg.eigvalsh(small).max()), 0.0)
    AdW = A @ dW
    C = AdW.T @ AdW + eps_rel * lam_max * (dW.T @ dW)
    sig2, V = np.linalg.eigh(C)                           # ascending
    sig = np.sqrt(np.maximum(sig2[::-1][:r], 0.0))
    Vr = V[:, ::-1][:, :r]
    L2 = sig[:, None] * Vr.T
    L1 = (dW @ Vr) * np.where(sig > 0, 1.0 / np.where(sig > 0, sig, 1.0), 0.0)[None, :]
    return L1, L2


def reconstruction_loss(A, dW, L1, L2) -> float:
    """Theorem 2 objective ||A (dW - L1 L2)||_F^2 in f64."""
    A = np.asarray(A, F64)
    return float(np.sum((A @ (dW - L1 @ L2)) ** 2))


def reconstruction_loss_from_gram(G, dW, L1, L2) -> float:
    """The same objective as <E, G E> with E = dW - L1 L2 (no T x n product)."""
    E = dW - L1 @ L2
    return float(np.sum(E * (np.asarray(G, F64) @ E)))


def naive_svd_factors(dW, r: int):
    """Plain truncated SVD of dW without whitening ("directly applying SVD fails")."""
    U, sig, Vt = np.linalg.svd(dW, full_matrices=False)
    return U[:, :r] * sig[None, :r], Vt[:r]


def effective_rank(M) -> float:
    """exp(-sum p_i ln p_i), p_i = sigma_i / sum sigma (fig:effective_rank)."""
    sig = np.linalg.svd(np.asarray(M, F64), compute_uv=False)
    p = sig / sig.sum()
    p = p[p > 0]
    return float(np.exp(-(p * np.log(p)).sum()))


def cmc_layer_factors(X, ids, s, W, wbits: int, r: int, eps_rel: float = 1e-8):
    """N2 end to end for one linear: for every non-text modality m present, A_m = X_m S_m^-1
    (f32 as the path computes it), dW_m = S_m W - Q(S_t W) with the text-smoothed base weight
    (PAPER.md:128-131), and (L1^m, L2^m) = cmc_factors(A_m, dW_m, r).
    Returns lists over m = 1..M-1 (None for an absent modality) and the residual losses."""
    s = np.asarray(s, F32)
    n_mod = s.shape[0]
    ids = _check_ids(ids, n_mod)
    xs = smooth_activations(decode(X), ids, s)
    qw_t, dw_t = quantize_weight(W, s[0], wbits)
    L1s, L2s, losses = [], [], []
    for m in range(1, n_mod):
        sel = ids == m
        if not sel.any():
            L1s.append(None), L2s.append(None), losses.append(None)
            continue
        A = xs[sel].astype(F64)
        dW = weight_residual(W, s[m], qw_t, dw_t)
        L1, L2 = cmc_factors(A, dW, r, eps_rel)
        L1s.append(L1), L2s.append(L2), losses.append(reconstruction_loss(A, dW, L1, L2))
    return L1s, L2s, losses


# --------------------------------------------------------------------------- N3 int4 groups
def quantize_weight_grouped(W, s, wbits: int, group: int):
    """N3 — Q(S W) with sub-channel groups: per output channel j and group g of `group`
    consecutive input channels, Delta_jg = max(div(max_{i in g} |ws_ij|, q_max), 1e-12f) and
    codes = clamp(rha(div(ws, Delta_jg))) — the O3 quantizer at group
    granularity (reading Q28: SURVEY §8(f) N3's g = 128).  d % group == 0.
    Returns (codes int8 [n x d] K-major, Delta f32 [n x d/group])."""
    Wf = decode(W)
    s = np.asarray(s, F32)
    d, n = Wf.shape
    if d % group:
        raise ValueError("d must be a multiple of the group size")
    ws = np.multiply(s[:, None], Wf, dtype=F32).T                 # [n x d]
    codes, delta = quantize_rows(np.ascontiguousarray(ws.reshape(n * (d // group), group)), wbits)
    return codes.reshape(n, d), delta.reshape(n, d // group)


def pack_int4(codes) -> np.ndarray:
    """Two's-complement nibbles, two per byte along K: byte k holds code 2k in the low nibble and
    code 2k+1 in the high nibble (reading Q28).  codes in [-8, 7], [n x d] -> uint8 [n x d/2]."""
    c = np.asarray(codes, np.int16) & 0xF
    return (c[:, 0::2] | (c[:, 1::2] << 4)).astype(np.uint8)


def unpack_int4(packed) -> np.ndarray:
    """Inverse of pack_int4 (sign-extends every nibble)."""
    p = np.asarray(packed, np.uint8).astype(np.int16)
    lo, hi = p & 0xF, p >> 4
    lo = np.where(lo >= 8, lo - 16, lo)
    hi = np.where(hi >= 8, hi - 16, hi)
    out = np.empty((p.shape[0], 2 * p.shape[1]), np.int8)
    out[:, 0::2], out[:, 1::2] = lo, hi
    return out


def linear_decode(X, s_t, codes, delta, abits: int, group: int) -> np.ndarray:
    """N3 decode-shaped forward for text tokens (the base modality; decoding is
    CMC-free): Y = Q(X S_t^-1) . Q_g(S_t W) with per-token activation scales and per-(channel,
    group) weight scales, f64 of the dequantized values.  Returns f64 [T x n]."""
    Xf = decode(X)
    inv = np.divide(F32(1.0), np.asarray(s_t, F32), dtype=F32)
    xs = np.multiply(Xf, inv[None, :], dtype=F32)
    qx, dx = quantize_rows(xs, abits)
    n, d = codes.shape
    What = (np.asarray(codes, F64).reshape(n, d // group, group) * np.asarray(delta, F64)[:, :, None]).reshape(n, d)
    return dequantize_rows(qx, dx) @ What.T


def linear_forward_grouped(X, ids, s, codes, delta, abits: int, group: int, L1=None, L2=None, rows=None):
    """N3 prefill — the routed forward of PAPER.md:177-185 with the group-quantized base weight
    Q_g(S_t W) (codes int [n x d] K-major, delta [n x d/group] from quantize_weight_grouped with s[0];
    reading Q28) for ANY token count and every modality:
        Y_t = Q(x_t S_m^-1) . Q_g(S_t W)                                 m = text
        Y_t = Q(x_t S_m^-1) . Q_g(S_t W) + x_t S_m^-1 . L1^m L2^m         m != text
    f64 of the dequantized values (per-token activation scales, per-(channel, group) weight
    scales).  rows: optional token subset.  With all tokens text and no CMC it is linear_decode;
    with group = d it is linear_forward with the O3 weight (pinned in tests/test_oracle_pins.py).
    Returns f64 [len(rows) x n]."""
    Xf = decode(X)
    ids = _check_ids(ids, np.asarray(s).shape[0])
    if rows is not None:
        rows = np.asarray(rows, np.int64)
        Xf, ids = Xf[rows], ids[rows]
    xs = smooth_activations(Xf, ids, s)
    qx, dx = quantize_rows(xs, abits)
    n, d = np.asarray(codes).shape
    What = (np.asarray(codes, F64).reshape(n, d // group, group) * np.asarray(delta, F64)[:, :, None]).reshape(n, d)
    Y = dequantize_rows(qx, dx) @ What.T
    if L1 is not None and L2 is not None:
        for m in range(1, np.asarray(s).shape[0]):
            sel = np.nonzero(ids == m)[0]
            if sel.size:
                Y[sel] += cmc_term(xs[sel], L1[m - 1], L2[m - 1])
    return Y

