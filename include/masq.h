/*
 * masq.h — C ABI of the B200-native MASQuant hot path (arXiv 2603.04800).
 *
 * The library implements the data-parallel hot path of MASQuant's
 * modality-aware smoothed quantized linear layer on sm_100a:
 *
 *   A1  masq_calibrate_stats   R^m_i = max_t |x^m_{t,i}|                  PAPER.md:35  (§4.1)
 *   A2  masq_init_factors      s^m_i = sqrt(R^m_i / max_j |w_{j,i}|)       PAPER.md:55-58 (§4.2)
 *   A3  masq_quantize_weight   Q(S W), per output channel                  PAPER.md:129, 244 (Eq. PTQ)
 *   A4  masq_quantize_activations  Q(X_m S_m^{-1}), per token
 *   A4-A7 masq_linear_forward  Y = Q(X_m S_m^-1) Q(S_t W) [+ X_m S_m^-1 L1^m L2^m if m != text]
 *                                                                          PAPER.md:177-185
 *   A8  masq_calib_loss        sum_m lambda_m MAE(Q(X_m S_m^-1) Q(S_m W), X_m W)
 *                                                                          PAPER.md:62-70
 *       masq_reference_output  X W (f32), the loss target, computed once per batch
 *   A3-A8 masq_calib_layer     one fused calibration pass of a linear (what bench.py runs)
 *
 * and the SURVEY §8(f) "next" rows on the same data:
 *   N1  masq_calib_loss_grad, masq_adam_init / masq_adam_step, masq_keep_best,
 *       masq_count_modalities                 S-optimisation (straight-through gradient, Adam)
 *   N2  masq_cmc_factors (= masq_cmc_gram + masq_cmc_factors_from_gram)
 *                                             whitened truncated-SVD CMC factors (Theorem 2)
 *   N3  masq_quantize_weight_int4, masq_unpack_int4, masq_linear_decode
 *                                             int4 weights in 128-channel groups, decode path
 *       masq_quantize_weight_w4g, masq_linear_forward_w4g
 *                                             the same weights packed for the prefill tcgen05 GEMM
 *   N4  masq_smooth_factors, masq_calibrate_meanabs, masq_range_stats
 *                                             SmoothQuant / unified / AWQ baselines, dominance
 *
 * Conventions (apply to every entry point unless stated):
 *  - Shapes follow the paper's problem statement: X is [T x d]
 *    row-major (token rows), W is [d x d_out] row-major (D_in x D_out), one
 *    modality id per token (uint8, 0 = text = the base modality, PAPER.md:129,
 *    561), n_mod = |M| in [1, 8].
 *  - Every array pointer is a DEVICE pointer owned by the caller, except
 *    `lambda` (host).  The library allocates nothing and keeps no global
 *    state (except the opt-in profiler below); scratch comes from the caller's workspace `ws` (size from
 *    masq_workspace_size, 256-byte aligned).  Calls on the same ws must be
 *    stream-ordered; concurrent calls need distinct ws.
 *  - Every call is asynchronous on `stream` (a cudaStream_t; NULL = legacy
 *    default stream).  Argument errors (NULL, shape, bits, alignment,
 *    workspace) are returned synchronously and nothing is launched.  Data
 *    errors found on the device (a modality id >= n_mod, a modality with no
 *    calibration tokens) set a sticky status word inside ws; masq_check()
 *    synchronizes the stream and returns/clears it.  CUDA launch errors ->
 *    MASQ_ERR_CUDA.  Nothing throws across the ABI.
 *  - Kernels are launched with programmatic stream serialization: a kernel
 *    may become resident while the previous kernel on the stream drains, but
 *    touches no global memory before that kernel has completed, so stream
 *    order holds for every buffer (the caller's and ws).  Environment
 *    MASQ_PDL=0 (read once per process) launches with plain serialization;
 *    results are byte-identical either way.  A kernel the caller launches
 *    right after a call WITH programmatic stream serialization must execute
 *    griddepcontrol.wait (cudaGridDependencySynchronize) before reading the
 *    call's outputs, as for any programmatic dependent.
 *  - Limits: d % 16 == 0, d_out % 32 == 0, T >= 0 (T == 0 is a no-op),
 *    bits in [2, 8] (A16 / W16 -> MASQ_ERR_UNSUPPORTED), r % 16 == 0 and
 *    r <= 256 (r == 0 disables CMC), all pointers 16-byte aligned.
 *  - Quantizer (readings Q1-Q7 in DESIGN.md): symmetric,
 *    z = 0, Delta = max(absmax / (2^{b-1}-1), 1e-12f), codes =
 *    clamp(round-half-away(x / Delta), -2^{b-1}, 2^{b-1}-1), all in IEEE f32
 *    with the operation order documented per call; integer codes and f32
 *    scales are bit-exact against the CPU oracle.
 */
#ifndef MASQ_H
#define MASQ_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef enum masq_status {
  MASQ_OK = 0,
  MASQ_ERR_NULL = 1,            /* a required pointer is NULL */
  MASQ_ERR_SHAPE = 2,           /* a dimension violates the limits above */
  MASQ_ERR_BITS = 3,            /* bit-width outside [2, 16] */
  MASQ_ERR_ALIGN = 4,           /* a pointer or leading dimension is misaligned */
  MASQ_ERR_WORKSPACE = 5,       /* ws NULL or ws_bytes < masq_workspace_size(...) */
  MASQ_ERR_BAD_MODALITY = 6,    /* (sticky) a token id >= n_mod */
  MASQ_ERR_EMPTY_MODALITY = 7,  /* (sticky) count[m] == 0 at init */
  MASQ_ERR_UNSUPPORTED = 8,     /* valid request outside this path (e.g. A16) */
  MASQ_ERR_CUDA = 9             /* a CUDA runtime / driver call failed */
} masq_status;

typedef enum masq_dtype { MASQ_F32 = 0, MASQ_BF16 = 1 } masq_dtype;

typedef void* masq_stream;      /* cudaStream_t */

/* Workspace queries: op is one of the MASQ_OP_* values.  The layouts of the calls that run the
 * forward or X W GEMM (FORWARD, LAYER, REFERENCE, LOSS | SELF_REF) include, for deep K (d >= 8192
 * for the int8 forward, d >= 4096 for X W), the GEMM's stream-K scratch: one 256 x 256 32-bit
 * partial tile and two flags per CTA pair of the device (~19 MB on 148 SMs). */
enum {
  MASQ_OP_STATS = 0, MASQ_OP_INIT = 1, MASQ_OP_QWEIGHT = 2, MASQ_OP_QACT = 3,
  MASQ_OP_FORWARD = 4, MASQ_OP_LOSS = 5, MASQ_OP_REFERENCE = 6, MASQ_OP_LOSS_GRAD = 7,
  MASQ_OP_MEANABS = 8, MASQ_OP_CMC = 9, MASQ_OP_DECODE = 10, MASQ_OP_LAYER = 11,
  MASQ_OP_CMC_GRAM = 12, MASQ_OP_CMC_FACTORS = 13,
  /* flag OR-ed into MASQ_OP_LOSS / MASQ_OP_LOSS_GRAD: the workspace also holds the loss
   * target X W (f32 [T x d_out]) for calls made with Yref == NULL */
  MASQ_OP_SELF_REF = 0x100
};
size_t masq_workspace_size(int32_t op, int64_t T, int64_t d, int64_t d_out,
                           int32_t n_mod, int32_t r);

/*
 * A1 — per-modality channel absmax.
 *   R[m*d + i]  = max(R_in[m*d+i], max_{t: id_t = m} |X[t*ld_x + i]|)     (f32, exact)
 *   count[m]   += #{t : id_t = m}                                          (int64)
 * reset != 0 zeroes R and count first (a new calibration set); reset == 0
 * continues a running max over batches (resumable calibration).
 * X: [T x d] (row stride ld_x elements) of dtype xt (bf16 or f32).
 * Tokens with id >= n_mod are skipped and raise MASQ_ERR_BAD_MODALITY (sticky).
 */
masq_status masq_calibrate_stats(const void* X, masq_dtype xt, int64_t ld_x, const uint8_t* mod_id,
                                 int64_t T, int64_t d, int32_t n_mod,
                                 float* R, int64_t* count, int32_t reset,
                                 void* ws, size_t ws_bytes, masq_stream stream);

/*
 * A2 — closed-form modality-aware factors (reading Q8: the
 * weight max is over output channels j of row i of W[d x d_out]).
 *   wmax[i]    = max_j |W[i*d_out + j]|
 *   s[m*d + i] = sqrtf( fmaxf(R[m*d+i], 1e-12f) / fmaxf(wmax[i], 1e-12f) )   (IEEE div, sqrt)
 * wmax_out (optional, may be NULL) receives wmax [d].
 * count[m] == 0 for some m raises MASQ_ERR_EMPTY_MODALITY (sticky).
 */
masq_status masq_init_factors(const float* R, const int64_t* count, const void* W, masq_dtype wt,
                              int64_t d, int64_t d_out, int32_t n_mod,
                              float* s, float* wmax_out,
                              void* ws, size_t ws_bytes, masq_stream stream);

/*
 * A3 — smoothing + per-output-channel quantization of the weight (reading Q1),
 * stored K-major for the integer GEMM:
 *   ws[i,j]   = s[i] * W[i*d_out + j]                               (f32 mul)
 *   dw[j]     = fmaxf( max_i |ws[i,j]| / (2^{wbits-1}-1), 1e-12f )
 *   qw[j*d+i] = clamp(rha(ws[i,j] / dw[j]), -2^{wbits-1}, 2^{wbits-1}-1)   (int8 container)
 * With s = s^text this is the single stored weight Q(S_t W).
 */
masq_status masq_quantize_weight(const void* W, masq_dtype wt, const float* s,
                                 int64_t d, int64_t d_out, int32_t wbits,
                                 int8_t* qw, float* dw,
                                 void* ws, size_t ws_bytes, masq_stream stream);

/*
 * A4 — routed smoothing + per-token quantization:
 *   inv[m,i]  = 1.0f / s[m*d+i];  xs = X[t,i] * inv[id_t, i]            (f32)
 *   dx[t]     = fmaxf( max_i |xs| / (2^{abits-1}-1), 1e-12f )
 *   qx[t*d+i] = clamp(rha(xs / dx[t]))                                   (int8)
 * tile_mask (optional, [ceil(T/128)] uint32, zeroed by the call) receives,
 * per 128-token tile, the bit set {1 << m} of modalities present.
 */
masq_status masq_quantize_activations(const void* X, masq_dtype xt, int64_t ld_x, const uint8_t* mod_id,
                                      int64_t T, int64_t d, int32_t n_mod, const float* s,
                                      int32_t abits, int8_t* qx, float* dx, uint32_t* tile_mask,
                                      void* ws, size_t ws_bytes, masq_stream stream);

/* Optional debug taps for masq_linear_forward (parity tests); every field may be NULL / 0. */
typedef struct masq_debug {
  int32_t* acc;        /* if non-NULL: write the int32 accumulators sum_i qx*qw [T x ld_acc]
                          instead of Y (CMC skipped) */
  int64_t ld_acc;
  int8_t* qx;          /* if non-NULL: receives the activation codes A4 produced, [T x d] int8 */
  float* dx;           /* if non-NULL: receives the per-token steps Delta_x, [T] f32 */
} masq_debug;

/*
 * A4-A7 — the routed inference equation:
 *   Y[t,:] = dx[t] * dw[:] * (qx[t,:] . qw[:,:]^T)                        m_t == 0 (text)
 *   Y[t,:] = same + (X_t S_m^-1) . L1^m . L2^m                             m_t != 0
 * s: [n_mod x d] factors (row m = s^m); qw/dw: the output of
 * masq_quantize_weight with s^text (qw [d_out x d] K-major, dw [d_out]).
 * L1: bf16 [(n_mod-1) x d x r] (L1^m = T^-1 U_r), row-major per modality;
 * L2: bf16 [(n_mod-1) x r x ld_l2] (L2^m = Sigma_r V_r^T), row-major per modality.
 * L1/L2 may be NULL iff r == 0.  s, qw, dw, L1, L2, Y: 16-byte aligned (MASQ_ERR_ALIGN).  The CMC term is computed in full precision
 * from the f32 smoothed activations (split-bf16 tensor-core products, fp32
 * accumulation, reading Q13).  Y: f32 [T x ld_y], original token order.
 * Column sharding: pass qw + j0*d, dw + j0, L2 + j0, Y + j0 and d_out = shard width.
 */
masq_status masq_linear_forward(const void* X, masq_dtype xt, int64_t ld_x, const uint8_t* mod_id,
                                int64_t T, int64_t d, int64_t d_out, int32_t n_mod,
                                const float* s, const int8_t* qw, const float* dw,
                                int32_t wbits, int32_t abits,
                                const void* L1, const void* L2, int64_t ld_l2, int32_t r,
                                float* Y, int64_t ld_y,
                                void* ws, size_t ws_bytes, const masq_debug* dbg, masq_stream stream);

/*
 * Loss target X W ("X_m W"; reading Q16): bf16 tensor-core
 * products accumulated in fp32.  X bf16 [T x ld_x], W bf16 [d x d_out];
 * Yref f32 [T x ld_ref].  Computed once per calibration batch and reused by
 * every masq_calib_loss pass of the S optimisation.
 */
masq_status masq_reference_output(const void* X, int64_t ld_x, const void* W, int64_t T, int64_t d,
                                  int64_t d_out, float* Yref, int64_t ld_ref,
                                  void* ws, size_t ws_bytes, masq_stream stream);

/*
 * A8 — fused calibration loss (Eq. mas_quant; readings Q9, Q10, Q12):
 *   for every modality m: qw^m = Q(S_m W) (A3 with s^m), qx = A4 (each token with its own s^m),
 *   sums[m]   = sum_{t: id_t = m} sum_j | dx[t] dw^m[j] (qx[t] . qw^m[j]) - Yref[t,j] |   (f64)
 *   counts[m] = #{t : id_t = m}
 *   loss[0]   = sum_m lambda[m] * sums[m] / (counts[m] * d_out)   over m with counts[m] > 0
 * lambda: HOST array [n_mod] (NULL -> all 1.0).  Yref: f32 [T x ld_ref]
 * from masq_reference_output (computed once per batch and reused across the S-optimisation
 * passes), or NULL: the call then computes X W itself (as masq_reference_output; X and W must
 * be bf16, else MASQ_ERR_UNSUPPORTED) into the workspace, which must be sized with
 * masq_workspace_size(MASQ_OP_LOSS | MASQ_OP_SELF_REF, ...) (else MASQ_ERR_WORKSPACE).
 * sums/counts/loss are device pointers; the sums are
 * reduced in a fixed order (deterministic).  For token-sharded multi-GPU use,
 * all-reduce sums and counts (SUM) and call masq_loss_finalize.
 */
masq_status masq_calib_loss(const void* X, masq_dtype xt, int64_t ld_x, const uint8_t* mod_id,
                            int64_t T, int64_t d, int64_t d_out, int32_t n_mod,
                            const float* s, const void* W, masq_dtype wt,
                            int32_t wbits, int32_t abits, const float* lambda,
                            const float* Yref, int64_t ld_ref,
                            double* sums, int64_t* counts, double* loss,
                            void* ws, size_t ws_bytes, masq_stream stream);

/*
 * N1 (the next row after A8) — the S-optimisation step's gradient: everything
 * masq_calib_loss computes, plus grad[m*d + l] = dL/dtheta^m_l with theta^m = ln s^m (SPEC.md:
 * 307-316: log-space parameters, rounding treated as identity = straight-through).  Reading
 * Q24: ONLY round() is straight-through; the dynamic scales Delta = max|.|/q_max
 * are differentiated through their first arg-max element (a floored Delta has zero derivative).
 * Per modality m, with A = X_m S_m^-1, Ahat = Q(A), B = S_m W, Bhat = Q(B),
 * G = lambda_m/(N_m n) sign(Ahat Bhat - X_m W):
 *   grad_l = sum_j (Ahat^T G)_lj B_lj - sum_j (A^T G)_lj Bhat_lj
 *          + sum_{j: k_j = l} beta_j - sum_{t: k_t = l} alpha_t,
 *   beta_j = sum_i (Ahat^T G)_ij (Bhat - B)_ij,   alpha_t = sum_j G_tj ((Ahat - A) Bhat)_tj,
 * k_j = first arg-max_i |B_ij| (weight column scale), k_t = first arg-max_i |A_ti| (token scale).
 * grad: device f64 [n_mod x d], summed in a fixed order (bit-reproducible).  X and W must be
 * bf16.  Yref may be NULL (as masq_calib_loss; workspace MASQ_OP_LOSS_GRAD | MASQ_OP_SELF_REF).  count_norm (device i64 [n_mod], optional): the token
 * counts N_m used in scale_m = lambda_m/(N_m n); NULL = this call's own counts.  Token-sharded
 * multi-GPU use passes the GLOBAL counts (known after the A1 exchange) so that a plain SUM
 * all-reduce of grad over ranks is the gradient of the whole batch.
 */
masq_status masq_calib_loss_grad(const void* X, masq_dtype xt, int64_t ld_x, const uint8_t* mod_id,
                                 int64_t T, int64_t d, int64_t d_out, int32_t n_mod,
                                 const float* s, const void* W, masq_dtype wt,
                                 int32_t wbits, int32_t abits, const float* lambda,
                                 const float* Yref, int64_t ld_ref,
                                 double* sums, int64_t* counts, double* loss, double* grad,
                                 const int64_t* count_norm, void* ws, size_t ws_bytes, masq_stream stream);

/* Adam in log space: m1 = b1 m1 + (1-b1) g; m2 = b2 m2 + (1-b2) g^2;
 * theta -= lr * (m1/(1-b1^step)) / (sqrt(m2/(1-b2^step)) + eps); s_out (optional, f32) = exp(theta).
 * All arrays device, [count]; step >= 1. */
masq_status masq_adam_step(double* theta, const double* grad, double* m1, double* m2, int64_t count,
                           int32_t step, double lr, double beta1, double beta2, double eps,
                           float* s_out, masq_stream stream);

/* Adam state from factors: theta = ln s (f64 of the f32 s), m1 = m2 = 0.  Device arrays [count]. */
masq_status masq_adam_init(const float* s, double* theta, double* m1, double* m2, int64_t count,
                           masq_stream stream);

/* Best-so-far iterate ("the returned factors are the best-so-far iterate"): if
 * loss[0] is finite and < best_loss[0] (or best_loss[0] is NaN), copy s -> s_best ([count] f32)
 * and set best_loss[0] = loss[0].  improved (optional, device i32) receives 1 / 0.  All device
 * pointers; stream-ordered, no host sync. */
masq_status masq_keep_best(const double* loss, double* best_loss, const float* s, float* s_best,
                           int64_t count, int32_t* improved, masq_stream stream);

/* ---------------------------------------------------------------- N2: CMC factor construction
 * (PAPER.md:126-160 eq:l1l2, Theorem 2).
 * For every non-text modality m = 1..n_mod-1, with A_m = X_m S_m^-1 (f32 smoothing as the path
 * computes it) and dW_m = S_m W - Q(S_t W) (qw_text [d_out x d] int8 / dw_text [d_out] f32 are
 * the text-smoothed base weight from masq_quantize_weight(s[0])):
 *   eig(A_m^T A_m) = P Lambda P^T, T = (P (Lambda + eps_rel*lambda_max)^1/2)^T   (reading Q27)
 *   SVD(T dW_m) ~ U_r Sigma_r V_r^T,  L1^m = T^-1 U_r [d x r],  L2^m = Sigma_r V_r^T [r x d_out]
 * in f64 (cuBLAS GEMM/SYRK and the cuSOLVER symmetric eigensolver, loaded on first use; no
 * linear-algebra libraries -> MASQ_ERR_UNSUPPORTED).  Outputs in the layout masq_linear_forward
 * consumes: L1 [(n_mod-1) x d x r], L2 [(n_mod-1) x r x d_out], dtype lt (MASQ_F32 / MASQ_BF16),
 * columns of L1 / rows of L2 in descending singular-value order.  resid (optional, device f64
 * [n_mod-1]) = ||A_m (dW_m - L1 L2)||_F^2 (Theorem 2's objective).  A modality with no tokens
 * gets zero factors.  1 <= r <= min(d, d_out).  One-off calibration work: O(d^3) eigensolves
 * and O(d^2 (T + d_out)) f64 GEMMs per modality; the workspace holds f64 [T x d], 2 x [d x d]
 * and 2 x [d x d_out] buffers. */
masq_status masq_cmc_factors(const void* X, masq_dtype xt, int64_t ld_x, const uint8_t* mod_id,
                             int64_t T, int64_t d, int64_t d_out, int32_t n_mod,
                             const float* s, const void* W, masq_dtype wt,
                             const int8_t* qw_text, const float* dw_text, int32_t r, double eps_rel,
                             void* L1, void* L2, masq_dtype lt, double* resid,
                             void* ws, size_t ws_bytes, masq_stream stream);

/* ---------------------------------------------------------------- N3: packed int4 + decode
 * (SURVEY §8(f)).  W4 with sub-channel groups of 128 input channels (reading Q28): per output
 * channel j and group g, Delta_jg = max(max_{i in g} |f32(s_i w_ij)| / 7, 1e-12) and codes
 * rha(ws / Delta_jg) in [-8, 7] (the A3 quantizer at group granularity).  packed: d_out*d/2
 * bytes in the decode kernel's register order (nibbles hold code + 8; tile (jt, g) = 512
 * bytes for output channels 8jt..8jt+7 and inputs 128g..128g+127; see csrc/decode.cu);
 * scales f32 tile-major [d_out/8][d/128][8] (Delta of channel 8jt+c, group g at (jt*(d/128)+g)*8+c).
 * d % 128 == 0, d_out % 8 == 0, group == 128. */
masq_status masq_quantize_weight_int4(const void* W, masq_dtype wt, const float* s, int64_t d, int64_t d_out,
                                      int32_t group, uint8_t* packed, float* scales, masq_stream stream);
/* codes int8 [d_out x d] (K-major) from the packed format (inspection / tests). */
masq_status masq_unpack_int4(const uint8_t* packed, int64_t d, int64_t d_out, int32_t group, int8_t* codes,
                             masq_stream stream);
/* Decode-shaped W4A8 forward for 1 <= T <= 16 text tokens (text is the base
 * modality, so decoding carries no CMC): Y[t, j] = Q(x_t S_t^-1) . Q_g(S_t W)_:j, per-token int8
 * activations (abits), per-(channel, group) weight scales; f32 Y [T x ld_y].  Weight-bandwidth
 * bound: streams d_out*d/2 bytes of codes + 4*d_out*d/128 bytes of scales once. */
masq_status masq_linear_decode(const void* X, masq_dtype xt, int64_t ld_x, int64_t T, int64_t d, int64_t d_out,
                               const float* s_t, const uint8_t* packed, const float* scales, int32_t group,
                               int32_t abits, float* Y, int64_t ld_y, void* ws, size_t ws_bytes,
                               masq_stream stream);

/* Prefill-shaped W4A8 forward with PACKED int4 weights and 128-channel group scales, any T, with
 * CMC (reading Q28):
 *   Y[t, j] = dx[t] * sum_g Delta_jg * (qx[t, g-th 128 channels] . code[j, g-th 128 channels])
 *             (+ (X_t S_m^-1) L1^m L2^m for m_t != text, as masq_linear_forward)
 * on the tensor cores: the packed nibbles are expanded to int8 in shared memory and every group is
 * one kind::i8 k-block into its own TMEM accumulator, promoted in f32 with the group's scale.
 * Weight format (masq_quantize_weight_w4g): packed uint8 [d/128][d_out][64] (group-major: the 64
 * bytes of group g of channel j at (g d_out + j) 64, so 128 channels of a group are one contiguous
 * 8 KB block), byte 16c + i = code[j][128g + 32c + i] & 0xF | (code[j][128g + 32c + 16 + i] & 0xF)
 * << 4 (two's complement nibbles); scales f32 [d_out x d/128] (Delta_jg = max(max|s_i w_ij|/7,
 * 1e-12), the A3 quantizer at group granularity).  The codes and scales equal those of
 * masq_quantize_weight_int4 (the decode format); only the byte order differs.
 * d % 128 == 0, d_out % 32 == 0, group == 128; workspace masq_workspace_size(MASQ_OP_FORWARD, ...).
 * masq_debug.acc: int32 sum over the groups of the unscaled group accumulators (CMC skipped). */
masq_status masq_quantize_weight_w4g(const void* W, masq_dtype wt, const float* s, int64_t d, int64_t d_out,
                                     int32_t group, uint8_t* packed, float* scales, masq_stream stream);
masq_status masq_linear_forward_w4g(const void* X, masq_dtype xt, int64_t ld_x, const uint8_t* mod_id,
                                    int64_t T, int64_t d, int64_t d_out, int32_t n_mod,
                                    const float* s, const uint8_t* packed, const float* scales, int32_t group,
                                    int32_t abits, const void* L1, const void* L2, int64_t ld_l2, int32_t r,
                                    float* Y, int64_t ld_y, void* ws, size_t ws_bytes,
                                    const masq_debug* dbg, masq_stream stream);

/* The two phases of masq_cmc_factors, for token-sharded / multi-batch runs: G[(m-1) d d] (+)=
 * A_m^T A_m for every non-text modality m (f64, lower triangle; accumulate != 0 adds to G) —
 * all-reduce G with SUM across ranks / batches — then the factors and the Theorem-2 residual
 * <E, G E> from G alone (the activations enter only through their Gram matrix).  "Lower" is in
 * column-major (cuBLAS) order, i.e. the upper triangle of a row-major [d x d] array. */
masq_status masq_cmc_gram(const void* X, masq_dtype xt, int64_t ld_x, const uint8_t* mod_id, int64_t T,
                          int64_t d, int32_t n_mod, const float* s, double* G, int32_t accumulate,
                          void* ws, size_t ws_bytes, masq_stream stream);
masq_status masq_cmc_factors_from_gram(const double* G, int64_t d, int64_t d_out, int32_t n_mod,
                                       const float* s, const void* W, masq_dtype wt,
                                       const int8_t* qw_text, const float* dw_text, int32_t r,
                                       double eps_rel, void* L1, void* L2, masq_dtype lt, double* resid,
                                       void* ws, size_t ws_bytes, masq_stream stream);

/* ---------------------------------------------------------------- N4: baseline factor methods
 * — the closed forms the paper compares MASQuant against, on the same data. */

/* s[r*d + i] = max(num[r*d+i], 1e-12)^beta / max(den[i], 1e-12)^(1-beta), evaluated in f64 and
 * rounded once to f32 (reading Q26).  SmoothQuant: num = R^m (or the unified
 * max_m R^m), den = max_j |w_ji| (masq_init_factors' wmax_out).  AWQ
 * (PAPER.md:24-28): num = mean_t |x_t,i|, den = NULL (treated as 1).  beta in [0, 1] (f64;
 * anything else -> MASQ_ERR_SHAPE).
 * All device arrays: num / s [rows x d], den [d]. */
masq_status masq_smooth_factors(const float* num, int64_t rows, int64_t d, const float* den, double beta,
                                float* s, masq_stream stream);

/* AWQ's activation statistic: sumabs[m*d + i] (+)= sum over tokens of modality m
 * of |x_t,i| (f64; f32 partials over 64-token slabs, fixed-order f64 reduction, so the result is
 * deterministic), count[m] (+)= tokens of m; optional f32 outputs mean[m*d+i] = sumabs/count and
 * mean_unified[i] = sum_m sumabs / sum_m count (the unified statistic over all tokens).
 * reset != 0 zeroes sumabs / count first; otherwise the call accumulates (multi-batch).
 * A bad id sets MASQ_ERR_BAD_MODALITY in the sticky status (the token is skipped). */
masq_status masq_calibrate_meanabs(const void* X, masq_dtype xt, int64_t ld_x, const uint8_t* mod_id,
                                   int64_t T, int64_t d, int32_t n_mod, double* sumabs, int64_t* count,
                                   float* mean, float* mean_unified, int32_t reset,
                                   void* ws, size_t ws_bytes, masq_stream stream);

/* count[m] (+)= number of tokens with id m (i64, device); reset != 0 zeroes first.  Bad ids set
 * MASQ_ERR_BAD_MODALITY in the sticky status.  Workspace: masq_workspace_size(MASQ_OP_STATS, ...).
 * (Token-sharded N1 runs use it to normalise each batch's gradient by the global counts.) */
masq_status masq_count_modalities(const uint8_t* mod_id, int64_t T, int32_t n_mod, int64_t* count,
                                  int32_t reset, void* ws, size_t ws_bytes, masq_stream stream);

/* Channel statistics across modalities from R [n_mod x d] (each output optional):
 * alpha[i] = R[dominant][i] / max(R[other][i], 1e-12) (f32 division; Theorem 1 range
 * ratio); r_unified[i] = max_m R[m][i]; dom_counts[m] = number of
 * channels whose maximum modality m attains (ties go to the first such m) and
 * dom_counts[n_mod] = number of tied channels. */
masq_status masq_range_stats(const float* R, int32_t n_mod, int64_t d, int32_t dominant, int32_t other,
                             float* alpha, float* r_unified, int64_t* dom_counts, masq_stream stream);

/*
 * One calibration pass of a linear layer in one call (A3 for every modality, A4-A7, A8): the
 * results of masq_quantize_weight(s[0]) + masq_linear_forward + masq_reference_output +
 * masq_calib_loss (codes, Y, Yref and counts bit-identical; loss sums to rounding), with the
 * shared work done once: every modality's weight codes come from one read of W (set 0 = the
 * forward's Q(S_t W)); the activations are quantized once in token order for the forward and
 * gathered into the modality-grouped order for the loss (A4's codes are row-wise); and since
 * S_0 = S_t, a text row's forward output IS its loss-side quantized output, so the forward
 * epilogue sums the text rows' |y - yref| and the loss GEMM runs on the non-text rows only.  X and W bf16.  Outputs: Y [T x ld_y] and Yref
 * [T x ld_ref] f32; optional qw_text [d_out x d] int8 / dw_text [d_out] f32 (the text-smoothed
 * base weight for serving); sums / counts / loss as masq_calib_loss.  CMC as masq_linear_forward
 * (L1 / L2 bf16, r = 0 disables).
 */
masq_status masq_calib_layer(const void* X, int64_t ld_x, const uint8_t* mod_id, int64_t T, int64_t d,
                             int64_t d_out, int32_t n_mod, const float* s, const void* W,
                             int32_t wbits, int32_t abits, const void* L1, const void* L2, int64_t ld_l2,
                             int32_t r, const float* lambda, float* Y, int64_t ld_y, float* Yref,
                             int64_t ld_ref, int8_t* qw_text, float* dw_text, double* sums,
                             int64_t* counts, double* loss, void* ws, size_t ws_bytes, masq_stream stream);

/* loss[0] = sum_m lambda[m] * sums[m] / (counts[m] * d_out) on the device (after an all-reduce). */
masq_status masq_loss_finalize(const double* sums, const int64_t* counts, const float* lambda,
                               int32_t n_mod, int64_t d_out, double* loss, masq_stream stream);

/* Synchronizes `stream`, returns the sticky device status stored in ws and clears it. */
masq_status masq_check(void* ws, masq_stream stream);

const char* masq_status_string(masq_status s);

/*
 * Opt-in kernel timing (measurement only; off by default; the one piece of process-global
 * state).  masq_profile_enable(1) starts recording a cudaEvent pair on the launching stream
 * around every kernel the library launches (and discards earlier records); it returns the
 * previous state.  masq_profile_collect() waits for the recorded events and aggregates them
 * by kernel name: names[i*32 .. i*32+31] (NUL-terminated), total_ms[i], launches[i] for
 * i < return value (at most max_entries); it clears the records.  A name may cover a short
 * sequence of library kernels (routing: the count and scatter passes); launches[i] counts them
 * all, total_ms[i] is the bracketed time.  Returns -1 on a CUDA error.
 */
int32_t masq_profile_enable(int32_t on);
/* Restricts the recording to the kernels reported under `name` (e.g. "gemm_ref"); NULL or ""
 * records every kernel again.  Every other launch then runs between unbracketed neighbours (no
 * event record serialising it with them).  Returns 0. */
int32_t masq_profile_only(const char* name);
int32_t masq_profile_collect(int32_t max_entries, char* names, double* total_ms, int64_t* launches);

/* Library identification: "<version> sm_100a". */
const char* masq_version(void);

#ifdef __cplusplus
}
#endif

#endif /* MASQ_H */
