// internal.h — host-side contracts between the C ABI (api.cu) and the kernel translation
// units (elem.cu, gemm.cu, zgemm.cu).  Not part of the public ABI.
#pragma once
#include <algorithm>
#include <utility>
#include <cstddef>
#include <cstdint>
#include <cuda.h>
#include <cuda_runtime.h>

#include "../../include/masq.h"

namespace masq {

constexpr int kMaxMod = 8;
constexpr int kTileM = 128;        // GEMM M tile (token rows)
constexpr int kTileN = 256;        // GEMM N tile (output channels)
constexpr int kUnitM = 256;        // GEMM M unit of a CTA pair (cta_group::2); loss segments align to it
constexpr int kStatusBytes = 256;

// sticky device status bits (stored in ws[0..3])
constexpr uint32_t kStBadModality = 1u << 0;
constexpr uint32_t kStEmptyModality = 1u << 1;

inline size_t align256(size_t x) { return (x + 255) & ~size_t(255); }
inline int64_t ceil_div(int64_t a, int64_t b) { return (a + b - 1) / b; }
inline int64_t rpad_of(int64_t r) { return r > 0 ? ceil_div(r, 64) * 64 : 0; }

struct WsLayout {
  size_t status = 0, inv_s = 0, qx = 0, dx = 0, mask = 0, z = 0, l1t = 0, l2t = 0, xsplit = 0;
  size_t qw_all = 0, dw_all = 0, amax = 0, partials = 0, wt = 0, perm = 0, tile_mod = 0, cnt = 0, total = 0;
  size_t gsign = 0, planes = 0, gpartial = 0, yref = 0;
  // N1 scale terms
  size_t dq = 0, de = 0, dq2 = 0, de2 = 0, apart = 0, bpart = 0, kj = 0, keys = 0, vals = 0, bucket = 0, skeys = 0, svals = 0,
         stemp = 0, stemp_bytes = 0;
  // N2 CMC factors (f64)
  size_t g = 0, c = 0, lam = 0, sig2 = 0, sq = 0, isq = 0, dw64 = 0, m64 = 0, l1t64 = 0, urs = 0, l2t64 = 0,
         work = 0, info = 0, dot = 0;
  size_t lwork = 0;   // doubles
  size_t gall = 0;    // CMC: the (n_mod-1) Gram matrices of the one-call path
  size_t gram_part = 0, gram_r = 0, gram_ex = 0, slices = 0;   // CMC: exact Gram scratch (gram.cu)
  // N3 decode
  size_t ids0 = 0, dpart = 0;
  // fused layer call: token-order codes next to the grouped ones
  size_t qx_tok = 0, dx_tok = 0, fpart = 0, ipos = 0, zpart = 0;
  // stream-K partials / flags of the forward and X.W GEMMs
  size_t skpart = 0, skflag = 0;
};
// f32_x: the forward needs bf16 hi/lo planes of X for the CMC GEMM
WsLayout ws_layout(int32_t op, int64_t T, int64_t d, int64_t n, int32_t n_mod, int32_t r, bool f32_x = true);

// cudaFuncSetAttribute(MaxDynamicSharedMemorySize) once per (kernel, device, size): the attribute
// is per device, so one host thread driving several GPUs must set it on each (gemm.cu)
cudaError_t set_max_dyn_smem(const void* func, int bytes);

// Kernel launch with programmatic stream serialization (MASQ_PDL, default on): the kernel may
// become resident while the previous kernel of the stream drains, and runs its prologue (barrier
// init, TMEM allocation, descriptor prefetch) there; every kernel launched this way executes
// sm100::pdl_wait() in each thread before touching global memory, so stream order holds for all
// data.  Kernels not launched this way serialise as usual.
bool pdl_enabled();
int gemm_sk_min_kb();   // stream-K: minimum k-blocks per GEMM unit (MASQ_SK_MINKB, default 64)
#define MASQ_LAUNCH(call)                      \
  do {                                         \
    const cudaError_t le_ = (call);            \
    if (le_ != cudaSuccess) return le_;        \
  } while (0)
template <typename... KArgs, typename... Args>
inline cudaError_t launch_k(void (*kern)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t st,
                            Args&&... args) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = at;
  cfg.numAttrs = pdl_enabled() ? 1 : 0;
  return cudaLaunchKernelEx(&cfg, kern, std::forward<Args>(args)...);
}

// ---------------------------------------------------------------- opt-in kernel timing (prof.cu)
// RAII: records a cudaEvent pair around a kernel launch when masq_profile_enable(1) is active.
class ProfScope {
 public:
  // launches: library kernels the scope brackets (counted into masq_profile_collect's launches)
  ProfScope(const char* name, cudaStream_t st, int launches = 1);
  ~ProfScope();
  ProfScope(const ProfScope&) = delete;
  ProfScope& operator=(const ProfScope&) = delete;

 private:
  const char* name_;
  cudaStream_t st_;
  void* a_ = nullptr;
  int launches_ = 1;
};

// ---------------------------------------------------------------- elementwise kernels (elem.cu)
cudaError_t launch_stats(const void* X, masq_dtype xt, int64_t ld_x, const uint8_t* ids, int64_t T, int64_t d,
                         int n_mod, float* R, int64_t* count, uint32_t* status, cudaStream_t st);
cudaError_t launch_init(const float* R, const int64_t* count, const void* W, masq_dtype wt, int64_t d, int64_t n,
                        int n_mod, float* s, float* wmax, uint32_t* status, cudaStream_t st);
// weight quantization of n_sets factor vectors s[k*d..] -> qw[k*n*d..], dw[k*n..]
cudaError_t launch_wquant(const void* W, masq_dtype wt, const float* s, int n_sets, int64_t d, int64_t n,
                          int wbits, int8_t* qw, float* dw, uint32_t* amax_scratch, cudaStream_t st);
// amax_scratch: [2 x n_sets x n] u32 — the column maxima max_i |s_i w_ij| (f32 bits, kept after
// the call), then the f32 reciprocals of the scales used by the quantizer
cudaError_t launch_inv(const float* s, int64_t count, float* inv, cudaStream_t st);
// qg[p] = qt[perm[p]] (rows of d bytes, d % 16 == 0), dg[p] = dt[perm[p]]; zeros for perm < 0
// fused layer call: A4 once, writing the token-order codes and the grouped copy of the non-text
// rows (ipos[t] = grouped row of token t from launch_route); zeroes the grouped padding rows of
// modalities >= 1.  cudaErrorNotSupported when the TMA row kernel does not apply.
// A4 for the decode path: every token modality 0, 1/s formed in the kernel (no ids, no inverse
// factors); cudaErrorNotSupported when the TMA row kernel does not apply
cudaError_t launch_aquant_direct(const void* X, masq_dtype xt, int64_t ld_x, int64_t T, int64_t d, const float* s,
                                 int abits, int8_t* qx, float* dx, uint32_t* status, cudaStream_t st);
cudaError_t launch_aquant_dual(const void* X, masq_dtype xt, int64_t ld_x, const uint8_t* ids, int64_t T, int64_t d,
                               int n_mod, const float* inv_s, int abits, int8_t* qx, float* dx, uint32_t* mask,
                               uint32_t* status, const int32_t* perm, const uint32_t* tile_mod, const int32_t* ipos,
                               int64_t Tg, int8_t* qg, float* dg, cudaStream_t st, const float* s_raw = nullptr);
cudaError_t launch_gather_rows(const int8_t* qt, const float* dt, const int32_t* perm, int64_t Tg, int64_t d, int8_t* qg,
                               float* dg, cudaStream_t st);
// perm (optional): output row p quantizes input token perm[p] (-1: padding row, left untouched);
// T_out = number of output rows (T when perm == NULL)
cudaError_t launch_aquant(const void* X, masq_dtype xt, int64_t ld_x, const uint8_t* ids, int64_t T, int64_t d,
                          int n_mod, const float* inv_s, int abits, int8_t* qx, float* dx, uint32_t* mask,
                          uint32_t* status, cudaStream_t st, const int32_t* perm = nullptr, int64_t T_out = -1,
                          const float* s_raw = nullptr);
// (inv_s == nullptr: 1/s is formed in the bf16 TMA row kernel from s_raw; cudaErrorNotSupported
//  when that kernel does not apply, and the caller computes the inverse factors and retries)
// rows grouped by modality, each segment padded to a multiple of kUnitM (256) rows:
// perm[Tg] (grouped row -> token, -1 padding), tile_mod[Tg/256] (modality of the unit, ~0u empty)
inline int64_t grouped_rows(int64_t T, int n_mod) { return ceil_div(T, kUnitM) * kUnitM + (int64_t)n_mod * kUnitM; }
// routing scratch: per-chunk modality counts stored after the Tg perm entries (callers size perm
// as grouped_rows(T, n_mod) + route_scratch_ints(T))
// multi-CTA routing: 8 tokens per thread, 256 threads per CTA (2048 tokens); 64 threads (512
// tokens) up to 8192 tokens, where the two passes are latency-bound on a handful of CTAs
inline int64_t route_chunk(int64_t T) { return T <= 8192 ? 512 : 2048; }
inline int64_t route_blocks(int64_t T) { return std::max<int64_t>(1, ceil_div(T, route_chunk(T))); }
inline int64_t route_scratch_ints(int64_t T) { return route_blocks(T) * kMaxMod; }
// counts (optional): per-modality token counts [n_mod] (int64)
cudaError_t launch_route(const uint8_t* ids, int64_t T, int n_mod, int32_t* perm, uint32_t* tile_mod,
                         int64_t* counts, cudaStream_t st, int32_t* ipos = nullptr);
// L2 [(M-1) x r x ld] -> L2t [(M-1)*n x 2*rpad] (the same L2^T for the Zhi and Zlo K-blocks)
cudaError_t launch_pack_l2(const uint16_t* L2, int64_t ld_l2, int n_nt, int64_t n, int r, int rpad, uint16_t* L2t,
                           cudaStream_t st);
// bf16 W [d x n] -> Wt [n x d]
cudaError_t launch_transpose_bf16(const uint16_t* W, int64_t d, int64_t n, uint16_t* Wt, cudaStream_t st);
// sums[m] = fixed-order sum of partials[u * epi + e] over units u with tile_mod[u / num_n] == m;
// counts_in: per-modality token counts from launch_route
// extra (optional): n_extra per-(unit, CTA) partials of modality 0 added after the grouped ones
cudaError_t launch_loss_reduce(const double* partials, int64_t n_units, int num_n, int epi, const uint32_t* tile_mod,
                               const int64_t* counts_in, int n_mod, int64_t n, const float* lambda_host,
                               double* sums, int64_t* counts, double* loss, cudaStream_t st,
                               const double* extra = nullptr, int64_t n_extra = 0,
                               // free doubles after the partials (two-level reduction when large)
                               double* scratch = nullptr, int64_t scratch_cap = 0,
                               // units of modality < m_lo are skipped (their partials never written)
                               int m_lo = 0);
cudaError_t launch_loss_finalize(const double* sums, const int64_t* counts, const float* lambda_host, int n_mod,
                                 int64_t n, double* loss, cudaStream_t st);

// ---------------------------------------------------------------- tensor maps (tmap.cu)
// 2-D row-major tensor [rows x cols] of elem_bytes elements, row pitch ld elements,
// box [box_rows x box_cols], 128-byte swizzle when swizzle128 (box_cols*elem_bytes must be 128).
bool make_tmap_2d(CUtensorMap* map, const void* base, CUtensorMapDataType dt, int elem_bytes, uint64_t rows,
                  uint64_t cols, uint64_t ld, uint32_t box_rows, uint32_t box_cols, bool swizzle128);

// ---------------------------------------------------------------- GEMM (gemm.cu)
enum GemmMode { kModeFwd = 0, kModeAcc = 1, kModeLoss = 2, kModeRef = 3, kModeAlpha = 4, kModeAlphaI8 = 5 };

struct GemmArgs {
  int mode;
  int64_t T, n, d;                 // rows, output columns, K
  const int8_t* qx;                // int8 A [T x d]   (kModeFwd/Acc/Loss)
  const uint16_t* xbf;             // bf16 A [T x ld_x] (kModeRef; kModeAlpha: the D plane)
  int64_t ld_x;
  const void* b;                   // int8 qw [(n_b) x d] or bf16 Wt [n x d]
  int64_t b_rows;                  // rows of the B tensor (n, or n_mod*n for the loss)
  const float* dx;
  const float* dw;                 // [n] or [n_mod * n] for the loss
  const uint32_t* tile_mask;       // per 128-row tile (fwd: modality bit set; loss: modality index)
  const int32_t* perm;             // loss: grouped row -> token
  int n_mod;
  void* out;                       // Y f32 / acc int32 [T x ld_out]
  int64_t ld_out;
  // CMC (kModeFwd, r > 0)
  int rpad;                        // 0 -> no CMC
  const uint16_t* z;               // [T x (M-1)*2*rpad] bf16 (hi | lo per modality)
  const uint16_t* l2t;             // [(M-1)*n x 2*rpad] bf16
  // loss
  const float* yref;
  int64_t ld_ref;
  double* partials;                // [n_mod][tiles][4]
  uint16_t* gsign;                 // loss, optional (N1): bf16 sign(yq - yref), grouped rows [T x n]
  // kModeAlpha (N1): acc = D . codes_m^T (bf16 codes of Q(S_m W), K-major [n_mod*n x d]);
  // apart[row * apart_ld + apart_off + 2*nt + half] = sum_j gsign[row][j] * dw_m[j] * acc[row][j]
  // over the CTA's columns (two passes: D's int8 codes and their residual's)
  float* apart;
  int apart_ld = 0, apart_off = 0;
  // fused layer call: the forward also sums the text rows' loss (|y - yref|, text rows only:
  // their forward output is the loss's quantized output) into partials, and the loss GEMM then
  // skips the text units
  const uint8_t* ids;
  int fwd_loss = 0;
  int skip_m0 = 0;
  // stream-K remainder (kModeFwd / Acc / Ref; optional, nullptr = off): the units past the last
  // full wave are split along K over all CTA pairs; sk_part holds the non-owner partial
  // accumulators (gemm_sk_bytes), sk_flag one ready flag per (pair, CTA)
  uint32_t* sk_part = nullptr;
  uint32_t* sk_flag = nullptr;
};
cudaError_t launch_gemm(const GemmArgs& a, cudaStream_t st);
size_t gemm_sk_part_bytes();   // workspace for GemmArgs::sk_part (device-independent upper bound)
size_t gemm_sk_flag_bytes();
int gemm_epilogue_warps();

// ---------------------------------------------------------------- N1 gradient (grad.cu)
// planes [2][Tg][d] bf16: D = Ahat - X S^-1 and X, in grouped row order
// ktkey[Tg]: m*d + (first arg-max_i |xs_ti|) of every grouped row (-1: padding / floored scale)
cudaError_t launch_gradprep(const uint16_t* X, int64_t ld_x, const uint8_t* mod_id, const int32_t* perm,
                            const int8_t* qx, const float* dx, const float* inv, int64_t Tg, int64_t d, int abits,
                            uint16_t* planes, int32_t* ktkey, int8_t* dq, float* de, int8_t* dq2, float* de2,
                            cudaStream_t st);
// partial[m][jt][i] (sum_j of the direct terms), bpart[m][4*it + q][j] (beta_j over 32 rows i),
// kj[m][j] = min i with |f32(s_i w_ij)| == colmax[m][j] (atomicMin; preset to INT_MAX)
cudaError_t launch_gradgemm(const uint16_t* planes, int64_t Tg, const uint16_t* gsign, const int8_t* qw_all,
                            const uint32_t* tile_mod, int n_mod, int64_t d, int64_t n, const float* s,
                            const float* inv, const uint16_t* W, const float* dw, const uint32_t* colmax,
                            double* partial, float* bpart, int32_t* kj, cudaStream_t st);
int gradgemm_ntiles_j(int64_t n);
int gradgemm_ntiles_i(int64_t d);
// keys/vals [n_mod*n + Tg]: (m*d + k_j, +beta_j) for every weight column, (ktkey[t], -alpha_t) for
// every grouped row; alpha_t = sum of apart[t][0..na), beta = sum of bpart over the nb row groups
cudaError_t launch_gradkeys(const float* bpart, int nb, const int32_t* kj, const uint32_t* colmax, int wbits,
                            const float* apart, int na, const int32_t* ktkey, int n_mod, int64_t d, int64_t n,
                            int64_t Tg, int32_t* keys, double* vals, cudaStream_t st);
size_t bucket_temp_bytes(int64_t nkeys);
// contrib[l] = sum of vals over keys == l (l in [0, nl)), summed in key order after a stable radix
// sort (deterministic); skeys / svals / temp are workspace
cudaError_t launch_bucket(const int32_t* keys, const double* vals, int64_t nkeys, int64_t nl, uint32_t* skeys,
                          double* svals, void* temp, size_t temp_bytes, double* contrib, cudaStream_t st);
cudaError_t launch_gradreduce(const double* partial, const double* contrib, const int64_t* counts,
                              const float* lambda_host, int n_mod, int nj, int64_t d, int64_t n, double* grad,
                              cudaStream_t st);
cudaError_t launch_adam_init(const float* s, double* theta, double* m1, double* m2, int64_t count, cudaStream_t st);
cudaError_t launch_keep_best(const double* loss, double* best, const float* s, float* s_best, int64_t count,
                             int32_t* improved, cudaStream_t st);
cudaError_t launch_adam(double* theta, const double* grad, double* m1, double* m2, int64_t count, int step, double lr,
                        double b1, double b2, double eps, float* s_out, cudaStream_t st);
int num_sms();

// ---------------------------------------------------------------- N2 CMC factors (cmc.cu)
struct CmcArgs {
  const void* X;
  masq_dtype xt;
  int64_t ld_x;
  const uint8_t* ids;
  int64_t T, d, n;
  int n_mod, r;
  const float* inv;              // [M][d] f32 reciprocals of s
  const float* s;                // [M][d]
  const void* W;
  masq_dtype wt;
  const int8_t* qw_t;            // text codes [n x d]
  const float* dw_t;             // text scales [n]
  double eps_rel;
  void* L1;                      // [(M-1) x d x r]
  void* L2;                      // [(M-1) x r x n]
  masq_dtype lt;
  double* resid;                 // optional [(M-1)]
  double *G, *C, *lam, *sig2, *sq, *isq, *dW, *Mb, *L1t, *Urs, *L2t, *work, *dot;
  int* info;
  size_t lwork;
  // tensor-core Gram (gram.cu)
  int32_t* perm;
  uint32_t* tile_mod;
  int64_t* cnt;
  float* R;
  int32_t* ex;
  int8_t* slices;
  double* gram_part;
  uint32_t* status;
};
bool cmc_linalg_available();
size_t cmc_syevd_lwork(int64_t d, int64_t n);
bool cmc_eig_route();
int cmc_dot_blocks();
cudaError_t launch_cmc_gram(const CmcArgs& a, double* G, int accumulate, cudaStream_t st);
// G[m-1] (+)= A_m^T A_m for m = 1..n_mod-1 on the int8 tensor cores, exact (gram.cu: three int8
// slices per value on a per-channel power-of-two scale, int32 accumulation, f64 combination; both
// triangles written); perm / tile_mod from launch_route, inv = 1/s; R / cnt / ex / slices / part
// are scratch (cmc_gram_slice_bytes, cmc_gram_part_bytes)
size_t cmc_gram_part_bytes(int64_t T, int64_t d, int n_mod);
size_t cmc_gram_slice_bytes(int64_t T, int64_t d, int n_mod);
cudaError_t launch_cmc_gram_tc(const void* X, masq_dtype xt, int64_t ld_x, const uint8_t* ids, int64_t T,
                               int64_t d, int n_mod, const float* inv, const int32_t* perm,
                               const uint32_t* tile_mod, float* R, int64_t* cnt, int32_t* ex, int8_t* slices,
                               double* part, uint32_t* status, double* G, int accumulate, cudaStream_t st);
cudaError_t launch_cmc_from_gram(const CmcArgs& a, const double* G, cudaStream_t st);

// ---------------------------------------------------------------- N3 int4 decode (decode.cu)
int decode_kchunks(int64_t d);
int decode_max_tokens();
cudaError_t launch_wq4(const void* W, masq_dtype wt, const float* s, int64_t d, int64_t n, uint8_t* packed,
                       float* scales, cudaStream_t st);
cudaError_t launch_unpack4(const uint8_t* packed, int64_t d, int64_t n, int8_t* codes, cudaStream_t st);
cudaError_t launch_decode(const int8_t* qa, const float* dx, int T, int64_t d, int64_t n, const uint8_t* packed,
                          const float* scales, float* part, float* Y, int64_t ldy, cudaStream_t st);

// ---------------------------------------------------------------- N3 prefill W4 grouped GEMM (w4g.cu)
struct W4gArgs {
  int64_t T, n, d;
  const int8_t* qx;                // activation codes [T x d]
  const float* dx;                 // [T]
  const uint8_t* packed;           // [n x d/2] (w4g layout)
  const float* scales;             // [n x d/128]
  const uint32_t* tile_mask;       // per 128-token tile modality bits (CMC)
  int n_mod, rpad;
  const uint16_t* z;               // [T x (M-1)*2*rpad]
  const uint16_t* l2t;             // [(M-1)*n x 2*rpad]
  void* out;
  int64_t ld_out;
  int acc_mode;
};
cudaError_t launch_w4g_gemm(const W4gArgs& a, cudaStream_t st);
// W4 grouped quantizer: layout 0 = decode (decode.cu format), 1 = prefill (w4g.cu format)
cudaError_t launch_wq4_layout(const void* W, masq_dtype wt, const float* s, int64_t d, int64_t n, uint8_t* packed,
                              float* scales, int layout, cudaStream_t st);

// ---------------------------------------------------------------- N4 baselines (baseline.cu)
int meanabs_slabs(int64_t T);
cudaError_t launch_smooth_factors(const float* num, int64_t rows, int64_t d, const float* den, double beta, float* s,
                                  cudaStream_t st);
cudaError_t launch_meanabs(const void* X, masq_dtype xt, int64_t ld_x, const uint8_t* ids, int64_t T, int64_t d,
                           int n_mod, double* S, int64_t* cnt, float* mean, float* uni, float* part,
                           uint32_t* status, cudaStream_t st);
cudaError_t launch_count_modalities(const uint8_t* ids, int64_t T, int n_mod, int64_t* cnt, uint32_t* status,
                                   cudaStream_t st);
cudaError_t launch_range_stats(const float* R, int n_mod, int64_t d, int dominant, int other, float* alpha,
                               float* runi, int64_t* dom, cudaStream_t st);

// ---------------------------------------------------------------- CMC first factor (zgemm.cu)
// L1s planes: [2][(M-1)*rpad][d] bf16, plane 0 = hi, 1 = lo of diag(1/s^m) L1^m (transposed)
// s: the factors [n_mod][d]; 1/s is formed in the kernel (IEEE division, as inv_kernel)
// l1_fold + the L2 packing of launch_pack_l2 in one launch (the forward calls' CMC factor packing);
// mask != nullptr: the same launch writes the per-128-row-tile modality bit sets of ids[0, T)
// (instead of a zeroing pass + the activation quantizer's atomics)
cudaError_t launch_cmc_pack(const uint16_t* L1, const float* s, int64_t d, int r, int rpad, int n_nt, uint16_t* L1s,
                            const uint16_t* L2, int64_t ld_l2, int64_t n, uint16_t* L2t, const uint8_t* ids, int64_t T,
                            int n_mod, uint32_t* mask, cudaStream_t st);
cudaError_t launch_l1_fold(const uint16_t* L1, const float* s, int64_t d, int r, int rpad, int n_nt,
                           uint16_t* L1s, cudaStream_t st);
// f32 X -> bf16 hi / lo planes [T x d]
cudaError_t launch_split_f32(const float* X, int64_t ld_x, int64_t T, int64_t d, uint16_t* hi, uint16_t* lo,
                             cudaStream_t st);
// Z[t, (m-1)*2*rpad + k] = hi(x_t . L1'^m)_k, [.. + rpad + k] = lo(...) for rows with id_t == m,
// zeros for the other rows of tiles that contain modality m.  A0 (and A1 for f32 X) are bf16 planes.
cudaError_t launch_zgemm(const uint16_t* A0, int64_t ld_a, const uint16_t* A1, const uint8_t* ids, int64_t T,
                         int64_t d, int n_mod, const uint16_t* L1s, int rpad, const uint32_t* tile_mask, uint16_t* Z,
                         cudaStream_t st, float* zpart = nullptr);
// split-K of the CMC first factor for small T (too few 128-row tiles to fill the GPU): number of
// K splits and the f32 partial workspace it needs (0 when not split)
int zgemm_splits(int64_t T, int64_t d);
size_t zgemm_part_bytes(int64_t T, int64_t d, int n_mod, int rpad);

}  // namespace masq
