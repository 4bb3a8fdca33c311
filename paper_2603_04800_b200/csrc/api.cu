#include <cstdio>
#include <cstdlib>
// api.cu — the C ABI (include/masq.h): argument validation, workspace carving and the launch
// sequence of every entry point.  All compute runs in the kernels of elem.cu, zgemm.cu, gemm.cu.
#include <cstring>

#include "internal.h"

namespace masq {

WsLayout ws_layout(int32_t op, int64_t T, int64_t d, int64_t n, int32_t n_mod, int32_t r, bool f32_x) {
  WsLayout L;
  size_t off = 0;
  auto take = [&](size_t bytes) {
    const size_t o = off;
    off += align256(bytes);
    return o;
  };
  const int64_t tiles_m = ceil_div(std::max<int64_t>(T, 1), kTileM);
  const int64_t rp = rpad_of(r);
  const int64_t nnt = std::max(n_mod - 1, 0);
  L.status = take(kStatusBytes);
  const bool self_ref = (op & MASQ_OP_SELF_REF) != 0;     // loss target X W computed into ws
  op &= ~MASQ_OP_SELF_REF;
  switch (op) {
    case MASQ_OP_STATS:
    case MASQ_OP_INIT:
      break;
    case MASQ_OP_CMC:
    case MASQ_OP_CMC_GRAM:
    case MASQ_OP_CMC_FACTORS: {
      if (op != MASQ_OP_CMC_FACTORS) {
        // exact tensor-core Gram (gram.cu): routing, channel maxima / exponents, the three int8
        // slice planes of X S^-1 (transposed), f64 partial tiles
        const int64_t Tg = grouped_rows(T, n_mod);
        L.inv_s = take(sizeof(float) * n_mod * d);
        L.perm = take(sizeof(int32_t) * (Tg + route_scratch_ints(T)));
        L.tile_mod = take(sizeof(uint32_t) * (Tg / kUnitM));
        L.cnt = take(sizeof(int64_t) * n_mod);
        L.gram_r = take(sizeof(float) * n_mod * d);
        L.gram_ex = take(sizeof(int32_t) * n_mod * d);
        L.slices = take(cmc_gram_slice_bytes(T, d, n_mod));
        L.gram_part = take(cmc_gram_part_bytes(T, d, n_mod));
      }
      if (op == MASQ_OP_CMC) L.gall = take(sizeof(double) * (size_t)(n_mod > 1 ? n_mod - 1 : 1) * d * d);
      if (op != MASQ_OP_CMC_GRAM) {
        L.g = take(sizeof(double) * (size_t)d * d);
        const int64_t ce = cmc_eig_route() ? d : std::min(d, n);     // the eigensolved matrix
        L.c = take(sizeof(double) * (size_t)ce * ce);
        L.lam = take(sizeof(double) * d);
        L.sig2 = take(sizeof(double) * d);
        L.sq = take(sizeof(double) * d);
        L.isq = take(sizeof(double) * d);
        L.dw64 = take(sizeof(double) * (size_t)d * n);
        L.m64 = take(sizeof(double) * (size_t)d * n);
        L.l1t64 = take(sizeof(double) * (size_t)d * r);
        L.urs = take(sizeof(double) * (size_t)d * r);
        L.l2t64 = take(sizeof(double) * (size_t)r * n);
        L.lwork = cmc_syevd_lwork(d, n);
        L.work = take(sizeof(double) * (L.lwork + 1));
        L.info = take(sizeof(int) * 2);
        L.dot = take(sizeof(double) * cmc_dot_blocks());
      }
      break;
    }
    case MASQ_OP_LAYER: {
      const int64_t Tg = grouped_rows(T, n_mod);
      L.inv_s = take(sizeof(float) * n_mod * d);
      L.qx_tok = take((size_t)T * d);
      L.dx_tok = take(sizeof(float) * T);
      L.mask = take(sizeof(uint32_t) * tiles_m);
      L.qx = take((size_t)Tg * d);
      L.dx = take(sizeof(float) * Tg);
      L.perm = take(sizeof(int32_t) * (Tg + route_scratch_ints(T)));
      L.tile_mod = take(sizeof(uint32_t) * (Tg / kUnitM));
      L.cnt = take(sizeof(int64_t) * n_mod);
      L.qw_all = take((size_t)n_mod * n * d);
      L.dw_all = take(sizeof(float) * n_mod * n);
      L.amax = take(2 * sizeof(uint32_t) * n_mod * n);
      L.partials = take(sizeof(double) * (Tg / kUnitM) * ceil_div(n, kTileN) * 16);
      L.fpart = take(sizeof(double) * ceil_div(T, kUnitM) * ceil_div(n, kTileN) * 2);
      L.ipos = take(sizeof(int32_t) * T);
      if (rp > 0 && nnt > 0) {
        L.z = take(sizeof(uint16_t) * (size_t)T * nnt * 2 * rp);
        L.zpart = take(zgemm_part_bytes(T, d, n_mod, (int)rp));
        L.l1t = take(sizeof(uint16_t) * 2 * (size_t)nnt * rp * d);
        L.l2t = take(sizeof(uint16_t) * (size_t)nnt * n * 2 * rp);
      }
      break;
    }
    case MASQ_OP_DECODE:
      L.inv_s = take(sizeof(float) * d);
      L.ids0 = take((size_t)T);
      L.qx = take((size_t)T * d);
      L.dx = take(sizeof(float) * T);
      L.dpart = take(sizeof(float) * (size_t)decode_kchunks(d) * (n / 8) * 128);
      break;
    case MASQ_OP_MEANABS:
      L.partials = take(sizeof(float) * (size_t)meanabs_slabs(T) * n_mod * d);
      break;
    case MASQ_OP_QWEIGHT:
      L.amax = take(2 * sizeof(uint32_t) * n);
      break;
    case MASQ_OP_QACT:
      L.inv_s = take(sizeof(float) * n_mod * d);
      break;
    case MASQ_OP_FORWARD:
      L.inv_s = take(sizeof(float) * n_mod * d);
      L.qx = take((size_t)T * d);
      L.dx = take(sizeof(float) * T);
      L.mask = take(sizeof(uint32_t) * tiles_m);
      if (rp > 0 && nnt > 0) {
        L.z = take(sizeof(uint16_t) * (size_t)T * nnt * 2 * rp);
        L.zpart = take(zgemm_part_bytes(T, d, n_mod, (int)rp));
        L.l1t = take(sizeof(uint16_t) * 2 * (size_t)nnt * rp * d);
        L.l2t = take(sizeof(uint16_t) * (size_t)nnt * n * 2 * rp);
        if (f32_x) L.xsplit = take(sizeof(uint16_t) * 2 * (size_t)T * d);
      }
      break;
    case MASQ_OP_LOSS: {
      const int64_t Tg = grouped_rows(T, n_mod);              // modality-grouped, tile-padded rows
      L.inv_s = take(sizeof(float) * n_mod * d);
      L.qx = take((size_t)Tg * d);
      L.dx = take(sizeof(float) * Tg);
      L.perm = take(sizeof(int32_t) * (Tg + route_scratch_ints(T)));
      L.tile_mod = take(sizeof(uint32_t) * (Tg / kUnitM));
      L.cnt = take(sizeof(int64_t) * n_mod);
      L.qw_all = take((size_t)n_mod * n * d);
      L.dw_all = take(sizeof(float) * n_mod * n);
      L.amax = take(2 * sizeof(uint32_t) * n_mod * n);
      L.partials = take(sizeof(double) * (Tg / kUnitM) * ceil_div(n, kTileN) * 16);
      break;
    }
    case MASQ_OP_REFERENCE:
      break;
    case MASQ_OP_LOSS_GRAD: {
      const int64_t Tg = grouped_rows(T, n_mod);
      L.inv_s = take(sizeof(float) * n_mod * d);
      L.qx = take((size_t)Tg * d);
      L.dx = take(sizeof(float) * Tg);
      L.perm = take(sizeof(int32_t) * (Tg + route_scratch_ints(T)));
      L.tile_mod = take(sizeof(uint32_t) * (Tg / kUnitM));
      L.cnt = take(sizeof(int64_t) * n_mod);
      L.qw_all = take((size_t)n_mod * n * d);
      L.dw_all = take(sizeof(float) * n_mod * n);
      L.amax = take(2 * sizeof(uint32_t) * n_mod * n);
      L.partials = take(sizeof(double) * (Tg / kUnitM) * ceil_div(n, kTileN) * 16);
      L.gsign = take(sizeof(uint16_t) * (size_t)Tg * n);
      L.planes = take(sizeof(uint16_t) * 2 * (size_t)Tg * d);
      L.gpartial = take(sizeof(double) * n_mod * gradgemm_ntiles_j(n) * d);
      L.dq = take((size_t)Tg * d);
      L.de = take(sizeof(float) * Tg);
      L.dq2 = take((size_t)Tg * d);
      L.de2 = take(sizeof(float) * Tg);
      L.apart = take(sizeof(float) * (size_t)Tg * 4 * ceil_div(n, kTileN));
      L.bpart = take(sizeof(float) * (size_t)n_mod * 4 * gradgemm_ntiles_i(d) * n);
      L.kj = take(sizeof(int32_t) * (size_t)n_mod * n);
      const int64_t nkeys = (int64_t)n_mod * n + Tg;
      L.keys = take(sizeof(int32_t) * nkeys);
      L.vals = take(sizeof(double) * nkeys);
      L.bucket = take(sizeof(double) * (size_t)n_mod * d);          // per-channel scale-term contributions
      L.skeys = take(sizeof(uint32_t) * nkeys);
      L.svals = take(sizeof(double) * nkeys);
      L.stemp_bytes = bucket_temp_bytes(nkeys);
      L.stemp = take(L.stemp_bytes);
      break;
    }
    default:
      break;
  }
  // stream-K scratch of the forward / X.W GEMMs (after the op's own regions); only where the
  // GEMM can take the stream-K path (>= 64 k-blocks per unit: d >= 8192 int8, d >= 4096 bf16)
  const bool sk_i8 = d >= (int64_t)gemm_sk_min_kb() * 128, sk_bf = d >= (int64_t)gemm_sk_min_kb() * 64;
  if ((op == MASQ_OP_FORWARD && sk_i8) || (op == MASQ_OP_LAYER && sk_bf) || (op == MASQ_OP_REFERENCE && sk_bf) ||
      (self_ref && sk_bf && (op == MASQ_OP_LOSS || op == MASQ_OP_LOSS_GRAD))) {
    L.skpart = take(gemm_sk_part_bytes());
    L.skflag = take(gemm_sk_flag_bytes());
  }
  // last, so every other offset is the same with and without the flag
  if (self_ref && (op == MASQ_OP_LOSS || op == MASQ_OP_LOSS_GRAD)) L.yref = take(sizeof(float) * (size_t)T * n);
  L.total = off;
  return L;
}

}  // namespace masq

using namespace masq;

namespace {
inline bool al16(const void* p) { return (reinterpret_cast<uintptr_t>(p) & 15u) == 0; }
inline cudaStream_t S(masq_stream s) { return reinterpret_cast<cudaStream_t>(s); }
inline uint8_t* W8(void* ws, size_t off) { return static_cast<uint8_t*>(ws) + off; }
inline uint32_t* status_of(void* ws) { return static_cast<uint32_t*>(ws); }
// the stream-K scratch of a GEMM whose workspace layout has one
inline void set_sk(GemmArgs& g, void* ws, const WsLayout& L) {
  if (L.skpart == 0 || L.skflag == 0) return;
  g.sk_part = reinterpret_cast<uint32_t*>(W8(ws, L.skpart));
  g.sk_flag = reinterpret_cast<uint32_t*>(W8(ws, L.skflag));
}
// MASQ_DEBUG=1 in the environment prints the failing call and the CUDA error to stderr
static bool masq_debug_on() {
  static int on = -1;
  if (on < 0) {
    const char* e = getenv("MASQ_DEBUG");
    on = e && atoi(e) ? 1 : 0;
  }
  return on == 1;
}
#define MASQ_CK(x)                                                                              \
  do {                                                                                          \
    const cudaError_t e_ = (x);                                                                 \
    if (e_ != cudaSuccess) {                                                                    \
      if (masq_debug_on()) fprintf(stderr, "[masq] %s:%d %s -> %s\n", __FILE__, __LINE__, #x,   \
                                   cudaGetErrorString(e_));                                     \
      return MASQ_ERR_CUDA;                                                                     \
    }                                                                                           \
  } while (0)

masq_status check_bits(int32_t b) {
  if (b >= 2 && b <= 8) return MASQ_OK;
  if (b > 8 && b <= 16) return MASQ_ERR_UNSUPPORTED;
  return MASQ_ERR_BITS;
}
masq_status check_common(int64_t T, int64_t d, int32_t n_mod) {
  if (T < 0 || d <= 0 || d % 16 != 0 || d >= (1LL << 31) || T >= (1LL << 31)) return MASQ_ERR_SHAPE;
  if (n_mod < 1 || n_mod > kMaxMod) return MASQ_ERR_SHAPE;
  return MASQ_OK;
}
// A4 with the inverse factors formed inside the bf16 row kernel; where that kernel does not apply
// (f32 X, very wide rows, unaligned X) the inverse factors are computed into inv_ws first
cudaError_t quantize_acts(const void* X, masq_dtype xt, int64_t ld_x, const uint8_t* ids, int64_t T, int64_t d,
                          int n_mod, const float* s, float* inv_ws, int abits, int8_t* qx, float* dx,
                          uint32_t* mask, uint32_t* status, cudaStream_t st) {
  static const bool sep = getenv("MASQ_SEPARATE_INV") != nullptr;   // measurement switch
  cudaError_t e = cudaErrorNotSupported;
  if (!sep) e = launch_aquant(X, xt, ld_x, ids, T, d, n_mod, nullptr, abits, qx, dx, mask, status, st, nullptr, -1, s);
  if (e != cudaErrorNotSupported) return e;
  e = launch_inv(s, (int64_t)n_mod * d, inv_ws, st);
  if (e != cudaSuccess) return e;
  return launch_aquant(X, xt, ld_x, ids, T, d, n_mod, inv_ws, abits, qx, dx, mask, status, st);
}

masq_status check_x(const void* X, masq_dtype xt, int64_t ld_x, int64_t d) {
  if (!X) return MASQ_ERR_NULL;
  if (xt != MASQ_BF16 && xt != MASQ_F32) return MASQ_ERR_UNSUPPORTED;
  if (ld_x < d) return MASQ_ERR_SHAPE;
  const int64_t bytes = ld_x * (xt == MASQ_BF16 ? 2 : 4);
  if (bytes % 16 != 0 || !al16(X)) return MASQ_ERR_ALIGN;
  return MASQ_OK;
}
masq_status check_ws(void* ws, size_t ws_bytes, const WsLayout& L) {
  if (!ws) return MASQ_ERR_WORKSPACE;
  if (ws_bytes < L.total || (reinterpret_cast<uintptr_t>(ws) & 255u) != 0) return MASQ_ERR_WORKSPACE;
  return MASQ_OK;
}
#define MASQ_TRY(x)                  \
  do {                               \
    masq_status s_ = (x);            \
    if (s_ != MASQ_OK) return s_;    \
  } while (0)
}  // namespace

extern "C" {

size_t masq_workspace_size(int32_t op, int64_t T, int64_t d, int64_t d_out, int32_t n_mod, int32_t r) {
  return ws_layout(op, T, d, d_out, n_mod, r).total;
}

masq_status masq_calibrate_stats(const void* X, masq_dtype xt, int64_t ld_x, const uint8_t* mod_id, int64_t T,
                                 int64_t d, int32_t n_mod, float* R, int64_t* count, int32_t reset, void* ws,
                                 size_t ws_bytes, masq_stream stream) {
  MASQ_TRY(check_common(T, d, n_mod));
  if (!R || !count) return MASQ_ERR_NULL;
  if (T > 0) {
    MASQ_TRY(check_x(X, xt, ld_x, d));
    if (!mod_id) return MASQ_ERR_NULL;
  }
  const WsLayout L = ws_layout(MASQ_OP_STATS, T, d, 0, n_mod, 0);
  MASQ_TRY(check_ws(ws, ws_bytes, L));
  if (reset) {
    MASQ_CK(cudaMemsetAsync(R, 0, sizeof(float) * n_mod * d, S(stream)));
    MASQ_CK(cudaMemsetAsync(count, 0, sizeof(int64_t) * n_mod, S(stream)));
  }
  MASQ_CK(launch_stats(X, xt, ld_x, mod_id, T, d, n_mod, R, count, status_of(ws), S(stream)));
  return MASQ_OK;
}

masq_status masq_init_factors(const float* R, const int64_t* count, const void* W, masq_dtype wt, int64_t d,
                              int64_t d_out, int32_t n_mod, float* s, float* wmax_out, void* ws, size_t ws_bytes,
                              masq_stream stream) {
  MASQ_TRY(check_common(0, d, n_mod));
  if (!R || !count || !W || !s) return MASQ_ERR_NULL;
  if (d_out <= 0 || d_out % 32 != 0) return MASQ_ERR_SHAPE;
  if (wt != MASQ_BF16 && wt != MASQ_F32) return MASQ_ERR_UNSUPPORTED;
  if (!al16(W)) return MASQ_ERR_ALIGN;
  MASQ_TRY(check_ws(ws, ws_bytes, ws_layout(MASQ_OP_INIT, 0, d, d_out, n_mod, 0)));
  MASQ_CK(launch_init(R, count, W, wt, d, d_out, n_mod, s, wmax_out, status_of(ws), S(stream)));
  return MASQ_OK;
}

masq_status masq_quantize_weight(const void* W, masq_dtype wt, const float* s, int64_t d, int64_t d_out,
                                 int32_t wbits, int8_t* qw, float* dw, void* ws, size_t ws_bytes,
                                 masq_stream stream) {
  MASQ_TRY(check_common(0, d, 1));
  MASQ_TRY(check_bits(wbits));
  if (!W || !s || !qw || !dw) return MASQ_ERR_NULL;
  if (d_out <= 0 || d_out % 32 != 0) return MASQ_ERR_SHAPE;
  if (wt != MASQ_BF16 && wt != MASQ_F32) return MASQ_ERR_UNSUPPORTED;
  if (!al16(W) || !al16(qw)) return MASQ_ERR_ALIGN;
  const WsLayout L = ws_layout(MASQ_OP_QWEIGHT, 0, d, d_out, 1, 0);
  MASQ_TRY(check_ws(ws, ws_bytes, L));
  MASQ_CK(launch_wquant(W, wt, s, 1, d, d_out, wbits, qw, dw, reinterpret_cast<uint32_t*>(W8(ws, L.amax)),
                        S(stream)));
  return MASQ_OK;
}

masq_status masq_quantize_activations(const void* X, masq_dtype xt, int64_t ld_x, const uint8_t* mod_id, int64_t T,
                                      int64_t d, int32_t n_mod, const float* s, int32_t abits, int8_t* qx,
                                      float* dx, uint32_t* tile_mask, void* ws, size_t ws_bytes,
                                      masq_stream stream) {
  MASQ_TRY(check_common(T, d, n_mod));
  MASQ_TRY(check_bits(abits));
  if (T == 0) return MASQ_OK;
  MASQ_TRY(check_x(X, xt, ld_x, d));
  if (!mod_id || !s || !qx || !dx) return MASQ_ERR_NULL;
  if (!al16(qx) || !al16(s)) return MASQ_ERR_ALIGN;
  const WsLayout L = ws_layout(MASQ_OP_QACT, T, d, 0, n_mod, 0);
  MASQ_TRY(check_ws(ws, ws_bytes, L));
  float* inv = reinterpret_cast<float*>(W8(ws, L.inv_s));
  MASQ_CK(quantize_acts(X, xt, ld_x, mod_id, T, d, n_mod, s, inv, abits, qx, dx, tile_mask, status_of(ws), S(stream)));
  return MASQ_OK;
}

masq_status masq_linear_forward(const void* X, masq_dtype xt, int64_t ld_x, const uint8_t* mod_id, int64_t T,
                                int64_t d, int64_t d_out, int32_t n_mod, const float* s, const int8_t* qw,
                                const float* dw, int32_t wbits, int32_t abits, const void* L1, const void* L2,
                                int64_t ld_l2, int32_t r, float* Y, int64_t ld_y, void* ws, size_t ws_bytes,
                                const masq_debug* dbg, masq_stream stream) {
  MASQ_TRY(check_common(T, d, n_mod));
  MASQ_TRY(check_bits(wbits));
  MASQ_TRY(check_bits(abits));
  if (d_out <= 0 || d_out % 32 != 0 || d_out >= (1LL << 31)) return MASQ_ERR_SHAPE;
  if (r < 0 || r > 256 || r % 16 != 0) return MASQ_ERR_SHAPE;
  const bool use_acc = dbg && dbg->acc;
  if (!s || !qw || !dw || (!Y && !use_acc)) return MASQ_ERR_NULL;
  const bool cmc = r > 0 && n_mod > 1 && !use_acc;
  if (cmc) {
    if (!L1 || !L2) return MASQ_ERR_NULL;
    if (ld_l2 < d_out || !al16(L1) || !al16(L2) || (ld_l2 % 8) != 0) return MASQ_ERR_ALIGN;
  }
  float* out = use_acc ? reinterpret_cast<float*>(dbg->acc) : Y;
  const int64_t ld_out = use_acc ? dbg->ld_acc : ld_y;
  if (ld_out < d_out || ld_out % 4 != 0 || !al16(out)) return MASQ_ERR_ALIGN;
  if (!al16(qw) || !al16(dw) || !al16(s)) return MASQ_ERR_ALIGN;
  if (T == 0) return MASQ_OK;
  MASQ_TRY(check_x(X, xt, ld_x, d));
  if (!mod_id) return MASQ_ERR_NULL;
  const WsLayout L = ws_layout(MASQ_OP_FORWARD, T, d, d_out, n_mod, cmc ? r : 0, xt == MASQ_F32);
  MASQ_TRY(check_ws(ws, ws_bytes, L));
  cudaStream_t st = S(stream);
  float* inv = reinterpret_cast<float*>(W8(ws, L.inv_s));
  int8_t* qx = reinterpret_cast<int8_t*>(W8(ws, L.qx));
  float* dx = reinterpret_cast<float*>(W8(ws, L.dx));
  uint32_t* mask = reinterpret_cast<uint32_t*>(W8(ws, L.mask));
  // the CMC path's tile masks come from the factor packing below (no zeroing pass, no atomics)
  MASQ_CK(quantize_acts(X, xt, ld_x, mod_id, T, d, n_mod, s, inv, abits, qx, dx, nullptr, status_of(ws), st));
  if (dbg && dbg->qx) MASQ_CK(cudaMemcpyAsync(dbg->qx, qx, (size_t)T * d, cudaMemcpyDeviceToDevice, st));
  if (dbg && dbg->dx) MASQ_CK(cudaMemcpyAsync(dbg->dx, dx, sizeof(float) * T, cudaMemcpyDeviceToDevice, st));
  GemmArgs g{};
  set_sk(g, ws, L);
  g.mode = use_acc ? kModeAcc : kModeFwd;
  g.T = T;
  g.n = d_out;
  g.d = d;
  g.qx = qx;
  g.b = qw;
  g.b_rows = d_out;
  g.dx = dx;
  g.dw = dw;
  g.tile_mask = cmc ? mask : nullptr;
  g.n_mod = n_mod;
  g.out = out;
  g.ld_out = ld_out;
  if (cmc) {
    const int rp = (int)rpad_of(r);
    uint16_t* l1t = reinterpret_cast<uint16_t*>(W8(ws, L.l1t));
    uint16_t* l2t = reinterpret_cast<uint16_t*>(W8(ws, L.l2t));
    uint16_t* z = reinterpret_cast<uint16_t*>(W8(ws, L.z));
    MASQ_CK(launch_cmc_pack(static_cast<const uint16_t*>(L1), s, d, r, rp, n_mod - 1, l1t,
                            static_cast<const uint16_t*>(L2), ld_l2, d_out, l2t, mod_id, T, n_mod, mask, st));
    if (xt == MASQ_BF16) {
      MASQ_CK(launch_zgemm(static_cast<const uint16_t*>(X), ld_x, nullptr, mod_id, T, d, n_mod, l1t, rp, mask, z, st, reinterpret_cast<float*>(W8(ws, L.zpart))));
    } else {
      uint16_t* xh = reinterpret_cast<uint16_t*>(W8(ws, L.xsplit));
      uint16_t* xl = xh + (size_t)T * d;
      MASQ_CK(launch_split_f32(static_cast<const float*>(X), ld_x, T, d, xh, xl, st));
      MASQ_CK(launch_zgemm(xh, d, xl, mod_id, T, d, n_mod, l1t, rp, mask, z, st, reinterpret_cast<float*>(W8(ws, L.zpart))));
    }
    g.rpad = rp;
    g.z = z;
    g.l2t = l2t;
  }
  MASQ_CK(launch_gemm(g, st));
  return MASQ_OK;
}

masq_status masq_calib_layer(const void* X, int64_t ld_x, const uint8_t* mod_id, int64_t T, int64_t d, int64_t d_out,
                             int32_t n_mod, const float* s, const void* W, int32_t wbits, int32_t abits, const void* L1,
                             const void* L2, int64_t ld_l2, int32_t r, const float* lambda, float* Y, int64_t ld_y,
                             float* Yref, int64_t ld_ref, int8_t* qw_text, float* dw_text, double* sums,
                             int64_t* counts, double* loss, void* ws, size_t ws_bytes, masq_stream stream) {
  MASQ_TRY(check_common(T, d, n_mod));
  MASQ_TRY(check_bits(wbits));
  MASQ_TRY(check_bits(abits));
  if (d_out <= 0 || d_out % 32 != 0 || d_out >= (1LL << 31)) return MASQ_ERR_SHAPE;
  if (r < 0 || r > 256 || r % 16 != 0) return MASQ_ERR_SHAPE;
  if (!s || !W || !Y || !Yref || !sums || !counts || !loss) return MASQ_ERR_NULL;
  const bool cmc = r > 0 && n_mod > 1;
  if (cmc) {
    if (!L1 || !L2) return MASQ_ERR_NULL;
    if (ld_l2 < d_out || !al16(L1) || !al16(L2) || (ld_l2 % 8) != 0) return MASQ_ERR_ALIGN;
  }
  if (ld_y < d_out || ld_y % 4 != 0 || !al16(Y)) return MASQ_ERR_ALIGN;
  if (ld_ref < d_out || ld_ref % 4 != 0 || !al16(Yref)) return MASQ_ERR_ALIGN;
  if (!al16(W) || !al16(s)) return MASQ_ERR_ALIGN;
  if ((qw_text && !al16(qw_text)) || (dw_text && !al16(dw_text))) return MASQ_ERR_ALIGN;
  const WsLayout L = ws_layout(MASQ_OP_LAYER, T, d, d_out, n_mod, cmc ? r : 0);
  MASQ_TRY(check_ws(ws, ws_bytes, L));
  cudaStream_t st = S(stream);
  if (T == 0) {
    MASQ_CK(cudaMemsetAsync(sums, 0, sizeof(double) * n_mod, st));
    MASQ_CK(cudaMemsetAsync(counts, 0, sizeof(int64_t) * n_mod, st));
    MASQ_CK(cudaMemsetAsync(loss, 0, sizeof(double), st));
    return MASQ_OK;
  }
  MASQ_TRY(check_x(X, MASQ_BF16, ld_x, d));
  if (!mod_id) return MASQ_ERR_NULL;
  float* inv = reinterpret_cast<float*>(W8(ws, L.inv_s));
  int8_t* qt = reinterpret_cast<int8_t*>(W8(ws, L.qx_tok));
  float* dt = reinterpret_cast<float*>(W8(ws, L.dx_tok));
  uint32_t* mask = reinterpret_cast<uint32_t*>(W8(ws, L.mask));
  int8_t* qg = reinterpret_cast<int8_t*>(W8(ws, L.qx));
  float* dg = reinterpret_cast<float*>(W8(ws, L.dx));
  int32_t* perm = reinterpret_cast<int32_t*>(W8(ws, L.perm));
  uint32_t* tmod = reinterpret_cast<uint32_t*>(W8(ws, L.tile_mod));
  int64_t* cnt = reinterpret_cast<int64_t*>(W8(ws, L.cnt));
  int8_t* qw = reinterpret_cast<int8_t*>(W8(ws, L.qw_all));
  float* dw = reinterpret_cast<float*>(W8(ws, L.dw_all));
  uint32_t* amax = reinterpret_cast<uint32_t*>(W8(ws, L.amax));
  double* partials = reinterpret_cast<double*>(W8(ws, L.partials));
  const int64_t Tg = grouped_rows(T, n_mod);
  const int num_n = (int)ceil_div(d_out, kTileN);
  const int64_t tiles = (Tg / kUnitM) * num_n;
  const int epi = gemm_epilogue_warps();
  // shared front half: factors, routing, every modality's weight codes (set 0 = the forward's
  // Q(S_t W)), the token-order activation codes (forward) and their grouped copy (loss)
  int32_t* ipos = reinterpret_cast<int32_t*>(W8(ws, L.ipos));
  MASQ_CK(launch_route(mod_id, T, n_mod, perm, tmod, cnt, st, ipos));
  MASQ_CK(launch_wquant(W, MASQ_BF16, s, n_mod, d, d_out, wbits, qw, dw, amax, st));
  // the loss GEMM below skips the text units, so only the non-text rows need the grouped copy;
  // the row kernel forms 1/s itself (no inverse-factor launch)
  const cudaError_t qe = launch_aquant_dual(X, MASQ_BF16, ld_x, mod_id, T, d, n_mod, nullptr, abits, qt, dt, nullptr,
                                            status_of(ws), perm, tmod, ipos, Tg, qg, dg, st, s);
  if (qe == cudaErrorNotSupported) {
    MASQ_CK(launch_inv(s, (int64_t)n_mod * d, inv, st));
    MASQ_CK(launch_aquant(X, MASQ_BF16, ld_x, mod_id, T, d, n_mod, inv, abits, qt, dt, nullptr, status_of(ws), st));
    MASQ_CK(launch_gather_rows(qt, dt, perm, Tg, d, qg, dg, st));
  } else {
    MASQ_CK(qe);
  }
  // A8 target first: the forward's epilogue reads it for the text rows
  GemmArgs gr{};
  set_sk(gr, ws, L);
  gr.mode = kModeRef;
  gr.T = T;
  gr.n = d_out;
  gr.d = d;
  gr.xbf = static_cast<const uint16_t*>(X);
  gr.ld_x = ld_x;
  gr.b = W;
  gr.b_rows = d;
  gr.n_mod = 1;
  gr.out = Yref;
  gr.ld_out = ld_ref;
  MASQ_CK(launch_gemm(gr, st));
  // A4-A7 forward; text rows' output is also the loss's quantized output (S_0 = S_t), so the
  // epilogue sums their |y - yref| and the loss GEMM below skips the text units
  double* fpart = reinterpret_cast<double*>(W8(ws, L.fpart));
  const int64_t fwd_units = ceil_div(T, kUnitM) * num_n;
  GemmArgs g{};
  set_sk(g, ws, L);
  g.mode = kModeFwd;
  g.T = T;
  g.n = d_out;
  g.d = d;
  g.qx = qt;
  g.b = qw;
  g.b_rows = d_out;
  g.dx = dt;
  g.dw = dw;
  g.tile_mask = cmc ? mask : nullptr;
  g.n_mod = n_mod;
  g.out = Y;
  g.ld_out = ld_y;
  g.ids = mod_id;
  g.fwd_loss = 1;
  g.yref = Yref;
  g.ld_ref = ld_ref;
  g.partials = fpart;
  if (cmc) {
    const int rp = (int)rpad_of(r);
    uint16_t* l1t = reinterpret_cast<uint16_t*>(W8(ws, L.l1t));
    uint16_t* l2t = reinterpret_cast<uint16_t*>(W8(ws, L.l2t));
    uint16_t* z = reinterpret_cast<uint16_t*>(W8(ws, L.z));
    MASQ_CK(launch_cmc_pack(static_cast<const uint16_t*>(L1), s, d, r, rp, n_mod - 1, l1t,
                            static_cast<const uint16_t*>(L2), ld_l2, d_out, l2t, mod_id, T, n_mod, mask, st));
    MASQ_CK(launch_zgemm(static_cast<const uint16_t*>(X), ld_x, nullptr, mod_id, T, d, n_mod, l1t, rp, mask, z, st, reinterpret_cast<float*>(W8(ws, L.zpart))));
    g.rpad = rp;
    g.z = z;
    g.l2t = l2t;
  }
  MASQ_CK(launch_gemm(g, st));
  // no zeroing of the loss partials: the loss GEMM writes both slots of every unit it runs, and
  // the units it skips (text, skip_m0; padding) are skipped by the reduction too (m_lo = 1)
  GemmArgs gl{};
  gl.mode = kModeLoss;
  gl.T = Tg;
  gl.n = d_out;
  gl.d = d;
  gl.qx = qg;
  gl.b = qw;
  gl.b_rows = (int64_t)n_mod * d_out;
  gl.dx = dg;
  gl.dw = dw;
  gl.tile_mask = tmod;
  gl.perm = perm;
  gl.n_mod = n_mod;
  gl.yref = Yref;
  gl.ld_ref = ld_ref;
  gl.partials = partials;
  gl.skip_m0 = 1;
  MASQ_CK(launch_gemm(gl, st));
  MASQ_CK(launch_loss_reduce(partials, tiles, num_n, epi, tmod, cnt, n_mod, d_out, lambda, sums, counts, loss, st,
                             fpart, fwd_units * 2, partials + tiles * epi, tiles * (16 - epi), 1));
  if (qw_text) MASQ_CK(cudaMemcpyAsync(qw_text, qw, (size_t)d_out * d, cudaMemcpyDeviceToDevice, st));
  if (dw_text) MASQ_CK(cudaMemcpyAsync(dw_text, dw, sizeof(float) * d_out, cudaMemcpyDeviceToDevice, st));
  return MASQ_OK;
}

masq_status masq_reference_output(const void* X, int64_t ld_x, const void* W, int64_t T, int64_t d, int64_t d_out,
                                  float* Yref, int64_t ld_ref, void* ws, size_t ws_bytes, masq_stream stream) {
  MASQ_TRY(check_common(T, d, 1));
  if (d_out <= 0 || d_out % 32 != 0) return MASQ_ERR_SHAPE;
  if (!W || !Yref) return MASQ_ERR_NULL;
  if (ld_ref < d_out || ld_ref % 4 != 0 || !al16(Yref) || !al16(W)) return MASQ_ERR_ALIGN;
  if (T == 0) return MASQ_OK;
  MASQ_TRY(check_x(X, MASQ_BF16, ld_x, d));
  const WsLayout L = ws_layout(MASQ_OP_REFERENCE, T, d, d_out, 1, 0);
  MASQ_TRY(check_ws(ws, ws_bytes, L));
  GemmArgs g{};
  set_sk(g, ws, L);
  g.mode = kModeRef;
  g.T = T;
  g.n = d_out;
  g.d = d;
  g.xbf = static_cast<const uint16_t*>(X);
  g.ld_x = ld_x;
  g.b = W;                                              // read as stored (MN-major B operand)
  g.b_rows = d;
  g.n_mod = 1;
  g.out = Yref;
  g.ld_out = ld_ref;
  MASQ_CK(launch_gemm(g, S(stream)));
  return MASQ_OK;
}

}  // extern "C"

namespace {
masq_status loss_core(const void* X, masq_dtype xt, int64_t ld_x, const uint8_t* mod_id, int64_t T, int64_t d,
                      int64_t d_out, int32_t n_mod, const float* s, const void* W, masq_dtype wt, int32_t wbits,
                      int32_t abits, const float* lambda, const float* Yref, int64_t ld_ref, double* sums,
                      int64_t* counts, double* loss, double* grad, const int64_t* count_norm, void* ws,
                      size_t ws_bytes, masq_stream stream) {
  MASQ_TRY(check_common(T, d, n_mod));
  MASQ_TRY(check_bits(wbits));
  MASQ_TRY(check_bits(abits));
  if (d_out <= 0 || d_out % 32 != 0) return MASQ_ERR_SHAPE;
  if (!s || !W || !sums || !counts || !loss) return MASQ_ERR_NULL;
  if (wt != MASQ_BF16 && wt != MASQ_F32) return MASQ_ERR_UNSUPPORTED;
  if (grad && (xt != MASQ_BF16 || wt != MASQ_BF16)) return MASQ_ERR_UNSUPPORTED;
  if (!al16(W) || !al16(s)) return MASQ_ERR_ALIGN;
  const WsLayout L = ws_layout(grad ? MASQ_OP_LOSS_GRAD : MASQ_OP_LOSS, T, d, d_out, n_mod, 0);
  MASQ_TRY(check_ws(ws, ws_bytes, L));
  cudaStream_t st = S(stream);
  if (T == 0) {
    MASQ_CK(cudaMemsetAsync(sums, 0, sizeof(double) * n_mod, st));
    MASQ_CK(cudaMemsetAsync(counts, 0, sizeof(int64_t) * n_mod, st));
    MASQ_CK(cudaMemsetAsync(loss, 0, sizeof(double), st));
    if (grad) MASQ_CK(cudaMemsetAsync(grad, 0, sizeof(double) * n_mod * d, st));
    return MASQ_OK;
  }
  MASQ_TRY(check_x(X, xt, ld_x, d));
  if (!mod_id) return MASQ_ERR_NULL;
  if (!Yref) {
    // the target X_m W is part of the loss; without a caller-supplied Yref it is
    // computed here (bf16 tensor-core products, fp32 accumulation, reading Q16) into the
    // workspace, which must then be sized with MASQ_OP_SELF_REF
    if (xt != MASQ_BF16 || wt != MASQ_BF16) return MASQ_ERR_UNSUPPORTED;
    const WsLayout Ls = ws_layout((grad ? MASQ_OP_LOSS_GRAD : MASQ_OP_LOSS) | MASQ_OP_SELF_REF, T, d, d_out, n_mod, 0);
    MASQ_TRY(check_ws(ws, ws_bytes, Ls));
    float* yr = reinterpret_cast<float*>(W8(ws, Ls.yref));
    GemmArgs gr{};
    set_sk(gr, ws, Ls);
    gr.mode = kModeRef;
    gr.T = T;
    gr.n = d_out;
    gr.d = d;
    gr.xbf = static_cast<const uint16_t*>(X);
    gr.ld_x = ld_x;
    gr.b = W;
    gr.b_rows = d;
    gr.n_mod = 1;
    gr.out = yr;
    gr.ld_out = d_out;
    MASQ_CK(launch_gemm(gr, st));
    Yref = yr;
    ld_ref = d_out;
  }
  if (ld_ref < d_out || ld_ref % 4 != 0 || !al16(Yref)) return MASQ_ERR_ALIGN;
  float* inv = reinterpret_cast<float*>(W8(ws, L.inv_s));
  int8_t* qx = reinterpret_cast<int8_t*>(W8(ws, L.qx));
  float* dx = reinterpret_cast<float*>(W8(ws, L.dx));
  int32_t* perm = reinterpret_cast<int32_t*>(W8(ws, L.perm));
  uint32_t* tmod = reinterpret_cast<uint32_t*>(W8(ws, L.tile_mod));
  int64_t* cnt = reinterpret_cast<int64_t*>(W8(ws, L.cnt));
  int8_t* qw = reinterpret_cast<int8_t*>(W8(ws, L.qw_all));
  float* dw = reinterpret_cast<float*>(W8(ws, L.dw_all));
  uint32_t* amax = reinterpret_cast<uint32_t*>(W8(ws, L.amax));
  double* partials = reinterpret_cast<double*>(W8(ws, L.partials));
  uint16_t* gsign = grad ? reinterpret_cast<uint16_t*>(W8(ws, L.gsign)) : nullptr;
  const int64_t Tg = grouped_rows(T, n_mod);
  const int num_n = (int)ceil_div(d_out, kTileN);
  const int64_t tiles = (Tg / kUnitM) * num_n;
  const int epi = gemm_epilogue_warps();
  MASQ_CK(launch_inv(s, (int64_t)n_mod * d, inv, st));
  MASQ_CK(launch_route(mod_id, T, n_mod, perm, tmod, cnt, st));
  MASQ_CK(launch_aquant(X, xt, ld_x, mod_id, T, d, n_mod, inv, abits, qx, dx, nullptr, status_of(ws), st, perm, Tg));
  MASQ_CK(launch_wquant(W, wt, s, n_mod, d, d_out, wbits, qw, dw, amax, st));
  MASQ_CK(cudaMemsetAsync(partials, 0, sizeof(double) * tiles * epi, st));
  GemmArgs g{};
  g.mode = kModeLoss;
  g.T = Tg;
  g.n = d_out;
  g.d = d;
  g.qx = qx;
  g.b = qw;
  g.b_rows = (int64_t)n_mod * d_out;
  g.dx = dx;
  g.dw = dw;
  g.tile_mask = tmod;
  g.perm = perm;
  g.n_mod = n_mod;
  g.yref = Yref;
  g.ld_ref = ld_ref;
  g.partials = partials;
  g.gsign = gsign;
  MASQ_CK(launch_gemm(g, st));
  MASQ_CK(launch_loss_reduce(partials, tiles, num_n, epi, tmod, cnt, n_mod, d_out, lambda, sums, counts, loss, st,
                             nullptr, 0, partials + tiles * epi, tiles * (16 - epi)));
  if (grad) {
    uint16_t* planes = reinterpret_cast<uint16_t*>(W8(ws, L.planes));
    double* gpart = reinterpret_cast<double*>(W8(ws, L.gpartial));
    int8_t* dq = reinterpret_cast<int8_t*>(W8(ws, L.dq));
    float* de = reinterpret_cast<float*>(W8(ws, L.de));
    float* apart = reinterpret_cast<float*>(W8(ws, L.apart));
    float* bpart = reinterpret_cast<float*>(W8(ws, L.bpart));
    int32_t* kj = reinterpret_cast<int32_t*>(W8(ws, L.kj));
    int32_t* keys = reinterpret_cast<int32_t*>(W8(ws, L.keys));
    double* vals = reinterpret_cast<double*>(W8(ws, L.vals));
    double* bucket = reinterpret_cast<double*>(W8(ws, L.bucket));
    const int64_t nj = (int64_t)n_mod * d_out, nkeys = nj + Tg;
    int32_t* ktkey = keys + nj;
    const uint32_t* colmax = amax;                     // first half of the scratch: column maxima
    int8_t* dq2 = reinterpret_cast<int8_t*>(W8(ws, L.dq2));
    float* de2 = reinterpret_cast<float*>(W8(ws, L.de2));
    MASQ_CK(launch_gradprep(static_cast<const uint16_t*>(X), ld_x, mod_id, perm, qx, dx, inv, Tg, d, abits, planes,
                            ktkey, dq, de, dq2, de2, st));
    MASQ_CK(cudaMemsetAsync(kj, 0x7F, sizeof(int32_t) * nj, st));
    MASQ_CK(launch_gradgemm(planes, Tg, gsign, qw, tmod, n_mod, d, d_out, s, inv, static_cast<const uint16_t*>(W), dw,
                            colmax, gpart, bpart, kj, st));
    GemmArgs ga{};
    ga.mode = kModeAlphaI8;                            // D (int8, row step Delta_t / 254) . codes^T
    ga.T = Tg;
    ga.n = d_out;
    ga.d = d;
    ga.qx = dq;
    ga.b = qw;
    ga.b_rows = (int64_t)n_mod * d_out;
    ga.dx = de;
    ga.dw = dw;
    ga.tile_mask = tmod;
    ga.n_mod = n_mod;
    ga.gsign = gsign;
    ga.apart = apart;
    ga.apart_ld = 4 * num_n;
    ga.apart_off = 0;
    MASQ_CK(launch_gemm(ga, st));
    ga.qx = dq2;                                       // the residual's codes on the step e_t / 254
    ga.dx = de2;
    ga.apart_off = 2 * num_n;
    MASQ_CK(launch_gemm(ga, st));
    MASQ_CK(launch_gradkeys(bpart, 4 * gradgemm_ntiles_i(d), kj, colmax, wbits, apart, 4 * num_n, ktkey, n_mod, d,
                            d_out, Tg, keys, vals, st));
    MASQ_CK(launch_bucket(keys, vals, nkeys, (int64_t)n_mod * d, reinterpret_cast<uint32_t*>(W8(ws, L.skeys)),
                          reinterpret_cast<double*>(W8(ws, L.svals)), W8(ws, L.stemp), L.stemp_bytes, bucket, st));
    MASQ_CK(launch_gradreduce(gpart, bucket, count_norm ? count_norm : cnt, lambda, n_mod,
                              gradgemm_ntiles_j(d_out), d, d_out, grad, st));
  }
  return MASQ_OK;
}
}  // namespace

extern "C" {

masq_status masq_calib_loss(const void* X, masq_dtype xt, int64_t ld_x, const uint8_t* mod_id, int64_t T, int64_t d,
                            int64_t d_out, int32_t n_mod, const float* s, const void* W, masq_dtype wt,
                            int32_t wbits, int32_t abits, const float* lambda, const float* Yref, int64_t ld_ref,
                            double* sums, int64_t* counts, double* loss, void* ws, size_t ws_bytes,
                            masq_stream stream) {
  return loss_core(X, xt, ld_x, mod_id, T, d, d_out, n_mod, s, W, wt, wbits, abits, lambda, Yref, ld_ref, sums,
                   counts, loss, nullptr, nullptr, ws, ws_bytes, stream);
}

masq_status masq_calib_loss_grad(const void* X, masq_dtype xt, int64_t ld_x, const uint8_t* mod_id, int64_t T,
                                 int64_t d, int64_t d_out, int32_t n_mod, const float* s, const void* W,
                                 masq_dtype wt, int32_t wbits, int32_t abits, const float* lambda, const float* Yref,
                                 int64_t ld_ref, double* sums, int64_t* counts, double* loss, double* grad,
                                 const int64_t* count_norm, void* ws, size_t ws_bytes, masq_stream stream) {
  if (!grad) return MASQ_ERR_NULL;
  return loss_core(X, xt, ld_x, mod_id, T, d, d_out, n_mod, s, W, wt, wbits, abits, lambda, Yref, ld_ref, sums,
                   counts, loss, grad, count_norm, ws, ws_bytes, stream);
}

masq_status masq_adam_step(double* theta, const double* grad, double* m1, double* m2, int64_t count, int32_t step,
                           double lr, double beta1, double beta2, double eps, float* s_out, masq_stream stream) {
  if (!theta || !grad || !m1 || !m2) return MASQ_ERR_NULL;
  if (count < 0 || step < 1) return MASQ_ERR_SHAPE;
  if (count == 0) return MASQ_OK;
  MASQ_CK(launch_adam(theta, grad, m1, m2, count, step, lr, beta1, beta2, eps, s_out, S(stream)));
  return MASQ_OK;
}

masq_status masq_adam_init(const float* s, double* theta, double* m1, double* m2, int64_t count,
                           masq_stream stream) {
  if (!s || !theta || !m1 || !m2) return MASQ_ERR_NULL;
  if (count < 0) return MASQ_ERR_SHAPE;
  if (count == 0) return MASQ_OK;
  MASQ_CK(launch_adam_init(s, theta, m1, m2, count, S(stream)));
  return MASQ_OK;
}

masq_status masq_keep_best(const double* loss, double* best_loss, const float* s, float* s_best, int64_t count,
                           int32_t* improved, masq_stream stream) {
  if (!loss || !best_loss || !s || !s_best) return MASQ_ERR_NULL;
  if (count < 0) return MASQ_ERR_SHAPE;
  MASQ_CK(launch_keep_best(loss, best_loss, s, s_best, count, improved, S(stream)));
  return MASQ_OK;
}

namespace {
CmcArgs cmc_factor_args(const WsLayout& L, void* ws, int64_t d, int64_t d_out, int32_t n_mod, const float* s,
                        const void* W, masq_dtype wt, const int8_t* qw_text, const float* dw_text, int32_t r,
                        double eps_rel, void* L1, void* L2, masq_dtype lt, double* resid) {
  CmcArgs a{};
  a.d = d;
  a.n = d_out;
  a.n_mod = n_mod;
  a.r = r;
  a.s = s;
  a.W = W;
  a.wt = wt;
  a.qw_t = qw_text;
  a.dw_t = dw_text;
  a.eps_rel = eps_rel;
  a.L1 = L1;
  a.L2 = L2;
  a.lt = lt;
  a.resid = resid;
  a.G = reinterpret_cast<double*>(W8(ws, L.g));
  a.C = reinterpret_cast<double*>(W8(ws, L.c));
  a.lam = reinterpret_cast<double*>(W8(ws, L.lam));
  a.sig2 = reinterpret_cast<double*>(W8(ws, L.sig2));
  a.sq = reinterpret_cast<double*>(W8(ws, L.sq));
  a.isq = reinterpret_cast<double*>(W8(ws, L.isq));
  a.dW = reinterpret_cast<double*>(W8(ws, L.dw64));
  a.Mb = reinterpret_cast<double*>(W8(ws, L.m64));
  a.L1t = reinterpret_cast<double*>(W8(ws, L.l1t64));
  a.Urs = reinterpret_cast<double*>(W8(ws, L.urs));
  a.L2t = reinterpret_cast<double*>(W8(ws, L.l2t64));
  a.work = reinterpret_cast<double*>(W8(ws, L.work));
  a.info = reinterpret_cast<int*>(W8(ws, L.info));
  a.dot = reinterpret_cast<double*>(W8(ws, L.dot));
  a.lwork = L.lwork;
  return a;
}

masq_status cmc_factor_checks(int64_t d, int64_t d_out, int32_t n_mod, const float* s, const void* W, masq_dtype wt,
                              const int8_t* qw_text, const float* dw_text, int32_t r, double eps_rel,
                              const void* L1, const void* L2, masq_dtype lt) {
  MASQ_TRY(check_common(0, d, n_mod));
  if (n_mod < 2) return MASQ_ERR_SHAPE;
  if (d_out <= 0 || r < 1 || r > d || r > d_out || !(eps_rel >= 0.0)) return MASQ_ERR_SHAPE;
  if (d > 2147483647 / 8 || d_out > 2147483647 / 8) return MASQ_ERR_SHAPE;
  if (!s || !W || !qw_text || !dw_text || !L1 || !L2) return MASQ_ERR_NULL;
  if (wt != MASQ_BF16 && wt != MASQ_F32) return MASQ_ERR_UNSUPPORTED;
  if (lt != MASQ_BF16 && lt != MASQ_F32) return MASQ_ERR_UNSUPPORTED;
  if (!cmc_linalg_available()) return MASQ_ERR_UNSUPPORTED;
  return MASQ_OK;
}

masq_status cmc_gram_core(const void* X, masq_dtype xt, int64_t ld_x, const uint8_t* mod_id, int64_t T, int64_t d,
                          int32_t n_mod, const float* s, double* G, int32_t accumulate, const WsLayout& L, void* ws,
                          cudaStream_t st) {
  CmcArgs a{};
  a.X = X;
  a.xt = xt;
  a.ld_x = ld_x;
  a.ids = mod_id;
  a.T = T;
  a.d = d;
  a.n_mod = n_mod;
  a.inv = reinterpret_cast<float*>(W8(ws, L.inv_s));
  a.perm = reinterpret_cast<int32_t*>(W8(ws, L.perm));
  a.tile_mod = reinterpret_cast<uint32_t*>(W8(ws, L.tile_mod));
  a.cnt = reinterpret_cast<int64_t*>(W8(ws, L.cnt));
  a.R = reinterpret_cast<float*>(W8(ws, L.gram_r));
  a.ex = reinterpret_cast<int32_t*>(W8(ws, L.gram_ex));
  a.slices = reinterpret_cast<int8_t*>(W8(ws, L.slices));
  a.gram_part = reinterpret_cast<double*>(W8(ws, L.gram_part));
  a.status = status_of(ws);
  if (T > 0) MASQ_CK(launch_inv(s, (int64_t)n_mod * d, const_cast<float*>(a.inv), st));
  const cudaError_t e = launch_cmc_gram(a, G, accumulate, st);
  if (e == cudaErrorNotSupported) return MASQ_ERR_UNSUPPORTED;
  MASQ_CK(e);
  return MASQ_OK;
}
}  // namespace

masq_status masq_cmc_gram(const void* X, masq_dtype xt, int64_t ld_x, const uint8_t* mod_id, int64_t T, int64_t d,
                          int32_t n_mod, const float* s, double* G, int32_t accumulate, void* ws, size_t ws_bytes,
                          masq_stream stream) {
  MASQ_TRY(check_common(T, d, n_mod));
  if (n_mod < 2) return MASQ_ERR_SHAPE;
  if (d > 2147483647 / 8 || T > 2147483647) return MASQ_ERR_SHAPE;
  if (!s || !G) return MASQ_ERR_NULL;
  if (T > 0) {
    MASQ_TRY(check_x(X, xt, ld_x, d));
    if (!mod_id) return MASQ_ERR_NULL;
  }
  if (!cmc_linalg_available()) return MASQ_ERR_UNSUPPORTED;
  const WsLayout L = ws_layout(MASQ_OP_CMC_GRAM, T, d, 0, n_mod, 0);
  MASQ_TRY(check_ws(ws, ws_bytes, L));
  return cmc_gram_core(X, xt, ld_x, mod_id, T, d, n_mod, s, G, accumulate, L, ws, S(stream));
}

masq_status masq_cmc_factors_from_gram(const double* G, int64_t d, int64_t d_out, int32_t n_mod, const float* s,
                                       const void* W, masq_dtype wt, const int8_t* qw_text, const float* dw_text,
                                       int32_t r, double eps_rel, void* L1, void* L2, masq_dtype lt, double* resid,
                                       void* ws, size_t ws_bytes, masq_stream stream) {
  MASQ_TRY(cmc_factor_checks(d, d_out, n_mod, s, W, wt, qw_text, dw_text, r, eps_rel, L1, L2, lt));
  if (!G) return MASQ_ERR_NULL;
  const WsLayout L = ws_layout(MASQ_OP_CMC_FACTORS, 0, d, d_out, n_mod, r);
  if (L.lwork == 0) return MASQ_ERR_UNSUPPORTED;
  MASQ_TRY(check_ws(ws, ws_bytes, L));
  const CmcArgs a = cmc_factor_args(L, ws, d, d_out, n_mod, s, W, wt, qw_text, dw_text, r, eps_rel, L1, L2, lt, resid);
  const cudaError_t e = launch_cmc_from_gram(a, G, S(stream));
  if (e == cudaErrorNotSupported) return MASQ_ERR_UNSUPPORTED;
  MASQ_CK(e);
  return MASQ_OK;
}

masq_status masq_cmc_factors(const void* X, masq_dtype xt, int64_t ld_x, const uint8_t* mod_id, int64_t T, int64_t d,
                             int64_t d_out, int32_t n_mod, const float* s, const void* W, masq_dtype wt,
                             const int8_t* qw_text, const float* dw_text, int32_t r, double eps_rel, void* L1,
                             void* L2, masq_dtype lt, double* resid, void* ws, size_t ws_bytes, masq_stream stream) {
  MASQ_TRY(check_common(T, d, n_mod));
  MASQ_TRY(cmc_factor_checks(d, d_out, n_mod, s, W, wt, qw_text, dw_text, r, eps_rel, L1, L2, lt));
  if (T > 2147483647) return MASQ_ERR_SHAPE;
  if (T > 0) {
    MASQ_TRY(check_x(X, xt, ld_x, d));
    if (!mod_id) return MASQ_ERR_NULL;
  }
  const WsLayout L = ws_layout(MASQ_OP_CMC, T, d, d_out, n_mod, r);
  if (L.lwork == 0) return MASQ_ERR_UNSUPPORTED;
  MASQ_TRY(check_ws(ws, ws_bytes, L));
  cudaStream_t st = S(stream);
  double* G = reinterpret_cast<double*>(W8(ws, L.gall));
  MASQ_TRY(cmc_gram_core(X, xt, ld_x, mod_id, T, d, n_mod, s, G, 0, L, ws, st));
  const CmcArgs a = cmc_factor_args(L, ws, d, d_out, n_mod, s, W, wt, qw_text, dw_text, r, eps_rel, L1, L2, lt, resid);
  const cudaError_t e = launch_cmc_from_gram(a, G, st);
  if (e == cudaErrorNotSupported) return MASQ_ERR_UNSUPPORTED;
  MASQ_CK(e);
  return MASQ_OK;
}

masq_status masq_quantize_weight_int4(const void* W, masq_dtype wt, const float* s, int64_t d, int64_t d_out,
                                      int32_t group, uint8_t* packed, float* scales, masq_stream stream) {
  if (!W || !s || !packed || !scales) return MASQ_ERR_NULL;
  if (group != 128) return MASQ_ERR_UNSUPPORTED;
  if (d <= 0 || d % 128 != 0 || d_out <= 0 || d_out % 8 != 0) return MASQ_ERR_SHAPE;
  if (wt != MASQ_BF16 && wt != MASQ_F32) return MASQ_ERR_UNSUPPORTED;
  if (!al16(packed)) return MASQ_ERR_ALIGN;
  MASQ_CK(launch_wq4(W, wt, s, d, d_out, packed, scales, S(stream)));
  return MASQ_OK;
}

masq_status masq_unpack_int4(const uint8_t* packed, int64_t d, int64_t d_out, int32_t group, int8_t* codes,
                             masq_stream stream) {
  if (!packed || !codes) return MASQ_ERR_NULL;
  if (group != 128) return MASQ_ERR_UNSUPPORTED;
  if (d <= 0 || d % 128 != 0 || d_out <= 0 || d_out % 8 != 0) return MASQ_ERR_SHAPE;
  MASQ_CK(launch_unpack4(packed, d, d_out, codes, S(stream)));
  return MASQ_OK;
}

masq_status masq_linear_decode(const void* X, masq_dtype xt, int64_t ld_x, int64_t T, int64_t d, int64_t d_out,
                               const float* s_t, const uint8_t* packed, const float* scales, int32_t group,
                               int32_t abits, float* Y, int64_t ld_y, void* ws, size_t ws_bytes,
                               masq_stream stream) {
  if (T < 0 || T > decode_max_tokens()) return MASQ_ERR_SHAPE;
  if (group != 128) return MASQ_ERR_UNSUPPORTED;
  if (d <= 0 || d % 128 != 0 || d_out <= 0 || d_out % 8 != 0) return MASQ_ERR_SHAPE;
  MASQ_TRY(check_bits(abits));
  if (!s_t || !packed || !scales || !Y) return MASQ_ERR_NULL;
  if (ld_y < d_out || !al16(packed) || !al16(s_t) || !al16(scales)) return MASQ_ERR_ALIGN;
  const WsLayout L = ws_layout(MASQ_OP_DECODE, T, d, d_out, 1, 0);
  MASQ_TRY(check_ws(ws, ws_bytes, L));
  if (T == 0) return MASQ_OK;
  MASQ_TRY(check_x(X, xt, ld_x, d));
  cudaStream_t st = S(stream);
  float* inv = reinterpret_cast<float*>(W8(ws, L.inv_s));
  uint8_t* ids0 = reinterpret_cast<uint8_t*>(W8(ws, L.ids0));
  int8_t* qa = reinterpret_cast<int8_t*>(W8(ws, L.qx));
  float* dx = reinterpret_cast<float*>(W8(ws, L.dx));
  const cudaError_t qe = launch_aquant_direct(X, xt, ld_x, T, d, s_t, abits, qa, dx, status_of(ws), st);
  if (qe == cudaErrorNotSupported) {
    MASQ_CK(cudaMemsetAsync(ids0, 0, (size_t)T, st));
    MASQ_CK(launch_inv(s_t, d, inv, st));
    MASQ_CK(launch_aquant(X, xt, ld_x, ids0, T, d, 1, inv, abits, qa, dx, nullptr, status_of(ws), st, nullptr, T));
  } else {
    MASQ_CK(qe);
  }
  MASQ_CK(launch_decode(qa, dx, (int)T, d, d_out, packed, scales, reinterpret_cast<float*>(W8(ws, L.dpart)), Y,
                        ld_y, st));
  return MASQ_OK;
}

masq_status masq_quantize_weight_w4g(const void* W, masq_dtype wt, const float* s, int64_t d, int64_t d_out,
                                     int32_t group, uint8_t* packed, float* scales, masq_stream stream) {
  if (!W || !s || !packed || !scales) return MASQ_ERR_NULL;
  if (group != 128) return MASQ_ERR_UNSUPPORTED;
  if (d <= 0 || d % 128 != 0 || d_out <= 0 || d_out % 32 != 0 || d >= (1LL << 31) || d_out >= (1LL << 31))
    return MASQ_ERR_SHAPE;
  if (wt != MASQ_BF16 && wt != MASQ_F32) return MASQ_ERR_UNSUPPORTED;
  if (!al16(packed) || !al16(W)) return MASQ_ERR_ALIGN;
  MASQ_CK(launch_wq4_layout(W, wt, s, d, d_out, packed, scales, 1, S(stream)));
  return MASQ_OK;
}

masq_status masq_linear_forward_w4g(const void* X, masq_dtype xt, int64_t ld_x, const uint8_t* mod_id, int64_t T,
                                    int64_t d, int64_t d_out, int32_t n_mod, const float* s, const uint8_t* packed,
                                    const float* scales, int32_t group, int32_t abits, const void* L1, const void* L2,
                                    int64_t ld_l2, int32_t r, float* Y, int64_t ld_y, void* ws, size_t ws_bytes,
                                    const masq_debug* dbg, masq_stream stream) {
  MASQ_TRY(check_common(T, d, n_mod));
  MASQ_TRY(check_bits(abits));
  if (group != 128) return MASQ_ERR_UNSUPPORTED;
  if (d % 128 != 0 || d_out <= 0 || d_out % 32 != 0 || d_out >= (1LL << 31)) return MASQ_ERR_SHAPE;
  if (r < 0 || r > 256 || r % 16 != 0) return MASQ_ERR_SHAPE;
  const bool use_acc = dbg && dbg->acc;
  if (!s || !packed || !scales || (!Y && !use_acc)) return MASQ_ERR_NULL;
  const bool cmc = r > 0 && n_mod > 1 && !use_acc;
  if (cmc) {
    if (!L1 || !L2) return MASQ_ERR_NULL;
    if (ld_l2 < d_out || !al16(L1) || !al16(L2) || (ld_l2 % 8) != 0) return MASQ_ERR_ALIGN;
  }
  void* out = use_acc ? static_cast<void*>(dbg->acc) : static_cast<void*>(Y);
  const int64_t ld_out = use_acc ? dbg->ld_acc : ld_y;
  if (ld_out < d_out || !al16(out) || !al16(packed) || !al16(s)) return MASQ_ERR_ALIGN;
  if (T == 0) return MASQ_OK;
  MASQ_TRY(check_x(X, xt, ld_x, d));
  if (!mod_id) return MASQ_ERR_NULL;
  const WsLayout L = ws_layout(MASQ_OP_FORWARD, T, d, d_out, n_mod, cmc ? r : 0, xt == MASQ_F32);
  MASQ_TRY(check_ws(ws, ws_bytes, L));
  cudaStream_t st = S(stream);
  float* inv = reinterpret_cast<float*>(W8(ws, L.inv_s));
  int8_t* qx = reinterpret_cast<int8_t*>(W8(ws, L.qx));
  float* dx = reinterpret_cast<float*>(W8(ws, L.dx));
  uint32_t* mask = reinterpret_cast<uint32_t*>(W8(ws, L.mask));
  // the CMC path's tile masks come from the factor packing below (no zeroing pass, no atomics)
  MASQ_CK(quantize_acts(X, xt, ld_x, mod_id, T, d, n_mod, s, inv, abits, qx, dx, nullptr, status_of(ws), st));
  if (dbg && dbg->qx) MASQ_CK(cudaMemcpyAsync(dbg->qx, qx, (size_t)T * d, cudaMemcpyDeviceToDevice, st));
  if (dbg && dbg->dx) MASQ_CK(cudaMemcpyAsync(dbg->dx, dx, sizeof(float) * T, cudaMemcpyDeviceToDevice, st));
  W4gArgs g{};
  g.T = T;
  g.n = d_out;
  g.d = d;
  g.qx = qx;
  g.dx = dx;
  g.packed = packed;
  g.scales = scales;
  g.tile_mask = cmc ? mask : nullptr;
  g.n_mod = n_mod;
  g.out = out;
  g.ld_out = ld_out;
  g.acc_mode = use_acc ? 1 : 0;
  if (cmc) {
    const int rp = (int)rpad_of(r);
    uint16_t* l1t = reinterpret_cast<uint16_t*>(W8(ws, L.l1t));
    uint16_t* l2t = reinterpret_cast<uint16_t*>(W8(ws, L.l2t));
    uint16_t* z = reinterpret_cast<uint16_t*>(W8(ws, L.z));
    MASQ_CK(launch_cmc_pack(static_cast<const uint16_t*>(L1), s, d, r, rp, n_mod - 1, l1t,
                            static_cast<const uint16_t*>(L2), ld_l2, d_out, l2t, mod_id, T, n_mod, mask, st));
    if (xt == MASQ_BF16) {
      MASQ_CK(launch_zgemm(static_cast<const uint16_t*>(X), ld_x, nullptr, mod_id, T, d, n_mod, l1t, rp, mask, z, st,
                           reinterpret_cast<float*>(W8(ws, L.zpart))));
    } else {
      uint16_t* xh = reinterpret_cast<uint16_t*>(W8(ws, L.xsplit));
      uint16_t* xl = xh + (size_t)T * d;
      MASQ_CK(launch_split_f32(static_cast<const float*>(X), ld_x, T, d, xh, xl, st));
      MASQ_CK(launch_zgemm(xh, d, xl, mod_id, T, d, n_mod, l1t, rp, mask, z, st,
                           reinterpret_cast<float*>(W8(ws, L.zpart))));
    }
    g.rpad = rp;
    g.z = z;
    g.l2t = l2t;
  }
  MASQ_CK(launch_w4g_gemm(g, st));
  return MASQ_OK;
}

masq_status masq_smooth_factors(const float* num, int64_t rows, int64_t d, const float* den, double beta, float* s,
                                masq_stream stream) {
  if (!num || !s) return MASQ_ERR_NULL;
  if (rows < 0 || d < 0 || !(beta >= 0.0 && beta <= 1.0)) return MASQ_ERR_SHAPE;
  if (rows == 0 || d == 0) return MASQ_OK;
  MASQ_CK(launch_smooth_factors(num, rows, d, den, beta, s, S(stream)));
  return MASQ_OK;
}

masq_status masq_calibrate_meanabs(const void* X, masq_dtype xt, int64_t ld_x, const uint8_t* mod_id, int64_t T,
                                   int64_t d, int32_t n_mod, double* sumabs, int64_t* count, float* mean,
                                   float* mean_unified, int32_t reset, void* ws, size_t ws_bytes,
                                   masq_stream stream) {
  MASQ_TRY(check_common(T, d, n_mod));
  if (!sumabs || !count) return MASQ_ERR_NULL;
  if (T > 0) {
    MASQ_TRY(check_x(X, xt, ld_x, d));
    if (!mod_id) return MASQ_ERR_NULL;
  }
  const WsLayout L = ws_layout(MASQ_OP_MEANABS, T, d, 0, n_mod, 0);
  MASQ_TRY(check_ws(ws, ws_bytes, L));
  cudaStream_t st = S(stream);
  if (reset) {
    MASQ_CK(cudaMemsetAsync(sumabs, 0, sizeof(double) * n_mod * d, st));
    MASQ_CK(cudaMemsetAsync(count, 0, sizeof(int64_t) * n_mod, st));
  }
  if (T == 0) return MASQ_OK;
  MASQ_CK(launch_meanabs(X, xt, ld_x, mod_id, T, d, n_mod, sumabs, count, mean, mean_unified,
                         reinterpret_cast<float*>(W8(ws, L.partials)), status_of(ws), st));
  return MASQ_OK;
}

masq_status masq_count_modalities(const uint8_t* mod_id, int64_t T, int32_t n_mod, int64_t* count, int32_t reset,
                                  void* ws, size_t ws_bytes, masq_stream stream) {
  MASQ_TRY(check_common(T, 16, n_mod));
  if (!count || (T > 0 && !mod_id)) return MASQ_ERR_NULL;
  MASQ_TRY(check_ws(ws, ws_bytes, ws_layout(MASQ_OP_STATS, T, 16, 0, n_mod, 0)));
  cudaStream_t st = S(stream);
  if (reset) MASQ_CK(cudaMemsetAsync(count, 0, sizeof(int64_t) * n_mod, st));
  if (T > 0) MASQ_CK(launch_count_modalities(mod_id, T, n_mod, count, status_of(ws), st));
  return MASQ_OK;
}

masq_status masq_range_stats(const float* R, int32_t n_mod, int64_t d, int32_t dominant, int32_t other,
                             float* alpha, float* r_unified, int64_t* dom_counts, masq_stream stream) {
  MASQ_TRY(check_common(0, d, n_mod));
  if (!R) return MASQ_ERR_NULL;
  if (alpha && (dominant < 0 || dominant >= n_mod || other < 0 || other >= n_mod)) return MASQ_ERR_SHAPE;
  MASQ_CK(launch_range_stats(R, n_mod, d, dominant, other, alpha, r_unified, dom_counts, S(stream)));
  return MASQ_OK;
}

masq_status masq_loss_finalize(const double* sums, const int64_t* counts, const float* lambda, int32_t n_mod,
                               int64_t d_out, double* loss, masq_stream stream) {
  if (!sums || !counts || !loss) return MASQ_ERR_NULL;
  if (n_mod < 1 || n_mod > kMaxMod || d_out <= 0) return MASQ_ERR_SHAPE;
  MASQ_CK(launch_loss_finalize(sums, counts, lambda, n_mod, d_out, loss, S(stream)));
  return MASQ_OK;
}

masq_status masq_check(void* ws, masq_stream stream) {
  if (!ws) return MASQ_ERR_WORKSPACE;
  if (cudaStreamSynchronize(S(stream)) != cudaSuccess) return MASQ_ERR_CUDA;
  uint32_t st = 0;
  if (cudaMemcpy(&st, ws, sizeof(st), cudaMemcpyDeviceToHost) != cudaSuccess) return MASQ_ERR_CUDA;
  const uint32_t zero = 0;
  if (cudaMemcpy(ws, &zero, sizeof(zero), cudaMemcpyHostToDevice) != cudaSuccess) return MASQ_ERR_CUDA;
  if (st & kStBadModality) return MASQ_ERR_BAD_MODALITY;
  if (st & kStEmptyModality) return MASQ_ERR_EMPTY_MODALITY;
  return MASQ_OK;
}

const char* masq_status_string(masq_status s) {
  switch (s) {
    case MASQ_OK: return "ok";
    case MASQ_ERR_NULL: return "a required pointer is NULL";
    case MASQ_ERR_SHAPE: return "dimension outside the supported limits";
    case MASQ_ERR_BITS: return "bit-width outside [2, 16]";
    case MASQ_ERR_ALIGN: return "pointer or leading dimension misaligned (16-byte rows required)";
    case MASQ_ERR_WORKSPACE: return "workspace missing, misaligned or smaller than masq_workspace_size()";
    case MASQ_ERR_BAD_MODALITY: return "token tagged with unknown modality (id >= n_mod)";
    case MASQ_ERR_EMPTY_MODALITY: return "modality with zero calibration tokens";
    case MASQ_ERR_UNSUPPORTED: return "valid request outside this path (e.g. 16-bit operands)";
    case MASQ_ERR_CUDA: return "CUDA runtime or driver call failed";
  }
  return "unknown status";
}

const char* masq_version(void) { return "0.1.0 sm_100a"; }

}  // extern "C"
