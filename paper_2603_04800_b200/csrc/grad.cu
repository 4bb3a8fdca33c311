// grad.cu — N1: straight-through gradient of the calibration loss w.r.t.
// theta^m = ln s^m, and the log-space Adam step.
//
// With the rows of modality m grouped as in the loss GEMM (perm), G = sign(Ahat Bhat - X W)
// (emitted by the loss epilogue, bf16, 0 on padding rows), A = X S^-1 (xs), Ahat = Q(A),
// B = S W, Bhat = Q(B), the oracle's
//   grad_i = scale_m * sum_j [ (Ahat^T G)_ij B_ij - (A^T G)_ij Bhat_ij ]
// is evaluated as the algebraically equal
//   grad_i = scale_m * sum_j [ (D^T G)_ij B_ij + inv_i (X^T G)_ij (B - Bhat)_ij ],  D = Ahat - A,
// whose two terms are the activation and weight quantisation residuals taken directly — no
// cancellation between two large near-equal products, so one bf16 plane of D suffices.
// Q' = D^T G and P = X^T G are tcgen05 kind::f16 GEMMs with the token axis as K: A operand
// planes [D | X] (bf16, MN-major: i contiguous), B operand G (MN-major: j contiguous), two fp32
// TMEM accumulators (Q' in columns 0..255, P in 256..511).  The epilogue reads W and the tile
// of Q(S_m W) (TMA) and reduces over j into one partial per (modality, j-tile, i); a
// fixed-order reduction forms the gradient (deterministic).
#include <cuda_bf16.h>

#include "internal.h"
#include "sm100.cuh"

namespace masq {
using namespace sm100;

namespace {
constexpr int GT = 192;                    // warp 0 TMA, warp 1 MMA, warps 2..5 epilogue
constexpr int GM = 128, GN = 256, GK = 64; // i rows, j columns, tokens per k-block
constexpr int APL = GM * GK * 2;           // one A plane tile: 128 i x 64 t bf16 = 16 KB
constexpr int BPL = GN * GK * 2;           // B tile: 256 j x 64 t bf16 = 32 KB
constexpr int NPL = 2;                     // planes D, X
constexpr int STAGE = NPL * APL + BPL;     // 64 KB
constexpr int GSTAGES = 3;
constexpr int QW_BYTES = GN * GM;          // qw tile [256 j][128 i] int8 = 32 KB
constexpr int G_SMEM = GSTAGES * STAGE + QW_BYTES + 256;
constexpr int G_ALLOC = G_SMEM + 1024;
constexpr uint32_t IDESC_G = idesc_bf16(GM, GN) | (1u << 15) | (1u << 16);   // A and B MN-major

struct GParams {
  int d, n, n_mod, Tg;
  int ni, nj, n_units;
  const uint32_t* tile_mod;      // modality of every 256-row grouped unit (~0u = empty)
  int n_tm;
  const float* s;                // [M][d]
  const float* inv;              // [M][d]
  const uint16_t* W;             // [d][n] bf16
  const float* dw;               // [M][n]
  double* partial;               // [M][nj][d]
};

__device__ __forceinline__ void seg_of(const GParams& p, int m, int& k0, int& nkb) {
  int first = -1, cnt = 0;
  for (int u = 0; u < p.n_tm; ++u)
    if (p.tile_mod[u] == (uint32_t)m) {
      if (first < 0) first = u;
      ++cnt;
    }
  k0 = first < 0 ? 0 : first * kUnitM;
  nkb = cnt * (kUnitM / GK);
}

__global__ void __launch_bounds__(GT, 1)
gradgemm_kernel(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB,
                const __grid_constant__ CUtensorMap tmQW, const GParams p) {
  extern __shared__ uint8_t smem_raw[];
  const uint32_t raw = smem_u32(smem_raw);
  uint8_t* smem = smem_raw + (((raw + 1023u) & ~1023u) - raw);
  uint8_t* qws = smem + GSTAGES * STAGE;
  uint64_t* full = reinterpret_cast<uint64_t*>(qws + QW_BYTES);
  uint64_t* empty = full + GSTAGES;
  uint64_t* tfull = empty + GSTAGES;
  uint64_t* tempty = tfull + 1;
  uint64_t* qfull = tempty + 1;
  uint64_t* qempty = qfull + 1;
  uint32_t* tslot = reinterpret_cast<uint32_t*>(qempty + 1);
  const uint32_t warp = warp_id(), lane = lane_id();
  if (warp == 0 && lane == 0) {
    tma_prefetch(&tmA);
    tma_prefetch(&tmB);
    tma_prefetch(&tmQW);
    for (int i = 0; i < GSTAGES; ++i) { mbar_init(&full[i], 1); mbar_init(&empty[i], 1); }
    mbar_init(tfull, 1);
    mbar_init(tempty, 4);
    mbar_init(qfull, 1);
    mbar_init(qempty, 4);
    fence_mbar_init();
  }
  if (warp == 1) tmem_alloc(tslot, 512);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tslot;

  auto decode = [&](int u, int& m, int& it, int& jt) {
    const int per_m = p.ni * p.nj;
    m = u / per_m;
    const int r = u - m * per_m;
    jt = r / p.ni;
    it = r - jt * p.ni;
  };

  if (warp == 0) {
    if (lane == 0) {
      uint32_t st = 0, ph = 0, local = 0;
      for (int u = blockIdx.x; u < p.n_units; u += gridDim.x) {
        int m, it, jt, k0, nkb;
        decode(u, m, it, jt);
        seg_of(p, m, k0, nkb);
        if (nkb == 0) continue;
        // the tile of Q(S_m W) for the epilogue: rows j (m*n + jt*256 ..), bytes i (it*128 ..)
        mbar_wait(qempty, (local & 1u) ^ 1u);
        mbar_expect_tx(qfull, QW_BYTES);
        tma_load_2d(qws, &tmQW, qfull, it * GM, m * p.n + jt * GN);
        ++local;
        for (int kb = 0; kb < nkb; ++kb) {
          mbar_wait(&empty[st], ph ^ 1u);
          mbar_expect_tx(&full[st], STAGE);
          uint8_t* base = smem + st * STAGE;
          const int t = k0 + kb * GK;
#pragma unroll
          for (int pl = 0; pl < NPL; ++pl)
#pragma unroll
            for (int h = 0; h < 2; ++h)
              tma_load_2d(base + pl * APL + h * (APL / 2), &tmA, &full[st], it * GM + h * 64, pl * p.Tg + t);
#pragma unroll
          for (int q = 0; q < 4; ++q)
            tma_load_2d(base + NPL * APL + q * (BPL / 4), &tmB, &full[st], jt * GN + q * 64, t);
          if (++st == GSTAGES) { st = 0; ph ^= 1u; }
        }
      }
    }
    __syncwarp();
  } else if (warp == 1) {
    if (lane == 0) {
      uint32_t st = 0, ph = 0, local = 0;
      for (int u = blockIdx.x; u < p.n_units; u += gridDim.x) {
        int m, it, jt, k0, nkb;
        decode(u, m, it, jt);
        seg_of(p, m, k0, nkb);
        if (nkb == 0) continue;
        mbar_wait(tempty, (local & 1u) ^ 1u);
        ++local;
        tc_fence_after();
        for (int kb = 0; kb < nkb; ++kb) {
          mbar_wait(&full[st], ph);
          tc_fence_after();
          const uint32_t base = smem_u32(smem + st * STAGE);
#pragma unroll
          for (int kk = 0; kk < 4; ++kk) {
            const uint64_t bd = umma_desc_sw128_mn(base + NPL * APL + kk * 2048, BPL / 4);
            const uint32_t acc0 = (kb | kk) != 0;
            mma_bf16(tmem, umma_desc_sw128_mn(base + 0 * APL + kk * 2048, APL / 2), bd, IDESC_G, acc0);
            mma_bf16(tmem + GN, umma_desc_sw128_mn(base + 1 * APL + kk * 2048, APL / 2), bd, IDESC_G, acc0);
          }
          mma_commit(&empty[st]);
          if (++st == GSTAGES) { st = 0; ph ^= 1u; }
        }
        mma_commit(tfull);
      }
    }
    __syncwarp();
  } else {
    const uint32_t q = warp & 3u;
    uint32_t local = 0;
    for (int u = blockIdx.x; u < p.n_units; u += gridDim.x) {
      int m, it, jt, k0, nkb;
      decode(u, m, it, jt);
      seg_of(p, m, k0, nkb);
      const int il = (int)(q * 32u + lane);
      const int i = it * GM + il;
      double* out = p.partial + ((size_t)m * p.nj + jt) * p.d;
      if (nkb == 0) {
        if (i < p.d) out[i] = 0.0;
        continue;
      }
      const int j0 = jt * GN;
      const int nch = min(8, (p.n - j0) / 32);
      float dwr[8];
#pragma unroll
      for (int c = 0; c < 8; ++c) dwr[c] = c < nch ? __ldg(p.dw + (size_t)m * p.n + j0 + c * 32 + lane) : 0.f;
      const bool iv = i < p.d;
      const float si = iv ? __ldg(p.s + (size_t)m * p.d + i) : 0.f;
      const float invi = iv ? __ldg(p.inv + (size_t)m * p.d + i) : 0.f;
      const uint32_t ph = local & 1u;
      ++local;
      mbar_wait(tfull, ph);
      mbar_wait(qfull, ph);
      tc_fence_after();
      const uint32_t tq = tmem + ((q * 32u) << 16);
      float acc = 0.f;
#pragma unroll 1
      for (int c = 0; c < nch; ++c) {
        uint32_t vq[32], vp[32];
        tmem_ld32(tq + c * 32, vq);
        tmem_ld32(tq + GN + c * 32, vp);
        uint4 w4[4];
        if (iv) {
          const uint4* wp = reinterpret_cast<const uint4*>(p.W + (size_t)i * p.n + j0 + c * 32);
#pragma unroll
          for (int k = 0; k < 4; ++k) w4[k] = __ldg(wp + k);
        } else {
#pragma unroll
          for (int k = 0; k < 4; ++k) w4[k] = make_uint4(0, 0, 0, 0);
        }
        tmem_wait_ld();
#pragma unroll
        for (int jj = 0; jj < 32; ++jj) {
          const uint32_t wv = (&w4[jj >> 3].x)[(jj >> 1) & 3];
          const float w = __uint_as_float((jj & 1) ? (wv & 0xFFFF0000u) : (wv << 16));
          const float dwj = __shfl_sync(0xffffffffu, dwr[c], jj);
          const int qv = (int)(int8_t)qws[(c * 32 + jj) * GM + il];
          const float bs = __fmul_rn(si, w);                       // (S_m W)_ij as quantized
          const float bh = __fmul_rn(dwj, (float)qv);              // Bhat_ij
          acc = fmaf(__uint_as_float(vq[jj]), bs, acc);
          acc = fmaf(__uint_as_float(vp[jj]) * invi, __fsub_rn(bs, bh), acc);
        }
      }
      if (iv) out[i] = (double)acc;
      tc_fence_before();
      __syncwarp();
      if (lane == 0) {
        mbar_arrive(tempty);
        mbar_arrive(qempty);
      }
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 1) {
    tc_fence_after();
    tmem_dealloc(tmem, 512);
  }
}

// planes for the gradient GEMM, in the loss's grouped row order: D = Ahat - xs and X (bf16)
__global__ void __launch_bounds__(256) gradprep_kernel(const uint16_t* __restrict__ X, int64_t ld_x,
                                                       const uint8_t* __restrict__ mod_id,
                                                       const int32_t* __restrict__ perm, const int8_t* __restrict__ qx,
                                                       const float* __restrict__ dx, const float* __restrict__ inv,
                                                       int64_t Tg, int64_t d, uint16_t* __restrict__ planes) {
  const int64_t p = (int64_t)blockIdx.x * 8 + (threadIdx.x >> 5);
  const int lane = threadIdx.x & 31;
  if (p >= Tg) return;
  const int32_t src = __ldg(perm + p);
  const float dxv = src >= 0 ? __ldg(dx + p) : 0.f;
  const float* invm = inv + (src >= 0 ? (int64_t)__ldg(mod_id + src) * d : 0);
  uint16_t* pd = planes + p * d;
  uint16_t* px = planes + (Tg + p) * d;
  for (int64_t c = (int64_t)lane * 8; c < d; c += 256) {
    uint4 xv = make_uint4(0, 0, 0, 0), dv = make_uint4(0, 0, 0, 0);
    if (src >= 0) {
      xv = __ldg(reinterpret_cast<const uint4*>(X + (int64_t)src * ld_x + c));
      const uint2 q8 = __ldg(reinterpret_cast<const uint2*>(qx + p * d + c));
      const float4 i0 = __ldg(reinterpret_cast<const float4*>(invm + c));
      const float4 i1 = __ldg(reinterpret_cast<const float4*>(invm + c + 4));
      const float iv[8] = {i0.x, i0.y, i0.z, i0.w, i1.x, i1.y, i1.z, i1.w};
      const uint32_t xw[4] = {xv.x, xv.y, xv.z, xv.w};
      const uint32_t qw[2] = {q8.x, q8.y};
      uint32_t o[4];
#pragma unroll
      for (int e = 0; e < 4; ++e) {
        uint16_t h[2];
#pragma unroll
        for (int k = 0; k < 2; ++k) {
          const int idx = 2 * e + k;
          const int8_t qv = (int8_t)((qw[idx >> 2] >> (8 * (idx & 3))) & 0xFF);
          const float x = __uint_as_float(k ? (xw[e] & 0xFFFF0000u) : (xw[e] << 16));
          const float ah = __fmul_rn(dxv, (float)qv);
          const float xs = __fmul_rn(x, iv[idx]);
          h[k] = __bfloat16_as_ushort(__float2bfloat16_rn(__fsub_rn(ah, xs)));
        }
        o[e] = (uint32_t)h[0] | ((uint32_t)h[1] << 16);
      }
      dv = make_uint4(o[0], o[1], o[2], o[3]);
    }
    *reinterpret_cast<uint4*>(pd + c) = dv;
    *reinterpret_cast<uint4*>(px + c) = xv;
  }
}

struct Lam8 {
  float v[kMaxMod];
};

// grad[m][i] = lambda_m / (counts_m * n) * sum_jt partial[m][jt][i]   (fixed order)
__global__ void gradreduce_kernel(const double* __restrict__ partial, const int64_t* __restrict__ counts, Lam8 lam,
                                  int n_mod, int nj, int64_t d, int64_t n, double* __restrict__ grad) {
  const int64_t idx = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (idx >= (int64_t)n_mod * d) return;
  const int m = (int)(idx / d);
  const int64_t i = idx - (int64_t)m * d;
  double a = 0.0;
  for (int jt = 0; jt < nj; ++jt) a += partial[((int64_t)m * nj + jt) * d + i];
  const int64_t c = counts[m];
  grad[idx] = c > 0 ? (double)lam.v[m] * a / ((double)c * (double)n) : 0.0;
}

__global__ void adam_kernel(double* __restrict__ theta, const double* __restrict__ grad, double* __restrict__ m1,
                            double* __restrict__ m2, int64_t count, int step, double lr, double b1, double b2,
                            double eps, float* __restrict__ s_out) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= count) return;
  const double g = grad[i];
  const double a = b1 * m1[i] + (1.0 - b1) * g;
  const double b = b2 * m2[i] + (1.0 - b2) * g * g;
  m1[i] = a;
  m2[i] = b;
  const double mh = a / (1.0 - pow(b1, (double)step));
  const double vh = b / (1.0 - pow(b2, (double)step));
  const double t = theta[i] - lr * mh / (sqrt(vh) + eps);
  theta[i] = t;
  if (s_out) s_out[i] = (float)exp(t);
}
}  // namespace

cudaError_t launch_gradprep(const uint16_t* X, int64_t ld_x, const uint8_t* mod_id, const int32_t* perm,
                            const int8_t* qx, const float* dx, const float* inv, int64_t Tg, int64_t d,
                            uint16_t* planes, cudaStream_t st) {
  ProfScope ps_("gradprep", st);
  gradprep_kernel<<<(unsigned)ceil_div(Tg, 8), 256, 0, st>>>(X, ld_x, mod_id, perm, qx, dx, inv, Tg, d, planes);
  return cudaGetLastError();
}

cudaError_t launch_gradgemm(const uint16_t* planes, int64_t Tg, const uint16_t* gsign, const int8_t* qw_all,
                            const uint32_t* tile_mod, int n_mod, int64_t d, int64_t n, const float* s,
                            const float* inv, const uint16_t* W, const float* dw, double* partial,
                            cudaStream_t st) {
  CUtensorMap ta, tb, tq;
  bool ok = make_tmap_2d(&ta, planes, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, (uint64_t)NPL * Tg, d, d, 64, 64, true);
  ok &= make_tmap_2d(&tb, gsign, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, Tg, n, n, 64, 64, true);
  ok &= make_tmap_2d(&tq, qw_all, CU_TENSOR_MAP_DATA_TYPE_UINT8, 1, (uint64_t)n_mod * n, d, d, GN, GM, false);
  if (!ok) return cudaErrorInvalidValue;
  static bool attr = false;
  if (!attr) {
    cudaError_t e = cudaFuncSetAttribute(gradgemm_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, G_ALLOC);
    if (e != cudaSuccess) return e;
    attr = true;
  }
  GParams p{};
  p.d = (int)d;
  p.n = (int)n;
  p.n_mod = n_mod;
  p.Tg = (int)Tg;
  p.ni = (int)ceil_div(d, GM);
  p.nj = (int)ceil_div(n, GN);
  p.n_units = p.ni * p.nj * n_mod;
  p.tile_mod = tile_mod;
  p.n_tm = (int)(Tg / kUnitM);
  p.s = s;
  p.inv = inv;
  p.W = W;
  p.dw = dw;
  p.partial = partial;
  const int grid = std::min(p.n_units, num_sms());
  ProfScope ps_("gradgemm", st);
  gradgemm_kernel<<<grid, GT, G_ALLOC, st>>>(ta, tb, tq, p);
  return cudaGetLastError();
}

int gradgemm_ntiles_j(int64_t n) { return (int)ceil_div(n, GN); }

cudaError_t launch_gradreduce(const double* partial, const int64_t* counts, const float* lambda_host, int n_mod,
                              int nj, int64_t d, int64_t n, double* grad, cudaStream_t st) {
  Lam8 l;
  for (int m = 0; m < kMaxMod; ++m) l.v[m] = (lambda_host && m < n_mod) ? lambda_host[m] : 1.0f;
  const int64_t count = (int64_t)n_mod * d;
  ProfScope ps_("gradreduce", st);
  gradreduce_kernel<<<(unsigned)ceil_div(count, 256), 256, 0, st>>>(partial, counts, l, n_mod, nj, d, n, grad);
  return cudaGetLastError();
}

cudaError_t launch_adam(double* theta, const double* grad, double* m1, double* m2, int64_t count, int step, double lr,
                        double b1, double b2, double eps, float* s_out, cudaStream_t st) {
  ProfScope ps_("adam", st);
  adam_kernel<<<(unsigned)ceil_div(count, 256), 256, 0, st>>>(theta, grad, m1, m2, count, step, lr, b1, b2, eps, s_out);
  return cudaGetLastError();
}

}  // namespace masq
