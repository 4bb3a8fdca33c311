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
// The scales are differentiated too (reading Q24: only round() is straight-through):
//   + sum_{j: k_j = l} beta_j - sum_{t: k_t = l} alpha_t,
//   beta_j = sum_i (Ahat^T G)_ij (Bhat - B)_ij   (this kernel's epilogue, per 32-row group),
//   alpha_t = sum_j G_tj (D Bhat)_tj              (gemm.cu kModeAlpha, D . codes^T),
// k_j / k_t the first arg-max rows / channels of |B| / |A|, summed into grad by a fixed-order
// bucket pass (deterministic).
// Q' = D^T G and P = X^T G are tcgen05 kind::f16 GEMMs with the token axis as K: A operand
// planes [D | X] (bf16, MN-major: i contiguous), B operand G (MN-major: j contiguous), two fp32
// TMEM accumulators (Q' in columns 0..255, P in 256..511).  The epilogue reads W and the tile
// of Q(S_m W) (TMA) and reduces over j into one partial per (modality, j-tile, i); a
// fixed-order reduction forms the gradient (deterministic).
#include <cub/device/device_radix_sort.cuh>
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
  const uint32_t* colmax;        // [M][n] f32 bits of max_i |s_i w_ij|
  double* partial;               // [M][nj][d]
  float* bpart;                  // [M][4 * ni][n]  (one row per 32-row warp group)
  int32_t* kj;                   // [M][n]
};

// 32 values per lane -> lane l returns the sum over the warp of v[l] (transpose-reduce, 31 shuffles)
__device__ __forceinline__ float warp_transpose_sum(float (&v)[32], uint32_t lane) {
#pragma unroll
  for (int off = 16; off >= 1; off >>= 1) {
    const bool upper = (lane & (uint32_t)off) != 0u;
#pragma unroll
    for (int k = 0; k < off; ++k) {
      const float send = upper ? v[k] : v[k + off];
      const float keep = upper ? v[k + off] : v[k];
      v[k] = keep + __shfl_xor_sync(0xffffffffu, send, off);
    }
  }
  return v[0];
}

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
    {
      // warp-wide loops (uniform state); one elected lane issues copies / MMAs
      uint32_t st = 0, ph = 0, local = 0;
      for (int u = blockIdx.x; u < p.n_units; u += gridDim.x) {
        int m, it, jt, k0, nkb;
        decode(u, m, it, jt);
        seg_of(p, m, k0, nkb);
        if (nkb == 0) continue;
        // the tile of Q(S_m W) for the epilogue: rows j (m*n + jt*256 ..), bytes i (it*128 ..)
        mbar_wait(qempty, (local & 1u) ^ 1u);
        if (elect_one()) {
          mbar_expect_tx(qfull, QW_BYTES);
          tma_load_2d(qws, &tmQW, qfull, it * GM, m * p.n + jt * GN);
        }
        __syncwarp();
        ++local;
        for (int kb = 0; kb < nkb; ++kb) {
          mbar_wait(&empty[st], ph ^ 1u);
          if (elect_one()) {
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
          }
          __syncwarp();
          if (++st == GSTAGES) { st = 0; ph ^= 1u; }
        }
      }
    }
    __syncwarp();
  } else if (warp == 1) {
    {
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
          if (elect_one()) {
            const uint32_t base = smem_u32(smem + st * STAGE);
            const uint64_t bd = umma_desc_sw128_mn(base + NPL * APL, BPL / 4);
            const uint64_t a0d = umma_desc_sw128_mn(base, APL / 2), a1d = umma_desc_sw128_mn(base + APL, APL / 2);
#pragma unroll
            for (int kk = 0; kk < 4; ++kk) {
              const uint32_t acc0 = (kb | kk) != 0;
              mma_bf16(tmem, a0d + 128 * kk, bd + 128 * kk, IDESC_G, acc0);
              mma_bf16(tmem + GN, a1d + 128 * kk, bd + 128 * kk, IDESC_G, acc0);
            }
            mma_commit(&empty[st]);
          }
          __syncwarp();
          if (++st == GSTAGES) { st = 0; ph ^= 1u; }
        }
        if (elect_one()) mma_commit(tfull);
        __syncwarp();
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
      if (nkb == 0) {                      // no tokens of modality m: zero contributions
        if (i < p.d) out[i] = 0.0;
        float* bz = p.bpart + ((size_t)m * 4 * p.ni + 4 * it + q) * p.n + jt * GN;
        const int nz = min(8, (p.n - jt * GN) / 32);
        for (int c = 0; c < nz; ++c) bz[c * 32 + lane] = 0.f;
        continue;
      }
      const int j0 = jt * GN;
      const int nch = min(8, (p.n - j0) / 32);
      float dwr[8];
      uint32_t cmr[8];
#pragma unroll
      for (int c = 0; c < 8; ++c) {
        dwr[c] = c < nch ? __ldg(p.dw + (size_t)m * p.n + j0 + c * 32 + lane) : 0.f;
        cmr[c] = c < nch ? __ldg(p.colmax + (size_t)m * p.n + j0 + c * 32 + lane) : 0xFFFFFFFFu;
      }
      float* bout = p.bpart + ((size_t)m * 4 * p.ni + 4 * it + q) * p.n + j0;
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
        float bj[32];
#pragma unroll
        for (int jj = 0; jj < 32; ++jj) {
          const uint32_t wv = (&w4[jj >> 3].x)[(jj >> 1) & 3];
          const float w = __uint_as_float((jj & 1) ? (wv & 0xFFFF0000u) : (wv << 16));
          const float dwj = __shfl_sync(0xffffffffu, dwr[c], jj);
          const uint32_t cmj = __shfl_sync(0xffffffffu, cmr[c], jj);
          const int qv = (int)(int8_t)qws[(c * 32 + jj) * GM + il];
          const float bs = __fmul_rn(si, w);                       // (S_m W)_ij as quantized
          const float bh = __fmul_rn(dwj, (float)qv);              // Bhat_ij
          const float q = __uint_as_float(vq[jj]), pv = __uint_as_float(vp[jj]);
          const float dbw = __fsub_rn(bs, bh);                     // B - Bhat
          acc = fmaf(q, bs, acc);
          acc = fmaf(pv * invi, dbw, acc);
          bj[jj] = -fmaf(pv, invi, q) * dbw;                       // (Ahat^T G)_ij (Bhat - B)_ij
          if (iv && (__float_as_uint(bs) & 0x7FFFFFFFu) == cmj) atomicMin(p.kj + (size_t)m * p.n + j0 + c * 32 + jj, i);
        }
        bout[c * 32 + lane] = warp_transpose_sum(bj, lane);
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
                                                       int64_t Tg, int64_t d, float qa, uint16_t* __restrict__ planes,
                                                       int32_t* __restrict__ ktkey, int8_t* __restrict__ dq,
                                                       float* __restrict__ de, int8_t* __restrict__ dq2,
                                                       float* __restrict__ de2) {
  const int64_t p = (int64_t)blockIdx.x * 8 + (threadIdx.x >> 5);
  const int lane = threadIdx.x & 31;
  if (p >= Tg) return;
  const int32_t src = __ldg(perm + p);
  const float dxv = src >= 0 ? __ldg(dx + p) : 0.f;
  const int mrow = src >= 0 ? (int)__ldg(mod_id + src) : 0;
  const float* invm = inv + (int64_t)mrow * d;
  uint32_t best = 0;                          // |xs| bits of the lane's first maximum
  int bidx = 0x7FFFFFFF;
  uint16_t* pd = planes + p * d;
  uint16_t* px = planes + (Tg + p) * d;
  // |D| <= Delta_t / 2 (a rounding residual), so D / (Delta_t / 254) fits int8: the alpha GEMM's
  // operand (int8 tensor path), scale e_t = Delta_t / 254.  Its rounding residual (<= e_t / 2) is
  // quantized again on e_t / 254 and contracted by a second pass of the same GEMM, so D enters
  // alpha_t to 1/254^2 of its range (one level alone is 1/254: ~1e-3 of the gradient when a
  // modality has a single token, whose alpha lands on one channel undiluted)
  const float estep = __fdiv_rn(dxv, 254.0f);
  const float einv = dxv > 0.f ? __fdiv_rn(254.0f, dxv) : 0.f;
  const float estep2 = __fdiv_rn(estep, 254.0f);
  const float einv2 = estep2 > 0.f ? __fdiv_rn(1.0f, estep2) : 0.f;
  if (lane == 0) {
    de[p] = estep;
    de2[p] = estep2;
  }
  for (int64_t c = (int64_t)lane * 8; c < d; c += 256) {
    uint4 xv = make_uint4(0, 0, 0, 0), dv = make_uint4(0, 0, 0, 0);
    uint2 qd = make_uint2(0, 0), qd2 = make_uint2(0, 0);
    if (src >= 0) {
      xv = __ldg(reinterpret_cast<const uint4*>(X + (int64_t)src * ld_x + c));
      const uint2 q8 = __ldg(reinterpret_cast<const uint2*>(qx + p * d + c));
      const float4 i0 = __ldg(reinterpret_cast<const float4*>(invm + c));
      const float4 i1 = __ldg(reinterpret_cast<const float4*>(invm + c + 4));
      const float iv[8] = {i0.x, i0.y, i0.z, i0.w, i1.x, i1.y, i1.z, i1.w};
      const uint32_t xw[4] = {xv.x, xv.y, xv.z, xv.w};
      const uint32_t qw[2] = {q8.x, q8.y};
      uint32_t o[4], qb[2] = {0u, 0u}, qb2[2] = {0u, 0u};
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
          const float dd = __fsub_rn(ah, xs);
          h[k] = __bfloat16_as_ushort(__float2bfloat16_rn(dd));
          const int qi = max(-127, min(127, __float2int_rn(dd * einv)));
          qb[idx >> 2] |= ((uint32_t)qi & 0xFFu) << (8 * (idx & 3));
          const float rr = fmaf(-(float)qi, estep, dd);             // second level: the residual
          const int q2 = max(-127, min(127, __float2int_rn(rr * einv2)));
          qb2[idx >> 2] |= ((uint32_t)q2 & 0xFFu) << (8 * (idx & 3));
          const uint32_t ab = __float_as_uint(xs) & 0x7FFFFFFFu;
          if (ab > best) { best = ab; bidx = (int)(c + idx); }
        }
        o[e] = (uint32_t)h[0] | ((uint32_t)h[1] << 16);
      }
      dv = make_uint4(o[0], o[1], o[2], o[3]);
      qd = make_uint2(qb[0], qb[1]);
      qd2 = make_uint2(qb2[0], qb2[1]);
    }
    *reinterpret_cast<uint4*>(pd + c) = dv;
    *reinterpret_cast<uint4*>(px + c) = xv;
    *reinterpret_cast<uint2*>(dq + p * d + c) = qd;
    *reinterpret_cast<uint2*>(dq2 + p * d + c) = qd2;
  }
  // first arg-max over the row: larger |xs| wins, ties -> smaller index
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    const uint32_t ob = __shfl_xor_sync(0xffffffffu, best, o);
    const int oi = __shfl_xor_sync(0xffffffffu, bidx, o);
    if (ob > best || (ob == best && oi < bidx)) { best = ob; bidx = oi; }
  }
  if (lane == 0) {
    // the scale derivative exists only when Delta_t = max/q_a is not floored (and the row is real)
    const bool live = src >= 0 && __fdiv_rn(__uint_as_float(best), qa) >= 1e-12f;
    ktkey[p] = live ? mrow * (int)d + bidx : -1;
  }
}

// beta keys / values: one CTA per (modality, 32 columns); thread (r0 = tid >> 5, lane = column)
// sums the row groups r = r0, r0 + 8, ...; the 8 partial sums are added in a fixed order
__global__ void __launch_bounds__(256) betakeys_kernel(const float* __restrict__ bpart, int nb,
                                                       const int32_t* __restrict__ kj,
                                                       const uint32_t* __restrict__ colmax, float qw, int64_t d,
                                                       int64_t n, int32_t* __restrict__ keys,
                                                       double* __restrict__ vals) {
  __shared__ double sh[8][32];
  const int64_t cb = (int64_t)blockIdx.x * 32;                 // column base in [0, n_mod * n)
  const int64_t m = cb / n, j = cb - m * n + (threadIdx.x & 31);
  const int r0 = threadIdx.x >> 5;
  double a = 0.0;
  for (int r = r0; r < nb; r += 8) a += (double)bpart[((int64_t)m * nb + r) * n + j];
  sh[r0][threadIdx.x & 31] = a;
  __syncthreads();
  if (threadIdx.x < 32) {
    double b = 0.0;
#pragma unroll
    for (int q = 0; q < 8; ++q) b += sh[q][threadIdx.x];
    const int64_t idx = m * n + j;
    const int32_t k = kj[idx];
    const bool live = k >= 0 && k < d && __fdiv_rn(__uint_as_float(colmax[idx]), qw) >= 1e-12f;
    keys[idx] = live ? (int32_t)(m * d + k) : -1;
    vals[idx] = b;
  }
}

// alpha keys / values: (ktkey[t], -alpha_t), alpha_t = the row's partials summed in order
__global__ void alphakeys_kernel(const float* __restrict__ apart, int na, const int32_t* __restrict__ ktkey,
                                 int64_t Tg, int32_t* __restrict__ keys, double* __restrict__ vals) {
  const int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= Tg) return;
  double a = 0.0;
  for (int r = 0; r < na; ++r) a += (double)apart[t * na + r];
  keys[t] = ktkey[t];
  vals[t] = -a;
}

struct Lam8 {
  float v[kMaxMod];
};

// contrib[l] = sum of vals over the run of keys == l in the (stably) sorted key list; keys -1
// sort last.  The warp whose 32 elements hold a run's first key sums the whole run: lane q takes
// elements start + q, start + q + 32, ... in order, then a fixed xor-shuffle tree -> the same
// association on every run, so the result is deterministic.  (A run can be as long as every
// column of the weight: the columns' arg-max rows concentrate on the outlier channels.)
__global__ void __launch_bounds__(256) runsum_kernel(const uint32_t* __restrict__ skeys,
                                                     const double* __restrict__ svals, int64_t nkeys, int64_t nl,
                                                     double* __restrict__ contrib) {
  const int lane = threadIdx.x & 31;
  const int64_t base = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) - lane;
  const int64_t i = base + lane;
  uint32_t k = 0xFFFFFFFFu;
  bool start = false;
  if (i < nkeys) {
    k = skeys[i];
    start = k < (uint32_t)nl && (i == 0 || skeys[i - 1] != k);
  }
  uint32_t bal = __ballot_sync(0xffffffffu, start);
  while (bal) {
    const int src = __ffs(bal) - 1;
    bal &= bal - 1;
    const uint32_t kk = __shfl_sync(0xffffffffu, k, src);
    double a = 0.0;
    for (int64_t j = base + src + lane; j < nkeys; j += 32) {
      if (skeys[j] != kk) break;                       // sorted: no later element of this lane matches
      a += svals[j];
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) a += __shfl_xor_sync(0xffffffffu, a, o);
    if (lane == 0) contrib[kk] = a;
  }
}

// grad[m][i] = lambda_m / (counts_m * n) * (sum_jt partial[m][jt][i] + contrib[m*d + i])  (fixed order)
__global__ void gradreduce_kernel(const double* __restrict__ partial, const double* __restrict__ contrib,
                                  const int64_t* __restrict__ counts, Lam8 lam, int n_mod, int nj, int64_t d,
                                  int64_t n, double* __restrict__ grad) {
  const int64_t idx = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (idx >= (int64_t)n_mod * d) return;
  const int m = (int)(idx / d);
  const int64_t i = idx - (int64_t)m * d;
  double a = 0.0;
  for (int jt = 0; jt < nj; ++jt) a += partial[((int64_t)m * nj + jt) * d + i];
  a += contrib[idx];
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
__global__ void adam_init_kernel(const float* __restrict__ s, double* __restrict__ theta, double* __restrict__ m1,
                                 double* __restrict__ m2, int64_t count) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= count) return;
  theta[i] = log((double)s[i]);
  m1[i] = 0.0;
  m2[i] = 0.0;
}

// best-so-far: if loss < best (or best is NaN), s_best = s and best = loss.  One CTA, so the
// decision is read by every thread before thread 0 overwrites best.
__global__ void __launch_bounds__(1024) keep_best_kernel(const double* __restrict__ loss, double* __restrict__ best,
                                                         const float* __restrict__ s, float* __restrict__ s_best,
                                                         int64_t count, int32_t* __restrict__ improved) {
  const double l = *loss, b = *best;
  const bool take = isfinite(l) && (l < b || isnan(b));
  if (take)
    for (int64_t i = threadIdx.x; i < count; i += blockDim.x) s_best[i] = s[i];
  __syncthreads();
  if (threadIdx.x == 0) {
    if (take) *best = l;
    if (improved) *improved = take ? 1 : 0;
  }
}
}  // namespace

cudaError_t launch_adam_init(const float* s, double* theta, double* m1, double* m2, int64_t count, cudaStream_t st) {
  ProfScope ps_("adam_init", st);
  adam_init_kernel<<<(unsigned)ceil_div(count, 256), 256, 0, st>>>(s, theta, m1, m2, count);
  return cudaGetLastError();
}

cudaError_t launch_keep_best(const double* loss, double* best, const float* s, float* s_best, int64_t count,
                             int32_t* improved, cudaStream_t st) {
  ProfScope ps_("keep_best", st);
  keep_best_kernel<<<1, 1024, 0, st>>>(loss, best, s, s_best, count, improved);
  return cudaGetLastError();
}

cudaError_t launch_gradprep(const uint16_t* X, int64_t ld_x, const uint8_t* mod_id, const int32_t* perm,
                            const int8_t* qx, const float* dx, const float* inv, int64_t Tg, int64_t d, int abits,
                            uint16_t* planes, int32_t* ktkey, int8_t* dq, float* de, int8_t* dq2, float* de2,
                            cudaStream_t st) {
  ProfScope ps_("gradprep", st);
  gradprep_kernel<<<(unsigned)ceil_div(Tg, 8), 256, 0, st>>>(X, ld_x, mod_id, perm, qx, dx, inv, Tg, d,
                                                             (float)((1 << (abits - 1)) - 1), planes, ktkey, dq, de,
                                                             dq2, de2);
  return cudaGetLastError();
}


cudaError_t launch_gradkeys(const float* bpart, int nb, const int32_t* kj, const uint32_t* colmax, int wbits,
                            const float* apart, int na, const int32_t* ktkey, int n_mod, int64_t d, int64_t n,
                            int64_t Tg, int32_t* keys, double* vals, cudaStream_t st) {
  ProfScope ps_("gradkeys", st, 2);
  betakeys_kernel<<<(unsigned)((int64_t)n_mod * n / 32), 256, 0, st>>>(bpart, nb, kj, colmax,
                                                                      (float)((1 << (wbits - 1)) - 1), d, n, keys,
                                                                      vals);
  const int64_t nj = (int64_t)n_mod * n;
  alphakeys_kernel<<<(unsigned)ceil_div(Tg, 256), 256, 0, st>>>(apart, na, ktkey, Tg, keys + nj, vals + nj);
  return cudaGetLastError();
}

size_t bucket_temp_bytes(int64_t nkeys) {
  size_t bytes = 0;
  cub::DeviceRadixSort::SortPairs(nullptr, bytes, (const uint32_t*)nullptr, (uint32_t*)nullptr, (const double*)nullptr,
                                  (double*)nullptr, (int)nkeys, 0, 32);
  return bytes;
}

cudaError_t launch_bucket(const int32_t* keys, const double* vals, int64_t nkeys, int64_t nl, uint32_t* skeys,
                          double* svals, void* temp, size_t temp_bytes, double* contrib, cudaStream_t st) {
  ProfScope ps_("bucket", st);
  cudaError_t e = cudaMemsetAsync(contrib, 0, sizeof(double) * nl, st);
  if (e != cudaSuccess) return e;
  // sort on the low B bits only, 2^B - 1 >= nl: valid keys (< nl) keep their order and the
  // invalid ones (-1, low bits all ones >= nl) still sort after them (radix sort is stable)
  int bits = 1;
  while (bits < 32 && ((1LL << bits) - 1) < nl) ++bits;
  size_t tb = temp_bytes;
  e = cub::DeviceRadixSort::SortPairs(temp, tb, reinterpret_cast<const uint32_t*>(keys), skeys, vals, svals,
                                      (int)nkeys, 0, bits, st);
  if (e != cudaSuccess) return e;
  runsum_kernel<<<(unsigned)ceil_div(nkeys, 256), 256, 0, st>>>(skeys, svals, nkeys, nl, contrib);
  return cudaGetLastError();
}

cudaError_t launch_gradgemm(const uint16_t* planes, int64_t Tg, const uint16_t* gsign, const int8_t* qw_all,
                            const uint32_t* tile_mod, int n_mod, int64_t d, int64_t n, const float* s,
                            const float* inv, const uint16_t* W, const float* dw, const uint32_t* colmax,
                            double* partial, float* bpart, int32_t* kj, cudaStream_t st) {
  CUtensorMap ta, tb, tq;
  bool ok = make_tmap_2d(&ta, planes, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, (uint64_t)NPL * Tg, d, d, 64, 64, true);
  ok &= make_tmap_2d(&tb, gsign, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, Tg, n, n, 64, 64, true);
  ok &= make_tmap_2d(&tq, qw_all, CU_TENSOR_MAP_DATA_TYPE_UINT8, 1, (uint64_t)n_mod * n, d, d, GN, GM, false);
  if (!ok) return cudaErrorInvalidValue;
  {
    cudaError_t e = set_max_dyn_smem(reinterpret_cast<const void*>(gradgemm_kernel), G_ALLOC);
    if (e != cudaSuccess) return e;
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
  p.colmax = colmax;
  p.partial = partial;
  p.bpart = bpart;
  p.kj = kj;
  const int grid = std::min(p.n_units, num_sms());
  ProfScope ps_("gradgemm", st);
  gradgemm_kernel<<<grid, GT, G_ALLOC, st>>>(ta, tb, tq, p);
  return cudaGetLastError();
}

int gradgemm_ntiles_j(int64_t n) { return (int)ceil_div(n, GN); }
int gradgemm_ntiles_i(int64_t d) { return (int)ceil_div(d, GM); }

cudaError_t launch_gradreduce(const double* partial, const double* contrib, const int64_t* counts,
                              const float* lambda_host, int n_mod, int nj, int64_t d, int64_t n, double* grad,
                              cudaStream_t st) {
  Lam8 l;
  for (int m = 0; m < kMaxMod; ++m) l.v[m] = (lambda_host && m < n_mod) ? lambda_host[m] : 1.0f;
  const int64_t count = (int64_t)n_mod * d;
  ProfScope ps_("gradreduce", st);
  gradreduce_kernel<<<(unsigned)ceil_div(count, 256), 256, 0, st>>>(partial, contrib, counts, l, n_mod, nj, d, n,
                                                                    grad);
  return cudaGetLastError();
}

cudaError_t launch_adam(double* theta, const double* grad, double* m1, double* m2, int64_t count, int step, double lr,
                        double b1, double b2, double eps, float* s_out, cudaStream_t st) {
  ProfScope ps_("adam", st);
  adam_kernel<<<(unsigned)ceil_div(count, 256), 256, 0, st>>>(theta, grad, m1, m2, count, step, lr, b1, b2, eps, s_out);
  return cudaGetLastError();
}

}  // namespace masq
