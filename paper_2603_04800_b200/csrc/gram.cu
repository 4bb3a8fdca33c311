// gram.cu — N2: the whitening Gram matrices G_m = (X_m S_m^-1)^T (X_m S_m^-1) of the
// CMC factor construction ("SVD(A^T A)" with A = X_m S_m^-1) on the tensor cores.
//
// A_m is the f32 smoothed activation the path computes (a = x * (1/s_m), IEEE mul).  Each value is
// split into a bf16 pair a = h + l (h = bf16(a), l = bf16(a - h); |a - h - l| <= 2^-17 |a|), and
//   G ~= H^T H + H^T L + L^T H + L^T L
// (all four products: dropping L^T L, <= 2^-18 |a||a'| per term but positive semidefinite, biases
// the Theorem-2 residual <E, G E> low by ~1e-6 of ||A dW||^2 — measured in a CPU emulation)
// is accumulated by tcgen05 kind::f16 MMAs in fp32 TMEM with the TOKEN axis as K (both operands
// MN-major, read from [tokens x d] planes).  Work unit = (modality, 128 x 256 tile of G, token
// chunk); only tiles on or above the block diagonal are computed (G is symmetric).  Every unit
// writes its fp32 partial tile; a reduction kernel adds the chunks of a tile in f64 in a fixed
// order (deterministic), and writes BOTH triangles of the row-major [d x d] G (each unordered
// pair {i, i'} comes from exactly one tile, so the matrix is exactly symmetric).
//
// Rows are taken in the loss's modality-grouped order (launch_route): modality m's tokens form one
// contiguous segment of the planes (padding rows zero), so a unit streams contiguous tokens.
#include <cuda_bf16.h>

#include "internal.h"
#include "sm100.cuh"

namespace masq {
using namespace sm100;

namespace {
constexpr int RT = 192;                       // warp 0 TMA, warp 1 MMA, warps 2..5 epilogue
constexpr int RM = 128, RN = 256, RK = 32;    // i rows, i' columns, tokens per k-block
constexpr int A_PL = RM * RK * 2;             // 8 KB: one plane of the A tile
constexpr int B_PL = RN * RK * 2;             // 16 KB: one plane of the B tile
constexpr int RSTAGE = 2 * A_PL + 2 * B_PL;   // 48 KB (H and L planes of both operands)
constexpr int RSTAGES = 4;
constexpr int R_SMEM = RSTAGES * RSTAGE + 256;
constexpr int R_ALLOC = R_SMEM + 1024;
constexpr uint32_t IDESC_R = idesc_bf16(RM, RN) | (1u << 15) | (1u << 16);   // A and B MN-major

struct RParams {
  int d, Tg, n_mod;
  const uint32_t* tile_mod;      // modality of every 256-row grouped unit (~0u = empty)
  int n_tm;
  int nti, ntj, n_tiles;         // tile grid (upper block triangle: it <= 2 jt + 1)
  int chunk_kb, max_chunks;      // k-blocks per token chunk; chunk slots per (modality, tile)
  int n_units;                   // (n_mod - 1) * n_tiles * max_chunks
  float* part;                   // [n_units][RN][RM] fp32 partial tiles (column-major in the tile)
};

__device__ __forceinline__ void seg_of(const RParams& p, int m, int& k0, int& nkb) {
  int first = -1, cnt = 0;
  for (int u = 0; u < p.n_tm; ++u)
    if (p.tile_mod[u] == (uint32_t)m) {
      if (first < 0) first = u;
      ++cnt;
    }
  k0 = first < 0 ? 0 : first * kUnitM;
  nkb = cnt * (kUnitM / RK);
}

// tile index -> (it, jt) over the upper block triangle, jt-major
__device__ __forceinline__ void tile_of(const RParams& p, int t, int& it, int& jt) {
  jt = 0;
  for (;;) {
    const int cnt = min(p.nti, 2 * jt + 2);
    if (t < cnt) break;
    t -= cnt;
    ++jt;
  }
  it = t;
}

struct Work {
  int m, it, jt, kb0, kb1, k0;
  bool live;
};

__device__ __forceinline__ Work decode(const RParams& p, int u) {
  Work w;
  const int per_m = p.n_tiles * p.max_chunks;
  w.m = 1 + u / per_m;
  const int r = u - (w.m - 1) * per_m;
  const int t = r / p.max_chunks, c = r - t * p.max_chunks;
  tile_of(p, t, w.it, w.jt);
  int nkb;
  seg_of(p, w.m, w.k0, nkb);
  w.kb0 = c * p.chunk_kb;
  w.kb1 = min(nkb, w.kb0 + p.chunk_kb);
  w.live = w.kb0 < w.kb1;
  return w;
}

__global__ void __launch_bounds__(RT, 1)
cmc_gram_kernel(const __grid_constant__ CUtensorMap tmP, const RParams p) {
  extern __shared__ uint8_t smem_raw[];
  const uint32_t raw = smem_u32(smem_raw);
  uint8_t* smem = smem_raw + (((raw + 1023u) & ~1023u) - raw);
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + RSTAGES * RSTAGE);
  uint64_t* empty = full + RSTAGES;
  uint64_t* tfull = empty + RSTAGES;       // [2]
  uint64_t* tempty = tfull + 2;            // [2]
  uint32_t* tslot = reinterpret_cast<uint32_t*>(tempty + 2);
  const uint32_t warp = warp_id(), lane = lane_id();
  if (warp == 0 && lane == 0) {
    tma_prefetch(&tmP);
    for (int i = 0; i < RSTAGES; ++i) { mbar_init(&full[i], 1); mbar_init(&empty[i], 1); }
    for (int i = 0; i < 2; ++i) { mbar_init(&tfull[i], 1); mbar_init(&tempty[i], 4); }
    fence_mbar_init();
  }
  if (warp == 1) tmem_alloc(tslot, 512);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tslot;

  if (warp == 0) {
    if (lane == 0) {
      // ------------------------------------------------------------ TMA producer
      uint32_t st = 0, ph = 0;
      for (int u = blockIdx.x; u < p.n_units; u += gridDim.x) {
        const Work w = decode(p, u);
        if (!w.live) continue;
        for (int kb = w.kb0; kb < w.kb1; ++kb) {
          mbar_wait(&empty[st], ph ^ 1u);
          mbar_expect_tx(&full[st], RSTAGE);
          uint8_t* base = smem + st * RSTAGE;
          const int t = w.k0 + kb * RK;
#pragma unroll
          for (int pl = 0; pl < 2; ++pl) {
#pragma unroll
            for (int h = 0; h < 2; ++h)
              tma_load_2d(base + pl * A_PL + h * (A_PL / 2), &tmP, &full[st], w.it * RM + h * 64, pl * p.Tg + t);
#pragma unroll
            for (int q = 0; q < 4; ++q)
              tma_load_2d(base + 2 * A_PL + pl * B_PL + q * (B_PL / 4), &tmP, &full[st], w.jt * RN + q * 64,
                          pl * p.Tg + t);
          }
          if (++st == RSTAGES) { st = 0; ph ^= 1u; }
        }
      }
    }
    __syncwarp();
  } else if (warp == 1) {
    if (lane == 0) {
      // ------------------------------------------------------------ MMA issuer
      uint32_t st = 0, ph = 0, local = 0;
      for (int u = blockIdx.x; u < p.n_units; u += gridDim.x) {
        const Work w = decode(p, u);
        if (!w.live) continue;
        const uint32_t buf = local & 1u, bph = (local >> 1) & 1u;
        ++local;
        mbar_wait(&tempty[buf], bph ^ 1u);
        tc_fence_after();
        const uint32_t acc = tmem + buf * RN;
        for (int kb = w.kb0; kb < w.kb1; ++kb) {
          mbar_wait(&full[st], ph);
          tc_fence_after();
          const uint32_t base = smem_u32(smem + st * RSTAGE);
#pragma unroll
          for (int kk = 0; kk < RK / 16; ++kk) {
            const uint64_t aH = umma_desc_sw128_mn(base + kk * 2048, A_PL / 2);
            const uint64_t aL = umma_desc_sw128_mn(base + A_PL + kk * 2048, A_PL / 2);
            const uint64_t bH = umma_desc_sw128_mn(base + 2 * A_PL + kk * 2048, B_PL / 4);
            const uint64_t bL = umma_desc_sw128_mn(base + 2 * A_PL + B_PL + kk * 2048, B_PL / 4);
            mma_bf16(acc, aH, bH, IDESC_R, (kb != w.kb0 || kk != 0) ? 1u : 0u);
            mma_bf16(acc, aH, bL, IDESC_R, 1u);
            mma_bf16(acc, aL, bH, IDESC_R, 1u);
            mma_bf16(acc, aL, bL, IDESC_R, 1u);
          }
          mma_commit(&empty[st]);
          if (++st == RSTAGES) { st = 0; ph ^= 1u; }
        }
        mma_commit(&tfull[buf]);
      }
    }
    __syncwarp();
  } else {
    // -------------------------------------------------------------- epilogue: TMEM -> partial tile
    const uint32_t q = warp & 3u;
    uint32_t local = 0;
    for (int u = blockIdx.x; u < p.n_units; u += gridDim.x) {
      const Work w = decode(p, u);
      if (!w.live) continue;
      const uint32_t buf = local & 1u, bph = (local >> 1) & 1u;
      ++local;
      mbar_wait(&tfull[buf], bph);
      tc_fence_after();
      const uint32_t taddr = tmem + ((q * 32u) << 16) + buf * RN;
      float* out = p.part + (size_t)u * RN * RM + q * 32 + lane;      // [col][row], row = q*32 + lane
#pragma unroll 1
      for (int c = 0; c < RN / 32; ++c) {
        uint32_t v[32];
        tmem_ld32(taddr + c * 32, v);
        tmem_wait_ld();
#pragma unroll
        for (int k = 0; k < 32; ++k) out[(size_t)(c * 32 + k) * RM] = __uint_as_float(v[k]);
      }
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(&tempty[buf]);
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 1) {
    tc_fence_after();
    tmem_dealloc(tmem, 512);
  }
}

// planes [2][Tg][d] bf16 of the non-text rows in grouped order: h = bf16(a), l = bf16(a - h),
// a = x * inv_m (f32); padding rows of non-text segments are zero; text rows are not written
template <typename XT>
__global__ void __launch_bounds__(256) gram_planes_kernel(const XT* __restrict__ X, int64_t ld_x,
                                                          const uint8_t* __restrict__ ids,
                                                          const int32_t* __restrict__ perm,
                                                          const uint32_t* __restrict__ tile_mod,
                                                          const float* __restrict__ inv, int64_t Tg, int64_t d,
                                                          uint16_t* __restrict__ planes) {
  const int64_t p = (int64_t)blockIdx.x * 8 + (threadIdx.x >> 5);
  const int lane = threadIdx.x & 31;
  if (p >= Tg) return;
  const uint32_t um = tile_mod[p / kUnitM];
  if (um == 0u || um == 0xFFFFFFFFu) return;                    // text unit or unused
  const int32_t src = perm[p];
  const float* invm = inv + (int64_t)um * d;
  uint16_t* ph = planes + p * d;
  uint16_t* pl = planes + (Tg + p) * d;
  for (int64_t c = (int64_t)lane * 8; c < d; c += 256) {
    uint4 hv = make_uint4(0, 0, 0, 0), lv = make_uint4(0, 0, 0, 0);
    if (src >= 0) {
      float x[8];
      if (sizeof(XT) == 2) {
        const uint4 xv = __ldg(reinterpret_cast<const uint4*>(reinterpret_cast<const uint16_t*>(X) + src * ld_x + c));
        const uint32_t xw[4] = {xv.x, xv.y, xv.z, xv.w};
#pragma unroll
        for (int k = 0; k < 8; ++k) x[k] = __uint_as_float((k & 1) ? (xw[k >> 1] & 0xFFFF0000u) : (xw[k >> 1] << 16));
      } else {
        const float4 a0 = __ldg(reinterpret_cast<const float4*>(reinterpret_cast<const float*>(X) + src * ld_x + c));
        const float4 a1 =
            __ldg(reinterpret_cast<const float4*>(reinterpret_cast<const float*>(X) + src * ld_x + c + 4));
        x[0] = a0.x; x[1] = a0.y; x[2] = a0.z; x[3] = a0.w;
        x[4] = a1.x; x[5] = a1.y; x[6] = a1.z; x[7] = a1.w;
      }
      const float4 i0 = __ldg(reinterpret_cast<const float4*>(invm + c));
      const float4 i1 = __ldg(reinterpret_cast<const float4*>(invm + c + 4));
      const float iv[8] = {i0.x, i0.y, i0.z, i0.w, i1.x, i1.y, i1.z, i1.w};
      uint32_t hw[4], lw[4];
#pragma unroll
      for (int e = 0; e < 4; ++e) {
        uint32_t hh[2], ll[2];
#pragma unroll
        for (int k = 0; k < 2; ++k) {
          const float a = __fmul_rn(x[2 * e + k], iv[2 * e + k]);
          const __nv_bfloat16 h = __float2bfloat16_rn(a);
          const float r = __fsub_rn(a, __bfloat162float(h));
          hh[k] = __bfloat16_as_ushort(h);
          ll[k] = __bfloat16_as_ushort(__float2bfloat16_rn(r));
        }
        hw[e] = hh[0] | (hh[1] << 16);
        lw[e] = ll[0] | (ll[1] << 16);
      }
      hv = make_uint4(hw[0], hw[1], hw[2], hw[3]);
      lv = make_uint4(lw[0], lw[1], lw[2], lw[3]);
    }
    *reinterpret_cast<uint4*>(ph + c) = hv;
    *reinterpret_cast<uint4*>(pl + c) = lv;
  }
}

// G[m-1] (+)= sum over the chunks (fixed order, f64) of the partial tiles; both triangles.
// Block = one 32 x 32 sub-block of a tile (8 x 4 per tile); grid.x = tile * 32 + sub, grid.y = m - 1.
__global__ void __launch_bounds__(256) gram_reduce_kernel(const RParams p, double* __restrict__ G, int accumulate) {
  __shared__ double sh[32][33];
  const int m = 1 + (int)blockIdx.y;
  const int t = (int)blockIdx.x >> 5, sub = (int)blockIdx.x & 31;
  int it, jt;
  tile_of(p, t, it, jt);
  const int r0 = (sub & 3) * 32, c0 = (sub >> 2) * 32;          // sub-block origin inside the 128 x 256 tile
  int k0, nkb;
  seg_of(p, m, k0, nkb);
  const int nch = min(p.max_chunks, (nkb + p.chunk_kb - 1) / p.chunk_kb);
  const int d = p.d;
  double* Gm = G + (size_t)(m - 1) * d * d;
  const int tx = threadIdx.x & 31, ty = threadIdx.x >> 5;
  const size_t ubase = ((size_t)(m - 1) * p.n_tiles + t) * p.max_chunks;
  for (int cc = ty; cc < 32; cc += 8) {
    const int col = c0 + cc, row = r0 + tx;
    double a = 0.0;
    for (int c = 0; c < nch; ++c) a += (double)p.part[((ubase + c) * RN + col) * RM + row];
    sh[cc][tx] = a;
  }
  __syncthreads();
  // (1) G[i'][i] with i = it*128 + r0 + tx (row fastest: contiguous), for i <= i'
  for (int cc = ty; cc < 32; cc += 8) {
    const int i = it * RM + r0 + tx, i2 = jt * RN + c0 + cc;
    if (i < d && i2 < d && i <= i2) {
      double* g = Gm + (size_t)i2 * d + i;
      *g = (accumulate ? *g : 0.0) + sh[cc][tx];
    }
  }
  // (2) G[i][i'] (i' fastest: contiguous), for i < i'
  for (int rr = ty; rr < 32; rr += 8) {
    const int i = it * RM + r0 + rr, i2 = jt * RN + c0 + tx;
    if (i < d && i2 < d && i < i2) {
      double* g = Gm + (size_t)i * d + i2;
      *g = (accumulate ? *g : 0.0) + sh[tx][rr];
    }
  }
}

RParams make_params(int64_t T, int64_t d, int n_mod, const uint32_t* tile_mod, float* part) {
  RParams p{};
  const int64_t Tg = grouped_rows(T, n_mod);
  p.d = (int)d;
  p.Tg = (int)Tg;
  p.n_mod = n_mod;
  p.tile_mod = tile_mod;
  p.n_tm = (int)(Tg / kUnitM);
  p.nti = (int)ceil_div(d, RM);
  p.ntj = (int)ceil_div(d, RN);
  p.n_tiles = 0;
  for (int jt = 0; jt < p.ntj; ++jt) p.n_tiles += std::min(p.nti, 2 * jt + 2);
  // token chunks: at least 2048 tokens, at most 4 chunk slots over the whole grouped batch
  const int64_t kb_total = ceil_div(Tg, RK);
  p.chunk_kb = (int)std::max<int64_t>(2048 / RK, ceil_div(kb_total, 4));
  p.max_chunks = (int)ceil_div(kb_total, p.chunk_kb);
  p.n_units = std::max(n_mod - 1, 0) * p.n_tiles * p.max_chunks;
  p.part = part;
  return p;
}
}  // namespace

size_t cmc_gram_part_bytes(int64_t T, int64_t d, int n_mod) {
  const RParams p = make_params(T, d, n_mod, nullptr, nullptr);
  return sizeof(float) * (size_t)p.n_units * RN * RM;
}

cudaError_t launch_cmc_gram_tc(const void* X, masq_dtype xt, int64_t ld_x, const uint8_t* ids, int64_t T,
                               int64_t d, int n_mod, const float* inv, const int32_t* perm,
                               const uint32_t* tile_mod, uint16_t* planes, float* part, double* G, int accumulate,
                               cudaStream_t st) {
  if (n_mod < 2) return cudaSuccess;
  const int64_t Tg = grouped_rows(T, n_mod);
  {
    ProfScope ps_("cmc_planes", st);
    const unsigned g = (unsigned)ceil_div(Tg, 8);
    if (xt == MASQ_BF16)
      gram_planes_kernel<<<g, 256, 0, st>>>(static_cast<const uint16_t*>(X), ld_x, ids, perm, tile_mod, inv, Tg, d,
                                            planes);
    else
      gram_planes_kernel<<<g, 256, 0, st>>>(static_cast<const float*>(X), ld_x, ids, perm, tile_mod, inv, Tg, d,
                                            planes);
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) return e;
  }
  CUtensorMap tp;
  if (!make_tmap_2d(&tp, planes, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, 2 * (uint64_t)Tg, d, d, RK, 64, true))
    return cudaErrorInvalidValue;
  const RParams p = make_params(T, d, n_mod, tile_mod, part);
  {
    cudaError_t e = set_max_dyn_smem(reinterpret_cast<const void*>(cmc_gram_kernel), R_ALLOC);
    if (e != cudaSuccess) return e;
  }
  {
    ProfScope ps_("cmc_gram", st);
    const int grid = (int)std::min<int64_t>(p.n_units, num_sms());
    cmc_gram_kernel<<<grid, RT, R_ALLOC, st>>>(tp, p);
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) return e;
  }
  ProfScope ps_("cmc_gram_reduce", st);
  dim3 grid((unsigned)p.n_tiles * 32, (unsigned)(n_mod - 1));
  gram_reduce_kernel<<<grid, 256, 0, st>>>(p, G, accumulate);
  return cudaGetLastError();
}

}  // namespace masq
