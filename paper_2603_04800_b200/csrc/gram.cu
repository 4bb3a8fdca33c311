// gram.cu — N2: the whitening Gram matrices G_m = A_m^T A_m, A_m = X_m S_m^-1, of the
// CMC factor construction ("SVD(A^T A)") on the int8 tensor cores, EXACTLY.
//
// Why exact: the whitening regulariser is eps * lambda_max with eps = 1e-8 (reading Q27), and a
// calibration batch often has fewer tokens of a modality than channels (3072 image tokens vs
// d = 3584 or 18944), so G is rank-deficient and its null-space eigenvalues must stay within
// ~1e-9 lambda_max of zero for the Cholesky factor of G + eps lambda_max I to exist.  fp32 tensor
// core accumulation of split-bf16 products leaves them at ~+-1e-6 lambda_max (measured: the
// factorisation fails); integer accumulation has no rounding at all.
//
// Representation: per modality and channel i a power-of-two scale 2^e_i with |a_ti| / 2^e_i < 64
// (e_i from the channel's max |a| = R^m_i * (1/s^m_i), exact: rounding is monotonic), and three
// int8 slices u = a / 2^e_i = S0 + S1 / 128 + S2 / 128^2 + r, |r| <= 2^-15, every step exact in f32
// (S0 = rint(u), S1 = rint((u - S0) * 128), S2 = rint(((u - S0) * 128 - S1) * 128); all in
// [-64, 64]).  So a_hat = 2^e (S0 + S1/128 + S2/128^2) differs from a by <= 2^-20 of the channel's
// max, and
//   G_hat_ij = 2^(e_i + e_j) * sum_{k=0..4} 128^-k * sum_{s + s' = k} sum_t S_s[t,i] S_s'[t,j]
// is the Gram of a_hat computed with no rounding except the final f64 combination (9 kind::i8
// products into 5 int32 TMEM accumulators, one per level k): positive semidefinite to f64
// rounding, and within ~1e-7 of G where it matters.
//
// Layout: the slices are written TRANSPOSED (channel rows, token columns in the loss's modality-
// grouped order from launch_route) so both MMA operands are ordinary K-major SWIZZLE_128B tiles
// with the token axis as K.  Work unit = (modality, 128 x 96 tile of G on or above the block
// diagonal, token chunk); each unit writes its f64 tile; a reduction adds the chunks in a fixed
// order (deterministic) and writes BOTH triangles of the row-major [d x d] G (each unordered pair
// {i, j} comes from exactly one tile, so G is exactly symmetric).
#include <cuda_bf16.h>

#include "internal.h"
#include "sm100.cuh"

namespace masq {
using namespace sm100;

namespace {
constexpr int RT = 192;                       // warp 0 TMA, warp 1 MMA, warps 2..5 epilogue
constexpr int RM = 128, RN = 96, RK = 128;    // i rows, j columns, tokens per k-block
constexpr int NSL = 3;                        // int8 slices per value
constexpr int NLV = 2 * NSL - 1;              // levels k = s + s'
constexpr int A_SL = RM * RK;                 // 16 KB: one slice of the A tile
constexpr int B_SL = RN * RK;                 // 12 KB
constexpr int RSTAGE = NSL * (A_SL + B_SL);   // 84 KB
constexpr int RSTAGES = 2;
constexpr int R_SMEM = RSTAGES * RSTAGE + 256;
constexpr int R_ALLOC = R_SMEM + 1024;
constexpr uint32_t IDESC_R = idesc_i8(RM, RN);
static_assert(NLV * RN <= 512, "TMEM columns");
static_assert(R_ALLOC <= 232448, "shared memory budget");

struct RParams {
  int d, Tg, n_mod;
  const uint32_t* tile_mod;      // modality of every 256-row grouped unit (~0u = empty)
  int n_tm;
  int nti, ntj, n_tiles;         // tile grid over the upper block triangle
  int chunk_kb, max_chunks;      // k-blocks per token chunk; chunk slots per (modality, tile)
  int n_units;                   // (n_mod - 1) * n_tiles * max_chunks
  const int32_t* ex;             // [n_mod][d] channel exponents e_i
  double* part;                  // [n_units][RN][RM] f64 tiles (column-major in the tile)
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

// tiles of jt-column block: it with 128 it <= 96 jt + 95 (some i <= j inside), jt-major
__device__ __host__ __forceinline__ int tiles_in_col(int nti, int jt) {
  const int lim = (RN * jt + RN - 1) / RM + 1;
  return lim < nti ? lim : nti;
}
__device__ __forceinline__ void tile_of(const RParams& p, int t, int& it, int& jt) {
  jt = 0;
  for (;;) {
    const int cnt = tiles_in_col(p.nti, jt);
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
cmc_gram_kernel(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB, const RParams p) {
  extern __shared__ uint8_t smem_raw[];
  const uint32_t raw = smem_u32(smem_raw);
  uint8_t* smem = smem_raw + (((raw + 1023u) & ~1023u) - raw);
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + RSTAGES * RSTAGE);
  uint64_t* empty = full + RSTAGES;
  uint64_t* tfull = empty + RSTAGES;
  uint64_t* tempty = tfull + 1;
  uint32_t* tslot = reinterpret_cast<uint32_t*>(tempty + 1);
  const uint32_t warp = warp_id(), lane = lane_id();
  if (warp == 0 && lane == 0) {
    tma_prefetch(&tmA);
    tma_prefetch(&tmB);
    for (int i = 0; i < RSTAGES; ++i) { mbar_init(&full[i], 1); mbar_init(&empty[i], 1); }
    mbar_init(tfull, 1);
    mbar_init(tempty, 4);
    fence_mbar_init();
  }
  if (warp == 1) tmem_alloc(tslot, 512);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tslot;

  if (warp == 0) {
    {
      // ------------------------------------------------------------ TMA producer
      // (warp-wide loops with uniform state; one elected lane issues copies / MMAs)
      uint32_t st = 0, ph = 0;
      for (int u = blockIdx.x; u < p.n_units; u += gridDim.x) {
        const Work w = decode(p, u);
        if (!w.live) continue;
        for (int kb = w.kb0; kb < w.kb1; ++kb) {
          mbar_wait(&empty[st], ph ^ 1u);
          if (elect_one()) {
            mbar_expect_tx(&full[st], RSTAGE);
            uint8_t* base = smem + st * RSTAGE;
            const int t = w.k0 + kb * RK;
#pragma unroll
            for (int s = 0; s < NSL; ++s) {
              tma_load_2d(base + s * A_SL, &tmA, &full[st], t, s * p.d + w.it * RM);
              tma_load_2d(base + NSL * A_SL + s * B_SL, &tmB, &full[st], t, s * p.d + w.jt * RN);
            }
          }
          __syncwarp();
          if (++st == RSTAGES) { st = 0; ph ^= 1u; }
        }
      }
    }
    __syncwarp();
  } else if (warp == 1) {
    {
      // ------------------------------------------------------------ MMA issuer
      uint32_t st = 0, ph = 0, local = 0;
      for (int u = blockIdx.x; u < p.n_units; u += gridDim.x) {
        const Work w = decode(p, u);
        if (!w.live) continue;
        mbar_wait(tempty, (local & 1u) ^ 1u);
        ++local;
        tc_fence_after();
        bool fresh[NLV];
#pragma unroll
        for (int k = 0; k < NLV; ++k) fresh[k] = true;
        for (int kb = w.kb0; kb < w.kb1; ++kb) {
          mbar_wait(&full[st], ph);
          tc_fence_after();
          if (elect_one()) {
            const uint32_t base = smem_u32(smem + st * RSTAGE);
            const uint64_t ad = umma_desc_sw128(base), bd = umma_desc_sw128(base + NSL * A_SL);
#pragma unroll
            for (int kk = 0; kk < RK / 32; ++kk) {
#pragma unroll
              for (int s = 0; s < NSL; ++s) {
#pragma unroll
                for (int s2 = 0; s2 < NSL; ++s2) {
                  const int lv = s + s2;
                  mma_i8(tmem + lv * RN, ad + (s * A_SL + kk * 32) / 16, bd + (s2 * B_SL + kk * 32) / 16, IDESC_R,
                         (fresh[lv] && kk == 0 && s == (lv < NSL ? 0 : lv - (NSL - 1))) ? 0u : 1u);
                }
              }
            }
            mma_commit(&empty[st]);
          }
          __syncwarp();
#pragma unroll
          for (int k = 0; k < NLV; ++k) fresh[k] = false;
          if (++st == RSTAGES) { st = 0; ph ^= 1u; }
        }
        if (elect_one()) mma_commit(tfull);
        __syncwarp();
      }
    }
    __syncwarp();
  } else {
    // -------------------------------------------------------------- epilogue: 5 levels -> f64 tile
    const uint32_t q = warp & 3u;
    uint32_t local = 0;
    for (int u = blockIdx.x; u < p.n_units; u += gridDim.x) {
      const Work w = decode(p, u);
      if (!w.live) continue;
      const int row = (int)(q * 32u + lane);
      const int i = w.it * RM + row;
      const int32_t* exm = p.ex + (size_t)w.m * p.d;
      const int ei = i < p.d ? __ldg(exm + i) : 0;
      mbar_wait(tfull, local & 1u);
      ++local;
      tc_fence_after();
      const uint32_t taddr = tmem + ((q * 32u) << 16);
      double* out = p.part + (size_t)u * RN * RM + row;            // [col][row]
#pragma unroll 1
      for (int c = 0; c < RN / 32; ++c) {
        double g[32];
#pragma unroll
        for (int k = 0; k < 32; ++k) g[k] = 0.0;
        double wl = 1.0;
#pragma unroll
        for (int lv = 0; lv < NLV; ++lv) {
          uint32_t v[32];
          tmem_ld32(taddr + lv * RN + c * 32, v);
          tmem_wait_ld();
#pragma unroll
          for (int k = 0; k < 32; ++k) g[k] = fma((double)(int)v[k], wl, g[k]);
          wl *= 0.0078125;                                             // 128^-1, exact
        }
#pragma unroll
        for (int k = 0; k < 32; ++k) {
          const int j = w.jt * RN + c * 32 + k;
          const int ej = j < p.d ? __ldg(exm + j) : 0;
          out[(size_t)(c * 32 + k) * RM] = ldexp(g[k], ei + ej);
        }
      }
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(tempty);
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 1) {
    tc_fence_after();
    tmem_dealloc(tmem, 512);
  }
}

// channel exponents e[m][i] = ilogb(max_t |a_ti|) - 5 (|a| / 2^e < 64), from R^m and 1/s^m
__global__ void gram_exp_kernel(const float* __restrict__ R, const float* __restrict__ inv, int64_t count,
                                int32_t* __restrict__ ex) {
  const int64_t k = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (k >= count) return;
  const float amax = __fmul_rn(R[k], inv[k]);
  ex[k] = amax > 0.f ? ilogbf(amax) - 5 : 0;
}

// slices S_s [NSL][d][Tg] (channel rows, grouped-token columns) of the non-text rows; padding rows
// give zeros; text columns are not written.  Block = 64 grouped rows x 128 channels, transposed
// through shared memory.
template <typename XT>
__global__ void __launch_bounds__(256) gram_slices_kernel(const XT* __restrict__ X, int64_t ld_x,
                                                          const int32_t* __restrict__ perm,
                                                          const uint32_t* __restrict__ tile_mod,
                                                          const float* __restrict__ inv,
                                                          const int32_t* __restrict__ ex, int64_t Tg, int64_t d,
                                                          int8_t* __restrict__ S) {
  __shared__ int8_t sh[NSL][128][64 + 4];
  const int64_t p0 = (int64_t)blockIdx.x * 64;
  const int64_t c0 = (int64_t)blockIdx.y * 128;
  const uint32_t um = tile_mod[p0 / kUnitM];                   // 64 rows never straddle a 256-row unit
  if (um == 0u || um == 0xFFFFFFFFu) return;
  const float* invm = inv + (int64_t)um * d;
  const int32_t* exm = ex + (int64_t)um * d;
  // load: thread (r = tid / 4, c = (tid % 4) * 32 .. +32): one row's 32 channels
  const int tid = threadIdx.x;
  for (int r = tid >> 2; r < 64; r += 64) {
    const int64_t prow = p0 + r;
    const int32_t src = perm[prow];
    const int cb = (tid & 3) * 32;
#pragma unroll 4
    for (int k = 0; k < 32; ++k) {
      const int64_t i = c0 + cb + k;
      int s0 = 0, s1 = 0, s2 = 0;
      if (src >= 0 && i < d) {
        const float x = (float)X[(int64_t)src * ld_x + i];
        const float a = __fmul_rn(x, __ldg(invm + i));
        const float u = ldexpf(a, -__ldg(exm + i));          // exact, |u| < 64
        const float f0 = rintf(u);
        const float r1 = (u - f0) * 128.0f;                  // exact
        const float f1 = rintf(r1);
        const float f2 = rintf((r1 - f1) * 128.0f);          // (r1 - f1) * 128 exact
        s0 = (int)f0;
        s1 = (int)f1;
        s2 = (int)f2;
      }
      sh[0][cb + k][r] = (int8_t)s0;
      sh[1][cb + k][r] = (int8_t)s1;
      sh[2][cb + k][r] = (int8_t)s2;
    }
  }
  __syncthreads();
  // store: per slice, 128 channel rows x 64 bytes; thread -> (slice row, 16-byte quarter)
  for (int e = tid; e < NSL * 128 * 4; e += 256) {
    const int s = e / 512, rem = e - s * 512, row = rem >> 2, qtr = rem & 3;
    const int64_t i = c0 + row;
    if (i >= d) continue;
    const int8_t* sp = &sh[s][row][qtr * 16];
    uint32_t w[4];
#pragma unroll
    for (int b = 0; b < 4; ++b)
      w[b] = (uint32_t)(uint8_t)sp[4 * b] | ((uint32_t)(uint8_t)sp[4 * b + 1] << 8) |
             ((uint32_t)(uint8_t)sp[4 * b + 2] << 16) | ((uint32_t)(uint8_t)sp[4 * b + 3] << 24);
    *reinterpret_cast<uint4*>(S + ((int64_t)s * d + i) * Tg + p0 + qtr * 16) = make_uint4(w[0], w[1], w[2], w[3]);
  }
}

// G[m-1] (+)= sum over the chunks (fixed order) of the f64 tiles; both triangles.
// Block = one 32 x 32 sub-block of a 128 x 96 tile (4 x 3); grid.x = tile * 12 + sub, grid.y = m - 1.
__global__ void __launch_bounds__(256) gram_reduce_kernel(const RParams p, double* __restrict__ G, int accumulate) {
  __shared__ double sh[32][33];
  const int m = 1 + (int)blockIdx.y;
  const int t = (int)blockIdx.x / 12, sub = (int)blockIdx.x % 12;
  int it, jt;
  tile_of(p, t, it, jt);
  const int r0 = (sub & 3) * 32, c0 = (sub >> 2) * 32;
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
    for (int c = 0; c < nch; ++c) a += p.part[((ubase + c) * RN + col) * RM + row];
    sh[cc][tx] = a;
  }
  __syncthreads();
  for (int cc = ty; cc < 32; cc += 8) {                        // G[j][i], i fastest, i <= j
    const int i = it * RM + r0 + tx, j = jt * RN + c0 + cc;
    if (i < d && j < d && i <= j) {
      double* g = Gm + (size_t)j * d + i;
      *g = (accumulate ? *g : 0.0) + sh[cc][tx];
    }
  }
  for (int rr = ty; rr < 32; rr += 8) {                        // G[i][j], j fastest, i < j
    const int i = it * RM + r0 + rr, j = jt * RN + c0 + tx;
    if (i < d && j < d && i < j) {
      double* g = Gm + (size_t)i * d + j;
      *g = (accumulate ? *g : 0.0) + sh[tx][rr];
    }
  }
}

RParams make_params(int64_t T, int64_t d, int n_mod, const uint32_t* tile_mod, const int32_t* ex, double* part) {
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
  for (int jt = 0; jt < p.ntj; ++jt) p.n_tiles += tiles_in_col(p.nti, jt);
  // token chunks only to fill the SMs when the tiles alone do not (>= 2048 tokens each); int32
  // accumulation is exact for any chunk here (|S| <= 64: 3 * 64^2 * 2^16 < 2^31 per level)
  const int64_t kb_total = ceil_div(Tg, RK);
  const int64_t tiles_all = (int64_t)std::max(n_mod - 1, 1) * p.n_tiles;
  const int64_t want = std::max<int64_t>(1, ceil_div(4 * 148, tiles_all));
  p.chunk_kb = (int)std::min<int64_t>(std::max<int64_t>(2048 / RK, ceil_div(kb_total, want)), 65536 / RK);
  p.max_chunks = (int)ceil_div(kb_total, p.chunk_kb);
  p.n_units = std::max(n_mod - 1, 0) * p.n_tiles * p.max_chunks;
  p.ex = ex;
  p.part = part;
  return p;
}
}  // namespace

size_t cmc_gram_part_bytes(int64_t T, int64_t d, int n_mod) {
  const RParams p = make_params(T, d, n_mod, nullptr, nullptr, nullptr);
  return sizeof(double) * (size_t)p.n_units * RN * RM;
}
size_t cmc_gram_slice_bytes(int64_t T, int64_t d, int n_mod) { return (size_t)NSL * d * grouped_rows(T, n_mod); }

cudaError_t launch_cmc_gram_tc(const void* X, masq_dtype xt, int64_t ld_x, const uint8_t* ids, int64_t T,
                               int64_t d, int n_mod, const float* inv, const int32_t* perm,
                               const uint32_t* tile_mod, float* R, int64_t* cnt, int32_t* ex, int8_t* slices,
                               double* part, uint32_t* status, double* G, int accumulate, cudaStream_t st) {
  if (n_mod < 2) return cudaSuccess;
  const int64_t Tg = grouped_rows(T, n_mod);
  // per-modality channel maxima of |x| -> exponents of the channel scales
  cudaError_t e = cudaMemsetAsync(R, 0, sizeof(float) * n_mod * d, st);
  if (e == cudaSuccess) e = cudaMemsetAsync(cnt, 0, sizeof(int64_t) * n_mod, st);
  if (e != cudaSuccess) return e;
  e = launch_stats(X, xt, ld_x, ids, T, d, n_mod, R, cnt, status, st);
  if (e != cudaSuccess) return e;
  {
    ProfScope ps_("cmc_slices", st, 2);
    gram_exp_kernel<<<(unsigned)ceil_div((int64_t)n_mod * d, 256), 256, 0, st>>>(R, inv, (int64_t)n_mod * d, ex);
    dim3 grid((unsigned)(Tg / 64), (unsigned)ceil_div(d, 128));
    if (xt == MASQ_BF16)
      gram_slices_kernel<<<grid, 256, 0, st>>>(static_cast<const __nv_bfloat16*>(X), ld_x, perm, tile_mod, inv, ex,
                                               Tg, d, slices);
    else
      gram_slices_kernel<<<grid, 256, 0, st>>>(static_cast<const float*>(X), ld_x, perm, tile_mod, inv, ex, Tg, d,
                                               slices);
    e = cudaGetLastError();
    if (e != cudaSuccess) return e;
  }
  CUtensorMap ta, tb;
  bool ok = make_tmap_2d(&ta, slices, CU_TENSOR_MAP_DATA_TYPE_UINT8, 1, (uint64_t)NSL * d, Tg, Tg, RM, RK, true);
  ok &= make_tmap_2d(&tb, slices, CU_TENSOR_MAP_DATA_TYPE_UINT8, 1, (uint64_t)NSL * d, Tg, Tg, RN, RK, true);
  if (!ok) return cudaErrorInvalidValue;
  const RParams p = make_params(T, d, n_mod, tile_mod, ex, part);
  e = set_max_dyn_smem(reinterpret_cast<const void*>(cmc_gram_kernel), R_ALLOC);
  if (e != cudaSuccess) return e;
  {
    ProfScope ps_("cmc_gram", st);
    const int grid = (int)std::min<int64_t>(p.n_units, num_sms());
    cmc_gram_kernel<<<grid, RT, R_ALLOC, st>>>(ta, tb, p);
    e = cudaGetLastError();
    if (e != cudaSuccess) return e;
  }
  ProfScope ps_("cmc_gram_reduce", st);
  dim3 grid((unsigned)p.n_tiles * 12, (unsigned)(n_mod - 1));
  gram_reduce_kernel<<<grid, 256, 0, st>>>(p, G, accumulate);
  return cudaGetLastError();
}

}  // namespace masq
