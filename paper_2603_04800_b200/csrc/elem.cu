// elem.cu — HBM-bound kernels of the MASQuant hot path (sm_100a):
//   stats (A1), factor init (A2), weight smoothing + quantization (A3),
//   routed activation smoothing + per-token quantization (A4), low-rank factor packing,
//   bf16 transpose, and the deterministic loss reduction (A8).
// Every quantizer step uses IEEE f32 ops in the order documented in include/masq.h
// (round-to-nearest mul/div/sqrt, no FMA contraction: explicit __fmul_rn/__fdiv_rn),
// so codes and scales are bit-exact against the CPU oracle.
#include <cuda_bf16.h>

#include "internal.h"

namespace masq {
namespace {

constexpr float kFloor = 1e-12f;

template <typename XT>
struct Vec;
template <>
struct Vec<__nv_bfloat16> {
  static constexpr int N = 8;
  __device__ __forceinline__ static void load(const __nv_bfloat16* p, float (&f)[8]) {
    const uint4 r = __ldg(reinterpret_cast<const uint4*>(p));
    const uint32_t w[4] = {r.x, r.y, r.z, r.w};
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      f[2 * i] = __uint_as_float(w[i] << 16);
      f[2 * i + 1] = __uint_as_float(w[i] & 0xFFFF0000u);
    }
  }
};
template <>
struct Vec<float> {
  static constexpr int N = 4;
  __device__ __forceinline__ static void load(const float* p, float (&f)[4]) {
    const float4 r = __ldg(reinterpret_cast<const float4*>(p));
    f[0] = r.x; f[1] = r.y; f[2] = r.z; f[3] = r.w;
  }
};

// round half away from zero, then clamp (reading Q5)
__device__ __forceinline__ int rha_clamp(float v, int qmin, int qmax) {
  const float t = truncf(v);
  const float fr = fabsf(__fsub_rn(v, t));
  float q = t;
  if (fr >= 0.5f) q = __fadd_rn(t, copysignf(1.0f, v));
  int qi = (int)q;
  return qi < qmin ? qmin : (qi > qmax ? qmax : qi);
}

// code = rha(xs / delta): fast path xs * (1/delta); near a half-integer (where the fast
// quotient could round differently from the IEEE quotient) recompute with div.rn.
__device__ __forceinline__ int quant_code(float xs, float delta, float rcp, int qmin, int qmax) {
  float v = __fmul_rn(xs, rcp);
  const float a = fabsf(v);
  const float fr = __fsub_rn(a, truncf(a));
  if (fabsf(fr - 0.5f) <= 1.52587890625e-05f * fmaxf(a, 1.0f)) v = __fdiv_rn(xs, delta);
  return rha_clamp(v, qmin, qmax);
}

// =============================================================== A1 stats
template <typename XT, int NM>
__global__ void __launch_bounds__(256) stats_kernel(const XT* __restrict__ X, int64_t ld_x,
                                                    const uint8_t* __restrict__ ids, int64_t T, int64_t d,
                                                    int rows_per_strip, float* __restrict__ R,
                                                    unsigned long long* __restrict__ count,
                                                    uint32_t* __restrict__ status) {
  constexpr int V = Vec<XT>::N;
  constexpr int U = 8;                      // rows in flight per thread
  constexpr int CH = 256 * V;               // channels per CTA
  __shared__ float sm[CH];
  __shared__ uint32_t s_present;
  const int64_t c0 = (int64_t)blockIdx.x * CH + threadIdx.x * V;
  const bool active = c0 < d;
  const int64_t t0 = (int64_t)blockIdx.y * rows_per_strip;
  const int64_t t1 = min(T, t0 + rows_per_strip);
  float acc[NM][V];
#pragma unroll
  for (int m = 0; m < NM; ++m)
#pragma unroll
    for (int e = 0; e < V; ++e) acc[m][e] = 0.f;
  uint32_t present = 0, bad = 0;
  unsigned long long cnt[NM];
#pragma unroll
  for (int m = 0; m < NM; ++m) cnt[m] = 0;

  for (int64_t t = t0; t < t1; t += U) {
    float f[U][V];
    int mid[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int64_t tt = t + u;
      mid[u] = tt < t1 ? (int)__ldg(ids + tt) : -1;
      if (active && tt < t1) Vec<XT>::load(X + tt * ld_x + c0, f[u]);
    }
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int m = mid[u];            // warp-uniform
      if (m < 0) continue;
      if (m >= NM) { bad = 1; continue; }
      present |= 1u << m;
#pragma unroll
      for (int mm = 0; mm < NM; ++mm) {
        if (m == mm) {
          ++cnt[mm];
          if (active) {
#pragma unroll
            for (int e = 0; e < V; ++e) acc[mm][e] = fmaxf(acc[mm][e], fabsf(f[u][e]));
          }
        }
      }
    }
  }
  if (threadIdx.x == 0) {
    s_present = present;
    if (bad) atomicOr(status, kStBadModality);
    if (blockIdx.x == 0) {
#pragma unroll
      for (int m = 0; m < NM; ++m)
        if (cnt[m]) atomicAdd(count + m, cnt[m]);
    }
  }
  __syncthreads();
  const uint32_t pres = s_present;
#pragma unroll
  for (int mm = 0; mm < NM; ++mm) {
    if (!((pres >> mm) & 1u)) continue;       // CTA-uniform
#pragma unroll
    for (int e = 0; e < V; ++e) sm[threadIdx.x * V + e] = acc[mm][e];
    __syncthreads();
    for (int c = threadIdx.x; c < CH; c += 256) {
      const int64_t col = (int64_t)blockIdx.x * CH + c;
      const float v = sm[c];
      if (col < d && v > 0.f) atomicMax(reinterpret_cast<unsigned int*>(R + (int64_t)mm * d + col), __float_as_uint(v));
    }
    __syncthreads();
  }
}

template <typename XT>
cudaError_t stats_dispatch(const XT* X, int64_t ld_x, const uint8_t* ids, int64_t T, int64_t d, int n_mod, float* R,
                           int64_t* count, uint32_t* status, cudaStream_t st) {
  constexpr int CH = 256 * Vec<XT>::N;
  const int gx = (int)ceil_div(d, CH);
  int strips = (int)std::max<int64_t>(1, std::min<int64_t>(ceil_div(num_sms() * 2, gx), ceil_div(T, 64)));
  const int rows = (int)ceil_div(T, strips);
  strips = (int)ceil_div(T, rows);
  dim3 grid(gx, strips);
  auto* c = reinterpret_cast<unsigned long long*>(count);
  switch (n_mod) {
#define MASQ_STATS_CASE(NM)                                                       \
  case NM: {                                                                      \
    ProfScope ps_("stats", st);                                                   \
    stats_kernel<XT, NM><<<grid, 256, 0, st>>>(X, ld_x, ids, T, d, rows, R, c, status); \
  } break;
    MASQ_STATS_CASE(1) MASQ_STATS_CASE(2) MASQ_STATS_CASE(3) MASQ_STATS_CASE(4)
    MASQ_STATS_CASE(5) MASQ_STATS_CASE(6) MASQ_STATS_CASE(7) MASQ_STATS_CASE(8)
#undef MASQ_STATS_CASE
    default: return cudaErrorInvalidValue;
  }
  return cudaGetLastError();
}

// =============================================================== A2 init
template <typename WT>
__global__ void __launch_bounds__(256) init_kernel(const float* __restrict__ R, const int64_t* __restrict__ count,
                                                   const WT* __restrict__ W, int64_t d, int64_t n, int n_mod,
                                                   float* __restrict__ s, float* __restrict__ wmax_out,
                                                   uint32_t* __restrict__ status) {
  constexpr int V = Vec<WT>::N;
  const int64_t i = (int64_t)blockIdx.x * 8 + (threadIdx.x >> 5);
  const int lane = threadIdx.x & 31;
  if (blockIdx.x == 0 && threadIdx.x == 0) {
    for (int m = 0; m < n_mod; ++m)
      if (count[m] == 0) atomicOr(status, kStEmptyModality);
  }
  if (i >= d) return;
  float wm = 0.f;
  for (int64_t j = (int64_t)lane * V; j < n; j += 32 * V) {
    float f[V];
    Vec<WT>::load(W + i * n + j, f);
#pragma unroll
    for (int e = 0; e < V; ++e) wm = fmaxf(wm, fabsf(f[e]));
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) wm = fmaxf(wm, __shfl_xor_sync(0xffffffffu, wm, o));
  if (lane < n_mod) {
    const float num = fmaxf(R[(int64_t)lane * d + i], kFloor);
    s[(int64_t)lane * d + i] = __fsqrt_rn(__fdiv_rn(num, fmaxf(wm, kFloor)));
  }
  if (lane == 0 && wmax_out) wmax_out[i] = wm;
}

// =============================================================== A3 weight quantization
// pass 1: amax[k*n + j] = max_i |s_k[i] * W[i, j]|   (u32 bit patterns of non-negative floats)
template <typename WT>
__global__ void __launch_bounds__(256) wcolmax_kernel(const WT* __restrict__ W, const float* __restrict__ s,
                                                      int64_t d, int64_t n, int rows_per_strip,
                                                      uint32_t* __restrict__ amax) {
  constexpr int V = Vec<WT>::N;
  const int k = blockIdx.z;
  const int64_t j0 = ((int64_t)blockIdx.x * 256 + threadIdx.x) * V;
  if (j0 >= n) return;
  const int64_t i0 = (int64_t)blockIdx.y * rows_per_strip;
  const int64_t i1 = min(d, i0 + rows_per_strip);
  const float* sk = s + (int64_t)k * d;
  float m[V];
#pragma unroll
  for (int e = 0; e < V; ++e) m[e] = 0.f;
  for (int64_t i = i0; i < i1; ++i) {
    float f[V];
    Vec<WT>::load(W + i * n + j0, f);
    const float si = __ldg(sk + i);
#pragma unroll
    for (int e = 0; e < V; ++e) m[e] = fmaxf(m[e], fabsf(__fmul_rn(si, f[e])));
  }
#pragma unroll
  for (int e = 0; e < V; ++e)
    if (m[e] > 0.f) atomicMax(amax + (int64_t)k * n + j0 + e, __float_as_uint(m[e]));
}

// pass 2: codes for a 128 (i) x 128 (j) tile, transposed through smem to K-major qw[j][i]
template <typename WT>
__global__ void __launch_bounds__(256) wquant_kernel(const WT* __restrict__ W, const float* __restrict__ s,
                                                     int64_t d, int64_t n, float qmaxf, int qmin, int qmax,
                                                     const uint32_t* __restrict__ amax, int8_t* __restrict__ qw,
                                                     float* __restrict__ dw) {
  constexpr int V = Vec<WT>::N;
  constexpr int TPR = 128 / V;            // threads per W row segment of 128 columns
  constexpr int RPI = 256 / TPR;          // rows per iteration
  __shared__ __align__(16) int8_t tile[128][128 + 16];
  const int k = blockIdx.z;
  const int64_t i0 = (int64_t)blockIdx.y * 128, j0 = (int64_t)blockIdx.x * 128;
  const int jc = (threadIdx.x % TPR) * V;
  const int ir = threadIdx.x / TPR;
  float dwv[V], rcp[V];
#pragma unroll
  for (int e = 0; e < V; ++e) {
    const int64_t j = j0 + jc + e;
    dwv[e] = j < n ? fmaxf(__fdiv_rn(__uint_as_float(amax[(int64_t)k * n + j]), qmaxf), kFloor) : 1.f;
    rcp[e] = __fdiv_rn(1.0f, dwv[e]);
  }
  const float* sk = s + (int64_t)k * d;
  for (int it = 0; it < 128 / RPI; ++it) {
    const int il = it * RPI + ir;
    const int64_t i = i0 + il;
    float f[V];
    if (i < d && j0 + jc < n) {
      Vec<WT>::load(W + i * n + j0 + jc, f);
      const float si = __ldg(sk + i);
#pragma unroll
      for (int e = 0; e < V; ++e) tile[jc + e][il] = (int8_t)quant_code(__fmul_rn(si, f[e]), dwv[e], rcp[e], qmin, qmax);
    }
  }
  __syncthreads();
  // write 128 rows (j) x 128 bytes (i); 8 threads x 16 B per row
  for (int it = 0; it < 4; ++it) {
    const int jl = it * 32 + (threadIdx.x >> 3);
    const int ic = (threadIdx.x & 7) * 16;
    const int64_t j = j0 + jl, i = i0 + ic;
    if (j < n && i < d) {
      *reinterpret_cast<uint4*>(qw + ((int64_t)k * n + j) * d + i) = *reinterpret_cast<const uint4*>(&tile[jl][ic]);
    }
  }
  if (blockIdx.y == 0 && threadIdx.x < 128) {
    const int64_t j = j0 + threadIdx.x;
    if (j < n) dw[(int64_t)k * n + j] = fmaxf(__fdiv_rn(__uint_as_float(amax[(int64_t)k * n + j]), qmaxf), kFloor);
  }
}

// =============================================================== A4 activation quantization
__global__ void inv_kernel(const float* __restrict__ s, int64_t count, float* __restrict__ inv) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i < count) inv[i] = __fdiv_rn(1.0f, s[i]);
}

// one warp per token row; two passes over the row (absmax, then codes; the 2nd read hits L1/L2)
template <typename XT>
__global__ void __launch_bounds__(256) aquant_kernel(const XT* __restrict__ X, int64_t ld_x,
                                                     const uint8_t* __restrict__ ids, int64_t T, int64_t d,
                                                     int n_mod, const float* __restrict__ inv_s, float qaf,
                                                     int qmin, int qmax, int8_t* __restrict__ qx,
                                                     float* __restrict__ dx, uint32_t* __restrict__ mask,
                                                     uint32_t* __restrict__ status, const int32_t* __restrict__ perm,
                                                     int64_t T_out) {
  constexpr int V = Vec<XT>::N;
  const int64_t row = (int64_t)blockIdx.x * 8 + (threadIdx.x >> 5);     // output row
  const int lane = threadIdx.x & 31;
  if (row >= T_out) return;
  const int64_t src = perm ? (int64_t)__ldg(perm + row) : row;          // input token
  if (src < 0) return;                                                   // padding row of a modality segment
  const int m = __ldg(ids + src);
  const XT* xr = X + src * ld_x;
  int8_t* qr = qx + row * d;
  if (m >= n_mod) {
    if (lane == 0) { atomicOr(status, kStBadModality); dx[row] = 0.f; }
    for (int64_t c = (int64_t)lane * V; c < d; c += 32 * V) {
      if (V == 8) *reinterpret_cast<uint2*>(qr + c) = make_uint2(0, 0);
      else *reinterpret_cast<uint32_t*>(qr + c) = 0u;
    }
    return;
  }
  const float* inv = inv_s + (int64_t)m * d;
  float amax = 0.f;
  for (int64_t c = (int64_t)lane * V; c < d; c += 32 * V) {
    float f[V];
    Vec<XT>::load(xr + c, f);
#pragma unroll
    for (int e = 0; e < V; e += 4) {
      const float4 iv = __ldg(reinterpret_cast<const float4*>(inv + c + e));
      amax = fmaxf(amax, fabsf(__fmul_rn(f[e + 0], iv.x)));
      amax = fmaxf(amax, fabsf(__fmul_rn(f[e + 1], iv.y)));
      amax = fmaxf(amax, fabsf(__fmul_rn(f[e + 2], iv.z)));
      amax = fmaxf(amax, fabsf(__fmul_rn(f[e + 3], iv.w)));
    }
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) amax = fmaxf(amax, __shfl_xor_sync(0xffffffffu, amax, o));
  const float delta = fmaxf(__fdiv_rn(amax, qaf), kFloor);
  const float rcp = __fdiv_rn(1.0f, delta);
  for (int64_t c = (int64_t)lane * V; c < d; c += 32 * V) {
    float f[V];
    Vec<XT>::load(xr + c, f);
    uint32_t packed[V / 4];
#pragma unroll
    for (int e = 0; e < V; e += 4) {
      const float4 iv = __ldg(reinterpret_cast<const float4*>(inv + c + e));
      const int q0 = quant_code(__fmul_rn(f[e + 0], iv.x), delta, rcp, qmin, qmax);
      const int q1 = quant_code(__fmul_rn(f[e + 1], iv.y), delta, rcp, qmin, qmax);
      const int q2 = quant_code(__fmul_rn(f[e + 2], iv.z), delta, rcp, qmin, qmax);
      const int q3 = quant_code(__fmul_rn(f[e + 3], iv.w), delta, rcp, qmin, qmax);
      packed[e / 4] = (uint32_t)(q0 & 0xFF) | ((uint32_t)(q1 & 0xFF) << 8) | ((uint32_t)(q2 & 0xFF) << 16) |
                      ((uint32_t)(q3 & 0xFF) << 24);
    }
    if (V == 8) *reinterpret_cast<uint2*>(qr + c) = make_uint2(packed[0], packed[V / 4 - 1]);
    else *reinterpret_cast<uint32_t*>(qr + c) = packed[0];
  }
  if (lane == 0) {
    dx[row] = delta;
    if (mask) atomicOr(mask + (row >> 7), 1u << m);
  }
}

// ------------------------------------------------- modality-grouped row order for the loss GEMM
// Stable counting sort of the tokens by modality; each modality segment starts on a 128-row
// tile boundary so every loss tile holds a single modality (uses that modality's Q(S_m W)).
__global__ void __launch_bounds__(1024) route_kernel(const uint8_t* __restrict__ ids, int64_t T, int n_mod,
                                                     int32_t* __restrict__ perm, uint32_t* __restrict__ tile_mod,
                                                     int64_t n_tiles) {
  __shared__ int s_cnt[1024];
  __shared__ int s_tot[kMaxMod], s_seg[kMaxMod + 1];
  const int tid = threadIdx.x;
  const int64_t chunk = (T + 1023) / 1024;
  const int64_t t0 = tid * chunk, t1 = min(T, t0 + chunk);
  int cnt[kMaxMod];
#pragma unroll
  for (int m = 0; m < kMaxMod; ++m) cnt[m] = 0;
  for (int64_t t = t0; t < t1; ++t) {
    const int m = ids[t];
#pragma unroll
    for (int mm = 0; mm < kMaxMod; ++mm) cnt[mm] += (m == mm);
  }
  int excl[kMaxMod];
  for (int m = 0; m < n_mod; ++m) {                 // block exclusive scan, one modality at a time
    s_cnt[tid] = cnt[m];
    __syncthreads();
    for (int off = 1; off < 1024; off <<= 1) {
      const int v = tid >= off ? s_cnt[tid - off] : 0;
      __syncthreads();
      s_cnt[tid] += v;
      __syncthreads();
    }
    excl[m] = s_cnt[tid] - cnt[m];
    if (tid == 1023) s_tot[m] = s_cnt[tid];
    __syncthreads();
  }
  if (tid == 0) {
    int acc = 0;
    for (int m = 0; m < n_mod; ++m) {
      s_seg[m] = acc;
      acc += (s_tot[m] + kTileM - 1) / kTileM * kTileM;
    }
    s_seg[n_mod] = acc;
  }
  __syncthreads();
  int pos[kMaxMod];
  for (int m = 0; m < n_mod; ++m) pos[m] = s_seg[m] + excl[m];
  for (int64_t t = t0; t < t1; ++t) {
    const int m = ids[t];
    if (m < n_mod) perm[pos[m]++] = (int32_t)t;
  }
  for (int64_t tile = tid; tile < n_tiles; tile += 1024) {
    const int64_t r = tile * kTileM;
    uint32_t v = 0xFFFFFFFFu;
    for (int m = 0; m < n_mod; ++m)
      if (r >= s_seg[m] && r < s_seg[m + 1] && s_tot[m] > 0) v = (uint32_t)m;
    tile_mod[tile] = v;
  }
}

// =============================================================== packing / transpose
// out[c * ld_out + r] = in[r * ld_in + c]  (bf16), optional duplicate at out + dup_off
__global__ void transpose_bf16_kernel(const uint16_t* __restrict__ in, int64_t rows, int64_t cols, int64_t ld_in,
                                      int64_t in_batch, uint16_t* __restrict__ out, int64_t ld_out,
                                      int64_t out_batch, int64_t dup_off) {
  __shared__ uint16_t t[32][33];
  const int64_t b = blockIdx.z;
  const int64_t r0 = (int64_t)blockIdx.y * 32, c0 = (int64_t)blockIdx.x * 32;
  const uint16_t* ib = in + b * in_batch;
  uint16_t* ob = out + b * out_batch;
  for (int k = threadIdx.y; k < 32; k += blockDim.y) {
    const int64_t r = r0 + k, c = c0 + threadIdx.x;
    t[k][threadIdx.x] = (r < rows && c < cols) ? ib[r * ld_in + c] : (uint16_t)0;
  }
  __syncthreads();
  for (int k = threadIdx.y; k < 32; k += blockDim.y) {
    const int64_t c = c0 + k, r = r0 + threadIdx.x;
    if (c < cols && r < rows) {
      const uint16_t v = t[threadIdx.x][k];
      ob[c * ld_out + r] = v;
      if (dup_off >= 0) ob[c * ld_out + r + dup_off] = v;
    }
  }
}

// =============================================================== A8 reduction
struct Lambda8 {
  float v[kMaxMod];
};

__global__ void __launch_bounds__(256) loss_reduce_kernel(const double* __restrict__ partials, int64_t n_tiles,
                                                          int num_n, int epi, const uint32_t* __restrict__ tile_mod,
                                                          const uint8_t* __restrict__ ids, int64_t T, int n_mod,
                                                          int64_t n, Lambda8 lam, double* __restrict__ sums,
                                                          int64_t* __restrict__ counts, double* __restrict__ loss) {
  __shared__ double red[256];
  __shared__ long long cred[256];
  __shared__ double s_sum[kMaxMod];
  __shared__ long long s_cnt[kMaxMod];
  for (int m = 0; m < n_mod; ++m) {
    double a = 0.0;
    long long c = 0;
    for (int64_t lt = threadIdx.x; lt < n_tiles; lt += 256) {     // fixed order -> deterministic
      if (tile_mod[lt / num_n] != (uint32_t)m) continue;
      for (int e = 0; e < epi; ++e) a += partials[lt * epi + e];
    }
    for (int64_t t = threadIdx.x; t < T; t += 256) c += (ids[t] == m);
    red[threadIdx.x] = a;
    cred[threadIdx.x] = c;
    __syncthreads();
    for (int o = 128; o > 0; o >>= 1) {
      if (threadIdx.x < o) {
        red[threadIdx.x] += red[threadIdx.x + o];
        cred[threadIdx.x] += cred[threadIdx.x + o];
      }
      __syncthreads();
    }
    if (threadIdx.x == 0) { s_sum[m] = red[0]; s_cnt[m] = cred[0]; }
    __syncthreads();
  }
  if (threadIdx.x == 0) {
    double L = 0.0;
    for (int m = 0; m < n_mod; ++m) {
      sums[m] = s_sum[m];
      counts[m] = s_cnt[m];
      if (s_cnt[m] > 0) L += (double)lam.v[m] * s_sum[m] / ((double)s_cnt[m] * (double)n);
    }
    loss[0] = L;
  }
}

__global__ void loss_finalize_kernel(const double* sums, const int64_t* counts, Lambda8 lam, int n_mod, int64_t n,
                                     double* loss) {
  double L = 0.0;
  for (int m = 0; m < n_mod; ++m)
    if (counts[m] > 0) L += (double)lam.v[m] * sums[m] / ((double)counts[m] * (double)n);
  loss[0] = L;
}

Lambda8 make_lambda(const float* lam, int n_mod) {
  Lambda8 l;
  for (int m = 0; m < kMaxMod; ++m) l.v[m] = (lam && m < n_mod) ? lam[m] : 1.0f;
  return l;
}

}  // namespace

// =============================================================== launchers
cudaError_t launch_stats(const void* X, masq_dtype xt, int64_t ld_x, const uint8_t* ids, int64_t T, int64_t d,
                         int n_mod, float* R, int64_t* count, uint32_t* status, cudaStream_t st) {
  if (T <= 0) return cudaSuccess;
  if (xt == MASQ_BF16)
    return stats_dispatch(static_cast<const __nv_bfloat16*>(X), ld_x, ids, T, d, n_mod, R, count, status, st);
  return stats_dispatch(static_cast<const float*>(X), ld_x, ids, T, d, n_mod, R, count, status, st);
}

cudaError_t launch_init(const float* R, const int64_t* count, const void* W, masq_dtype wt, int64_t d, int64_t n,
                        int n_mod, float* s, float* wmax, uint32_t* status, cudaStream_t st) {
  const int grid = (int)ceil_div(d, 8);
  ProfScope ps_("init", st);
  if (wt == MASQ_BF16)
    init_kernel<<<grid, 256, 0, st>>>(R, count, static_cast<const __nv_bfloat16*>(W), d, n, n_mod, s, wmax, status);
  else
    init_kernel<<<grid, 256, 0, st>>>(R, count, static_cast<const float*>(W), d, n, n_mod, s, wmax, status);
  return cudaGetLastError();
}

cudaError_t launch_wquant(const void* W, masq_dtype wt, const float* s, int n_sets, int64_t d, int64_t n, int wbits,
                          int8_t* qw, float* dw, uint32_t* amax, cudaStream_t st) {
  cudaError_t e = cudaMemsetAsync(amax, 0, sizeof(uint32_t) * n_sets * n, st);
  if (e != cudaSuccess) return e;
  const int qmax = (1 << (wbits - 1)) - 1, qmin = -(1 << (wbits - 1));
  const int V = wt == MASQ_BF16 ? 8 : 4;
  const int gx = (int)ceil_div(n, 256 * V);
  int strips = (int)std::max<int64_t>(1, std::min<int64_t>(ceil_div(num_sms() * 4, gx * n_sets), ceil_div(d, 32)));
  const int rows = (int)ceil_div(d, strips);
  strips = (int)ceil_div(d, rows);
  dim3 g1(gx, strips, n_sets), g2((unsigned)ceil_div(n, 128), (unsigned)ceil_div(d, 128), n_sets);
  if (wt == MASQ_BF16) {
    auto* w = static_cast<const __nv_bfloat16*>(W);
    { ProfScope ps_("wcolmax", st); wcolmax_kernel<<<g1, 256, 0, st>>>(w, s, d, n, rows, amax); }
    { ProfScope ps_("wquant", st); wquant_kernel<<<g2, 256, 0, st>>>(w, s, d, n, (float)qmax, qmin, qmax, amax, qw, dw); }
  } else {
    auto* w = static_cast<const float*>(W);
    { ProfScope ps_("wcolmax", st); wcolmax_kernel<<<g1, 256, 0, st>>>(w, s, d, n, rows, amax); }
    { ProfScope ps_("wquant", st); wquant_kernel<<<g2, 256, 0, st>>>(w, s, d, n, (float)qmax, qmin, qmax, amax, qw, dw); }
  }
  return cudaGetLastError();
}

cudaError_t launch_inv(const float* s, int64_t count, float* inv, cudaStream_t st) {
  ProfScope ps_("inv", st);
  inv_kernel<<<(unsigned)ceil_div(count, 256), 256, 0, st>>>(s, count, inv);
  return cudaGetLastError();
}

cudaError_t launch_aquant(const void* X, masq_dtype xt, int64_t ld_x, const uint8_t* ids, int64_t T, int64_t d,
                          int n_mod, const float* inv_s, int abits, int8_t* qx, float* dx, uint32_t* mask,
                          uint32_t* status, cudaStream_t st, const int32_t* perm, int64_t T_out) {
  if (T <= 0) return cudaSuccess;
  if (T_out < 0) T_out = T;
  if (mask) {
    cudaError_t e = cudaMemsetAsync(mask, 0, sizeof(uint32_t) * ceil_div(T, kTileM), st);
    if (e != cudaSuccess) return e;
  }
  const int qmax = (1 << (abits - 1)) - 1, qmin = -(1 << (abits - 1));
  const unsigned grid = (unsigned)ceil_div(T_out, 8);
  ProfScope ps_("aquant", st);
  if (xt == MASQ_BF16)
    aquant_kernel<<<grid, 256, 0, st>>>(static_cast<const __nv_bfloat16*>(X), ld_x, ids, T, d, n_mod, inv_s,
                                        (float)qmax, qmin, qmax, qx, dx, mask, status, perm, T_out);
  else
    aquant_kernel<<<grid, 256, 0, st>>>(static_cast<const float*>(X), ld_x, ids, T, d, n_mod, inv_s, (float)qmax,
                                        qmin, qmax, qx, dx, mask, status, perm, T_out);
  return cudaGetLastError();
}

cudaError_t launch_route(const uint8_t* ids, int64_t T, int n_mod, int32_t* perm, uint32_t* tile_mod,
                         cudaStream_t st) {
  const int64_t Tg = grouped_rows(T, n_mod);
  cudaError_t e = cudaMemsetAsync(perm, 0xFF, sizeof(int32_t) * Tg, st);
  if (e != cudaSuccess) return e;
  ProfScope ps_("route", st);
  route_kernel<<<1, 1024, 0, st>>>(ids, T, n_mod, perm, tile_mod, Tg / kTileM);
  return cudaGetLastError();
}

static cudaError_t transpose(const uint16_t* in, int64_t rows, int64_t cols, int64_t ld_in, int64_t in_batch,
                             uint16_t* out, int64_t ld_out, int64_t out_batch, int64_t dup_off, int batches,
                             cudaStream_t st) {
  dim3 grid((unsigned)ceil_div(cols, 32), (unsigned)ceil_div(rows, 32), batches), block(32, 8);
  ProfScope ps_("transpose", st);
  transpose_bf16_kernel<<<grid, block, 0, st>>>(in, rows, cols, ld_in, in_batch, out, ld_out, out_batch, dup_off);
  return cudaGetLastError();
}

cudaError_t launch_pack_l2(const uint16_t* L2, int64_t ld_l2, int n_nt, int64_t n, int r, int rpad, uint16_t* L2t,
                           cudaStream_t st) {
  if (r < rpad) {
    cudaError_t e = cudaMemsetAsync(L2t, 0, sizeof(uint16_t) * n_nt * n * 2 * rpad, st);
    if (e != cudaSuccess) return e;
  }
  // L2^m [r x n] (ld_l2) -> L2t rows m*n + j, cols [k] and [rpad + k]
  return transpose(L2, r, n, ld_l2, (int64_t)r * ld_l2, L2t, 2 * rpad, n * 2 * rpad, rpad, n_nt, st);
}

cudaError_t launch_transpose_bf16(const uint16_t* W, int64_t d, int64_t n, uint16_t* Wt, cudaStream_t st) {
  return transpose(W, d, n, n, 0, Wt, d, 0, -1, 1, st);
}

cudaError_t launch_loss_reduce(const double* partials, int64_t n_tiles, int num_n, int epi, const uint32_t* tile_mod,
                               const uint8_t* ids, int64_t T, int n_mod, int64_t n, const float* lambda_host,
                               double* sums, int64_t* counts, double* loss, cudaStream_t st) {
  ProfScope ps_("loss_reduce", st);
  loss_reduce_kernel<<<1, 256, 0, st>>>(partials, n_tiles, num_n, epi, tile_mod, ids, T, n_mod, n,
                                        make_lambda(lambda_host, n_mod), sums, counts, loss);
  return cudaGetLastError();
}

cudaError_t launch_loss_finalize(const double* sums, const int64_t* counts, const float* lambda_host, int n_mod,
                                 int64_t n, double* loss, cudaStream_t st) {
  ProfScope ps_("loss_finalize", st);
  loss_finalize_kernel<<<1, 1, 0, st>>>(sums, counts, make_lambda(lambda_host, n_mod), n_mod, n, loss);
  return cudaGetLastError();
}

}  // namespace masq
