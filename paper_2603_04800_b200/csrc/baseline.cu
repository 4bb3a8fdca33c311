// baseline.cu — N4: the baseline factor methods the paper compares MASQuant
// against, on the same device data.
//   smooth_factors  s_i = num_i^beta / den_i^(1-beta)   (PAPER.md:19-23 SmoothQuant, with
//                   num = R (or the unified max_m R^m); PAPER.md:24-28 AWQ with
//                   num = mean_t |x_t,i| and no denominator), f64 pow, one rounding to f32 (Q26)
//   meanabs         sum_t |x^m_t,i| per modality (f64, deterministic: f32 slab partials, fixed-
//                   order f64 reduction), counts, f32 means per modality and over all tokens
//   range_stats     alpha = R^m / max(R^m', 1e-12) (Theorem 1), unified max_m R^m,
//                   dominance counts per modality + tied (fig:modality_dominance)
#include <cuda_bf16.h>

#include "internal.h"

namespace masq {
namespace {

constexpr float kFloorB = 1e-12f;
constexpr int kSlab = 64;                      // tokens per meanabs partial

__global__ void smooth_factors_kernel(const float* __restrict__ num, int64_t rows, int64_t d,
                                      const float* __restrict__ den, double beta, float* __restrict__ s) {
  const int64_t idx = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (idx >= rows * d) return;
  const int64_t i = idx % d;
  double r = pow((double)fmaxf(num[idx], kFloorB), beta);
  if (den) r = r / pow((double)fmaxf(den[i], kFloorB), 1.0 - beta);
  s[idx] = (float)r;
}

template <typename XT>
__device__ __forceinline__ void load8(const XT* p, float (&f)[8]);
template <>
__device__ __forceinline__ void load8<__nv_bfloat16>(const __nv_bfloat16* p, float (&f)[8]) {
  const uint4 r = __ldg(reinterpret_cast<const uint4*>(p));
  const uint32_t w[4] = {r.x, r.y, r.z, r.w};
#pragma unroll
  for (int k = 0; k < 4; ++k) {
    f[2 * k] = __uint_as_float(w[k] << 16);
    f[2 * k + 1] = __uint_as_float(w[k] & 0xFFFF0000u);
  }
}
template <>
__device__ __forceinline__ void load8<float>(const float* p, float (&f)[8]) {
  const float4 a = __ldg(reinterpret_cast<const float4*>(p));
  const float4 b = __ldg(reinterpret_cast<const float4*>(p + 4));
  f[0] = a.x; f[1] = a.y; f[2] = a.z; f[3] = a.w; f[4] = b.x; f[5] = b.y; f[6] = b.z; f[7] = b.w;
}

// one thread = 8 consecutive channels over one slab of kSlab tokens; per-modality f32 sums
template <typename XT, int NM>
__global__ void __launch_bounds__(256) meanabs_kernel(const XT* __restrict__ X, int64_t ld_x,
                                                      const uint8_t* __restrict__ ids, int64_t T, int64_t d,
                                                      float* __restrict__ part) {
  const int64_t c = ((int64_t)blockIdx.x * 256 + threadIdx.x) * 8;
  const int64_t t0 = (int64_t)blockIdx.y * kSlab;
  if (c >= d) return;
  float acc[NM][8];
#pragma unroll
  for (int m = 0; m < NM; ++m)
#pragma unroll
    for (int e = 0; e < 8; ++e) acc[m][e] = 0.f;
  const int64_t t1 = min(T, t0 + kSlab);
  for (int64_t t = t0; t < t1; ++t) {
    const int m = __ldg(ids + t);
    float f[8];
    load8<XT>(X + t * ld_x + c, f);
#pragma unroll
    for (int mm = 0; mm < NM; ++mm)
      if (mm == m)
#pragma unroll
        for (int e = 0; e < 8; ++e) acc[mm][e] += fabsf(f[e]);
  }
#pragma unroll
  for (int m = 0; m < NM; ++m) {
    float* o = part + ((int64_t)blockIdx.y * NM + m) * d + c;
    *reinterpret_cast<float4*>(o) = make_float4(acc[m][0], acc[m][1], acc[m][2], acc[m][3]);
    *reinterpret_cast<float4*>(o + 4) = make_float4(acc[m][4], acc[m][5], acc[m][6], acc[m][7]);
  }
}

__global__ void count_ids_kernel(const uint8_t* __restrict__ ids, int64_t T, int n_mod, int64_t* __restrict__ cnt,
                                 uint32_t* __restrict__ status) {
  __shared__ unsigned long long sc[kMaxMod];
  if (threadIdx.x < kMaxMod) sc[threadIdx.x] = 0ull;
  __syncthreads();
  for (int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; t < T; t += (int64_t)gridDim.x * blockDim.x) {
    const int m = ids[t];
    if (m < n_mod) atomicAdd(&sc[m], 1ull);
    else atomicOr(status, kStBadModality);
  }
  __syncthreads();
  if (threadIdx.x < n_mod && sc[threadIdx.x]) atomicAdd(reinterpret_cast<unsigned long long*>(cnt + threadIdx.x),
                                                        sc[threadIdx.x]);
}

// S[m][i] (+)= sum over slabs (fixed order); mean[m][i] = f32(S / N_m); uni[i] = f32(sum_m S / sum_m N)
__global__ void meanabs_finalize_kernel(const float* __restrict__ part, int nslab, int n_mod, int64_t d,
                                        double* __restrict__ S, const int64_t* __restrict__ cnt,
                                        float* __restrict__ mean, float* __restrict__ uni) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= d) return;
  double tot = 0.0;
  int64_t ntot = 0;
  for (int m = 0; m < n_mod; ++m) {
    double a = 0.0;
    for (int b = 0; b < nslab; ++b) a += (double)part[((int64_t)b * n_mod + m) * d + i];
    const double sm = S[(int64_t)m * d + i] + a;
    S[(int64_t)m * d + i] = sm;
    const int64_t n = cnt[m];
    if (mean) mean[(int64_t)m * d + i] = n > 0 ? (float)(sm / (double)n) : 0.f;
    tot += sm;
    ntot += n;
  }
  if (uni) uni[i] = ntot > 0 ? (float)(tot / (double)ntot) : 0.f;
}

__global__ void range_stats_kernel(const float* __restrict__ R, int n_mod, int64_t d, int dominant, int other,
                                   float* __restrict__ alpha, float* __restrict__ runi,
                                   unsigned long long* __restrict__ dom) {
  __shared__ unsigned int sc[kMaxMod + 1];
  if (threadIdx.x <= kMaxMod) sc[threadIdx.x] = 0u;
  __syncthreads();
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i < d) {
    if (alpha) alpha[i] = __fdiv_rn(R[(int64_t)dominant * d + i], fmaxf(R[(int64_t)other * d + i], kFloorB));
    float top = R[i];
    int win = 0, nwin = 1;
    for (int m = 1; m < n_mod; ++m) {
      const float v = R[(int64_t)m * d + i];
      if (v > top) { top = v; win = m; nwin = 1; }
      else if (v == top) ++nwin;
    }
    if (runi) runi[i] = top;
    if (dom) {
      atomicAdd(&sc[win], 1u);
      if (nwin > 1) atomicAdd(&sc[n_mod], 1u);
    }
  }
  __syncthreads();
  if (dom && threadIdx.x <= n_mod && sc[threadIdx.x]) atomicAdd(dom + threadIdx.x, (unsigned long long)sc[threadIdx.x]);
}

template <typename XT>
cudaError_t meanabs_dispatch(const XT* X, int64_t ld_x, const uint8_t* ids, int64_t T, int64_t d, int n_mod,
                             float* part, cudaStream_t st) {
  dim3 grid((unsigned)ceil_div(d, 256 * 8), (unsigned)ceil_div(T, kSlab));
#define MA(NM) meanabs_kernel<XT, NM><<<grid, 256, 0, st>>>(X, ld_x, ids, T, d, part)
  switch (n_mod) {
    case 1: MA(1); break;
    case 2: MA(2); break;
    case 3: MA(3); break;
    case 4: MA(4); break;
    case 5: MA(5); break;
    case 6: MA(6); break;
    case 7: MA(7); break;
    default: MA(8); break;
  }
#undef MA
  return cudaGetLastError();
}
}  // namespace

int meanabs_slabs(int64_t T) { return (int)ceil_div(T, kSlab); }

cudaError_t launch_smooth_factors(const float* num, int64_t rows, int64_t d, const float* den, double beta, float* s,
                                  cudaStream_t st) {
  ProfScope ps_("smooth_factors", st);
  smooth_factors_kernel<<<(unsigned)ceil_div(rows * d, 256), 256, 0, st>>>(num, rows, d, den, beta, s);
  return cudaGetLastError();
}

cudaError_t launch_meanabs(const void* X, masq_dtype xt, int64_t ld_x, const uint8_t* ids, int64_t T, int64_t d,
                           int n_mod, double* S, int64_t* cnt, float* mean, float* uni, float* part,
                           uint32_t* status, cudaStream_t st) {
  {
    ProfScope ps_("meanabs", st);
    cudaError_t e = xt == MASQ_BF16
                        ? meanabs_dispatch(static_cast<const __nv_bfloat16*>(X), ld_x, ids, T, d, n_mod, part, st)
                        : meanabs_dispatch(static_cast<const float*>(X), ld_x, ids, T, d, n_mod, part, st);
    if (e != cudaSuccess) return e;
    count_ids_kernel<<<(unsigned)std::min<int64_t>(ceil_div(T, 256), 1024), 256, 0, st>>>(ids, T, n_mod, cnt, status);
  }
  ProfScope ps2_("meanabs_fin", st);
  meanabs_finalize_kernel<<<(unsigned)ceil_div(d, 256), 256, 0, st>>>(part, meanabs_slabs(T), n_mod, d, S, cnt, mean,
                                                                       uni);
  return cudaGetLastError();
}

cudaError_t launch_count_modalities(const uint8_t* ids, int64_t T, int n_mod, int64_t* cnt, uint32_t* status,
                                   cudaStream_t st) {
  ProfScope ps_("count_modalities", st);
  count_ids_kernel<<<(unsigned)std::max<int64_t>(1, std::min<int64_t>(ceil_div(T, 256), 1024)), 256, 0, st>>>(
      ids, T, n_mod, cnt, status);
  return cudaGetLastError();
}

cudaError_t launch_range_stats(const float* R, int n_mod, int64_t d, int dominant, int other, float* alpha,
                               float* runi, int64_t* dom, cudaStream_t st) {
  if (dom) {
    cudaError_t e = cudaMemsetAsync(dom, 0, sizeof(int64_t) * (n_mod + 1), st);
    if (e != cudaSuccess) return e;
  }
  ProfScope ps_("range_stats", st);
  range_stats_kernel<<<(unsigned)ceil_div(d, 256), 256, 0, st>>>(R, n_mod, d, dominant, other, alpha, runi,
                                                                  reinterpret_cast<unsigned long long*>(dom));
  return cudaGetLastError();
}

}  // namespace masq
