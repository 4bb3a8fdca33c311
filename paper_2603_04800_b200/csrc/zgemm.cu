// zgemm.cu — CMC first factor (A5): Z^m = (X_m S_m^{-1}) . L1^m on the tensor cores (sm_100a).
//
// the correction X_m S_m^{-1} . L1^m L2^m is applied in full precision.  The
// smoothed activations xs = x * (1/s^m) are f32; they enter kind::f16 MMAs as an exact
// split xs = hi + lo with hi = bf16(xs), lo = bf16(xs - hi) (reading Q13), accumulated in
// fp32 TMEM.  The result is written back split again, Z = Zhi + Zlo, laid out as
//   Z[t, (m-1)*2*rpad + k]        = Zhi,   Z[t, (m-1)*2*rpad + rpad + k] = Zlo,
// so the main GEMM can add [Zhi | Zlo] . [L2^T ; L2^T] as extra K-blocks.
//
// One CTA per (128-token tile, non-text modality m present in the tile).  The A operand is
// produced by the CTA's threads straight from X (smooth + split + swizzled st.shared, never
// written to HBM); the B operand L1^T chunk [rpad x 64] arrives by TMA.  Two-stage ring:
// threads fill stage s while the tensor core consumes stage s^1.
#include <cuda_bf16.h>

#include "internal.h"
#include "sm100.cuh"

namespace masq {
using namespace sm100;

namespace {
constexpr int ZT = 128;                 // threads
constexpr int ZA = 128 * 128;           // one A (hi or lo) stage: 128 rows x 64 bf16
constexpr int ZB = 256 * 128;           // B stage capacity: rpad (<= 256) rows x 64 bf16
constexpr int Z_SMEM = 2 * (2 * ZA + ZB) + 128;
constexpr int Z_ALLOC = Z_SMEM + 1024;

template <typename XT>
struct ZLoad;
template <>
struct ZLoad<__nv_bfloat16> {
  __device__ __forceinline__ static void load8(const __nv_bfloat16* p, float (&f)[8]) {
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
struct ZLoad<float> {
  __device__ __forceinline__ static void load8(const float* p, float (&f)[8]) {
    const float4 a = __ldg(reinterpret_cast<const float4*>(p));
    const float4 b = __ldg(reinterpret_cast<const float4*>(p) + 1);
    f[0] = a.x; f[1] = a.y; f[2] = a.z; f[3] = a.w; f[4] = b.x; f[5] = b.y; f[6] = b.z; f[7] = b.w;
  }
};

__device__ __forceinline__ uint32_t pack_bf16(float a, float b) {
  const uint32_t lo = __bfloat16_as_ushort(__float2bfloat16_rn(a));
  const uint32_t hi = __bfloat16_as_ushort(__float2bfloat16_rn(b));
  return lo | (hi << 16);
}

template <typename XT>
__global__ void __launch_bounds__(ZT, 1)
zgemm_kernel(const __grid_constant__ CUtensorMap tmL1, const XT* __restrict__ X, int64_t ld_x,
             const uint8_t* __restrict__ ids, int T, int d, int n_mod, const float* __restrict__ inv_s, int rpad,
             uint32_t tmem_cols, const uint32_t* __restrict__ tile_mask, uint16_t* __restrict__ Z) {
  const int mt = blockIdx.x;
  const int m = blockIdx.y + 1;
  if (!((tile_mask[mt] >> m) & 1u)) return;                   // CTA-uniform early exit

  extern __shared__ uint8_t smem_raw[];
  const uint32_t raw = smem_u32(smem_raw);
  uint8_t* smem = smem_raw + (((raw + 1023u) & ~1023u) - raw);
  uint8_t* sAh = smem;                    // [2][ZA]
  uint8_t* sAl = smem + 2 * ZA;           // [2][ZA]
  uint8_t* sB = smem + 4 * ZA;            // [2][ZB]
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + 4 * ZA + 2 * ZB);
  uint64_t* done = full + 2;
  uint32_t* tslot = reinterpret_cast<uint32_t*>(done + 2);

  const int tid = threadIdx.x;
  const uint32_t warp = warp_id(), lane = lane_id();
  if (tid == 0) {
    tma_prefetch(&tmL1);
    for (int i = 0; i < 2; ++i) { mbar_init(&full[i], 1); mbar_init(&done[i], 1); }
    fence_mbar_init();
  }
  if (warp == 0) tmem_alloc(tslot, tmem_cols);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tslot;

  // this thread's 8 rows (r = tid/8 + 16*i) and 16-byte column chunk (tid % 8)
  const int chunk = tid & 7;
  bool rowok[8];
#pragma unroll
  for (int i = 0; i < 8; ++i) {
    const int g = mt * 128 + (tid >> 3) + 16 * i;
    rowok[i] = g < T && __ldg(ids + g) == (uint8_t)m;
  }
  const float* inv = inv_s + (int64_t)m * d;
  const uint32_t idesc = idesc_bf16(128, rpad);
  const int nk = (d + 63) / 64;
  const uint32_t bbytes = (uint32_t)rpad * 128u;

  for (int kc = 0; kc < nk; ++kc) {
    const int s = kc & 1;
    if (kc >= 2) mbar_wait(&done[s], ((kc - 2) >> 1) & 1);   // stage s free again
    if (tid == 0) {
      mbar_expect_tx(&full[s], bbytes);
      tma_load_2d(sB + s * ZB, &tmL1, &full[s], kc * 64, (m - 1) * rpad);
    }
    const int col = kc * 64 + chunk * 8;
    float iv[8];
    if (col < d) {
      const float4 a = __ldg(reinterpret_cast<const float4*>(inv + col));
      const float4 b = __ldg(reinterpret_cast<const float4*>(inv + col) + 1);
      iv[0] = a.x; iv[1] = a.y; iv[2] = a.z; iv[3] = a.w; iv[4] = b.x; iv[5] = b.y; iv[6] = b.z; iv[7] = b.w;
    }
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      const int r = (tid >> 3) + 16 * i;
      uint4 vh = make_uint4(0, 0, 0, 0), vl = make_uint4(0, 0, 0, 0);
      if (rowok[i] && col < d) {
        float f[8];
        ZLoad<XT>::load8(X + (int64_t)(mt * 128 + r) * ld_x + col, f);
        float h[8], l[8];
#pragma unroll
        for (int e = 0; e < 8; ++e) {
          const float xs = __fmul_rn(f[e], iv[e]);
          h[e] = __bfloat162float(__float2bfloat16_rn(xs));
          l[e] = __fsub_rn(xs, h[e]);
        }
        vh = make_uint4(pack_bf16(h[0], h[1]), pack_bf16(h[2], h[3]), pack_bf16(h[4], h[5]), pack_bf16(h[6], h[7]));
        vl = make_uint4(pack_bf16(l[0], l[1]), pack_bf16(l[2], l[3]), pack_bf16(l[4], l[5]), pack_bf16(l[6], l[7]));
      }
      const uint32_t off = (uint32_t)r * 128u + (((uint32_t)chunk ^ ((uint32_t)r & 7u)) << 4);
      *reinterpret_cast<uint4*>(sAh + s * ZA + off) = vh;
      *reinterpret_cast<uint4*>(sAl + s * ZA + off) = vl;
    }
    fence_proxy_async_smem();
    __syncthreads();
    if (tid == 0) {
      mbar_wait(&full[s], (kc >> 1) & 1);
      tc_fence_after();
      const uint32_t ah = smem_u32(sAh + s * ZA), al = smem_u32(sAl + s * ZA), b = smem_u32(sB + s * ZB);
#pragma unroll
      for (int k = 0; k < 4; ++k)
        mma_bf16(tmem, umma_desc_sw128(ah + k * 32), umma_desc_sw128(b + k * 32), idesc, (kc | k) != 0);
#pragma unroll
      for (int k = 0; k < 4; ++k)
        mma_bf16(tmem, umma_desc_sw128(al + k * 32), umma_desc_sw128(b + k * 32), idesc, 1u);
      mma_commit(&done[s]);
    }
  }
  // wait for the last commit (it covers all earlier MMAs)
  mbar_wait(&done[(nk - 1) & 1], ((nk - 1) >> 1) & 1);
  tc_fence_after();

  const int row = mt * 128 + (int)(warp * 32 + lane);
  const uint32_t taddr = tmem + ((warp * 32u) << 16);
  uint16_t* zr = Z + (int64_t)row * ((n_mod - 1) * 2 * rpad) + (int64_t)(m - 1) * 2 * rpad;
  for (int c = 0; c < rpad / 32; ++c) {
    uint32_t v[32];
    tmem_ld32(taddr + c * 32, v);
    tmem_wait_ld();
    if (row < T) {
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        uint32_t ph[4], pl[4];
#pragma unroll
        for (int e = 0; e < 4; ++e) {
          const float z0 = __uint_as_float(v[8 * q + 2 * e]), z1 = __uint_as_float(v[8 * q + 2 * e + 1]);
          const float h0 = __bfloat162float(__float2bfloat16_rn(z0));
          const float h1 = __bfloat162float(__float2bfloat16_rn(z1));
          ph[e] = pack_bf16(h0, h1);
          pl[e] = pack_bf16(__fsub_rn(z0, h0), __fsub_rn(z1, h1));
        }
        *reinterpret_cast<uint4*>(zr + c * 32 + q * 8) = make_uint4(ph[0], ph[1], ph[2], ph[3]);
        *reinterpret_cast<uint4*>(zr + rpad + c * 32 + q * 8) = make_uint4(pl[0], pl[1], pl[2], pl[3]);
      }
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 0) {
    tc_fence_after();
    tmem_dealloc(tmem, tmem_cols);
  }
}

template <typename XT>
cudaError_t zlaunch(const CUtensorMap& tm, const XT* X, int64_t ld_x, const uint8_t* ids, int64_t T, int64_t d,
                    int n_mod, const float* inv_s, int rpad, const uint32_t* mask, uint16_t* Z, cudaStream_t st) {
  static bool attr = false;
  if (!attr) {
    cudaError_t e = cudaFuncSetAttribute(zgemm_kernel<XT>, cudaFuncAttributeMaxDynamicSharedMemorySize, Z_ALLOC);
    if (e != cudaSuccess) return e;
    attr = true;
  }
  uint32_t cols = 32;
  while ((int)cols < rpad) cols <<= 1;
  dim3 grid((unsigned)ceil_div(T, 128), (unsigned)(n_mod - 1));
  ProfScope ps_("zgemm", st);
  zgemm_kernel<XT><<<grid, ZT, Z_ALLOC, st>>>(tm, X, ld_x, ids, (int)T, (int)d, n_mod, inv_s, rpad, cols, mask, Z);
  return cudaGetLastError();
}
}  // namespace

cudaError_t launch_zgemm(const void* X, masq_dtype xt, int64_t ld_x, const uint8_t* ids, int64_t T, int64_t d,
                         int n_mod, const float* inv_s, const uint16_t* L1t, int rpad, const uint32_t* tile_mask,
                         uint16_t* Z, cudaStream_t st) {
  if (T <= 0 || n_mod < 2 || rpad <= 0) return cudaSuccess;
  CUtensorMap tm;
  if (!make_tmap_2d(&tm, L1t, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, (uint64_t)(n_mod - 1) * rpad, d, d,
                    (uint32_t)rpad, 64, true))
    return cudaErrorInvalidValue;
  if (xt == MASQ_BF16)
    return zlaunch(tm, static_cast<const __nv_bfloat16*>(X), ld_x, ids, T, d, n_mod, inv_s, rpad, tile_mask, Z, st);
  return zlaunch(tm, static_cast<const float*>(X), ld_x, ids, T, d, n_mod, inv_s, rpad, tile_mask, Z, st);
}

}  // namespace masq
