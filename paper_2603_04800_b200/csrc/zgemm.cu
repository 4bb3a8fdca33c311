// zgemm.cu — CMC first factor (A5): Z^m = (X_m S_m^{-1}) . L1^m on the tensor cores (sm_100a).
//
// PAPER.md:183 applies the correction X_m S_m^{-1} . L1^m L2^m in full precision.  We use
// (X S_m^{-1}) L1^m = X (S_m^{-1} L1^m): the reciprocal smoothing is folded into the tiny
// factor L1'^m = diag(1/s^m) L1^m (d x r), which is split exactly enough into two bf16
// planes L1'hi + L1'lo (reading Q13).  A bf16 X then enters kind::f16 MMAs straight from
// TMA, unmodified and exact; an f32 X is first split into bf16 hi/lo planes.
//   Z[t, :] = sum over A planes a, B planes b (a=lo & b=lo dropped) of X_a[t] . L1'_b^T
// accumulated in fp32 TMEM, then written split again (Zhi | Zlo) per modality so that the
// main GEMM can add [Zhi | Zlo] . [L2^T ; L2^T] as extra K-blocks.  Rows whose modality is
// not m are written as zeros (mixed tiles stay exact).
//
// One CTA per (128-token tile, group of non-text modalities whose ranks fit N <= 256),
// warp-specialised: warp 0 = TMA producer, warp 1 = MMA issuer, warps 2..5 = epilogue.
#include <cuda_bf16.h>

#include "internal.h"
#include "sm100.cuh"

namespace masq {
using namespace sm100;

namespace {
constexpr int ZT = 192;
constexpr int XCH = 128 * 128;       // A chunk: 128 rows x 64 bf16
// ksub (kernel argument): 64-column sub-blocks per ring stage; two adjacent SWIZZLE_128B boxes
// give 256-byte row segments of X per stage (one box alone reads 128 B per row at a d * 2-byte
// stride); one when a stage of two would not leave two ring stages (large ranks)
constexpr int KSUB_MAX = 2;
constexpr int SMEM_CAP = 200 * 1024;

__device__ __forceinline__ uint32_t pack_bf16(float a, float b) {
  const uint32_t lo = __bfloat16_as_ushort(__float2bfloat16_rn(a));
  const uint32_t hi = __bfloat16_as_ushort(__float2bfloat16_rn(b));
  return lo | (hi << 16);
}

// grid (num m-tiles, num passes); pass p covers non-text modalities [1 + p*per, 1 + min((p+1)*per, M-1))
__global__ void __launch_bounds__(ZT, 1)
zgemm_kernel(const __grid_constant__ CUtensorMap tmA0, const __grid_constant__ CUtensorMap tmA1,
             const __grid_constant__ CUtensorMap tmB, const uint8_t* __restrict__ ids, int T, int d, int n_mod,
             int rpad, int per, int a_planes, uint32_t tmem_cols, int stages,
             const uint32_t* __restrict__ tile_mask, uint16_t* __restrict__ Z, float* __restrict__ zpart,
             int splits, int pair, int ksub) {
  sm100::pdl_wait();     // launch_k: tile_mask / X of the previous kernels
  const int mt = blockIdx.x;
  const int m0 = 1 + blockIdx.y * per;
  const int m1 = min(m0 + per, n_mod);           // exclusive
  // the forward GEMM works on 256-row units (tile pairs): write every modality block present in
  // either tile of the pair, so the CMC K-blocks of the unit read zeros (never stale data)
  const int n_tiles = (T + 127) / 128;
  const uint32_t tmask = tile_mask[mt] | ((mt ^ 1) < n_tiles ? tile_mask[mt ^ 1] : 0u);
  uint32_t want = 0;
  for (int mm = m0; mm < m1; ++mm) want |= 1u << mm;
  if (!(tmask & want)) return;                   // CTA-uniform: no modality of this pass here
  if (!(tile_mask[mt] & want)) {
    // none of this tile's tokens belongs to the pass, only its pair tile's: the unit's CMC K-blocks
    // need zero Z rows here, not a product (no X read, no MMA).  Split-K: the combine kernel
    // writes them (rows of other modalities are zero there)
    if (splits > 1 && !pair) return;
    if (blockIdx.z != 0) return;
    const int zld = (n_mod - 1) * 2 * rpad;
    const int chunks = (2 * rpad) / 8;                          // 16-byte chunks per modality block
    for (int mm = m0; mm < m1; ++mm) {
      if (!((tmask >> mm) & 1u)) continue;
      for (int e = threadIdx.x; e < 128 * chunks; e += blockDim.x) {
        const int rl = e / chunks, c = e - rl * chunks;
        const int g = mt * 128 + rl;
        if (g < T)
          *reinterpret_cast<uint4*>(Z + (int64_t)g * zld + (int64_t)(mm - 1) * 2 * rpad + c * 8) = make_uint4(0, 0, 0, 0);
      }
    }
    return;
  }

  const int N = per * rpad;                      // accumulator columns (= B box rows)
  const bool combined = 2 * N <= 256;            // [hi; lo] planes as one B operand
  const int BB = N * 128;                        // one B plane chunk
  const int SBS = a_planes * XCH + 2 * BB;       // one 64-column sub-block of a stage
  const int SB = ((ksub * SBS) + 1023) & ~1023;

  extern __shared__ uint8_t smem_raw[];
  const uint32_t raw = smem_u32(smem_raw);
  uint8_t* smem = smem_raw + (((raw + 1023u) & ~1023u) - raw);
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + stages * SB);
  uint64_t* empty = full + stages;
  uint64_t* done = empty + stages;
  uint32_t* tslot = reinterpret_cast<uint32_t*>(done + 1);

  const uint32_t warp = warp_id(), lane = lane_id();
  if (warp == 0 && lane == 0) {
    tma_prefetch(&tmA0);
    tma_prefetch(&tmB);
    for (int i = 0; i < stages; ++i) { mbar_init(&full[i], 1); mbar_init(&empty[i], 1); }
    mbar_init(done, 1);
    fence_mbar_init();
  }
  if (warp == 1) tmem_alloc(tslot, tmem_cols);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tslot;
  sm100::pdl_trigger();                          // this CTA's TMEM is held
  // split-K (small T): CTA z takes k-chunks [kc0, kc1) and writes an f32 partial; a combine kernel
  // adds the partials in split order
  const int nk_all = (d + 64 * ksub - 1) / (64 * ksub);
  const int kc0 = (int)((int64_t)nk_all * blockIdx.z / splits);
  const int kc1 = (int)((int64_t)nk_all * (blockIdx.z + 1) / splits);
  const int nk = kc1 - kc0;
  const int lo_row0 = (n_mod - 1) * rpad;        // lo plane starts after the hi plane

  if (warp == 0) {
    // warp-wide loops (uniform state); one elected lane issues the copies / MMAs
    {
      uint32_t st = 0, ph = 0;
      for (int kc = kc0; kc < kc1; ++kc) {
        mbar_wait(&empty[st], ph ^ 1u);
        if (elect_one()) {
          mbar_expect_tx(&full[st], ksub * SBS);
#pragma unroll
          for (int sb = 0; sb < KSUB_MAX; ++sb) {
            if (sb >= ksub) break;
            const int col = (kc * ksub + sb) * 64;         // past d: TMA zero-fills the whole box
            uint8_t* base = smem + st * SB + sb * SBS;
            tma_load_2d(base, &tmA0, &full[st], col, mt * 128);
            if (a_planes == 2) tma_load_2d(base + XCH, &tmA1, &full[st], col, mt * 128);
            uint8_t* bb = base + a_planes * XCH;
            tma_load_2d(bb, &tmB, &full[st], col, (m0 - 1) * rpad);
            tma_load_2d(bb + BB, &tmB, &full[st], col, lo_row0 + (m0 - 1) * rpad);
          }
        }
        __syncwarp();
        if (++st == (uint32_t)stages) { st = 0; ph ^= 1u; }
      }
    }
    __syncwarp();
  } else if (warp == 1) {
    {
      // B = [L1'hi ; L1'lo] (2N rows, the two TMA boxes are contiguous): one N = 2N MMA per
      // k-step accumulates X.L1'hi into columns [0, N) and X.L1'lo into [N, 2N); the epilogue
      // adds the halves
      // (ranks above 128: two N-column MMAs into the same accumulator, as before)
      const uint32_t idesc = idesc_bf16(128, combined ? 2 * N : N);
      uint32_t st = 0, ph = 0;
      for (int kc = 0; kc < nk; ++kc) {
        mbar_wait(&full[st], ph);
        tc_fence_after();
        if (elect_one()) {
#pragma unroll
          for (int sb = 0; sb < KSUB_MAX; ++sb) {
            if (sb >= ksub) break;
            const uint32_t base = smem_u32(smem + st * SB + sb * SBS);
            const uint64_t ad = umma_desc_sw128(base), ad2 = umma_desc_sw128(base + XCH);
            const uint64_t bdh = umma_desc_sw128(base + a_planes * XCH), bdl = umma_desc_sw128(base + a_planes * XCH + BB);
#pragma unroll
            for (int k = 0; k < 4; ++k) {
              mma_bf16(tmem, ad + 2 * k, bdh + 2 * k, idesc, (kc | sb | k) != 0);
              if (!combined) mma_bf16(tmem, ad + 2 * k, bdl + 2 * k, idesc, 1u);
              if (a_planes == 2) mma_bf16(tmem, ad2 + 2 * k, bdh + 2 * k, idesc, 1u);
            }
          }
          mma_commit(&empty[st]);
        }
        __syncwarp();
        if (++st == (uint32_t)stages) { st = 0; ph ^= 1u; }
      }
      if (elect_one()) mma_commit(done);
      __syncwarp();
    }
    __syncwarp();
  } else {
    // ---------------------------------------------------------------- epilogue: TMEM -> Z (masked, split)
    const uint32_t q = warp & 3u;
    const int g = mt * 128 + (int)(q * 32u + lane);
    const int mid = g < T ? (int)__ldg(ids + g) : -1;
    mbar_wait(done, 0);
    tc_fence_after();
    const uint32_t taddr = tmem + ((q * 32u) << 16);
    const int zld = (n_mod - 1) * 2 * rpad;
    const int nnt = n_mod - 1;
    for (int mm = m0; mm < m1 && !pair; ++mm) {
      if (!((tmask >> mm) & 1u)) continue;                     // block never read by the GEMM
      if (splits > 1) {                                        // raw f32 partial of this K range
        float* zp = zpart + (((int64_t)blockIdx.z * gridDim.x * 128 + g) * nnt + (mm - 1)) * rpad;
        for (int c = 0; c < rpad / 32; ++c) {
          uint32_t v[32], w[32];
          tmem_ld32(taddr + (mm - m0) * rpad + c * 32, v);
          if (combined) tmem_ld32(taddr + N + (mm - m0) * rpad + c * 32, w);
          tmem_wait_ld();
          if (combined) {
#pragma unroll
            for (int e = 0; e < 32; ++e)
              v[e] = __float_as_uint(__fadd_rn(__uint_as_float(v[e]), __uint_as_float(w[e])));
          }
          if (g < T) {
#pragma unroll
            for (int qq = 0; qq < 8; ++qq)
              *reinterpret_cast<uint4*>(zp + c * 32 + qq * 4) = make_uint4(v[4 * qq], v[4 * qq + 1], v[4 * qq + 2], v[4 * qq + 3]);
          }
        }
        continue;
      }
      const bool mine = mid == mm;
      uint16_t* zr = Z + (int64_t)g * zld + (int64_t)(mm - 1) * 2 * rpad;
      for (int c = 0; c < rpad / 32; ++c) {
        uint32_t v[32], w[32];
        tmem_ld32(taddr + (mm - m0) * rpad + c * 32, v);
        if (combined) {
          tmem_ld32(taddr + N + (mm - m0) * rpad + c * 32, w);
          tmem_wait_ld();
#pragma unroll
          for (int e = 0; e < 32; ++e) v[e] = __float_as_uint(__fadd_rn(__uint_as_float(v[e]), __uint_as_float(w[e])));
        }
        tmem_wait_ld();
        if (g < T) {
#pragma unroll
          for (int qq = 0; qq < 4; ++qq) {
            uint32_t ph2[4], pl[4];
#pragma unroll
            for (int e = 0; e < 4; ++e) {
              const float z0 = mine ? __uint_as_float(v[8 * qq + 2 * e]) : 0.f;
              const float z1 = mine ? __uint_as_float(v[8 * qq + 2 * e + 1]) : 0.f;
              const float h0 = __bfloat162float(__float2bfloat16_rn(z0));
              const float h1 = __bfloat162float(__float2bfloat16_rn(z1));
              ph2[e] = pack_bf16(h0, h1);
              pl[e] = pack_bf16(__fsub_rn(z0, h0), __fsub_rn(z1, h1));
            }
            *reinterpret_cast<uint4*>(zr + c * 32 + qq * 8) = make_uint4(ph2[0], ph2[1], ph2[2], ph2[3]);
            *reinterpret_cast<uint4*>(zr + rpad + c * 32 + qq * 8) = make_uint4(pl[0], pl[1], pl[2], pl[3]);
          }
        }
      }
    }
  }
  if (pair) {
    // cluster pair = the two K halves of one 128-row tile: rank 1 adds its f32 accumulator into
    // rank 0's (now idle) ring through DSMEM, rank 0 sums (own + partner, fixed order) and writes Z
    const uint32_t rank = cluster_ctarank();
    float* pbuf = reinterpret_cast<float*>(smem);              // [128 rows][N] f32 (<= 64 KB)
    cluster_sync();                                            // both CTAs' MMAs are complete
    if (warp >= 2 && rank == 1) {
      const uint32_t q = warp & 3u;
      const int rl = (int)(q * 32u + lane);
      const uint32_t taddr = tmem + ((q * 32u) << 16);
      for (int mm = m0; mm < m1; ++mm) {
        if (!((tmask >> mm) & 1u)) continue;
        for (int c = 0; c < rpad / 32; ++c) {
          const int col = (mm - m0) * rpad + c * 32;
          uint32_t v[32], w[32];
          tmem_ld32(taddr + col, v);
          tmem_ld32(taddr + N + col, w);                       // pair mode is the combined [hi; lo] form
          tmem_wait_ld();
#pragma unroll
          for (int e = 0; e < 32; ++e) v[e] = __float_as_uint(__fadd_rn(__uint_as_float(v[e]), __uint_as_float(w[e])));
          uint32_t raddr;
          asm volatile("mapa.shared::cluster.u32 %0, %1, 0;" : "=r"(raddr) : "r"(smem_u32(pbuf + (size_t)rl * N + col)));
#pragma unroll
          for (int qq = 0; qq < 8; ++qq)
            asm volatile("st.shared::cluster.v4.b32 [%0], {%1, %2, %3, %4};" ::"r"(raddr + 16u * qq),
                         "r"(v[4 * qq]), "r"(v[4 * qq + 1]), "r"(v[4 * qq + 2]), "r"(v[4 * qq + 3])
                         : "memory");
        }
      }
    }
    cluster_sync();                                            // partner partials visible in rank 0
    if (warp >= 2 && rank == 0) {
      const uint32_t q = warp & 3u;
      const int rl = (int)(q * 32u + lane);
      const int g = mt * 128 + rl;
      const uint32_t taddr = tmem + ((q * 32u) << 16);
      const int zld = (n_mod - 1) * 2 * rpad;
      const int mid = g < T ? (int)__ldg(ids + g) : -1;
      for (int mm = m0; mm < m1; ++mm) {
        if (!((tmask >> mm) & 1u)) continue;
        const bool mine = mid == mm;
        uint16_t* zr = Z + (int64_t)g * zld + (int64_t)(mm - 1) * 2 * rpad;
        for (int c = 0; c < rpad / 32; ++c) {
          const int col = (mm - m0) * rpad + c * 32;
          uint32_t v[32], w[32];
          tmem_ld32(taddr + col, v);
          tmem_ld32(taddr + N + col, w);
          tmem_wait_ld();
          const float* pr = pbuf + (size_t)rl * N + col;
          if (g < T) {
#pragma unroll
            for (int qq = 0; qq < 4; ++qq) {
              const float4 pa = *reinterpret_cast<const float4*>(pr + 8 * qq);
              const float4 pb = *reinterpret_cast<const float4*>(pr + 8 * qq + 4);
              const float pp[8] = {pa.x, pa.y, pa.z, pa.w, pb.x, pb.y, pb.z, pb.w};
              uint32_t ph2[4], pl[4];
#pragma unroll
              for (int e = 0; e < 4; ++e) {
                const int k0 = 8 * qq + 2 * e;
                const float o0 = __fadd_rn(__uint_as_float(v[k0]), __uint_as_float(w[k0]));
                const float o1 = __fadd_rn(__uint_as_float(v[k0 + 1]), __uint_as_float(w[k0 + 1]));
                const float z0 = mine ? __fadd_rn(o0, pp[2 * e]) : 0.f;
                const float z1 = mine ? __fadd_rn(o1, pp[2 * e + 1]) : 0.f;
                const float h0 = __bfloat162float(__float2bfloat16_rn(z0));
                const float h1 = __bfloat162float(__float2bfloat16_rn(z1));
                ph2[e] = pack_bf16(h0, h1);
                pl[e] = pack_bf16(__fsub_rn(z0, h0), __fsub_rn(z1, h1));
              }
              *reinterpret_cast<uint4*>(zr + c * 32 + qq * 8) = make_uint4(ph2[0], ph2[1], ph2[2], ph2[3]);
              *reinterpret_cast<uint4*>(zr + rpad + c * 32 + qq * 8) = make_uint4(pl[0], pl[1], pl[2], pl[3]);
            }
          }
        }
      }
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 1) {
    tc_fence_after();
    tmem_dealloc(tmem, tmem_cols);
  }
}

// L1s[p][(m-1)*rpad + k][i] = plane p of inv_s[m][i] * L1^m[i][k] (p = 0 hi, 1 lo); zero for k >= r
__global__ void l1_fold_kernel(const uint16_t* __restrict__ L1, const float* __restrict__ s_f, int64_t d, int r,
                               int rpad, int n_nt, uint16_t* __restrict__ L1s) {
  sm100::pdl_wait();     // launch_k: the previous kernel's writes are visible
  sm100::pdl_trigger();
  __shared__ float t[32][33];
  const int mb = blockIdx.z;                    // non-text modality index (m - 1)
  const int64_t i0 = (int64_t)blockIdx.x * 32;
  const int k0 = blockIdx.y * 32;
  const float* sm = s_f + (int64_t)(mb + 1) * d;
  const uint16_t* src = L1 + (int64_t)mb * d * r;
  for (int y = threadIdx.y; y < 32; y += blockDim.y) {
    const int64_t i = i0 + y;
    const int k = k0 + threadIdx.x;
    float v = 0.f;
    if (i < d && k < r) v = __fmul_rn(__uint_as_float((uint32_t)src[i * r + k] << 16), __fdiv_rn(1.0f, sm[i]));
    t[y][threadIdx.x] = v;
  }
  __syncthreads();
  for (int y = threadIdx.y; y < 32; y += blockDim.y) {
    const int k = k0 + y;
    const int64_t i = i0 + threadIdx.x;
    if (k < rpad && i < d) {
      const float v = t[threadIdx.x][y];
      const __nv_bfloat16 h = __float2bfloat16_rn(v);
      const __nv_bfloat16 l = __float2bfloat16_rn(__fsub_rn(v, __bfloat162float(h)));
      const int64_t row = (int64_t)mb * rpad + k;
      L1s[row * d + i] = __bfloat16_as_ushort(h);
      L1s[((int64_t)n_nt * rpad + row) * d + i] = __bfloat16_as_ushort(l);
    }
  }
}

// f32 X -> bf16 hi / lo planes (exact split to ~2^-17)
__global__ void split_f32_kernel(const float* __restrict__ X, int64_t ld_x, int64_t T, int64_t d,
                                 uint16_t* __restrict__ hi, uint16_t* __restrict__ lo) {
  sm100::pdl_wait();     // launch_k: the previous kernel's writes are visible
  sm100::pdl_trigger();
  const int64_t idx = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (idx >= T * d) return;
  const int64_t t = idx / d, i = idx - t * d;
  const float v = X[t * ld_x + i];
  const __nv_bfloat16 h = __float2bfloat16_rn(v);
  hi[idx] = __bfloat16_as_ushort(h);
  lo[idx] = __bfloat16_as_ushort(__float2bfloat16_rn(__fsub_rn(v, __bfloat162float(h))));
}
// split-K combine: Z rows of the blocks the forward reads = hi/lo of sum_s zpart[s] (fixed order),
// zeros for rows of other modalities; one thread per (row, non-text modality, 4 columns)
__global__ void __launch_bounds__(256) zcombine_kernel(const float* __restrict__ zpart, int splits, int64_t T_pad,
                                                       const uint8_t* __restrict__ ids, int64_t T, int n_mod,
                                                       int rpad, const uint32_t* __restrict__ tile_mask,
                                                       uint16_t* __restrict__ Z) {
  sm100::pdl_wait();     // launch_k: the previous kernel's writes are visible
  sm100::pdl_trigger();
  const int nnt = n_mod - 1;
  const int q4 = rpad / 4;
  const int64_t idx = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (idx >= T * nnt * q4) return;
  const int c4 = (int)(idx % q4);
  const int64_t w = idx / q4;
  const int64_t g = w / nnt;
  const int mm = (int)(w - g * nnt) + 1;
  const int64_t n_tiles = (T + 127) / 128, mt = g >> 7;
  const uint32_t tmask = tile_mask[mt] | ((mt ^ 1) < n_tiles ? tile_mask[mt ^ 1] : 0u);
  if (!((tmask >> mm) & 1u)) return;
  const bool mine = (int)__ldg(ids + g) == mm;
  float4 v[16];                                   // splits <= 16: all loads in flight, then the ordered sum
#pragma unroll
  for (int sp = 0; sp < 16; ++sp)
    if (sp < splits)
      v[sp] = __ldg(reinterpret_cast<const float4*>(zpart + ((sp * T_pad + g) * nnt + (mm - 1)) * rpad) + c4);
  float z[4] = {0.f, 0.f, 0.f, 0.f};
#pragma unroll
  for (int sp = 0; sp < 16; ++sp)
    if (sp < splits) {
      z[0] += v[sp].x;
      z[1] += v[sp].y;
      z[2] += v[sp].z;
      z[3] += v[sp].w;
    }
  uint16_t h[4], l[4];
#pragma unroll
  for (int e = 0; e < 4; ++e) {
    const float x = mine ? z[e] : 0.f;
    const __nv_bfloat16 hb = __float2bfloat16_rn(x);
    h[e] = __bfloat16_as_ushort(hb);
    l[e] = __bfloat16_as_ushort(__float2bfloat16_rn(__fsub_rn(x, __bfloat162float(hb))));
  }
  uint16_t* zr = Z + g * (int64_t)nnt * 2 * rpad + (int64_t)(mm - 1) * 2 * rpad + c4 * 4;
  *reinterpret_cast<uint2*>(zr) = make_uint2(h[0] | ((uint32_t)h[1] << 16), h[2] | ((uint32_t)h[3] << 16));
  *reinterpret_cast<uint2*>(zr + rpad) = make_uint2(l[0] | ((uint32_t)l[1] << 16), l[2] | ((uint32_t)l[3] << 16));
}
}  // namespace

int zgemm_splits(int64_t T, int64_t d) {
  const int64_t tiles = ceil_div(T, 128), nk = ceil_div(d, 64 * KSUB_MAX);
  static const int env_sp = [] {                         // measurement knob: forced split count
    const char* e = getenv("MASQ_ZGEMM_SPLITS");
    return e ? atoi(e) : 0;
  }();
  if (env_sp > 0) return (int)std::max<int64_t>(1, std::min<int64_t>(env_sp, nk / 2));
  if (tiles <= 0 || tiles * 2 > num_sms()) return 1;     // enough tiles to fill the GPU
  int64_t sp = num_sms() / tiles;
  sp = std::min<int64_t>(sp, 16);
  sp = std::min<int64_t>(sp, nk / 2);                    // >= 2 k-chunks (256 columns) per split
  return (int)std::max<int64_t>(sp, 1);
}

size_t zgemm_part_bytes(int64_t T, int64_t d, int n_mod, int rpad) {
  const int sp = zgemm_splits(T, d);
  if (sp <= 1 || n_mod < 2 || rpad <= 0) return 0;
  return sizeof(float) * (size_t)sp * ceil_div(T, 128) * 128 * (n_mod - 1) * rpad;
}

// the CMC factor packing of a forward call in one launch: blocks [0, g1) fold L1 as l1_fold_kernel,
// blocks [g1, ...) transpose L2^m [r x n] into L2t rows m*n + j, columns k and rpad + k (the
// [L2^T ; L2^T] operand of the GEMM's CMC k-blocks).  Both read only the factors, not X.
__global__ void cmc_pack_kernel(const uint16_t* __restrict__ L1, const float* __restrict__ s_f, int64_t d, int r,
                                int rpad, int n_nt, uint16_t* __restrict__ L1s, int g1x, int g1y,
                                const uint16_t* __restrict__ L2, int64_t ld_l2, int64_t n, uint16_t* __restrict__ L2t,
                                int g2x, int g2y, const uint8_t* __restrict__ ids, int64_t T, int n_mod,
                                uint32_t* __restrict__ mask) {
  sm100::pdl_wait();     // launch_k: the previous kernel's writes are visible
  sm100::pdl_trigger();
  __shared__ float t[32][33];
  const int g1 = g1x * g1y * n_nt;
  const int g2 = g2x * g2y * n_nt;
  int b = blockIdx.x;
  if (b >= g1 + g2) {
    // the per-128-row-tile modality bit sets the CMC first factor and the GEMM's CMC k-blocks read
    // (one warp per tile, written whole: no zeroing pass, no atomics); ids >= n_mod set no bit
    // (the activation quantizer flags them)
    const int64_t tile = (int64_t)(b - g1 - g2) * 8 + threadIdx.y;
    if (tile * 128 >= T) return;
    uint32_t bits = 0;
#pragma unroll
    for (int e = 0; e < 4; ++e) {
      const int64_t row = tile * 128 + threadIdx.x * 4 + e;
      if (row < T) {
        const int m = (int)__ldg(ids + row);
        if (m < n_mod) bits |= 1u << m;
      }
    }
    bits = __reduce_or_sync(0xffffffffu, bits);
    if (threadIdx.x == 0) mask[tile] = bits;
    return;
  }
  if (b < g1) {
    const int mb = b / (g1x * g1y);
    b -= mb * g1x * g1y;
    const int64_t i0 = (int64_t)(b % g1x) * 32;
    const int k0 = (b / g1x) * 32;
    const float* sm = s_f + (int64_t)(mb + 1) * d;
    const uint16_t* src = L1 + (int64_t)mb * d * r;
    for (int y = threadIdx.y; y < 32; y += blockDim.y) {
      const int64_t i = i0 + y;
      const int k = k0 + threadIdx.x;
      float v = 0.f;
      if (i < d && k < r) v = __fmul_rn(__uint_as_float((uint32_t)src[i * r + k] << 16), __fdiv_rn(1.0f, sm[i]));
      t[y][threadIdx.x] = v;
    }
    __syncthreads();
    for (int y = threadIdx.y; y < 32; y += blockDim.y) {
      const int k = k0 + y;
      const int64_t i = i0 + threadIdx.x;
      if (k < rpad && i < d) {
        const float v = t[threadIdx.x][y];
        const __nv_bfloat16 h = __float2bfloat16_rn(v);
        const __nv_bfloat16 l = __float2bfloat16_rn(__fsub_rn(v, __bfloat162float(h)));
        const int64_t row = (int64_t)mb * rpad + k;
        L1s[row * d + i] = __bfloat16_as_ushort(h);
        L1s[((int64_t)n_nt * rpad + row) * d + i] = __bfloat16_as_ushort(l);
      }
    }
    return;
  }
  b -= g1;
  const int mb = b / (g2x * g2y);
  b -= mb * g2x * g2y;
  const int64_t c0 = (int64_t)(b % g2x) * 32, r0 = (int64_t)(b / g2x) * 32;   // columns j, rows k of L2^m
  const uint16_t* ib = L2 + (int64_t)mb * r * ld_l2;
  uint16_t* ob = L2t + (int64_t)mb * n * 2 * rpad;
  uint16_t (*tt)[33] = reinterpret_cast<uint16_t(*)[33]>(&t[0][0]);
  for (int k = threadIdx.y; k < 32; k += blockDim.y) {
    const int64_t rr = r0 + k, c = c0 + threadIdx.x;
    tt[k][threadIdx.x] = (rr < r && c < n) ? ib[rr * ld_l2 + c] : (uint16_t)0;
  }
  __syncthreads();
  for (int k = threadIdx.y; k < 32; k += blockDim.y) {
    const int64_t c = c0 + k, rr = r0 + threadIdx.x;
    if (c < n && rr < r) {
      const uint16_t v = tt[threadIdx.x][k];
      ob[c * 2 * rpad + rr] = v;
      ob[c * 2 * rpad + rr + rpad] = v;
    }
  }
}

cudaError_t launch_cmc_pack(const uint16_t* L1, const float* s_f, int64_t d, int r, int rpad, int n_nt, uint16_t* L1s,
                            const uint16_t* L2, int64_t ld_l2, int64_t n, uint16_t* L2t, const uint8_t* ids, int64_t T,
                            int n_mod, uint32_t* mask, cudaStream_t st) {
  if (r < rpad) {
    cudaError_t e = cudaMemsetAsync(L1s, 0, sizeof(uint16_t) * 2 * (size_t)n_nt * rpad * d, st);
    if (e == cudaSuccess) e = cudaMemsetAsync(L2t, 0, sizeof(uint16_t) * n_nt * n * 2 * rpad, st);
    if (e != cudaSuccess) return e;
  }
  const int g1x = (int)ceil_div(d, 32), g1y = (int)ceil_div(r, 32);
  const int g2x = (int)ceil_div(n, 32), g2y = (int)ceil_div(r, 32);
  const int64_t g3 = mask ? ceil_div(ceil_div(T, 128), 8) : 0;
  const int64_t blocks = (int64_t)(g1x * g1y + g2x * g2y) * n_nt + g3;
  ProfScope ps_("cmc_pack", st);
  MASQ_LAUNCH(launch_k(cmc_pack_kernel, dim3((unsigned)blocks), dim3(32, 8), 0, st, L1, s_f, d, r, rpad, n_nt, L1s, g1x,
                       g1y, L2, ld_l2, n, L2t, g2x, g2y, ids, T, n_mod, mask));
  return cudaGetLastError();
}

cudaError_t launch_l1_fold(const uint16_t* L1, const float* s_f, int64_t d, int r, int rpad, int n_nt,
                           uint16_t* L1s, cudaStream_t st) {
  if (r < rpad) {
    cudaError_t e = cudaMemsetAsync(L1s, 0, sizeof(uint16_t) * 2 * (size_t)n_nt * rpad * d, st);
    if (e != cudaSuccess) return e;
  }
  dim3 grid((unsigned)ceil_div(d, 32), (unsigned)ceil_div(r, 32), n_nt), block(32, 8);
  ProfScope ps_("l1_fold", st);
  MASQ_LAUNCH(launch_k(l1_fold_kernel, dim3(grid), dim3(block), 0, st, L1, s_f, d, r, rpad, n_nt, L1s));
  return cudaGetLastError();
}

cudaError_t launch_split_f32(const float* X, int64_t ld_x, int64_t T, int64_t d, uint16_t* hi, uint16_t* lo,
                             cudaStream_t st) {
  const int64_t n = T * d;
  ProfScope ps_("split_f32", st);
  MASQ_LAUNCH(launch_k(split_f32_kernel, dim3((unsigned)ceil_div(n, 256)), dim3(256), 0, st, X, ld_x, T, d, hi, lo));
  return cudaGetLastError();
}

cudaError_t launch_zgemm(const uint16_t* A0, int64_t ld_a, const uint16_t* A1, const uint8_t* ids, int64_t T,
                         int64_t d, int n_mod, const uint16_t* L1s, int rpad, const uint32_t* tile_mask, uint16_t* Z,
                         cudaStream_t st, float* zpart) {
  if (T <= 0 || n_mod < 2 || rpad <= 0) return cudaSuccess;
  const int n_nt = n_mod - 1;
  // modalities per pass: 2 * per * rpad <= 256 MMA columns (the combined [hi; lo] form), else
  // per * rpad <= 256 with two MMAs per k-step
  const int per = rpad <= 128 ? std::max(1, std::min(n_nt, 128 / rpad)) : std::max(1, std::min(n_nt, 256 / rpad));
  const int passes = (int)ceil_div(n_nt, per);
  const int a_planes = A1 ? 2 : 1;
  CUtensorMap ta0, ta1, tb;
  bool ok = make_tmap_2d(&ta0, A0, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, T, d, ld_a, 128, 64, true);
  ok &= make_tmap_2d(&ta1, A1 ? A1 : A0, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, T, d, ld_a, 128, 64, true);
  const int N = per * rpad;
  ok &= make_tmap_2d(&tb, L1s, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, (uint64_t)2 * n_nt * rpad, d, d, (uint32_t)N, 64,
                     true);
  if (!ok) return cudaErrorInvalidValue;
  const int SBS = a_planes * XCH + 2 * N * 128;
  // measured (c3 step): two sub-blocks per stage make the pair-mode CTAs 1 per SM and lose
  // (zgemm 0.26 -> 0.36 ms per step), so one is the default
  int ksub = 1;
  static const int env_ks = [] {                         // measurement knob: sub-blocks per stage
    const char* e = getenv("MASQ_ZGEMM_KSUB");
    return e ? atoi(e) : 0;
  }();
  if (env_ks >= 1 && env_ks <= KSUB_MAX) ksub = env_ks;
  const int SB = ((ksub * SBS) + 1023) & ~1023;
  // cluster-pair split-K (two K halves per 128-row tile, reduced through DSMEM) when the tiles
  // alone leave SMs idle but no global split is taken: 3 stages so two CTAs fit per SM
  static const bool no_pair = [] {
    const char* e = getenv("MASQ_ZGEMM_PAIR");
    return e && e[0] == '0';
  }();
  const int64_t tiles = ceil_div(T, 128);
  const bool pair = !no_pair && zpart != nullptr && zgemm_splits(T, d) == 1 && a_planes == 1 && 2 * N <= 256 &&
                    tiles <= num_sms() && ceil_div(d, 64 * KSUB_MAX) >= 4;
  int stages = (SMEM_CAP - 2048) / SB;
  stages = stages > 8 ? 8 : stages;
  if (pair) stages = std::min(stages, 3);
  static const int env_st = [] {                         // measurement knob: ring stages
    const char* e = getenv("MASQ_ZGEMM_STAGES");
    return e ? atoi(e) : 0;
  }();
  if (env_st > 0) stages = std::min(stages, env_st);
  if (stages < 2) return cudaErrorInvalidValue;
  const int smem = stages * SB + 2048;
  cudaError_t e = set_max_dyn_smem(reinterpret_cast<const void*>(zgemm_kernel), smem);
  if (e != cudaSuccess) return e;
  const int acc_cols = 2 * N <= 256 ? 2 * N : N;
  uint32_t cols = 32;
  while ((int)cols < acc_cols) cols <<= 1;
  const int splits = pair ? 2 : (zpart ? zgemm_splits(T, d) : 1);
  dim3 grid((unsigned)ceil_div(T, 128), (unsigned)passes, (unsigned)splits);
  {
    ProfScope ps_("zgemm", st);
    if (pair) {
      cudaLaunchConfig_t cfg = {};
      cfg.gridDim = grid;
      cfg.blockDim = dim3(ZT);
      cfg.dynamicSmemBytes = (size_t)smem;
      cfg.stream = st;
      cudaLaunchAttribute at[2];
      at[0].id = cudaLaunchAttributeClusterDimension;
      at[0].val.clusterDim.x = 1;
      at[0].val.clusterDim.y = 1;
      at[0].val.clusterDim.z = 2;
      at[1].id = cudaLaunchAttributeProgrammaticStreamSerialization;   // as launch_k
      at[1].val.programmaticStreamSerializationAllowed = 1;
      cfg.attrs = at;
      cfg.numAttrs = pdl_enabled() ? 2 : 1;
      e = cudaLaunchKernelEx(&cfg, zgemm_kernel, ta0, ta1, tb, ids, (int)T, (int)d, n_mod, rpad, per, a_planes, cols,
                             stages, tile_mask, Z, (float*)nullptr, 2, 1, ksub);
      if (e != cudaSuccess) return e;
    } else {
      MASQ_LAUNCH(launch_k(zgemm_kernel, dim3(grid), dim3(ZT), smem, st, ta0, ta1, tb, ids, (int)T, (int)d, n_mod, rpad, per, a_planes, cols,
                                           stages, tile_mask, Z, zpart, splits, 0, ksub));
    }
  }
  if (splits > 1 && !pair) {
    e = cudaGetLastError();
    if (e != cudaSuccess) return e;
    const int64_t threads = T * n_nt * (rpad / 4);
    ProfScope ps_("zcombine", st);
    MASQ_LAUNCH(launch_k(zcombine_kernel, dim3((unsigned)ceil_div(threads, 256)), dim3(256), 0, st, zpart, splits, ceil_div(T, 128) * 128, ids, T,
                                                                      n_mod, rpad, tile_mask, Z));
  }
  return cudaGetLastError();
}

}  // namespace masq
