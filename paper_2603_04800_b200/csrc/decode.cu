// decode.cu — N3: packed int4 weights with 128-channel groups and a
// decode-shaped (T <= 16 tokens) W4A8 forward for text tokens (with text as
// the base modality, decoding needs no CMC).
//
// Weight format (reading Q28).  Codes of Q_g(S_t W) (per output channel j and group of 128 input
// channels) are stored as biased nibbles code + 8 (0..15) in the register order of the legacy
// warp MMA mma.sync.m16n8k32 B fragment, so that one 16-byte load per lane yields the B fragments
// of four consecutive k-steps (one group) for an 8-column tile:
//   tile (jt, g) = 512 bytes at ((jt * ngroups) + g) * 512;  lane L = 4*gid + tig holds 4 words;
//   word ks (k-step), byte e: low nibble  = code[j = 8 jt + gid][k = 128 g + 32 ks + 4 tig + e] + 8
//                             high nibble = code[j][k + 16] + 8
// so b0 = w & 0x0F0F0F0F and b1 = (w >> 4) & 0x0F0F0F0F are unsigned bytes fed to the s8 x u8 MMA,
// and the bias is removed exactly by starting each group's int32 accumulator at -8 * (sum of the
// group's activation codes of that token row).  Scales: f32 tile-major
// [n/8][ngroups][8] (the 8 columns of tile jt for group g at (jt*ngroups + g)*8), so that a tile's
// codes and scales for a K-chunk are two contiguous byte ranges.
//
// The decode GEMM is weight-bandwidth-bound: one CTA per SM owns a K-chunk of 4096 input
// channels (32 groups, 4 per consumer warp) whose activation A fragments stay in registers for
// the whole kernel; a producer warp streams the CTA's 8-column weight tiles (16 KB of codes + 1
// KB of scales, contiguous) with 1D TMA bulk copies into a 6-stage shared-memory ring (~100 KB
// in flight per SM); every group's int32 MMA sums are scaled by the group's weight scale into an
// f32 accumulator; warps combine through shared memory; with more than one K-chunk (d > 4096)
// the chunk partials are summed in a fixed order by a second small kernel (deterministic).
#include <cuda_bf16.h>

#include <cstdlib>

#include "internal.h"
#include "sm100.cuh"

namespace masq {
using namespace sm100;
namespace {

constexpr int kGroup = 128;
constexpr int kDecWarps = 8;
constexpr int kGroupsPerWarp = 4;
constexpr int kKChunk = kDecWarps * kGroupsPerWarp * kGroup;    // 4096 input channels per CTA
constexpr int kMaxDecodeT = 16;

constexpr int kTileCodes = (kKChunk / kGroup) * 512;              // 16 KB
constexpr int kTileScales = (kKChunk / kGroup) * 8 * 4;           // 1 KB

constexpr int kDecThreads = 32 * (kDecWarps + 1);
template <int kSub, int kStages, int kRed = 2>
struct DecCfg {
  static constexpr int kStageBytes = kSub * (kTileCodes + kTileScales);
  static constexpr int kSmem = kStages * kStageBytes + 2 * kStages * 8 + kRed * kSub * kDecWarps * 32 * 4 * 4 + 64;
  static_assert(kSmem <= 232448, "decode shared memory");
};

__device__ __forceinline__ int rha_code(float x, float delta, int qmin, int qmax) {
  const float v = __fdiv_rn(x, delta);
  const float t = truncf(v);
  const float fr = fabsf(__fsub_rn(v, t));
  const float q = fr >= 0.5f ? __fadd_rn(t, copysignf(1.0f, v)) : t;
  const int qi = (int)q;
  return qi < qmin ? qmin : (qi > qmax ? qmax : qi);
}

template <typename WT>
__device__ __forceinline__ float ldw(const WT* p);
template <>
__device__ __forceinline__ float ldw<__nv_bfloat16>(const __nv_bfloat16* p) { return __bfloat162float(*p); }
template <>
__device__ __forceinline__ float ldw<float>(const float* p) { return *p; }

// one CTA = 16 output channels (two 8-column tiles) x one group of 128 input channels;
// thread k reads row k of the group (16 columns), block max per column, exact codes, packing
// LAYOUT 0: the decode kernel's fragment order (above); LAYOUT 1: the prefill GEMM's group-major
// format (w4g.cu): packed[(g*n + j)*64 + 16c + i] = code[j][128g+32c+i] | code[j][128g+32c+16+i] << 4
// (two's complement nibbles), scales[j][g]
template <typename WT, int LAYOUT>
__global__ void __launch_bounds__(128) wq4_kernel(const WT* __restrict__ W, const float* __restrict__ s, int64_t d,
                                                  int64_t n, uint8_t* __restrict__ packed,
                                                  float* __restrict__ scales) {
  __shared__ float red[4][16];
  __shared__ float dsh[16];
  __shared__ int8_t codes[16][kGroup + 4];
  const int k = threadIdx.x;
  const int g = blockIdx.y;
  const int64_t j0 = (int64_t)blockIdx.x * 16;
  const int64_t row = (int64_t)g * kGroup + k;
  const float si = s[row];
  float ws[16];
#pragma unroll
  for (int c = 0; c < 16; ++c) ws[c] = (j0 + c < n) ? __fmul_rn(si, ldw<WT>(W + row * n + j0 + c)) : 0.f;
  const int warp = k >> 5, lane = k & 31;
#pragma unroll
  for (int c = 0; c < 16; ++c) {
    float m = fabsf(ws[c]);
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) m = fmaxf(m, __shfl_xor_sync(0xffffffffu, m, o));
    if (lane == 0) red[warp][c] = m;
  }
  __syncthreads();
  if (k < 16) {
    const float m = fmaxf(fmaxf(red[0][k], red[1][k]), fmaxf(red[2][k], red[3][k]));
    const float dl = fmaxf(__fdiv_rn(m, 7.0f), 1e-12f);
    dsh[k] = dl;
    if (j0 + k < n) {
      if (LAYOUT == 0) scales[(((j0 + k) >> 3) * (d / kGroup) + g) * 8 + ((j0 + k) & 7)] = dl;
      else scales[(j0 + k) * (d / kGroup) + g] = dl;
    }
  }
  __syncthreads();
#pragma unroll
  for (int c = 0; c < 16; ++c) codes[c][k] = (int8_t)rha_code(ws[c], dsh[c], -8, 7);
  __syncthreads();
  if (LAYOUT == 1) {
    // thread k: channel j0 + (k >> 3), bytes 8 (k & 7) .. + 7 of the group's 64
    const int c = k >> 3, b0 = (k & 7) * 8;
    if (j0 + c >= n) return;
    uint32_t w2[2] = {0u, 0u};
#pragma unroll
    for (int e = 0; e < 8; ++e) {
      const int b = b0 + e, cc = b >> 4, i = b & 15;
      const uint32_t lo = (uint32_t)codes[c][32 * cc + i] & 0xFu;
      const uint32_t hi = (uint32_t)codes[c][32 * cc + 16 + i] & 0xFu;
      w2[e >> 2] |= (lo | (hi << 4)) << (8 * (e & 3));
    }
    *reinterpret_cast<uint2*>(packed + ((int64_t)g * n + j0 + c) * 64 + b0) = make_uint2(w2[0], w2[1]);
    return;
  }
  // 2 tiles x 32 lanes x 4 words: thread k -> tile k >> 6, lane (k >> 1) & 31, words 2 (k & 1) + {0, 1}
  const int tile = k >> 6, L = (k >> 1) & 31, gid = L >> 2, tig = L & 3;
  const int64_t jt = (j0 >> 3) + tile;
  if (jt * 8 >= n) return;
  const int64_t ngroups = d / kGroup;
  uint32_t w2[2];
#pragma unroll
  for (int h = 0; h < 2; ++h) {
    const int ks = 2 * (k & 1) + h;
    uint32_t w = 0;
#pragma unroll
    for (int e = 0; e < 4; ++e) {
      const int kk = 32 * ks + 4 * tig + e;
      const uint32_t lo = (uint32_t)(codes[8 * tile + gid][kk] + 8);
      const uint32_t hi = (uint32_t)(codes[8 * tile + gid][kk + 16] + 8);
      w |= (lo | (hi << 4)) << (8 * e);
    }
    w2[h] = w;
  }
  uint2* dst = reinterpret_cast<uint2*>(packed + ((jt * ngroups + g) * 512) + L * 16 + (k & 1) * 8);
  *dst = make_uint2(w2[0], w2[1]);
}

__global__ void unpack4_kernel(const uint8_t* __restrict__ packed, int64_t d, int64_t n, int8_t* __restrict__ codes) {
  const int64_t idx = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;    // one word
  const int64_t ngroups = d / kGroup;
  const int64_t words = (n / 8) * ngroups * 128;
  if (idx >= words) return;
  const int64_t tile = idx >> 7;
  const int L = (int)((idx >> 2) & 31), ks = (int)(idx & 3);
  const int64_t jt = tile / ngroups, g = tile - jt * ngroups;
  const uint32_t w = reinterpret_cast<const uint32_t*>(packed)[idx];
  const int gid = L >> 2, tig = L & 3;
  const int64_t j = jt * 8 + gid;
#pragma unroll
  for (int e = 0; e < 4; ++e) {
    const int64_t k = g * kGroup + 32 * ks + 4 * tig + e;
    const int lo = (int)((w >> (8 * e)) & 0xF), hi = (int)((w >> (8 * e + 4)) & 0xF);
    codes[j * d + k] = (int8_t)(lo - 8);
    codes[j * d + k + 16] = (int8_t)(hi - 8);
  }
}

__device__ __forceinline__ void mma_s8u8(int (&c)[4], const uint32_t (&a)[4], uint32_t b0, uint32_t b1) {
  asm volatile(
      "mma.sync.aligned.m16n8k32.row.col.s32.s8.u8.s32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, "
      "{%0,%1,%2,%3};\n"
      : "+r"(c[0]), "+r"(c[1]), "+r"(c[2]), "+r"(c[3])
      : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b0), "r"(b1));
}

// grid (x: CTAs streaming 32-column super tiles, y: K-chunks of 4096 channels); warps 0-7
// consume, warp 8 (one lane) produces.  A stage holds up to 4 sub-tiles (8 columns each) of the
// CTA's K-chunk: codes at [sub][group][512 B], scales at [sub][group][8 f32].
template <int kSub, int kStages, int kRed = 2>
__global__ void __launch_bounds__(kDecThreads) decode_kernel(const int8_t* __restrict__ qa,
                                                             const float* __restrict__ dx, int T, int64_t d,
                                                             int64_t n, const uint8_t* __restrict__ packed,
                                                             const float* __restrict__ scales,
                                                             float* __restrict__ part, float* __restrict__ Y,
                                                             int64_t ldy) {
  constexpr int kStageBytes = DecCfg<kSub, kStages, kRed>::kStageBytes;
  extern __shared__ __align__(128) uint8_t dsm[];
  uint8_t* ring = dsm;
  uint64_t* full = reinterpret_cast<uint64_t*>(dsm + kStages * kStageBytes);
  uint64_t* empty = full + kStages;
  float* red = reinterpret_cast<float*>(empty + kStages);          // [2][kSub][8 warps][32][4]
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int64_t ngroups = d / kGroup;
  const int ky = (int)gridDim.y;
  const int64_t gbase = (int64_t)blockIdx.y * (kKChunk / kGroup);
  const int64_t remc = ngroups - gbase;
  const int ngc = remc < (kKChunk / kGroup) ? (int)remc : (kKChunk / kGroup);   // groups of this chunk
  const int64_t ntiles = n / 8;
  const int64_t nsuper = (ntiles + kSub - 1) / kSub;
  if (threadIdx.x == 0) {
    for (int i = 0; i < kStages; ++i) {
      mbar_init(&full[i], 1);
      mbar_init(&empty[i], kDecWarps);
    }
    fence_mbar_init();
  }
  __syncthreads();
  if (warp == kDecWarps) {
    if (lane == 0) {
      uint32_t st = 0, ph = 0;
      const uint32_t cb = (uint32_t)ngc * 512u, sb = (uint32_t)ngc * 32u;
      for (int64_t js = blockIdx.x; js < nsuper; js += gridDim.x) {
        const int64_t jt0 = js * kSub;
        const int ns = (int)(ntiles - jt0 < kSub ? ntiles - jt0 : kSub);
        mbar_wait(&empty[st], ph ^ 1u);
        mbar_expect_tx(&full[st], (uint32_t)ns * (cb + sb));
        uint8_t* dst = ring + st * kStageBytes;
        for (int sub = 0; sub < ns; ++sub) {
          const int64_t jt = jt0 + sub;
          bulk_load_1d(dst + sub * kTileCodes, packed + (jt * ngroups + gbase) * 512, cb, &full[st]);
          bulk_load_1d(dst + kSub * kTileCodes + sub * kTileScales, scales + (jt * ngroups + gbase) * 8, sb,
                       &full[st]);
        }
        if (++st == kStages) { st = 0; ph ^= 1u; }
      }
    }
    return;
  }
  // programmatic dependent launch: the producer above streams weights (inputs of earlier calls)
  // while the activation quantizer that precedes this kernel may still run; the consumers wait
  // for it here, before touching its codes and scales
  asm volatile("griddepcontrol.wait;" ::: "memory");
  const int gid = lane >> 2, tig = lane & 3;
  const int gw = warp * kGroupsPerWarp;                            // first group of this warp in the chunk
  const int remw = ngc - gw;
  const int ng = remw <= 0 ? 0 : (remw < kGroupsPerWarp ? remw : kGroupsPerWarp);
  uint32_t af[kGroupsPerWarp][4][4];
#pragma unroll
  for (int gg = 0; gg < kGroupsPerWarp; ++gg)
#pragma unroll
    for (int ks = 0; ks < 4; ++ks) {
      const int64_t k = (gbase + gw + gg) * kGroup + 32 * ks + 4 * tig;
      const bool ok = gg < ng;
      af[gg][ks][0] = (ok && gid < T) ? __ldg(reinterpret_cast<const uint32_t*>(qa + (int64_t)gid * d + k)) : 0u;
      af[gg][ks][1] = (ok && gid + 8 < T) ? __ldg(reinterpret_cast<const uint32_t*>(qa + (int64_t)(gid + 8) * d + k)) : 0u;
      af[gg][ks][2] = (ok && gid < T) ? __ldg(reinterpret_cast<const uint32_t*>(qa + (int64_t)gid * d + k + 16)) : 0u;
      af[gg][ks][3] = (ok && gid + 8 < T) ? __ldg(reinterpret_cast<const uint32_t*>(qa + (int64_t)(gid + 8) * d + k + 16))
                                          : 0u;
    }
  // bias correction: -8 * sum of the group's activation codes, for rows gid and gid + 8
  int nlo[kGroupsPerWarp], nhi[kGroupsPerWarp];
#pragma unroll
  for (int gg = 0; gg < kGroupsPerWarp; ++gg) {
    int sl = 0, sh = 0;
#pragma unroll
    for (int ks = 0; ks < 4; ++ks) {
      sl = __dp4a((int)af[gg][ks][0], 0x01010101, sl);
      sl = __dp4a((int)af[gg][ks][2], 0x01010101, sl);
      sh = __dp4a((int)af[gg][ks][1], 0x01010101, sh);
      sh = __dp4a((int)af[gg][ks][3], 0x01010101, sh);
    }
    sl += __shfl_xor_sync(0xffffffffu, sl, 1);
    sl += __shfl_xor_sync(0xffffffffu, sl, 2);
    sh += __shfl_xor_sync(0xffffffffu, sh, 1);
    sh += __shfl_xor_sync(0xffffffffu, sh, 2);
    nlo[gg] = -8 * sl;
    nhi[gg] = -8 * sh;
  }
  const float d0 = gid < T ? dx[gid] : 0.f, d1 = gid + 8 < T ? dx[gid + 8] : 0.f;
  const uint32_t boff = (uint32_t)gw * 512u + (uint32_t)lane * 16u;
  const uint32_t soff = kSub * kTileCodes + ((uint32_t)gw * 8u + 2u * (uint32_t)tig) * 4u;
  uint32_t st = 0, ph = 0, it = 0;
  for (int64_t js = blockIdx.x; js < nsuper; js += gridDim.x, ++it) {
    const int64_t jt0 = js * kSub;
    const int ns = (int)(ntiles - jt0 < kSub ? ntiles - jt0 : kSub);
    mbar_wait(&full[st], ph);
    const uint8_t* sbase = ring + st * kStageBytes;
    // kRed == 1: one partials buffer; the reducers of the previous stage must be done with it
    if (kRed == 1 && it > 0) asm volatile("bar.sync 1, %0;" ::"n"(32 * kDecWarps) : "memory");
    float* rb = red + (kRed == 2 ? (it & 1u) : 0u) * (kSub * kDecWarps * 32 * 4);
#pragma unroll
    for (int sub = 0; sub < kSub; ++sub) {
      float acc[4] = {0.f, 0.f, 0.f, 0.f};
      if (sub < ns && ng == kGroupsPerWarp) {                       // full warp chunk: no per-group guards
        uint4 bw[kGroupsPerWarp];
        float2 sc[kGroupsPerWarp];
#pragma unroll
        for (int gg = 0; gg < kGroupsPerWarp; ++gg) {
          bw[gg] = *reinterpret_cast<const uint4*>(sbase + sub * kTileCodes + boff + gg * 512);
          sc[gg] = *reinterpret_cast<const float2*>(sbase + soff + sub * kTileScales + gg * 32);
        }
        int c[kGroupsPerWarp][4];
#pragma unroll
        for (int gg = 0; gg < kGroupsPerWarp; ++gg) {
          c[gg][0] = c[gg][1] = nlo[gg];
          c[gg][2] = c[gg][3] = nhi[gg];
        }
#pragma unroll
        for (int ks = 0; ks < 4; ++ks)
#pragma unroll
          for (int gg = 0; gg < kGroupsPerWarp; ++gg) {
            const uint32_t w = ks == 0 ? bw[gg].x : ks == 1 ? bw[gg].y : ks == 2 ? bw[gg].z : bw[gg].w;
            mma_s8u8(c[gg], af[gg][ks], w & 0x0F0F0F0Fu, (w >> 4) & 0x0F0F0F0Fu);
          }
#pragma unroll
        for (int gg = 0; gg < kGroupsPerWarp; ++gg) {
          acc[0] = fmaf((float)c[gg][0], sc[gg].x, acc[0]);
          acc[1] = fmaf((float)c[gg][1], sc[gg].y, acc[1]);
          acc[2] = fmaf((float)c[gg][2], sc[gg].x, acc[2]);
          acc[3] = fmaf((float)c[gg][3], sc[gg].y, acc[3]);
        }
      } else if (sub < ns) {                                       // the chunk's tail warp
        for (int gg = 0; gg < ng; ++gg) {
          const uint4 bw = *reinterpret_cast<const uint4*>(sbase + sub * kTileCodes + boff + gg * 512);
          const float2 sc = *reinterpret_cast<const float2*>(sbase + soff + sub * kTileScales + gg * 32);
          int c[4] = {nlo[gg], nlo[gg], nhi[gg], nhi[gg]};
          const uint32_t w[4] = {bw.x, bw.y, bw.z, bw.w};
#pragma unroll
          for (int ks = 0; ks < 4; ++ks) mma_s8u8(c, af[gg][ks], w[ks] & 0x0F0F0F0Fu, (w[ks] >> 4) & 0x0F0F0F0Fu);
          acc[0] = fmaf((float)c[0], sc.x, acc[0]);
          acc[1] = fmaf((float)c[1], sc.y, acc[1]);
          acc[2] = fmaf((float)c[2], sc.x, acc[2]);
          acc[3] = fmaf((float)c[3], sc.y, acc[3]);
        }
      }
      *reinterpret_cast<float4*>(rb + ((sub * kDecWarps + warp) * 32 + lane) * 4) =
          make_float4(acc[0], acc[1], acc[2], acc[3]);
    }
    __syncwarp();
    if (lane == 0) mbar_arrive(&empty[st]);                        // this warp is done with the stage
    if (++st == kStages) { st = 0; ph ^= 1u; }
    asm volatile("bar.sync 1, %0;" ::"n"(32 * kDecWarps) : "memory");
    if (warp < ns) {                                               // warp w reduces sub-tile w
      const int64_t jt = jt0 + warp;
      float v[4] = {0.f, 0.f, 0.f, 0.f};
#pragma unroll
      for (int w = 0; w < kDecWarps; ++w) {
        const float4 q = *reinterpret_cast<const float4*>(rb + ((warp * kDecWarps + w) * 32 + lane) * 4);
        v[0] += q.x;
        v[1] += q.y;
        v[2] += q.z;
        v[3] += q.w;
      }
      // C fragment: v0, v1 -> row gid, cols 2 tig + {0, 1}; v2, v3 -> row gid + 8
      const int64_t j = jt * 8 + 2 * tig;
      if (ky > 1) {
        *reinterpret_cast<float4*>(part + ((int64_t)blockIdx.y * ntiles + jt) * 128 + lane * 4) =
            make_float4(v[0], v[1], v[2], v[3]);
      } else {
        if (gid < T) {
          Y[(int64_t)gid * ldy + j] = v[0] * d0;
          Y[(int64_t)gid * ldy + j + 1] = v[1] * d0;
        }
        if (gid + 8 < T) {
          Y[(int64_t)(gid + 8) * ldy + j] = v[2] * d1;
          Y[(int64_t)(gid + 8) * ldy + j + 1] = v[3] * d1;
        }
      }
    }
  }
}

// Y = dx[t] * sum over K-chunks (fixed order) of the chunk partials; thread = (tile, lane)
__global__ void decode_combine_kernel(const float* __restrict__ part, int ky, int64_t ntiles, int T,
                                      const float* __restrict__ dx, float* __restrict__ Y, int64_t ldy) {
  const int64_t idx = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (idx >= ntiles * 32) return;
  const int64_t jt = idx >> 5;
  const int lane = (int)(idx & 31), gid = lane >> 2, tig = lane & 3;
  float v[4] = {0.f, 0.f, 0.f, 0.f};
  for (int y = 0; y < ky; ++y) {
    const float4 q = *reinterpret_cast<const float4*>(part + ((int64_t)y * ntiles + jt) * 128 + lane * 4);
    v[0] += q.x;
    v[1] += q.y;
    v[2] += q.z;
    v[3] += q.w;
  }
  const int64_t j = jt * 8 + 2 * tig;
  if (gid < T) {
    const float d0 = dx[gid];
    Y[(int64_t)gid * ldy + j] = v[0] * d0;
    Y[(int64_t)gid * ldy + j + 1] = v[1] * d0;
  }
  if (gid + 8 < T) {
    const float d1 = dx[gid + 8];
    Y[(int64_t)(gid + 8) * ldy + j] = v[2] * d1;
    Y[(int64_t)(gid + 8) * ldy + j + 1] = v[3] * d1;
  }
}

}  // namespace

int decode_kchunks(int64_t d) { return (int)ceil_div(d, kKChunk); }
int decode_max_tokens() { return kMaxDecodeT; }

cudaError_t launch_wq4_layout(const void* W, masq_dtype wt, const float* s, int64_t d, int64_t n, uint8_t* packed,
                              float* scales, int layout, cudaStream_t st) {
  dim3 grid((unsigned)ceil_div(n, 16), (unsigned)(d / kGroup));
  ProfScope ps_(layout ? "wq4g" : "wq4", st);
  if (wt == MASQ_BF16) {
    if (layout) wq4_kernel<__nv_bfloat16, 1><<<grid, 128, 0, st>>>(static_cast<const __nv_bfloat16*>(W), s, d, n, packed, scales);
    else wq4_kernel<__nv_bfloat16, 0><<<grid, 128, 0, st>>>(static_cast<const __nv_bfloat16*>(W), s, d, n, packed, scales);
  } else {
    if (layout) wq4_kernel<float, 1><<<grid, 128, 0, st>>>(static_cast<const float*>(W), s, d, n, packed, scales);
    else wq4_kernel<float, 0><<<grid, 128, 0, st>>>(static_cast<const float*>(W), s, d, n, packed, scales);
  }
  return cudaGetLastError();
}

cudaError_t launch_wq4(const void* W, masq_dtype wt, const float* s, int64_t d, int64_t n, uint8_t* packed,
                       float* scales, cudaStream_t st) {
  return launch_wq4_layout(W, wt, s, d, n, packed, scales, 0, st);
}

cudaError_t launch_unpack4(const uint8_t* packed, int64_t d, int64_t n, int8_t* codes, cudaStream_t st) {
  const int64_t words = (n / 8) * (d / kGroup) * 128;
  unpack4_kernel<<<(unsigned)ceil_div(words, 256), 256, 0, st>>>(packed, d, n, codes);
  return cudaGetLastError();
}

cudaError_t launch_decode(const int8_t* qa, const float* dx, int T, int64_t d, int64_t n, const uint8_t* packed,
                          const float* scales, float* part, float* Y, int64_t ldy, cudaStream_t st) {
  const int ky = decode_kchunks(d);
  const int64_t ntiles = n / 8;
  // (sub-tiles per stage, stages): MASQ_DECODE_CFG=<s><k> overrides (measurement only)
  static int cfg = -1;
  if (cfg < 0) {
    const char* e = getenv("MASQ_DECODE_CFG");
    cfg = e ? atoi(e) : 42;
  }
  static const bool pdl = getenv("MASQ_DECODE_PDL") == nullptr || getenv("MASQ_DECODE_PDL")[0] != '0';
  const int per = std::max(1, num_sms() / ky);                    // one CTA per SM in total
  dim3 grid((unsigned)std::min<int64_t>(ntiles, per), (unsigned)ky);
  cudaError_t err = cudaSuccess;
  {
    ProfScope ps_("decode_w4a8", st);
#define DEC(S, K, RD)                                                                                         \
  {                                                                                                           \
    err = set_max_dyn_smem(reinterpret_cast<const void*>(decode_kernel<S, K, RD>), DecCfg<S, K, RD>::kSmem);    \
    if (err != cudaSuccess) return err;                                                                       \
    cudaLaunchConfig_t cfg_ = {};                                                                             \
    cfg_.gridDim = grid;                                                                                      \
    cfg_.blockDim = dim3(kDecThreads);                                                                        \
    cfg_.dynamicSmemBytes = DecCfg<S, K, RD>::kSmem;                                                          \
    cfg_.stream = st;                                                                                         \
    cudaLaunchAttribute at_[1];                                                                               \
    at_[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;                                           \
    at_[0].val.programmaticStreamSerializationAllowed = pdl ? 1 : 0;                                          \
    cfg_.attrs = at_;                                                                                         \
    cfg_.numAttrs = 1;                                                                                        \
    err = cudaLaunchKernelEx(&cfg_, decode_kernel<S, K, RD>, qa, dx, T, d, n, packed, scales, part, Y, ldy);  \
    if (err != cudaSuccess) return err;                                                                       \
  }
    switch (cfg) {
      case 33: DEC(3, 3, 2) break;
      case 24: DEC(2, 4, 2) break;
      case 25: DEC(2, 5, 2) break;
      case 16: DEC(1, 6, 2) break;
      case 431: DEC(4, 3, 1) break;
      case 531: DEC(5, 2, 1) break;
      default: DEC(4, 2, 2) break;
    }
#undef DEC
  }
  if ((err = cudaGetLastError()) != cudaSuccess) return err;
  if (ky > 1) {
    ProfScope ps_("decode_combine", st);
    decode_combine_kernel<<<(unsigned)ceil_div(ntiles * 32, 256), 256, 0, st>>>(part, ky, ntiles, T, dx, Y, ldy);
  }
  return cudaGetLastError();
}

}  // namespace masq
