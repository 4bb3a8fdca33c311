// w4g.cu — N3: the prefill-shaped W4A8 forward with PACKED int4 weights and
// per-(output channel, 128-input-channel group) scales on the CTA-pair tcgen05 path
// (PAPER.md:241-246 WxAy quantization, PAPER.md:177-185 routed forward with CMC, PAPER.md:584 W4
// kernel; reading Q28: groups of 128, codes in [-8, 7], Delta_jg = max|s w| / 7).
//
//   Y[t, j] = dx[t] * sum_g Delta_jg * (sum_{i in g} qx[t, i] * code[j, i])   (+ CMC for m_t != text)
//
// Roles are swapped with respect to gemm.cu so that the per-group scale is per TMEM LANE: the
// weight tile is the MMA's A operand (M = 256 output channels per CTA pair, 128 per CTA = one
// TMEM lane each) and the tokens are N (128 per unit).  Every group of 128 input channels is one
// k-block and one fresh int32 accumulator (4 x kind::i8 K = 32 MMAs); the epilogue warps read it
// (tcgen05.ld) and promote it into f32 registers with the lane's own scale:  y += Delta_jg/16 * acc
// — no shuffles, one scalar per lane and group.  Four 128-column TMEM accumulators rotate so the
// MMAs of group g+1..g+3 overlap the promotion of group g.
//
// Packed format (this kernel's, masq_quantize_weight_w4g): K-major, d/2 bytes per output channel;
// in the 64 bytes of group g, byte 16c + i holds code[128g + 32c + i] in its low nibble and
// code[128g + 32c + 16 + i] in its high nibble (two's complement).  Converter warps expand one
// group per stage in shared memory: (w << 4) & 0xF0F0F0F0 and w & 0xF0F0F0F0 are the int8 values
// 16*code of 16 consecutive k (two ops per 8 codes, no sign extension, natural K order), written
// into the SWIZZLE_128B K-major A tile the MMA reads; the factor 16 is removed exactly in the
// epilogue (Delta / 16 is a power-of-two scaling).  |16 * sum_g| <= 16 * 8 * 127 * 128 < 2^22.
//
// CMC (non-text tokens): one more accumulator per unit whose tile holds non-text
// tokens: [Zhi | Zlo] . [L2^T ; L2^T] (kind::f16, A = the L2^T rows of the unit's channels, B = the
// tokens' Z rows), added in f32 after the dx scaling.  Y is written straight from registers (lane =
// channel, so a warp stores 32 consecutive floats of a token row).
#include <cstdio>
#include <type_traits>

#include "internal.h"
#include "sm100.cuh"

namespace masq {
using namespace sm100;

namespace {
constexpr int QM = 128;                 // output channels per CTA (TMEM lanes)
constexpr int QUM = 2 * QM;             // per CTA pair (MMA M)
constexpr int QN = 128;                 // tokens per unit (MMA N)
constexpr int QNH = QN / 2;             // token rows each CTA loads
constexpr int QK = 128;                 // one group = one k-block (128 int8 / 64 bf16)
constexpr int PK_BYTES = QM * 64;       // packed group tile (8 KB)
constexpr int QA_BYTES = QM * QK;       // unpacked / L2^T A tile (16 KB)
constexpr int QB_BYTES = QNH * QK;      // activation / Z B tile (8 KB)
constexpr int QSTAGES = 5;
constexpr int NBUF = 4;                 // 128-column TMEM accumulators
constexpr int CONV_WARPS = 2;               // each thread expands 2 rows per group
constexpr int EPI_WARPS = 8;
constexpr int QTHREADS = 64 + 32 * (CONV_WARPS + EPI_WARPS);
constexpr int SM_PK = 0;
constexpr int SM_A = SM_PK + QSTAGES * PK_BYTES;
constexpr int SM_B = SM_A + QSTAGES * QA_BYTES;
constexpr int SM_BAR = SM_B + QSTAGES * QB_BYTES;
constexpr int SM_USED = SM_BAR + 512;
constexpr int SM_ALLOC = SM_USED + 1024;
constexpr uint32_t IDESC_Q = idesc_i8(QUM, QN);
constexpr uint32_t IDESC_QC = idesc_bf16(QUM, QN);
constexpr uint16_t kPair = 0x3;
static_assert(SM_ALLOC <= 232448, "shared memory budget");

struct WParams {
  int T, n, d, ng;                      // tokens, output channels, input channels, groups (d / 128)
  int num_m, num_n, n_units, group;     // token tiles, channel tiles (256), units, raster group
  int n_mod, rpad, cmc_kb;
  const uint32_t* tile_mask;            // modality bit set per 128-token tile
  const float* dx;                      // [T]
  const float* scales;                  // [n][ng]
  void* out;                            // f32 Y or int32 accumulators [T][ld_out]
  long long ld_out;
  int acc_mode;                         // 1: int32 sum over groups (debug tap), no dx / CMC
};


struct WUnit {
  int mt, nt;
  uint32_t mask;
  bool cmc;
};

__device__ __forceinline__ WUnit w_unit(const WParams& p, int u) {
  // p.group consecutive channel tiles swept over all token tiles: the group's packed weights stay
  // L2-resident while each token tile's activations are read by the group's units back to back
  WUnit w;
  const int per_group = p.group * p.num_m;
  const int g = u / per_group;
  const int rem = u - g * per_group;
  const int nt0 = g * p.group;
  const int gsz = min(p.group, p.num_n - nt0);
  w.mt = rem / gsz;
  w.nt = nt0 + (rem - w.mt * gsz);
  w.mask = p.tile_mask ? p.tile_mask[w.mt] : 1u;
  w.cmc = !p.acc_mode && p.rpad > 0 && (w.mask & ~1u) != 0u;
  return w;
}

struct QRing {
  uint32_t stage = 0, phase = 0;
  __device__ __forceinline__ void advance() {
    if (++stage == QSTAGES) { stage = 0; phase ^= 1u; }
  }
};

template <bool ACC>
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(QTHREADS, 1)
w4g_gemm_kernel(const __grid_constant__ CUtensorMap tmPK, const __grid_constant__ CUtensorMap tmX,
                const __grid_constant__ CUtensorMap tmL2, const __grid_constant__ CUtensorMap tmZ, const WParams p) {
  extern __shared__ uint8_t smem_raw[];
  const uint32_t raw = smem_u32(smem_raw);
  uint8_t* smem = smem_raw + (((raw + 1023u) & ~1023u) - raw);
  uint8_t* sPK = smem + SM_PK;
  uint8_t* sA = smem + SM_A;
  uint8_t* sB = smem + SM_B;
  uint64_t* pfull = reinterpret_cast<uint64_t*>(smem + SM_BAR);   // own: packed tile landed
  uint64_t* full = pfull + QSTAGES;      // leader's: B (and CMC A) landed in both CTAs
  uint64_t* aready = full + QSTAGES;     // leader's: both CTAs' converters wrote A
  uint64_t* empty = aready + QSTAGES;    // both: the MMAs of the stage completed
  uint64_t* tfull = empty + QSTAGES;     // [NBUF] both: accumulator ready
  uint64_t* tempty = tfull + NBUF;       // [NBUF] leader's: both CTAs' epilogues drained it
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tempty + NBUF);

  const uint32_t warp = warp_id(), lane = lane_id();
  const uint32_t rank = cluster_ctarank();
  const bool leader = rank == 0;
  const int cid = (int)cluster_id_x(), ncl = (int)ncluster_x();

  if (warp == 0 && lane == 0) {
    tma_prefetch(&tmPK);
    tma_prefetch(&tmX);
    for (int i = 0; i < QSTAGES; ++i) {
      mbar_init(&pfull[i], 1);
      mbar_init(&full[i], 1);
      mbar_init(&aready[i], 2 * CONV_WARPS);
      mbar_init(&empty[i], 1);
    }
    for (int i = 0; i < NBUF; ++i) {
      mbar_init(&tfull[i], 1);
      mbar_init(&tempty[i], 2 * EPI_WARPS);
    }
    fence_mbar_init();
  }
  if (warp == 1) tmem_alloc_2sm(tmem_slot, 512);
  tc_fence_before();
  cluster_sync();
  tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;

  if (warp == 0) {
    if (lane == 0) {
      // ---------------------------------------------------------------- TMA producer (both CTAs)
      QRing ring;
      for (int u = cid; u < p.n_units; u += ncl) {
        const WUnit w = w_unit(p, u);
        const int crow = w.nt * QUM + (int)rank * QM;         // this CTA's output channels
        const int trow = w.mt * QN + (int)rank * QNH;         // this CTA's token rows
        for (int g = 0; g < p.ng; ++g) {
          mbar_wait(&empty[ring.stage], ring.phase ^ 1u);
          mbar_expect_tx(&pfull[ring.stage], PK_BYTES);
          tma_load_2d(sPK + ring.stage * PK_BYTES, &tmPK, &pfull[ring.stage], g * 64, crow);
          if (leader) mbar_expect_tx(&full[ring.stage], 2 * QB_BYTES);
          tma_load_2d_2sm(sB + ring.stage * QB_BYTES, &tmX, &full[ring.stage], g * QK, trow);
          ring.advance();
        }
        if (w.cmc) {
          for (int mm = 1; mm < p.n_mod; ++mm) {
            if (!((w.mask >> mm) & 1u)) continue;
            for (int kb = 0; kb < p.cmc_kb; ++kb) {
              mbar_wait(&empty[ring.stage], ring.phase ^ 1u);
              if (leader) mbar_expect_tx(&full[ring.stage], 2 * (QA_BYTES + QB_BYTES));
              tma_load_2d_2sm(sA + ring.stage * QA_BYTES, &tmL2, &full[ring.stage], kb * 64, (mm - 1) * p.n + crow);
              tma_load_2d_2sm(sB + ring.stage * QB_BYTES, &tmZ, &full[ring.stage], (mm - 1) * 2 * p.rpad + kb * 64,
                              trow);
              ring.advance();
            }
          }
        }
      }
    }
    __syncwarp();
  } else if (warp == 1) {
    if (leader && lane == 0) {
      // ---------------------------------------------------------------- MMA issuer (leader CTA)
      QRing ring;
      uint32_t aph = 0;                 // per-stage phase bits of aready (group stages only)
      uint32_t acnt = 0;                // accumulator buffers used so far
      const uint32_t a0 = smem_u32(sA), b0 = smem_u32(sB);
      for (int u = cid; u < p.n_units; u += ncl) {
        const WUnit w = w_unit(p, u);
        for (int g = 0; g < p.ng; ++g) {
          const uint32_t buf = acnt % NBUF, bph = (acnt / NBUF) & 1u;
          ++acnt;
          mbar_wait(&tempty[buf], bph ^ 1u);
          mbar_wait(&full[ring.stage], ring.phase);
          mbar_wait(&aready[ring.stage], (aph >> ring.stage) & 1u);
          aph ^= 1u << ring.stage;
          tc_fence_after();
          const uint32_t dtm = tmem_base + buf * QN;
#pragma unroll
          for (int k = 0; k < 4; ++k)
            mma_i8_2sm(dtm, umma_desc_sw128(a0 + ring.stage * QA_BYTES + k * 32),
                       umma_desc_sw128(b0 + ring.stage * QB_BYTES + k * 32), IDESC_Q, k != 0);
          mma_commit_2sm(&empty[ring.stage], kPair);
          mma_commit_2sm(&tfull[buf], kPair);
          ring.advance();
        }
        if (w.cmc) {
          const uint32_t buf = acnt % NBUF, bph = (acnt / NBUF) & 1u;
          ++acnt;
          mbar_wait(&tempty[buf], bph ^ 1u);
          tc_fence_after();
          const uint32_t dtm = tmem_base + buf * QN;
          bool first = true;
          for (int mm = 1; mm < p.n_mod; ++mm) {
            if (!((w.mask >> mm) & 1u)) continue;
            for (int kb = 0; kb < p.cmc_kb; ++kb) {
              mbar_wait(&full[ring.stage], ring.phase);
              tc_fence_after();
#pragma unroll
              for (int k = 0; k < 4; ++k) {
                mma_bf16_2sm(dtm, umma_desc_sw128(a0 + ring.stage * QA_BYTES + k * 32),
                             umma_desc_sw128(b0 + ring.stage * QB_BYTES + k * 32), IDESC_QC, first ? 0u : 1u);
                first = false;
              }
              mma_commit_2sm(&empty[ring.stage], kPair);
              ring.advance();
            }
          }
          mma_commit_2sm(&tfull[buf], kPair);
        }
      }
    }
    __syncwarp();
  } else if (warp < 2 + CONV_WARPS) {
    // ------------------------------------------------------------------ converters (both CTAs)
    // thread = two output channel rows of this CTA's tile: 64 packed bytes -> 128 int8 (16 x code)
    const uint32_t row0 = (warp - 2) * 32 + lane;
    QRing ring;
    uint32_t pph = 0;                   // per-stage phase bits of pfull (group stages only)
    for (int u = cid; u < p.n_units; u += ncl) {
      const WUnit w = w_unit(p, u);
      for (int g = 0; g < p.ng; ++g) {
        mbar_wait(&pfull[ring.stage], (pph >> ring.stage) & 1u);
        pph ^= 1u << ring.stage;
#pragma unroll
        for (int rr = 0; rr < QM / (32 * CONV_WARPS); ++rr) {
          const uint32_t row = row0 + rr * 32 * CONV_WARPS;
          const uint4* src = reinterpret_cast<const uint4*>(sPK + ring.stage * PK_BYTES + row * 64);
          const uint32_t dst = smem_u32(sA + ring.stage * QA_BYTES + row * QK);
#pragma unroll
          for (int c = 0; c < 4; ++c) {
            const uint4 x = src[c];
            const uint4 lo = make_uint4((x.x << 4) & 0xF0F0F0F0u, (x.y << 4) & 0xF0F0F0F0u,
                                        (x.z << 4) & 0xF0F0F0F0u, (x.w << 4) & 0xF0F0F0F0u);
            const uint4 hi = make_uint4(x.x & 0xF0F0F0F0u, x.y & 0xF0F0F0F0u, x.z & 0xF0F0F0F0u, x.w & 0xF0F0F0F0u);
            const uint32_t d0 = dst + ((((uint32_t)(2 * c)) ^ (row & 7u)) << 4);
            const uint32_t d1 = dst + ((((uint32_t)(2 * c + 1)) ^ (row & 7u)) << 4);
            asm volatile("st.shared.v4.b32 [%0], {%1, %2, %3, %4};" ::"r"(d0), "r"(lo.x), "r"(lo.y), "r"(lo.z),
                         "r"(lo.w)
                         : "memory");
            asm volatile("st.shared.v4.b32 [%0], {%1, %2, %3, %4};" ::"r"(d1), "r"(hi.x), "r"(hi.y), "r"(hi.z),
                         "r"(hi.w)
                         : "memory");
          }
        }
        fence_proxy_async_smem();
        __syncwarp();
        if (lane == 0) mbar_arrive_cluster(&aready[ring.stage], 0);
        ring.advance();
      }
      if (w.cmc) {
        for (int mm = 1; mm < p.n_mod; ++mm)
          if ((w.mask >> mm) & 1u)
            for (int kb = 0; kb < p.cmc_kb; ++kb) ring.advance();
      }
    }
  } else {
    // ------------------------------------------------------------------ epilogue (both CTAs)
    const uint32_t e = warp - 2 - CONV_WARPS;           // 0..7
    const uint32_t q = warp & 3u;                       // TMEM lane quarter
    const int h = (int)(e >> 2);                        // column half: tokens [64h, 64h + 64)
    uint32_t acnt = 0;
    for (int u = cid; u < p.n_units; u += ncl) {
      const WUnit w = w_unit(p, u);
      const int j = w.nt * QUM + (int)rank * QM + (int)q * 32 + (int)lane;    // this lane's channel
      const bool jv = j < p.n;
      const float* scp = p.scales + (size_t)(jv ? j : 0) * p.ng;
      // ACC: exact int32 sums over the groups (the debug tap); else f32 promotion with the scale
      typename std::conditional<ACC, int, float>::type y[64];
#pragma unroll
      for (int k = 0; k < 64; ++k) y[k] = 0;
      float sc_next = jv ? __ldg(scp) : 0.f;
      for (int g = 0; g < p.ng; ++g) {
        const uint32_t buf = acnt % NBUF, bph = (acnt / NBUF) & 1u;
        ++acnt;
        const float sc = sc_next * 0.0625f;               // Delta_jg / 16 (exact)
        if (g + 1 < p.ng) sc_next = jv ? __ldg(scp + g + 1) : 0.f;
        mbar_wait(&tfull[buf], bph);
        tc_fence_after();
        const uint32_t taddr = tmem_base + ((q * 32u) << 16) + buf * QN + h * 64;
#pragma unroll
        for (int half = 0; half < 2; ++half) {
          uint32_t v[32];
          tmem_ld32(taddr + half * 32, v);
          tmem_wait_ld();
          if (half == 1) {
            tc_fence_before();
            __syncwarp();
            if (lane == 0) mbar_arrive_cluster(&tempty[buf], 0);
          }
#pragma unroll
          for (int k = 0; k < 32; ++k) {
            if (ACC) y[half * 32 + k] += ((int)v[k]) >> 4;
            else y[half * 32 + k] = fmaf((float)(int)v[k], sc, y[half * 32 + k]);
          }
        }
      }
      const int t0 = w.mt * QN + h * 64;
      if constexpr (ACC) {
        int32_t* out = static_cast<int32_t*>(p.out);
#pragma unroll
        for (int k = 0; k < 64; ++k)
          if (jv && t0 + k < p.T) out[(size_t)(t0 + k) * p.ld_out + j] = (int)y[k];
      } else {
#pragma unroll
        for (int k = 0; k < 64; ++k) y[k] *= (t0 + k < p.T) ? __ldg(p.dx + t0 + k) : 0.f;
        if (w.cmc) {
          const uint32_t buf = acnt % NBUF, bph = (acnt / NBUF) & 1u;
          ++acnt;
          mbar_wait(&tfull[buf], bph);
          tc_fence_after();
          const uint32_t taddr = tmem_base + ((q * 32u) << 16) + buf * QN + h * 64;
#pragma unroll
          for (int half = 0; half < 2; ++half) {
            uint32_t v[32];
            tmem_ld32(taddr + half * 32, v);
            tmem_wait_ld();
            if (half == 1) {
              tc_fence_before();
              __syncwarp();
              if (lane == 0) mbar_arrive_cluster(&tempty[buf], 0);
            }
#pragma unroll
            for (int k = 0; k < 32; ++k) y[half * 32 + k] += __uint_as_float(v[k]);
          }
        }
        float* out = static_cast<float*>(p.out);
#pragma unroll
        for (int k = 0; k < 64; ++k)
          if (jv && t0 + k < p.T) out[(size_t)(t0 + k) * p.ld_out + j] = y[k];
      }
    }
  }

  tc_fence_before();
  cluster_sync();
  if (warp == 1) {
    tc_fence_after();
    tmem_dealloc_2sm(tmem_base, 512);
  }
}
}  // namespace

cudaError_t launch_w4g_gemm(const W4gArgs& g, cudaStream_t st) {
  if (g.T <= 0 || g.n <= 0) return cudaSuccess;
  CUtensorMap tpk, tx, tl2, tz;
  bool ok = make_tmap_2d(&tpk, g.packed, CU_TENSOR_MAP_DATA_TYPE_UINT8, 1, g.n, g.d / 2, g.d / 2, QM, 64, false);
  ok &= make_tmap_2d(&tx, g.qx, CU_TENSOR_MAP_DATA_TYPE_UINT8, 1, g.T, g.d, g.d, QNH, 128, true);
  const bool cmc = !g.acc_mode && g.rpad > 0 && g.n_mod > 1;
  if (cmc) {
    const int64_t zc = (int64_t)(g.n_mod - 1) * 2 * g.rpad;
    ok &= make_tmap_2d(&tz, g.z, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, g.T, zc, zc, QNH, 64, true);
    ok &= make_tmap_2d(&tl2, g.l2t, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, (uint64_t)(g.n_mod - 1) * g.n, 2 * g.rpad,
                       2 * g.rpad, QM, 64, true);
  } else {
    tz = tx;
    tl2 = tx;
  }
  if (!ok) return cudaErrorInvalidValue;
  WParams p{};
  p.T = (int)g.T;
  p.n = (int)g.n;
  p.d = (int)g.d;
  p.ng = (int)(g.d / QK);
  p.num_m = (int)ceil_div(g.T, QN);
  p.num_n = (int)ceil_div(g.n, QUM);
  p.n_units = p.num_m * p.num_n;
  p.group = 16;
  p.n_mod = g.n_mod;
  p.rpad = cmc ? g.rpad : 0;
  p.cmc_kb = cmc ? (2 * g.rpad) / 64 : 0;
  p.tile_mask = g.tile_mask;
  p.dx = g.dx;
  p.scales = g.scales;
  p.out = g.out;
  p.ld_out = g.ld_out;
  p.acc_mode = g.acc_mode;
  const void* fn = g.acc_mode ? reinterpret_cast<const void*>(w4g_gemm_kernel<true>)
                              : reinterpret_cast<const void*>(w4g_gemm_kernel<false>);
  {
    cudaError_t e = set_max_dyn_smem(fn, SM_ALLOC);
    if (e != cudaSuccess) return e;
  }
  const int clusters = (int)std::min<int64_t>(p.n_units, num_sms() / 2);
  ProfScope ps_(g.acc_mode ? "gemm_w4g_acc" : "gemm_w4g", st);
  if (g.acc_mode)
    w4g_gemm_kernel<true><<<2 * clusters, QTHREADS, SM_ALLOC, st>>>(tpk, tx, tl2, tz, p);
  else
    w4g_gemm_kernel<false><<<2 * clusters, QTHREADS, SM_ALLOC, st>>>(tpk, tx, tl2, tz, p);
  return cudaGetLastError();
}

}  // namespace masq
