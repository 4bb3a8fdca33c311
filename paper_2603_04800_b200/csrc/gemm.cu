// gemm.cu — persistent, warp-specialised, CTA-pair (cta_group::2) tcgen05 GEMM for the MASQuant
// hot path (sm_100a).
//
// One kernel template serves four epilogues:
//   kModeFwd  A6+A7: acc = qx . qw^T (kind::i8, s32 in TMEM); y = acc * dx[t] * dw[j];
//             units that contain non-text tokens get the CMC term
//             y += [Zhi | Zlo] . [L2^T ; L2^T] (kind::f16, fp32) accumulated on top of y,
//             which the epilogue writes back into the same TMEM columns first.
//   kModeAcc  debug tap: raw int32 accumulators.
//   kModeLoss A8: rows arrive grouped by modality (each 256-row unit holds one modality m,
//             perm maps a grouped row to its token), acc = qx . Q(S_m W)^T and the epilogue
//             sums |acc*dx*dw_m - Yref[perm[row]]| -> per-(unit, CTA, warp) partials.
//   kModeRef  Yref = X . W (kind::f16 bf16 -> fp32), the loss target.
//   kModeAlpha N1 scale term: rows grouped as for the loss, acc = D . codes(Q(S_m W))^T
//             (kind::f16, both K-major; D = Ahat - X S^-1 as bf16), and the epilogue reduces
//             sum_j sign(E)_tj * dw_m[j] * acc_tj per row into per-(row, CTA column half) partials.
//   kModeAlphaI8 the same contraction on the int8 path: D quantized per row with the fixed step
//             Delta_t / 254 (|D| <= Delta_t / 2), B = the int8 weight codes themselves; the
//             epilogue applies the row step (dx = e_t).
//
// A cluster of two CTAs (one per SM of a TPC) computes a 256 x 256 output unit with
// tcgen05.mma.cta_group::2 (M = 256, N = 256): CTA r loads rows [128r, 128r+128) of the A tile
// and rows [128r, 128r+128) of the B tile (2-SM TMA, bytes counted on the leader's barrier), so
// each SM streams 32 KB per k-block instead of 48 KB for a 1-CTA 128 x 256 tile.  The leader
// (rank 0) issues the MMAs and multicasts its commits to both CTAs; each CTA's TMEM holds its
// 128 rows x 256 columns.
//
// Optionally (CL = 4, MASQ_GEMM_CL) a cluster holds two such pairs working on adjacent n-tiles of
// the same 256-row m-unit: the A tile is then identical for both pairs, and the CTA of rank r in
// each pair TMA-loads half of it (64 rows) multicast into the rank-r CTAs of both pairs, so each
// SM reads 24 KB per k-block from L2 instead of 32 KB.  Every stage slot is then shared by the
// two pairs: the MMA commits that free it multicast to all four CTAs (empty barrier count 2).
// Measured 2-8% slower than CL = 2 on this part (only 33 four-CTA clusters are co-resident:
// 132 SMs), so CL = 2 is the default.
//
// Work items: whole units in a raster order (groups of >= 16 n-tiles swept over all m-units), and
// for deep K (>= 64 k-blocks) a stream-K remainder: the units past the last full wave of pairs
// are cut along K into <= 4 segments over the pairs; a segment that does not start at k-block 0
// writes its raw accumulators to the workspace and releases a flag, and the unit's owner (the
// pair holding k-block 0) adds them before its normal epilogue.
//
// Roles per CTA (320 threads, 1 CTA per SM, grid = CL x min(#work items, active clusters)):
//   warp 0        : TMA producer  (all CTAs; 6-stage ring of 16 KB A + 16 KB B; one elect.sync lane
//                   issues each stage's copies)
//   warp 1        : TMEM allocation (all CTAs); in the leader the whole warp runs the MMA loop and
//                   one elect.sync lane issues the MMAs and commits (warp-uniform operands: no
//                   per-operand R2UR waterfalls, profiles/r02b_mma_issue.md)
//   warps 2..9    : epilogue      (warp w owns TMEM lane quarter w%4 and column half (w-2)/4:
//                                  tcgen05.ld 32x32b -> dequant -> swizzled smem -> TMA store)
// TMEM holds two 256-column accumulators (512 columns) so the epilogue of unit i overlaps the
// main loop of unit i+1.  The CMC k-blocks of unit i are inserted into the k-block stream of
// unit i+1 (after min(20, 5/8 of its main k-blocks)), by which time both epilogues have converted unit i's
// int32 accumulator to f32 in place; no extra TMEM columns and no Y round trip are needed.
#include <cstdio>
#include <mutex>
#include <vector>
#include <cstdlib>

#include "internal.h"
#include "sm100.cuh"

namespace masq {
using namespace sm100;

namespace {
constexpr int BM = 128;                              // rows per CTA
constexpr int UM = 2 * BM;                           // rows per cluster unit
constexpr int BN = kTileN;                           // columns per unit (MMA N)
constexpr int BNH = BN / 2;                          // B rows held by each CTA
constexpr int BKB = 128;                             // k-block bytes (128 int8 / 64 bf16)
#ifndef MASQ_GEMM_STAGES
#define MASQ_GEMM_STAGES 6
#endif
#ifndef MASQ_GEMM_NSTG
#define MASQ_GEMM_NSTG 1
#endif
constexpr int STAGES = MASQ_GEMM_STAGES;
// Y staging tiles per epilogue warp; measured (tools/ab_gemm.sh): 6 stages x 1 staging tile beats
// 5 x 2 and 4 x 2 by 3-8% on the int8 GEMMs (ring depth matters more), and per-lane direct
// global stores of Y (no staging, 7 stages) lose 25-30%
constexpr int NSTG = MASQ_GEMM_NSTG;
constexpr int A_BYTES = BM * BKB;
constexpr int B_BYTES = BNH * BKB;
constexpr int EPI_WARPS = 8;
constexpr int THREADS = 64 + 32 * EPI_WARPS;
constexpr int STG_BYTES = 32 * 32 * 4;               // one 32-row x 32-column f32 staging tile per warp
constexpr int SMEM_A = 0;
constexpr int SMEM_B = SMEM_A + STAGES * A_BYTES;
constexpr int SMEM_STG = SMEM_B + STAGES * B_BYTES;
constexpr int SMEM_BAR = SMEM_STG + EPI_WARPS * NSTG * STG_BYTES;
constexpr int SMEM_USED = SMEM_BAR + 256;
constexpr int SMEM_ALLOC = SMEM_USED + 1024;
constexpr int kCmcDefer = 4;
constexpr int kSkMinKb = 4;                          // stream-K: k-blocks per segment, at least
constexpr int kSkMaxSeg = 4;                         // stream-K: segments per remainder unit, at most
// stream-K only for deep K: the owner's fix-up (waiting for and adding up to 3 partial tiles) costs
// more than the tail it removes at 28 (int8) / 56 (bf16) k-blocks and pays at 148 / 296 (measured,
// tools/sk_ab.sh: d = 18944 forward -12% at 4k tokens, -4% at 16k; d = 3584 +4-15%)
constexpr int kSkMinUnitKb = 64;
}  // namespace
// MASQ_SK_MINKB (measurement knob): the minimum k-blocks per unit for the stream-K remainder
int gemm_sk_min_kb() {
  static const int v = [] {
    const char* e = getenv("MASQ_SK_MINKB");
    const int x = e ? atoi(e) : 0;
    return x > 0 ? x : kSkMinUnitKb;
  }();
  return v;
}
namespace {
constexpr int kRasterL2MB = 32;                      // L2 budget of a raster group's B panels
constexpr int kRasterGroupMin = 16;                  // n-tiles per raster group, at least
constexpr uint32_t IDESC_I8 = idesc_i8(UM, BN);
constexpr uint32_t IDESC_BF16 = idesc_bf16(UM, BN);
constexpr uint32_t IDESC_BF16_BMN = idesc_bf16(UM, BN) | (1u << 16);   // B MN-major (X.W reads W as stored)
static_assert(SMEM_ALLOC <= 232448, "shared memory budget");

struct Params {
  int mode;
  int T, n, d;
  int num_m, num_n, num_kb, n_units;  // num_m = 256-row units
  int num_np, n_items;                // n-tile groups of the cluster's pairs, work items (m-unit x group)
  int n_tiles128;                     // forward: entries of the 128-row modality mask
  int group;                          // raster: n-tiles per group swept over all m-units
  int n_mod;
  const float* dx;
  const float* dw;
  const uint32_t* tile_mask;   // fwd: modality bit set per 128-row tile; loss: modality per 256-row unit
  const int32_t* perm;         // loss: grouped row -> token (-1 = padding)
  int rpad, cmc_kb;
  int cmc_defer;                      // main k-blocks of unit i+1 issued before unit i's CMC k-blocks
  const float* yref;
  long long ld_ref;
  double* partials;            // loss: [n_units][2] (one per CTA of the pair)
  uint16_t* gsign;             // loss (optional, N1): bf16 sign(yq - yref) [T x n], 0 on padding rows
  float* apart;                // alpha: [T][apart_ld] per-row partials, this pass at apart_off
  int apart_ld, apart_off;
  const uint8_t* ids;          // fwd with fwd_loss: modality id per row (text rows feed the loss)
  int fwd_loss;                // fwd: sum |y - yref| over text rows into partials[unit][rank]
  int skip_m0;                 // loss: skip the text units (their loss comes from the forward)
  // stream-K remainder: work items n_full.. are the sk_R units past the last full wave, their
  // sk_R * num_kb k-blocks cut into ranges of sk_per over pairs 0 .. sk_pairs-1
  int n_full, sk_R, sk_per, sk_pairs;
  int policy;                  // X.W operand L2 hints: bit 0 A evict_first, bit 1 B evict_last
  uint32_t* sk_part;           // [pair][CTA][128 rows][256 cols] 32-bit partial accumulators
  uint32_t* sk_flag;           // [pair][CTA] partial posted (zeroed before the launch)
};

struct Unit {
  int mt, nt, m;
  uint32_t mask;
};

// work item u -> (m-unit, n-tile group); pair `pair` of the cluster takes n-tile NP * group + pair
// (an n-tile >= num_n runs the k-loop for its partner's shared A stages and stores nothing)
template <int NP>
__device__ __forceinline__ bool decode_unit(const Params& p, int u, int pair, Unit& w) {
  int ntp;
  if (p.group > 0) {
    // grouped raster: p.group consecutive n-tile groups swept over all m-units
    const int per_group = p.group * p.num_m;
    const int g = u / per_group;
    const int rem = u - g * per_group;
    const int nt0 = g * p.group;
    const int gsz = min(p.group, p.num_np - nt0);
    w.mt = rem / gsz;
    ntp = nt0 + (rem - w.mt * gsz);
  } else {
    // m-grouped raster (-p.group consecutive m-units swept over all n-tiles): the A panels of the
    // group stay in L2 while B streams once per group
    const int gm = -p.group;
    const int per_group = gm * p.num_np;
    const int g = u / per_group;
    const int rem = u - g * per_group;
    const int mt0 = g * gm;
    const int gsz = min(gm, p.num_m - mt0);
    ntp = rem / gsz;
    w.mt = mt0 + (rem - ntp * gsz);
  }
  w.nt = NP * ntp + pair;
  w.m = 0;
  if (p.mode == kModeLoss || p.mode == kModeAlpha || p.mode == kModeAlphaI8) {
    w.mask = p.tile_mask[w.mt];
    if (w.mask == 0xFFFFFFFFu) return false;
    if (p.skip_m0 && w.mask == 0u) return false;
    w.m = (int)w.mask;
  } else if (p.tile_mask) {
    const int t0 = 2 * w.mt;
    w.mask = p.tile_mask[t0] | (t0 + 1 < p.n_tiles128 ? p.tile_mask[t0 + 1] : 0u);
  } else {
    w.mask = 1u;
  }
  return true;
}
// a cluster's work item: a whole unit, or (stream-K) a k-block segment of a remainder unit
struct Item {
  int u;                       // work item index (decode_unit)
  int kb0, kb1;                // k-block range
  int kind;                    // 0 whole unit; 1 owner: adds the partials of pairs c_lo..c_hi; 2 partial
  int c_lo, c_hi;
};
constexpr int kItemWhole = 0, kItemOwner = 1, kItemPart = 2;
// item i of cluster cid: whole units cid, cid + ncl, ... below n_full, then the (<= 2) segments
// of its stream-K range [cid * sk_per, (cid + 1) * sk_per) of the remainder's k-blocks, the later
// segment first.  A unit's owner is the pair holding its LAST k-block; it waits for the partials
// of the lower pairs c_lo..cid-1 holding its earlier k-blocks.  A pair's partial segment comes
// before its owner segment and never waits, and lower cluster ids are dispatched first, so the
// waits form no cycle and no chain, even when only some clusters are resident (another kernel
// on another stream holding SMs).  Every role walks the same sequence.
__device__ __forceinline__ bool get_item(const Params& p, int cid, int ncl, int i, Item& it) {
  const int n1 = p.n_full > cid ? (p.n_full - cid + ncl - 1) / ncl : 0;
  if (i < n1) {
    it.u = cid + i * ncl;
    it.kb0 = 0;
    it.kb1 = p.num_kb;
    it.kind = kItemWhole;
    return true;
  }
  const int j = i - n1;
  if (p.sk_R == 0 || cid >= p.sk_pairs || j > 1) return false;
  const long long tot = (long long)p.sk_R * p.num_kb;
  const long long g0 = (long long)cid * p.sk_per;
  const long long g1 = g0 + p.sk_per < tot ? g0 + p.sk_per : tot;
  if (g0 >= g1) return false;
  // the range's segments in reverse order: a second segment (the start of the next unit, never
  // its last k-block: a partial) first, so partials are posted before any owner waits
  const int r0 = (int)(g0 / p.num_kb);
  const bool two = g1 > (long long)(r0 + 1) * p.num_kb;
  if (j > (two ? 1 : 0)) return false;
  const int r = r0 + ((two && j == 0) ? 1 : 0);
  const long long us = (long long)r * p.num_kb, ue = us + p.num_kb;
  const long long a = g0 > us ? g0 : us, b = g1 < ue ? g1 : ue;
  if (a >= b) return false;
  it.u = p.n_full + r;
  it.kb0 = (int)(a - us);
  it.kb1 = (int)(b - us);
  if (it.kb1 < p.num_kb) {
    it.kind = kItemPart;
  } else {
    const int c0 = (int)(us / p.sk_per);                 // the pair holding the unit's k-block 0
    it.kind = c0 < cid ? kItemOwner : kItemWhole;
    it.c_lo = c0;
    it.c_hi = cid - 1;
  }
  return true;
}

__device__ __forceinline__ bool unit_has_cmc(const Params& p, const Unit& w) {
  return p.mode == kModeFwd && p.rpad > 0 && (w.mask & ~1u) != 0u;
}

struct Ring {
  uint32_t stage = 0, phase = 0;
  __device__ __forceinline__ void advance() {
    if (++stage == STAGES) { stage = 0; phase ^= 1u; }
  }
};

template <int MODE, int CL>
__global__ void __cluster_dims__(CL, 1, 1) __launch_bounds__(THREADS, 1)
masq_gemm_kernel(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB,
                 const __grid_constant__ CUtensorMap tmY, const __grid_constant__ CUtensorMap tmZ,
                 const __grid_constant__ CUtensorMap tmL2, const Params p) {
  extern __shared__ uint8_t smem_raw[];
  const uint32_t raw = smem_u32(smem_raw);
  uint8_t* smem = smem_raw + (((raw + 1023u) & ~1023u) - raw);
  uint8_t* smA = smem + SMEM_A;
  uint8_t* smB = smem + SMEM_B;
  uint8_t* smS = smem + SMEM_STG;
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + SMEM_BAR);  // leader's is used
  uint64_t* empty = full + STAGES;      // all: the multicast MMA commits of every pair free the stage
  uint64_t* tfull = empty + STAGES;     // [2] both: accumulator ready
  uint64_t* tempty = tfull + 2;         // [2] leader's: both epilogues drained the buffer
  uint64_t* conv = tempty + 2;          // [2] leader's: both epilogues wrote y_base back (CMC)
  uint64_t* cmcd = conv + 2;            // [2] both: CMC accumulated
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(cmcd + 2);
  double* red = reinterpret_cast<double*>(tmem_slot + 2);   // [EPI_WARPS] loss partials of one unit

  const uint32_t warp = warp_id();
  const uint32_t lane = lane_id();
  constexpr int NP = CL / 2;             // CTA pairs per cluster
  const uint32_t crank = cluster_ctarank();
  const uint32_t rank = crank & 1u;      // rank within the pair
  const int pair = (int)(crank >> 1);
  const bool leader = rank == 0;
  const uint32_t lead_cta = crank & ~1u;
  const uint16_t pmask = (uint16_t)(0x3u << (2 * pair));          // this pair's CTAs
  const uint16_t all_mask = (uint16_t)((1u << CL) - 1u);
  const uint16_t a_mask = (uint16_t)(NP == 2 ? ((1u << rank) | (1u << (2 + rank))) : 0u);   // rank-r CTA of each pair
  const int cid = (int)cluster_id_x(), ncl = (int)ncluster_x();

  if (warp == 0 && lane == 0) {
    tma_prefetch(&tmA);
    tma_prefetch(&tmB);
    if (MODE != kModeLoss && MODE != kModeAlpha && MODE != kModeAlphaI8) tma_prefetch(&tmY);
    for (int i = 0; i < STAGES; ++i) { mbar_init(&full[i], 1); mbar_init(&empty[i], NP); }
    for (int i = 0; i < 2; ++i) {
      mbar_init(&tfull[i], 1);
      mbar_init(&tempty[i], 2 * EPI_WARPS);
      mbar_init(&conv[i], 2 * EPI_WARPS);
      mbar_init(&cmcd[i], 1);
    }
    fence_mbar_init();
  }
  if (warp == 1) tmem_alloc_2sm(tmem_slot, 512);
  tc_fence_before();
  cluster_sync();                       // barriers of all CTAs initialised before any remote use
  tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;
  pdl_wait();                           // the previous kernel's outputs (launch_k) ...
  pdl_trigger();                        // ... and this grid's TMEM held: the next kernel may start

  constexpr int KELEMS = (MODE == kModeRef || MODE == kModeAlpha) ? 64 : 128;
  constexpr bool kGrouped = MODE == kModeLoss || MODE == kModeAlpha || MODE == kModeAlphaI8;
  constexpr bool kAlpha = MODE == kModeAlpha || MODE == kModeAlphaI8;

  if (warp == 0) {
    {
      // ------------------------------------------------------------ TMA producer (all CTAs)
      // warp-wide loop (uniform state), one elected lane issues each stage's copies
      // L2 hints per mode and depth (p.policy, set on the host): B is re-read by every m-unit of the
      // raster group (evict_last); A evict_first only for X.W at d = 3584
      const uint64_t pol_a = (p.policy & 1) ? policy_evict_first() : policy_evict_normal();
      const uint64_t pol_b = (p.policy & 2) ? policy_evict_last() : policy_evict_normal();
      Ring ring;
      bool pend = false;
      Unit pu{};
      auto arm = [&]() {                  // elected lane: the leader's barrier expects the stage's bytes
        if (leader) mbar_expect_tx(&full[ring.stage], 2 * (A_BYTES + B_BYTES));
      };
      // A side: CL = 2 loads its 128 rows; CL = 4 loads half of them into both pairs (multicast)
      auto load_a = [&](const CUtensorMap* tm, int c0, int arow, uint64_t pol) {
        if (NP == 2) {
          tma_load_2d_2sm_mc_hint(smA + ring.stage * A_BYTES + pair * (A_BYTES / 2), tm, &full[ring.stage], c0,
                                  arow + pair * (BM / 2), a_mask, pol);
        } else {
          tma_load_2d_2sm_hint(smA + ring.stage * A_BYTES, tm, &full[ring.stage], c0, arow, pol);
        }
      };
      auto load_cmc = [&](const Unit& w) {
        for (int mm = 1; mm < p.n_mod; ++mm) {
          if (!((w.mask >> mm) & 1u)) continue;
          for (int kb = 0; kb < p.cmc_kb; ++kb) {
            mbar_wait(&empty[ring.stage], ring.phase ^ 1u);
            if (elect_one()) {
              arm();
              load_a(&tmZ, (mm - 1) * 2 * p.rpad + kb * 64, w.mt * UM + (int)rank * BM, policy_evict_normal());
              tma_load_2d_2sm(smB + ring.stage * B_BYTES, &tmL2, &full[ring.stage], kb * 64,
                              (mm - 1) * p.n + w.nt * BN + (int)rank * BNH);
            }
            __syncwarp();
            ring.advance();
          }
        }
      };
      Item it;
      for (int i = 0; get_item(p, cid, ncl, i, it); ++i) {
        Unit w;
        if (!decode_unit<NP>(p, it.u, pair, w)) continue;
        const int brow = (kGrouped ? w.m * p.n : 0) + w.nt * BN + (int)rank * BNH;
        const int arow = w.mt * UM + (int)rank * BM;
        const int defer_at = min(p.cmc_defer, it.kb1 - it.kb0 - 1);
        for (int kb = it.kb0; kb < it.kb1; ++kb) {
          if (pend && kb - it.kb0 == defer_at) { load_cmc(pu); pend = false; }
          mbar_wait(&empty[ring.stage], ring.phase ^ 1u);
          if (elect_one()) {
            arm();
            load_a(&tmA, kb * KELEMS, arow, pol_a);
            if (MODE == kModeRef) {
              // W [d x n] as stored: two 64(n) x 64(k) boxes -> MN-major B tile [n-half][k][64 n]
              tma_load_2d_2sm_hint(smB + ring.stage * B_BYTES, &tmB, &full[ring.stage], brow, kb * KELEMS, pol_b);
              tma_load_2d_2sm_hint(smB + ring.stage * B_BYTES + B_BYTES / 2, &tmB, &full[ring.stage], brow + 64,
                                   kb * KELEMS, pol_b);
            } else {
              tma_load_2d_2sm_hint(smB + ring.stage * B_BYTES, &tmB, &full[ring.stage], kb * KELEMS, brow, pol_b);
            }
          }
          __syncwarp();
          ring.advance();
        }
        if (it.kind != kItemPart && unit_has_cmc(p, w)) { pend = true; pu = w; }
      }
      if (pend) load_cmc(pu);
    }
    __syncwarp();
  } else if (warp == 1) {
    if (leader) {
      // ------------------------------------------------------------ MMA issuer (leader CTA)
      // the whole warp runs the loop (its state stays warp-uniform, in uniform registers); one
      // elected lane issues each k-block's MMAs and the commit that tracks them
      Ring ring;
      uint32_t local = 0, cmc_cnt[2] = {0u, 0u};   // conv/cmcd phases count CMC uses per buffer
      bool pend = false;
      Unit pu{};
      uint32_t pbuf = 0, pph = 0;
      const uint32_t a0 = smem_u32(smA), b0 = smem_u32(smB);
      auto issue_cmc = [&](const Unit& w, uint32_t buf, uint32_t ph) {
        mbar_wait(&conv[buf], ph);
        tc_fence_after();
        for (int mm = 1; mm < p.n_mod; ++mm) {
          if (!((w.mask >> mm) & 1u)) continue;
          for (int kb = 0; kb < p.cmc_kb; ++kb) {
            mbar_wait(&full[ring.stage], ring.phase);
            tc_fence_after();
            if (elect_one()) {
              const uint64_t ad = umma_desc_sw128(a0 + ring.stage * A_BYTES);
              const uint64_t bd = umma_desc_sw128(b0 + ring.stage * B_BYTES);
#pragma unroll
              for (int k = 0; k < 4; ++k)
                mma_bf16_2sm(tmem_base + buf * BN, ad + 2 * k, bd + 2 * k, IDESC_BF16, 1u);
              mma_commit_2sm(&empty[ring.stage], all_mask);
            }
            __syncwarp();
            ring.advance();
          }
        }
        if (elect_one()) mma_commit_2sm(&cmcd[buf], pmask);
        __syncwarp();
      };
      Item it;
      for (int i = 0; get_item(p, cid, ncl, i, it); ++i) {
        Unit w;
        if (!decode_unit<NP>(p, it.u, pair, w)) continue;
        const uint32_t buf = local & 1u, ph = (local >> 1) & 1u;
        ++local;
        mbar_wait(&tempty[buf], ph ^ 1u);
        tc_fence_after();
        const uint32_t dtm = tmem_base + buf * BN;
        const int defer_at = min(p.cmc_defer, it.kb1 - it.kb0 - 1);
        for (int kb = it.kb0; kb < it.kb1; ++kb) {
          if (pend && kb - it.kb0 == defer_at) { issue_cmc(pu, pbuf, pph); pend = false; }
          mbar_wait(&full[ring.stage], ring.phase);
          tc_fence_after();
          if (elect_one()) {
            // descriptor start addresses advance by 16-byte units: +32 B per K step (K-major),
            // +2048 B per 16 K rows (MN-major B of X.W)
            const uint64_t ad = umma_desc_sw128(a0 + ring.stage * A_BYTES);
            if (MODE == kModeRef) {
              const uint64_t bd = umma_desc_sw128_mn(b0 + ring.stage * B_BYTES, B_BYTES / 2);
#pragma unroll
              for (int k = 0; k < 4; ++k)
                mma_bf16_2sm(dtm, ad + 2 * k, bd + 128 * k, IDESC_BF16_BMN, (kb != it.kb0 || k != 0) ? 1u : 0u);
            } else {
              const uint64_t bd = umma_desc_sw128(b0 + ring.stage * B_BYTES);
#pragma unroll
              for (int k = 0; k < 4; ++k) {
                const uint32_t acc = (kb != it.kb0 || k != 0) ? 1u : 0u;
                if (MODE == kModeAlpha) mma_bf16_2sm(dtm, ad + 2 * k, bd + 2 * k, IDESC_BF16, acc);
                else mma_i8_2sm(dtm, ad + 2 * k, bd + 2 * k, IDESC_I8, acc);
              }
            }
            mma_commit_2sm(&empty[ring.stage], all_mask);
          }
          __syncwarp();
          ring.advance();
        }
        if (elect_one()) mma_commit_2sm(&tfull[buf], pmask);
        __syncwarp();
        if (it.kind != kItemPart && unit_has_cmc(p, w)) {
          pend = true;
          pu = w;
          pbuf = buf;
          pph = cmc_cnt[buf] & 1u;
          ++cmc_cnt[buf];
        }
      }
      if (pend) issue_cmc(pu, pbuf, pph);
    }
    __syncwarp();
  } else {
    // -------------------------------------------------------------- epilogue warps (both CTAs)
    const uint32_t q = warp & 3u;                       // TMEM lane quarter this warp may access
    const uint32_t ew = warp - 2u;                      // 0..7
    const int c0 = (int)(ew >> 2) * 4;                  // this warp's 4 column chunks: c0 .. c0+3
    uint8_t* const sb0 = smS + ew * NSTG * STG_BYTES;
    uint32_t nst = 0;                                   // Y chunks this warp has staged so far
    uint32_t local = 0, cmc_cnt[2] = {0u, 0u};
    const uint64_t pol_y = policy_evict_first();          // Y is written once, never re-read here
    Item it;
    for (int i = 0; get_item(p, cid, ncl, i, it); ++i) {
      Unit w;
      if (!decode_unit<NP>(p, it.u, pair, w)) continue;
      const bool real = w.nt < p.num_n;                  // false: partner-only n-tile past the edge
      const uint32_t buf = local & 1u, ph = (local >> 1) & 1u;
      ++local;
      const int row0 = w.mt * UM + (int)rank * BM + (int)q * 32;
      const int row = row0 + (int)lane;
      const int col_base = w.nt * BN;
      const int nch = max(0, min(4, (p.n - col_base) / 32 - c0));   // valid chunks of this warp
      // ---- prefetch (overlaps the main loop): row scale, this warp's 128 column scales (lane l
      //      holds dw[col_base + (c0+c)*32 + l]), and for the loss the source token of the row
      float dxr = 0.f;
      if (MODE != kModeRef && MODE != kModeAlpha && row < p.T) dxr = p.dx[row];
      float dwr[4] = {0.f, 0.f, 0.f, 0.f};
      if (MODE != kModeRef && MODE != kModeAcc) {
        const float* dwp = p.dw + (kGrouped ? (size_t)w.m * p.n : 0) + col_base + c0 * 32 + lane;
#pragma unroll
        for (int c = 0; c < 4; ++c)
          if (c < nch) dwr[c] = __ldg(dwp + c * 32);
      }
      int src = -1;
      if (MODE == kModeLoss && row < p.T) src = __ldg(p.perm + row);
      // forward + text loss: this row's Yref row (text rows only; their forward output is the
      // loss's quantized output, PAPER.md:69 with S_m = S_t)
      const bool tl = MODE == kModeFwd && p.fwd_loss && row < p.T && __ldg(p.ids + row) == 0;
      double tpart = 0.0;
      auto text_loss = [&](const uint32_t (&v)[32], int c) {
        const float4* r4 = reinterpret_cast<const float4*>(p.yref + (size_t)row * p.ld_ref + col_base + (c0 + c) * 32);
        float acc = 0.f;
#pragma unroll
        for (int j = 0; j < 8; ++j) {
          const float4 y = __ldg(r4 + j);
          acc += fabsf(__uint_as_float(v[4 * j + 0]) - y.x) + fabsf(__uint_as_float(v[4 * j + 1]) - y.y) +
                 fabsf(__uint_as_float(v[4 * j + 2]) - y.z) + fabsf(__uint_as_float(v[4 * j + 3]) - y.w);
        }
        tpart += (double)acc;
      };
      // loss: issue the first chunk's Yref loads now, under the main loop of this unit
      float4 ycur[8];
      if (MODE == kModeLoss && src >= 0 && nch > 0) {
        const float4* r4 = reinterpret_cast<const float4*>(p.yref + (size_t)src * p.ld_ref + col_base + c0 * 32);
#pragma unroll
        for (int j = 0; j < 8; ++j) ycur[j] = __ldg(r4 + j);
      }

      mbar_wait(&tfull[buf], ph);
      tc_fence_after();
      const uint32_t taddr = tmem_base + ((q * 32u) << 16) + buf * BN + c0 * 32;
      if (it.kind == kItemPart) {
        // stream-K partial: the raw 32-bit accumulators of this CTA's 128 rows go to the pair's
        // slot; the owner of the unit adds them (int32 exactly; f32 in a fixed order)
        // slot layout [warp][chunk][j][lane][4]: each 16-byte store of a warp covers 512
        // contiguous bytes (the owner reads it back the same way)
        uint4* dst = reinterpret_cast<uint4*>(p.sk_part) + ((size_t)(cid * 2 + (int)rank) * EPI_WARPS + ew) * 4 * 8 * 32 + lane;
#pragma unroll
        for (int c = 0; c < 4; ++c) {
          if (c >= nch) break;
          uint32_t v[32];
          tmem_ld32(taddr + c * 32, v);
          tmem_wait_ld();
#pragma unroll
          for (int j = 0; j < 8; ++j) dst[(c * 8 + j) * 32] = make_uint4(v[4 * j], v[4 * j + 1], v[4 * j + 2], v[4 * j + 3]);
        }
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive_cluster(&tempty[buf], lead_cta);
        __threadfence();
        asm volatile("bar.sync 1, %0;" ::"n"(32 * EPI_WARPS) : "memory");
        if (ew == 0 && lane == 0)
          asm volatile("st.release.gpu.global.u32 [%0], 1;" ::"l"(p.sk_flag + cid * 2 + (int)rank) : "memory");
        continue;
      }
      if (it.kind == kItemOwner) {                       // the later segments' partials are posted
        if (lane == 0)
          for (int pc = it.c_lo; pc <= it.c_hi; ++pc) {
            const uint32_t* fl = p.sk_flag + pc * 2 + (int)rank;
            uint32_t v = 0;
            const long long t0 = clock64();
            do {
              asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(fl) : "memory");
              if (clock64() - t0 > 8000000000LL) __trap();
            } while (v == 0u);
          }
        __syncwarp();
      }
      // owner: + the posted partials of pairs c_lo..c_hi (same rows / columns), in that order
      auto add_parts = [&](uint32_t (&v)[32], int c) {
        if (it.kind != kItemOwner) return;
        for (int pc = it.c_lo; pc <= it.c_hi; ++pc) {
          const uint4* s4 = reinterpret_cast<const uint4*>(p.sk_part) +
                            ((size_t)(pc * 2 + (int)rank) * EPI_WARPS + ew) * 4 * 8 * 32 + c * 8 * 32 + lane;
          uint4 pa[8];
#pragma unroll
          for (int j = 0; j < 8; ++j) pa[j] = __ldcg(s4 + j * 32);
#pragma unroll
          for (int j = 0; j < 8; ++j) {
            const uint4 a = pa[j];
            const uint32_t x[4] = {a.x, a.y, a.z, a.w};
#pragma unroll
            for (int e = 0; e < 4; ++e) {
              uint32_t& t = v[4 * j + e];
              t = MODE == kModeRef ? __float_as_uint(__uint_as_float(t) + __uint_as_float(x[e])) : t + x[e];
            }
          }
        }
      };

      auto dequant = [&](uint32_t (&v)[32], int c) {
#pragma unroll
        for (int i = 0; i < 32; ++i) {
          const float s = __shfl_sync(0xffffffffu, dwr[c], i);
          v[i] = __float_as_uint(__fmul_rn(__fmul_rn((float)(int)v[i], dxr), s));
        }
      };
      auto store_chunk = [&](const uint32_t (&v)[32], int c) {
        // NSTG staging tiles per warp, used round robin: before refilling one, the TMA store
        // issued NSTG chunks ago (its last user) must have finished reading it
        uint8_t* sb = sb0 + (nst % NSTG) * STG_BYTES;
        const uint32_t sbase = smem_u32(sb) + lane * 128u;
        if (nst >= (uint32_t)NSTG) {
          if (lane == 0) bulk_wait_read<NSTG - 1>();
          __syncwarp();
        }
#pragma unroll
        for (int j = 0; j < 8; ++j) {
          const uint32_t dst = sbase + (((uint32_t)j ^ (lane & 7u)) << 4);
          asm volatile("st.shared.v4.b32 [%0], {%1, %2, %3, %4};" ::"r"(dst), "r"(v[4 * j]), "r"(v[4 * j + 1]),
                       "r"(v[4 * j + 2]), "r"(v[4 * j + 3])
                       : "memory");
        }
        fence_proxy_async_smem();
        __syncwarp();
        if (lane == 0) {
          tma_store_2d_hint(&tmY, sb, col_base + (c0 + c) * 32, row0, pol_y);
          bulk_commit();
        }
        ++nst;
      };

      if (MODE == kModeFwd && unit_has_cmc(p, w)) {
        // 1) int32 -> y_base (f32) in place, 2) let the MMA accumulate CMC on top, 3) store.
#pragma unroll
        for (int c = 0; c < 4; ++c) {
          if (c >= nch) break;
          uint32_t v[32];
          tmem_ld32(taddr + c * 32, v);
          tmem_wait_ld();
          add_parts(v, c);
          dequant(v, c);
          tmem_st32(taddr + c * 32, v);
        }
        tmem_wait_st();
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive_cluster(&conv[buf], lead_cta);
        mbar_wait(&cmcd[buf], cmc_cnt[buf] & 1u);
        ++cmc_cnt[buf];
        tc_fence_after();
#pragma unroll
        for (int c = 0; c < 4; ++c) {
          if (c >= nch) break;
          uint32_t v[32];
          tmem_ld32(taddr + c * 32, v);
          tmem_wait_ld();
          if (tl) text_loss(v, c);
          store_chunk(v, c);
        }
      } else if (MODE == kModeLoss) {
        double part = 0.0;
#pragma unroll
        for (int c = 0; c < 4; ++c) {
          if (c >= nch) break;
          uint32_t v[32];
          tmem_ld32(taddr + c * 32, v);
          float4 ynext[8];
          if (src >= 0 && c + 1 < nch) {                 // prefetch the next chunk's Yref row segment
            const float4* r4 = reinterpret_cast<const float4*>(p.yref + (size_t)src * p.ld_ref + col_base +
                                                               (c0 + c + 1) * 32);
#pragma unroll
            for (int j = 0; j < 8; ++j) ynext[j] = __ldg(r4 + j);
          }
          tmem_wait_ld();
          dequant(v, c);
          if (p.gsign) {                                    // N1: G = sign(yq - yref), bf16, grouped rows
            uint32_t g[16];
#pragma unroll
            for (int k = 0; k < 16; ++k) {
              uint32_t lo = 0, hi = 0;
              if (src >= 0) {
                const float a0 = __uint_as_float(v[2 * k]) - (&ycur[k >> 1].x)[(2 * k) & 3];
                const float a1 = __uint_as_float(v[2 * k + 1]) - (&ycur[k >> 1].x)[(2 * k + 1) & 3];
                lo = a0 > 0.f ? 0x3F80u : (a0 < 0.f ? 0xBF80u : 0u);
                hi = a1 > 0.f ? 0x3F80u : (a1 < 0.f ? 0xBF80u : 0u);
              }
              g[k] = lo | (hi << 16);
            }
            uint4* gp = reinterpret_cast<uint4*>(p.gsign + (size_t)row * p.n + col_base + (c0 + c) * 32);
#pragma unroll
            for (int k = 0; k < 4; ++k) gp[k] = make_uint4(g[4 * k], g[4 * k + 1], g[4 * k + 2], g[4 * k + 3]);
          }
          if (src >= 0) {
            float acc = 0.f;
#pragma unroll
            for (int j = 0; j < 8; ++j) {
              acc += fabsf(__uint_as_float(v[4 * j + 0]) - ycur[j].x) +
                     fabsf(__uint_as_float(v[4 * j + 1]) - ycur[j].y) +
                     fabsf(__uint_as_float(v[4 * j + 2]) - ycur[j].z) +
                     fabsf(__uint_as_float(v[4 * j + 3]) - ycur[j].w);
            }
            part += (double)acc;
          }
#pragma unroll
          for (int j = 0; j < 8; ++j) ycur[j] = ynext[j];
        }
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) part += __shfl_xor_sync(0xffffffffu, part, o);
        // combine the 8 epilogue warps in a fixed order -> one partial per (unit, CTA)
        if (lane == 0) red[ew] = part;
        asm volatile("bar.sync 1, %0;" ::"n"(32 * EPI_WARPS) : "memory");
        if (ew == 0 && lane == 0 && real) {
          double tot = 0.0;
#pragma unroll
          for (int e = 0; e < EPI_WARPS; ++e) tot += red[e];
          p.partials[(size_t)(w.mt * p.num_n + w.nt) * 2 + rank] = tot;
        }
        asm volatile("bar.sync 1, %0;" ::"n"(32 * EPI_WARPS) : "memory");
      } else if (kAlpha) {
        float part = 0.f;
#pragma unroll
        for (int c = 0; c < 4; ++c) {
          if (c >= nch) break;
          uint32_t v[32];
          tmem_ld32(taddr + c * 32, v);
          const uint4* gp = reinterpret_cast<const uint4*>(p.gsign + (size_t)row * p.n + col_base + (c0 + c) * 32);
          uint4 g4[4];
#pragma unroll
          for (int k = 0; k < 4; ++k) g4[k] = __ldg(gp + k);
          tmem_wait_ld();
#pragma unroll
          for (int i = 0; i < 32; ++i) {
            const uint32_t gw = (&g4[i >> 3].x)[(i >> 1) & 3];
            const float g = __uint_as_float((i & 1) ? (gw & 0xFFFF0000u) : (gw << 16));   // +-1 or 0
            const float dws = __shfl_sync(0xffffffffu, dwr[c], i);
            const float av = MODE == kModeAlphaI8 ? (float)(int)v[i] : __uint_as_float(v[i]);
            part = fmaf(g * dws, av, part);
          }
        }
        if (MODE == kModeAlphaI8) part *= dxr;                      // the row step e_t
        if (row < p.T && real) p.apart[(size_t)row * p.apart_ld + p.apart_off + 2 * w.nt + (ew >> 2)] = part;
      } else {
#pragma unroll
        for (int c = 0; c < 4; ++c) {
          if (c >= nch) break;
          uint32_t v[32];
          tmem_ld32(taddr + c * 32, v);
          tmem_wait_ld();
          add_parts(v, c);
          if (MODE == kModeFwd) dequant(v, c);
          if (MODE == kModeFwd && tl) text_loss(v, c);
          store_chunk(v, c);
        }
      }
      if (MODE == kModeFwd && p.fwd_loss) {
        // fixed-order combine of the 8 epilogue warps -> one text-loss partial per (unit, CTA)
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) tpart += __shfl_xor_sync(0xffffffffu, tpart, o);
        if (lane == 0) red[ew] = tpart;
        asm volatile("bar.sync 1, %0;" ::"n"(32 * EPI_WARPS) : "memory");
        if (ew == 0 && lane == 0 && real) {
          double tot = 0.0;
#pragma unroll
          for (int e = 0; e < EPI_WARPS; ++e) tot += red[e];
          p.partials[(size_t)(w.mt * p.num_n + w.nt) * 2 + rank] = tot;
        }
        asm volatile("bar.sync 1, %0;" ::"n"(32 * EPI_WARPS) : "memory");
      }
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive_cluster(&tempty[buf], lead_cta);
    }
    if (lane == 0) bulk_wait<0>();
    __syncwarp();
  }

  tc_fence_before();
  cluster_sync();                       // all CTAs done with TMEM and with each other's barriers
  if (warp == 1) {
    tc_fence_after();
    tmem_dealloc_2sm(tmem_base, 512);
  }
}

// co-resident clusters of CL CTAs for this kernel (4-CTA clusters need two TPCs of one GPC, so
// fewer than #SMs / 4 may fit); cached per (mode, CL, device)
template <int MODE, int CL>
int active_clusters() {
  static int cached[16] = {0};
  int dev = 0;
  cudaGetDevice(&dev);
  int& c = cached[dev & 15];
  if (c == 0) {
    int n = 0;
    if (CL == 2) {
      n = num_sms() / 2;
    } else {
      cudaLaunchConfig_t cfg{};
      cfg.gridDim = dim3(CL * (num_sms() / CL));
      cfg.blockDim = dim3(THREADS);
      cfg.dynamicSmemBytes = SMEM_ALLOC;
      cudaLaunchAttribute at[1];
      at[0].id = cudaLaunchAttributeClusterDimension;
      at[0].val.clusterDim.x = CL;
      at[0].val.clusterDim.y = 1;
      at[0].val.clusterDim.z = 1;
      cfg.attrs = at;
      cfg.numAttrs = 1;
      if (cudaOccupancyMaxActiveClusters(&n, masq_gemm_kernel<MODE, CL>, &cfg) != cudaSuccess || n <= 0) {
        cudaGetLastError();
        n = num_sms() / CL;
      }
      n = std::min(n, num_sms() / CL);
    }
    c = n;
    if (getenv("MASQ_GEMM_VERBOSE")) fprintf(stderr, "[masq] gemm mode %d: %d active clusters of %d CTAs\n", MODE, n, CL);
  }
  return c;
}

template <int MODE, int CL>
cudaError_t launch_mode(const CUtensorMap& a, const CUtensorMap& b, const CUtensorMap& y, const CUtensorMap& z,
                        const CUtensorMap& l2, Params p, int max_cl, bool sk_ok, cudaStream_t st) {
  {
    cudaError_t e = set_max_dyn_smem(reinterpret_cast<const void*>(masq_gemm_kernel<MODE, CL>), SMEM_ALLOC);
    if (e != cudaSuccess) return e;
  }
  const int avail = std::min(max_cl, active_clusters<MODE, CL>());
  int clusters = (int)std::min<int64_t>(p.n_items, avail);
  p.n_full = p.n_items;
  p.sk_R = p.sk_per = p.sk_pairs = 0;
  if (sk_ok && CL == 2 && p.num_kb >= gemm_sk_min_kb()) {
    // stream-K remainder: when the units past the last full wave would leave more than a quarter
    // of the pairs idle, their k-blocks are spread over all pairs instead (segments of >= kSkMinKb)
    const int W = p.n_items / avail, R = p.n_items - W * avail;
    if (R > 0 && 4 * R <= 3 * avail) {
      // segment length: an even share of the remainder over all pairs, but at least kSkMinKb and
      // at most kSkMaxSeg segments per unit (the owner adds the others' partials one by one);
      // below one unit (a pair holds at most two segments)
      const long long tot = (long long)R * p.num_kb;
      long long per = ceil_div(tot, (long long)avail);
      per = std::max<long long>(per, kSkMinKb);
      per = std::max<long long>(per, ceil_div((long long)p.num_kb, (long long)kSkMaxSeg));
      if (per < p.num_kb) {
        p.sk_per = (int)per;
        p.sk_pairs = (int)ceil_div(tot, (long long)p.sk_per);
        p.sk_R = R;
        p.n_full = W * avail;
        clusters = avail;
        cudaError_t e = cudaMemsetAsync(p.sk_flag, 0, sizeof(uint32_t) * 2 * p.sk_pairs, st);
        if (e != cudaSuccess) return e;
      }
    }
  }
  static const char* const kNames[6] = {"gemm_fwd", "gemm_acc", "gemm_loss", "gemm_ref", "gemm_alpha",
                                        "gemm_alpha_i8"};
  ProfScope ps_(kNames[MODE], st);
  return launch_k(masq_gemm_kernel<MODE, CL>, dim3(CL * clusters), dim3(THREADS), SMEM_ALLOC, st, a, b, y, z, l2, p);
}

// MASQ_GEMM_CL (measurement knob): 2 = one CTA pair per cluster, 4 = two pairs sharing the A tile
int gemm_cluster_size(int mode) {
  static const int env = [] {
    const char* e = getenv("MASQ_GEMM_CL");
    return e ? atoi(e) : 0;
  }();
  if (env == 2 || env == 4) return env;
  // measured (tools/cl_ab.sh): 4-CTA clusters fit 33 per GPU (132 SMs) against 74 pairs (148 SMs);
  // the multicast saves L2 reads but the 16 idle SMs cost more (2-8% slower at every c3 shape)
  (void)mode;
  return 2;
}

template <int MODE>
cudaError_t launch_cl(const CUtensorMap& a, const CUtensorMap& b, const CUtensorMap& y, const CUtensorMap& z,
                      const CUtensorMap& l2, const Params& p, int cl, int max_pairs, bool sk_ok, cudaStream_t st) {
  if (cl == 4) return launch_mode<MODE, 4>(a, b, y, z, l2, p, std::max(1, max_pairs / 2), false, st);
  return launch_mode<MODE, 2>(a, b, y, z, l2, p, max_pairs, sk_ok, st);
}
}  // namespace

size_t gemm_sk_part_bytes() { return (size_t)(num_sms() / 2) * 2 * BM * BN * sizeof(uint32_t); }
size_t gemm_sk_flag_bytes() { return (size_t)(num_sms() / 2) * 2 * sizeof(uint32_t); }

int gemm_epilogue_warps() { return 2; }   // loss partial slots per unit (one per CTA of the pair)

cudaError_t set_max_dyn_smem(const void* func, int bytes) {
  struct Entry {
    const void* f;
    int dev, bytes;
  };
  static std::mutex mu;
  static std::vector<Entry> done;
  int dev = 0;
  cudaError_t e = cudaGetDevice(&dev);
  if (e != cudaSuccess) return e;
  std::lock_guard<std::mutex> lock(mu);
  for (const Entry& x : done)
    if (x.f == func && x.dev == dev && x.bytes >= bytes) return cudaSuccess;
  e = cudaFuncSetAttribute(func, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes);
  if (e == cudaSuccess) done.push_back({func, dev, bytes});
  return e;
}

bool pdl_enabled() {
  static const bool on = [] {
    const char* e = getenv("MASQ_PDL");
    return !(e && e[0] == '0');
  }();
  return on;
}

int num_sms() {
  static int n = 0;
  if (n == 0) {
    int dev = 0;
    cudaGetDevice(&dev);
    if (cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess || n <= 0) n = 148;
  }
  return n;
}

cudaError_t launch_gemm(const GemmArgs& g, cudaStream_t st) {
  if (g.T <= 0 || g.n <= 0) return cudaSuccess;
  CUtensorMap ta, tb, ty, tz, tl2;
  const bool bf = g.mode == kModeRef || g.mode == kModeAlpha;
  const int cl = gemm_cluster_size(g.mode);
  const int abox = cl == 4 ? BM / 2 : BM;              // A rows per TMA box (CL = 4: half, multicast)
  bool ok = true;
  if (g.mode == kModeAlpha) {
    ok &= make_tmap_2d(&ta, g.xbf, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, g.T, g.d, g.ld_x, abox, 64, true);
    ok &= make_tmap_2d(&tb, g.b, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, g.b_rows, g.d, g.d, BNH, 64, true);
  } else if (bf) {
    ok &= make_tmap_2d(&ta, g.xbf, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, g.T, g.d, g.ld_x, abox, 64, true);
    // B = W [d x n] row-major (MN-major for the MMA): box 64 (n) x 64 (k)
    ok &= make_tmap_2d(&tb, g.b, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, g.d, g.n, g.n, 64, 64, true);
  } else {
    ok &= make_tmap_2d(&ta, g.qx, CU_TENSOR_MAP_DATA_TYPE_UINT8, 1, g.T, g.d, g.d, abox, 128, true);
    ok &= make_tmap_2d(&tb, g.b, CU_TENSOR_MAP_DATA_TYPE_UINT8, 1, g.b_rows, g.d, g.d, BNH, 128, true);
  }
  if (g.mode != kModeLoss && g.mode != kModeAlpha && g.mode != kModeAlphaI8) {
    ok &= make_tmap_2d(&ty, g.out, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 4, g.T, g.n, g.ld_out, 32, 32, true);
  } else {
    ty = ta;
  }
  const bool cmc = g.mode == kModeFwd && g.rpad > 0;
  if (cmc) {
    const int64_t zc = (int64_t)(g.n_mod - 1) * 2 * g.rpad;
    ok &= make_tmap_2d(&tz, g.z, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, g.T, zc, zc, abox, 64, true);
    ok &= make_tmap_2d(&tl2, g.l2t, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, (uint64_t)(g.n_mod - 1) * g.n,
                       2 * g.rpad, 2 * g.rpad, BNH, 64, true);
  } else {
    tz = ta;
    tl2 = tb;
  }
  if (!ok) return cudaErrorInvalidValue;

  Params p{};
  p.mode = g.mode;
  p.T = (int)g.T;
  p.n = (int)g.n;
  p.d = (int)g.d;
  p.num_m = (int)ceil_div(g.T, UM);
  p.num_n = (int)ceil_div(g.n, BN);
  p.num_kb = (int)ceil_div(g.d, bf ? 64 : 128);
  p.n_units = p.num_m * p.num_n;
  p.num_np = (int)ceil_div(p.num_n, cl / 2);
  p.n_items = p.num_m * p.num_np;
  p.n_tiles128 = (int)ceil_div(g.T, kTileM);
  {
    static int env_group = -1000;
    if (env_group == -1000) {
      const char* e = getenv("MASQ_RASTER_GROUP");         // tuning knob (measurement only;
      env_group = e ? atoi(e) : 0;                          // < 0: m-grouped with -value m-units)
    }
    if (env_group != 0) {
      p.group = env_group;
    } else {
      // n-tiles per raster group: at least 16, more when more B panels (256 columns x K) fit an
      // L2 budget (the group's B stays resident while every m-unit streams past it; A is re-read
      // once per group); groups balanced in size.  Measured (tools/elect_ab.sh, l2mb_sweep.sh):
      // the budget helps the 18-tile qkv (one int8 group, +5%), fewer than 16 tiles per group
      // loses at the deep-K down projection even with less DRAM traffic.
      // MASQ_RASTER_L2MB: budget knob (measurement only)
      static const int env_mb = [] {
        const char* e = getenv("MASQ_RASTER_L2MB");
        return e ? atoi(e) : 0;
      }();
      const double budget = (env_mb > 0 ? env_mb : kRasterL2MB) * 1048576.0;
      const double panel = (double)BN * (double)g.d * (bf ? 2.0 : 1.0);
      const int gmax = std::max(kRasterGroupMin, (int)(budget / panel));
      const int ngroups = (int)ceil_div(p.num_n, gmax);
      p.group = (int)ceil_div(p.num_n, ngroups);
    }
    if (p.group > 0) p.group = std::max(1, (int)ceil_div(p.group, cl / 2));   // in n-tile groups of the cluster
  }
  p.n_mod = g.n_mod;
  p.dx = g.dx;
  p.dw = g.dw;
  p.tile_mask = g.tile_mask;
  p.perm = g.perm;
  p.rpad = cmc ? g.rpad : 0;
  p.cmc_kb = cmc ? (2 * g.rpad) / 64 : 0;
  {
    // MASQ_CMC_DEFER (measurement knob): k-blocks of the next unit before the CMC MMAs; -1 = half
    static const int env_def = [] {
      const char* e = getenv("MASQ_CMC_DEFER");
      return e ? atoi(e) : -1000;
    }();
    // measured (tools/defer_sweep.sh, r = 64): at K = 3584 (28 int8 k-blocks) 16-20 beats 4 by
    // 1.5-2% (the epilogue's dequant pass is done by then, so the MMA issuer does not wait on it)
    // and 24+ loses (the second epilogue pass then delays the unit after next); deep K is flat
    const int dflt = std::min(20, std::max(kCmcDefer, p.num_kb * 5 / 8));
    p.cmc_defer = env_def == -1000 ? dflt : (env_def < 0 ? p.num_kb / 2 : env_def);
  }
  p.yref = g.yref;
  p.ld_ref = g.ld_ref;
  p.partials = g.partials;
  p.gsign = g.gsign;
  p.apart = g.apart;
  p.apart_ld = g.apart_ld > 0 ? g.apart_ld : 2 * p.num_n;
  p.apart_off = g.apart_off;
  p.ids = g.ids;
  p.fwd_loss = g.fwd_loss;
  p.skip_m0 = g.skip_m0;
  // MASQ_GEMM_CLUSTERS (measurement knob): fewer persistent CTA pairs than SM pairs, leaving SMs
  // to HBM-bound kernels of another stream
  static const int env_cl = [] {
    const char* e = getenv("MASQ_GEMM_CLUSTERS");
    return e ? atoi(e) : 0;
  }();
  const int max_pairs = env_cl > 0 ? std::min(env_cl, num_sms() / 2) : num_sms() / 2;
  static const bool sk_off = [] {                          // MASQ_STREAMK=0: measurement switch
    const char* e = getenv("MASQ_STREAMK");
    return e && e[0] == '0';
  }();
  const bool sk_ok = !sk_off && g.sk_part != nullptr && g.sk_flag != nullptr &&
                     (g.mode == kModeFwd || g.mode == kModeAcc || g.mode == kModeRef);
  p.sk_part = g.sk_part;
  p.sk_flag = g.sk_flag;
  // X.W L2 hints: A (X) evict_first keeps the raster group's B panels (evict_last) resident at
  // d = 3584; at deep K the A tile of a k-block is re-read by the other units of the wave after
  // it was evicted: there A keeps the normal policy (tools/refpol_sweep.sh, profiles/
  // r02b_refpol_sweep.txt: down projection 1.578 -> 1.506 ms, DRAM reads 6.39 -> 4.00 GB)
  static const int env_pol = [] {                          // MASQ_REF_POLICY: measurement knob
    const char* e = getenv("MASQ_REF_POLICY");
    return e ? atoi(e) : -1;
  }();
  // int8 GEMMs: B evict_last, A normal measured best or tied at every c3 shape (1-1.5%,
  // tools/i8pol_sweep.sh, profiles/r02b_i8pol_sweep.txt)
  static const int env_pol8 = [] {                         // MASQ_I8_POLICY: the same for the int8 GEMMs
    const char* e = getenv("MASQ_I8_POLICY");
    return e ? atoi(e) : 2;
  }();
  if (g.mode == kModeRef) p.policy = env_pol >= 0 ? env_pol : (p.num_kb >= 128 ? 2 : 3);
  else p.policy = env_pol8;
  switch (g.mode) {
    case kModeFwd: return launch_cl<kModeFwd>(ta, tb, ty, tz, tl2, p, cl, max_pairs, sk_ok, st);
    case kModeAcc: return launch_cl<kModeAcc>(ta, tb, ty, tz, tl2, p, cl, max_pairs, sk_ok, st);
    case kModeLoss: return launch_cl<kModeLoss>(ta, tb, ty, tz, tl2, p, cl, max_pairs, sk_ok, st);
    case kModeRef: return launch_cl<kModeRef>(ta, tb, ty, tz, tl2, p, cl, max_pairs, sk_ok, st);
    case kModeAlpha: return launch_cl<kModeAlpha>(ta, tb, ty, tz, tl2, p, cl, max_pairs, sk_ok, st);
    case kModeAlphaI8: return launch_cl<kModeAlphaI8>(ta, tb, ty, tz, tl2, p, cl, max_pairs, sk_ok, st);
    default: return cudaErrorInvalidValue;
  }
}

}  // namespace masq
