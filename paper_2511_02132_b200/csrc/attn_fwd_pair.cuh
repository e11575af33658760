// attn_fwd_pair.cuh -- head dim 65..128 forward on CTA pairs: one 128-row
// query tile per SM, the two tiles of a work unit computed by cta_group::2
// (M = 256) tensor-core MMAs, S and P double-buffered in TMEM.
//
// Same math, work units, queues and scheduler as attn_fwd_sm100.cuh (PAPER.md
// eq:fa :149-155, the online-softmax fix-up :172); what changes is how the SM
// overlaps the two tensor-core contractions with the softmax.  In the
// two-tiles-per-CTA kernel TMEM holds S0 S1 O0 O1 (4 x 128 columns), P_t
// aliases S_t, and each tile's iteration is a chain
//     softmax_t(j) -> O_t += P_t V_j -> S_t = Q_t K_(j+1) -> softmax_t(j+1)
// whose tensor part (1024 cycles) plus latencies leaves the tensor pipe idle
// ~30% of the time.  Here an SM owns ONE 128-row tile
// and TMEM holds S0 S1 [0,256), P0 P1 [256,384) (bf16 pairs, 64 columns
// each) and O [384,512).  Block g of the CTA (counted over all its units)
// uses S_(g%2) and P_(g%2) and is the softmax work of warpgroup g%2, so each
// softmax warpgroup owns one S and one P buffer.  P does not alias S, so the
// MMA warp issues S(g+2) into S_(g%2) as soon as that warpgroup has LOADED
// S(g) into registers, long before O += P(g) V(g): the tensor pipe never
// waits for a softmax to finish before the next S, and a warpgroup finds
// S(g+2) ready when it comes back.  Two blocks' exps and row maxima overlap
// on every SMSP; the running max m is handed from block to block through
// shared memory right after each block's row max (so the next block's exps
// can start); each warpgroup keeps its own partial row sum l (rescaled when
// m moves) and the two partials are merged once per unit by the warpgroup
// that writes the output.  The same threshold-rescale rule, P and O += P V
// as the two-tiles-per-CTA kernel; only l's summation order differs.
//
// The unit's two tiles (query blocks 2u, 2u+1) run on the two SMs of a
// cluster as ONE M = 256 tile: the leader CTA's MMA warp issues
// tcgen05.mma.cta_group::2, each SM
// supplies its own 128 rows of Q (A) and HALF of the B operand -- keys
// 64r..64r+63 of K_j for S, head-dim columns 64r..64r+63 of V_j for O += P V
// -- so each SM loads and the tensor core reads half of every K/V block
// (ncu, C2: tensor-pipe SMEM wavefronts 26% of peak vs 50% in the two-tile
// kernel).  Both SMs' TMA loads signal the leader's barriers (cta_group::2
// TMA); both SMs' softmax warps publish P to the leader; the leader's commits
// multicast to both.  The leader's scheduler warp pops units from the
// mapping's queues (the plain per-unit queues: B * Hq * U entries).
//
// CTA layout (384 threads, one CTA per SM, persistent; clusters of 2):
//   warp 0      TMA producer: own Q tile; own halves of K and V into a K
//               ring and a V ring, in the order K0 K1 K2 V0 K3 V1 ...
//   warp 1      S issuer (leader CTA): S(g) into S_(g%2) as soon as K(g) has
//               landed and block g-2 has left the buffer; idle in the peer
//   warp 2      TMEM allocator (both CTAs) + (leader) work scheduler
//   warp 3      O += P V issuer (leader CTA): O += P(g) V(g) as soon as both
//               SMs published P(g); idle in the peer.  Two issuers, so an S
//               never queues behind an O += P V that waits for a softmax
//   warps 4-7   softmax + fix-up (+ epilogue) of the even key blocks
//   warps 8-11  the same for the odd key blocks (block parity counted over
//               all the CTA's blocks; the warpgroup of a unit's last block
//               writes its output)
#pragma once
#include "attn_fwd_sm100.cuh"

namespace attn {
namespace pairk {

constexpr int D = 128;
constexpr int kColP = 256;  // TMEM column of P0 (P1 at +64)
constexpr int kColO = 384;  // TMEM column of O
#ifndef ATTN_PAIR_RING
#define ATTN_PAIR_RING 5  // half-block slots per ring (K ring, V ring)
#endif
constexpr int kRing = ATTN_PAIR_RING;
constexpr int kSlots = 2 * kRing;
#define ATTN_PAIR_WGS 2  // softmax warpgroups taking alternate key blocks, one S and one P buffer each
#ifndef ATTN_PAIR_UNIT_SYNC
#define ATTN_PAIR_UNIT_SYNC 1  // both warpgroups meet after every unit
#endif
constexpr int kQBytes = kBlockM * D * 2;        // one 128-row Q tile (this SM's rows of the M = 256 A)
constexpr int kHalfBytes = kBlockN / 2 * D * 2;  // this SM's half of a K or V block (16 KB)
constexpr int kOffQ = 0;
constexpr int kOffKV = kQBytes;
constexpr int kOffCtrl = kOffKV + kSlots * kHalfBytes;
constexpr int kOffRows = kOffCtrl + 512;
constexpr int kSmemBytes = kOffRows + 3072 + 1024;  // control block + row state + alignment slack
static_assert(kSmemBytes <= 232448, "shared memory exceeds 227 KB");
static_assert(kSlots <= 12, "K/V rings deeper than the barrier arrays");

struct __align__(16) Ctrl {
  uint64_t sched_full[kSchedRing];
  uint64_t sched_empty[kSchedRing];
  uint64_t q_full, q_empty;     // q_full: leader's, both Q halves (tx); q_empty: each CTA
  uint64_t kv_full[12];         // leader's: both SMs' halves of a slot landed (tx); K ring, then V ring
  uint64_t kv_empty[12];        // each CTA: the pair's MMAs are done with the slot
  uint64_t s_full[2];           // each CTA: S(g) in S_(g%2)
  uint64_t s_free[2];           // leader's: both SMs' warpgroup g%2 have S(g) in registers (8 warps)
  uint64_t p_full[2][2];        // leader's: half h of P(g) in P_(g%2), both SMs (8 warps)
  uint64_t pv_done[4];          // each CTA: O += P V of block g done, [g & 3]
  uint64_t o_full;              // each CTA: the unit's last O += P V done
  uint64_t o_empty;             // leader's: both SMs' epilogues have read O
  uint64_t m_ready[2];          // softmax -> softmax: m after the CTA's g-th block in mrow[g & 1]
  uint64_t lpart_ready[2];      // softmax -> softmax: one warpgroup's partial (l, m) of the unit in lpart[k & 1]
  int4 entry[kSchedRing];
  uint32_t tmem_base;
};
// block-to-block softmax state of the 128 rows (after Ctrl in SMEM)
struct RowState {
  float mrow[2][kBlockM];      // m after the CTA's g-th block, [g & 1]
  float lpart[2][2][kBlockM];  // [k & 1][l or m]: the non-final warpgroup's row sum of unit k and its max
};

// key blocks query block qb needs (0 if the block does not exist)
template <bool kCausal>
__device__ __forceinline__ int tile_blocks(int qb, int nblk) {
  if (qb >= nblk) return 0;
  return kCausal ? qb + 1 : nblk;
}

template <bool kCausal>
__global__ void __launch_bounds__(kThreads, 1)
    attn_fwd_pair_kernel(const __grid_constant__ CUtensorMap tm_q, const __grid_constant__ CUtensorMap tm_k,
                         const __grid_constant__ CUtensorMap tm_v, const KernelParams p) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* q_smem = smem + kOffQ;
  uint8_t* kv_smem = smem + kOffKV;
  Ctrl* ctrl = reinterpret_cast<Ctrl*>(smem + kOffCtrl);
  RowState* rs = reinterpret_cast<RowState*>(smem + kOffRows);
  static_assert(sizeof(Ctrl) <= 512, "control block exceeds 512 B");
  static_assert(sizeof(RowState) <= 3072, "row state exceeds 3 KB");
  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;
  const uint32_t crank = ptx::cluster_ctarank();
  constexpr uint16_t kMask = 3;

  if (threadIdx.x == 0) {
    for (int i = 0; i < kSchedRing; ++i) {
      ptx::mbar_init(&ctrl->sched_full[i], 1);
      // both producers, the leader's two MMA issuers, both CTAs' softmax warps
      ptx::mbar_init(&ctrl->sched_empty[i], 2 + 2 + 2 * 4 * ATTN_PAIR_WGS);
    }
    ptx::mbar_init(&ctrl->q_full, 1);
    ptx::mbar_init(&ctrl->q_empty, 1);
    for (int i = 0; i < kSlots; ++i) {
      ptx::mbar_init(&ctrl->kv_full[i], 1);
      ptx::mbar_init(&ctrl->kv_empty[i], 1);
    }
    for (int s = 0; s < 2; ++s) {
      ptx::mbar_init(&ctrl->s_full[s], 1);
      ptx::mbar_init(&ctrl->s_free[s], 2 * 4);
      for (int h = 0; h < 2; ++h) ptx::mbar_init(&ctrl->p_full[s][h], 2 * 4);
    }
    for (int i = 0; i < 4; ++i) ptx::mbar_init(&ctrl->pv_done[i], 1);
    for (int i = 0; i < 2; ++i) {
      ptx::mbar_init(&ctrl->m_ready[i], 4);
      ptx::mbar_init(&ctrl->lpart_ready[i], 4);
    }
    ptx::mbar_init(&ctrl->o_full, 1);
    ptx::mbar_init(&ctrl->o_empty, 2 * 4);
    ptx::fence_barrier_init();
  }
  if (warp == 0 && lane == 0) {
    ptx::tma_prefetch_desc(&tm_q);
    ptx::tma_prefetch_desc(&tm_k);
    ptx::tma_prefetch_desc(&tm_v);
  }
  if (warp == 2) {  // one warp of each CTA of the pair
    ptx::tmem_alloc_2(&ctrl->tmem_base, kTmemCols);
    ptx::tmem_relinquish_2();
  }
  ptx::tc_fence_before();
  __syncthreads();
  ptx::cluster_sync();  // peer barriers initialised before any remote arrive / TMA signal
  ptx::tc_fence_after();

  // ring position -> (slot, parity) of the K ring (which = 0) or the V ring
  struct Ring {
    int stage = 0;
    uint32_t phase = 0;
    __device__ __forceinline__ void advance() {
      if (++stage == kRing) { stage = 0; phase ^= 1; }
    }
  };

  if (warp == 0) {
    // ------------------------------------------------------------ TMA producer
    if (ATTN_SETMAXNREG) ptx::setmaxnreg_dec<kOtherRegs>();
    if (lane == 0) {
      SchedReader<2, Ctrl> sr;
      const uint64_t pol_q = ptx::policy_evict_first();
      const uint64_t pol_kv = ptx::policy_evict_normal();
      const uint32_t lead_q_full = ptx::mapa_shared(ptx::smem_u32(&ctrl->q_full), 0);
      uint32_t q_phase = 0;
      Ring rk, rv;
      int seq = 0;
      ATTN_CYC_DECL()
      // this SM's half of block j of K (which = 0: keys 64r..64r+63, all 128
      // columns, two 8 KB swizzle-atom columns) or V (which = 1: all 128 keys,
      // columns 64r..64r+63, one 16 KB atom column); the leader's kv_full
      // counts both SMs' bytes
      auto load_kv = [&](int j, int which, int kvbh) {
        Ring& rr = which ? rv : rk;
        const int slot = which * kRing + rr.stage;
        ATTN_CYC_START();
        ptx::mbar_wait(&ctrl->kv_empty[slot], rr.phase ^ 1);
        ATTN_CYC_ADD(0);
        ATTN_CYC_COUNT(7);
        if (crank == 0) ptx::mbar_arrive_expect_tx(&ctrl->kv_full[slot], 2 * kHalfBytes);
        const uint32_t full = ptx::mapa_shared(ptx::smem_u32(&ctrl->kv_full[slot]), 0);
        uint8_t* dst = kv_smem + slot * kHalfBytes;
        if (which == 0) {
#pragma unroll
          for (int c = 0; c < D / 64; ++c)
            ptx::tma_load_3d_2sm(dst + c * (kBlockN / 2) * 128, &tm_k, full, c * 64,
                                 j * kBlockN + (int)crank * (kBlockN / 2), kvbh, pol_kv);
        } else {
          ptx::tma_load_3d_2sm(dst, &tm_v, full, (int)crank * 64, j * kBlockN, kvbh, pol_kv);
        }
        rr.advance();
      };
      while (true) {
        const int4 e = sr.next(ctrl, true);
        if (!e.w) break;
        const int b = e.x, h = e.y, u = e.z;
        const int qb = 2 * u + (int)crank;
        const int n = max(tile_blocks<kCausal>(2 * u, p.nblk), tile_blocks<kCausal>(2 * u + 1, p.nblk));
        if (p.trace && crank == 0 && !ATTN_INSTRUMENTED) {
          const long long id = ((long long)b * p.Hq + h) * p.U + u;
          if (id < p.trace_cap) {
            const int sm = (int)ptx::smid();
            attn_trace_rec_t r;
            r.b = b; r.h = h; r.unit = u; r.smid = sm;
            r.domain = (sm < p.n_smid) ? (int)p.domain_of_smid[sm] : 0;
            r.queue = (e.w >> 1) & 63; r.stolen = (e.w >> 7) & 1; r.seq = seq;
            r.t_pop_ns = ptx::globaltimer();
            p.trace[id] = r;
          }
        }
        ++seq;
        // Q: both SMs always load their tile (rows >= N, or a whole missing
        // tile of a ragged unit, are zero-filled and their output discarded)
        ATTN_CYC_START();
        ptx::mbar_wait(&ctrl->q_empty, q_phase ^ 1);
        ATTN_CYC_ADD(2);
        q_phase ^= 1;
        if (crank == 0) ptx::mbar_arrive_expect_tx(&ctrl->q_full, 2 * kQBytes);
#pragma unroll
        for (int c = 0; c < D / 64; ++c)
          ptx::tma_load_3d_2sm(q_smem + c * kBlockM * 128, &tm_q, lead_q_full, c * 64, qb * kBlockM, b * p.Hq + h,
                               pol_q);
        const int kvbh = b * p.Hkv + h / p.G;
        // K runs two blocks ahead of V (the order the two issuers need them)
        for (int j = 0; j < min(2, n); ++j) load_kv(j, 0, kvbh);
        for (int j = 0; j < n; ++j) {
          if (j + 2 < n) load_kv(j + 2, 0, kvbh);
          load_kv(j, 1, kvbh);
        }
      }
      // drain: every slot's last fill released by the leader's commits, so no
      // multicast arrive is still in flight towards this CTA when it exits
      for (int i = 0; i < kRing; ++i) {
        ptx::mbar_wait(&ctrl->kv_empty[rk.stage], rk.phase ^ 1);
        ptx::mbar_wait(&ctrl->kv_empty[kRing + rv.stage], rv.phase ^ 1);
        rk.advance();
        rv.advance();
      }
      ATTN_CYC_WRITE12(p.trace, 0)
    }
  } else if (warp == 1 || warp == 3) {
    // ------------------------------------------------------- MMA issuers (leader)
    if (ATTN_SETMAXNREG) ptx::setmaxnreg_dec<kOtherRegs>();
    if (crank == 0) {
      const uint32_t tmem = *reinterpret_cast<volatile uint32_t*>(&ctrl->tmem_base);
      SchedReader<2, Ctrl> sr;
      Ring rr;
      uint32_t gb = 0;  // the pair's key blocks over all units
      ATTN_CYC_DECL()
      auto take = [&]() {
        const int slot = (warp == 1 ? 0 : kRing) + rr.stage;
        ptx::mbar_wait(&ctrl->kv_full[slot], rr.phase);
        rr.advance();
        return slot;
      };
      if (warp == 1) {
        // S(g) = Q K(g)^T into S_(g%2): M = 256 (both SMs' Q), N = 128 (keys
        // 0-63 from the leader's half slot, 64-127 from the peer's)
        constexpr uint32_t idesc_s = ptx::idesc_bf16_f32(2 * kBlockM, kBlockN, 0, 0);
        const uint64_t dq = ptx::smem_desc_sw128(ptx::smem_u32(q_smem), 16, 1024);
        const uint64_t dkv0 = ptx::smem_desc_sw128(ptx::smem_u32(kv_smem), 16, 1024);
        uint32_t q_phase = 0;
        while (true) {
          const int4 e = sr.next(ctrl, false);
          __syncwarp();
          if (lane == 0) sr.release_prev(ctrl);
          if (!e.w) break;
          const int u = e.z;
          const int n = max(tile_blocks<kCausal>(2 * u, p.nblk), tile_blocks<kCausal>(2 * u + 1, p.nblk));
          ptx::mbar_wait(&ctrl->q_full, q_phase);
          q_phase ^= 1;
          for (int j = 0; j < n; ++j, ++gb) {
            ATTN_CYC_START();
            // S_(g%2) free once both SMs' warpgroup g%2 loaded S(g-2)
            if (gb >= 2) ptx::mbar_wait_cluster(&ctrl->s_free[gb & 1], ((gb >> 1) - 1) & 1);
            ATTN_CYC_ADD(3);
            const int sk = take();
            ATTN_CYC_ADD(0);
            ATTN_CYC_COUNT(7);
            ptx::tc_fence_after();
            if (ptx::elect_one_sync()) {
              const uint64_t dk = dkv0 + (uint64_t)((sk * kHalfBytes) >> 4);
              const uint32_t d_tmem = tmem + 128u * (gb & 1);
#pragma unroll
              for (int k = 0; k < D / 16; ++k) {
                const uint32_t oq = ((k >> 2) * (kBlockM * 128) + (k & 3) * 32) >> 4;
                const uint32_t ok = ((k >> 2) * (kBlockN / 2 * 128) + (k & 3) * 32) >> 4;
                ptx::mma_ss_2(d_tmem, dq + oq, dk + ok, idesc_s, k > 0 ? 1u : 0u);
              }
              ptx::mma_commit_2mc(&ctrl->s_full[gb & 1], kMask);
              if (j == n - 1) ptx::mma_commit_2mc(&ctrl->q_empty, kMask);  // last read of this Q pair
              ptx::mma_commit_2mc(&ctrl->kv_empty[sk], kMask);
            }
            __syncwarp();
            ATTN_CYC_ADD(4);
          }
        }
        ATTN_CYC_WRITE12(p.trace, 1)
      } else {
        // O (+)= P(g) V(g): A = P_(g%2) from each SM's TMEM, B = V with its
        // 128 head-dim columns split between the SMs; P published in halves
        constexpr uint32_t idesc_o = ptx::idesc_bf16_f32(2 * kBlockM, D, 0, 1);
        const uint64_t dv0 = ptx::smem_desc_sw128(ptx::smem_u32(kv_smem), kBlockN * 128, 1024);
        uint32_t units_done = 0;  // units whose epilogue frees O (o_empty phases)
        while (true) {
          const int4 e = sr.next(ctrl, false);
          __syncwarp();
          if (lane == 0) sr.release_prev(ctrl);
          if (!e.w) break;
          const int u = e.z;
          const int n = max(tile_blocks<kCausal>(2 * u, p.nblk), tile_blocks<kCausal>(2 * u + 1, p.nblk));
          for (int j = 0; j < n; ++j, ++gb) {
            ATTN_CYC_START();
            const int sv = take();
            ATTN_CYC_ADD(0);
            if (j == 0 && units_done > 0)  // O of the previous unit read by both SMs' epilogues
              ptx::mbar_wait_cluster(&ctrl->o_empty, (units_done - 1) & 1);
            ATTN_CYC_ADD(5);
            ATTN_CYC_COUNT(7);
            const uint64_t dv = dv0 + (uint64_t)((sv * kHalfBytes) >> 4);
            const uint32_t a_tmem = tmem + kColP + 64u * (gb & 1);
#pragma unroll
            for (int h = 0; h < 2; ++h) {
              ATTN_CYC_START();
              ptx::mbar_wait_cluster(&ctrl->p_full[gb & 1][h], (gb >> 1) & 1);
              ATTN_CYC_ADD(1);
              ptx::tc_fence_after();
              if (ptx::elect_one_sync()) {
#pragma unroll
                for (int k = h * 4; k < (h + 1) * 4; ++k)
                  ptx::mma_ts_2(tmem + kColO, a_tmem + k * 8, dv + (uint64_t)((k * 16 * 128) >> 4), idesc_o,
                                (j > 0 || k > 0) ? 1u : 0u);
              }
              __syncwarp();
              ATTN_CYC_ADD(2);
            }
            if (ptx::elect_one_sync()) {
              ptx::mma_commit_2mc(&ctrl->pv_done[gb & 3], kMask);
              if (j == n - 1) ptx::mma_commit_2mc(&ctrl->o_full, kMask);
              ptx::mma_commit_2mc(&ctrl->kv_empty[sv], kMask);
            }
            __syncwarp();
          }
          ++units_done;
        }
        ATTN_CYC_WRITE12(p.trace, 3)
      }
    }
  } else if (warp == 2) {
    // --------------------------------------------------------------- scheduler
    if (ATTN_SETMAXNREG) ptx::setmaxnreg_dec<kOtherRegs>();
    if (lane == 0 && crank == 0) run_scheduler<2>(p, ctrl);  // the leader schedules for the pair
  } else if (warp >= 4 && warp < 4 + 4 * ATTN_PAIR_WGS) {
    // ------------------------------------------------ softmax / fix-up / epilogue
    if (ATTN_SETMAXNREG) ptx::setmaxnreg_inc<kSoftmaxRegs>();
    const uint32_t tmem = *reinterpret_cast<volatile uint32_t*>(&ctrl->tmem_base);
    const uint32_t wg = (uint32_t)(warp - 4) >> 2;  // this warpgroup takes the CTA's blocks g with g % 2 == wg
    const int quarter = warp & 3;            // TMEM lane quarter this warp may access
    const int row = quarter * 32 + lane;     // row within the 128-row tile
    const uint32_t trow = tmem + ((uint32_t)(quarter * 32) << 16);
    const float c = p.scale_log2;
    SchedReader<2, Ctrl> sr;
    uint32_t o_phase = 0;
    uint32_t g = 0;                     // the CTA's blocks over all units (both warpgroups count all)
    uint32_t un = 0;                    // units with two or more blocks so far (lpart hand-overs)
    float l_w = 0.f, m_w = -INFINITY;   // this warpgroup's partial row sum and the max it is relative to
    ATTN_CYC_DECL()
    while (true) {
      const int4 e = sr.next(ctrl, false);
      __syncwarp();
      if (lane == 0) sr.release_prev(ctrl);
      if (!e.w) break;
      const int u = e.z;
      const int qb = 2 * u + (int)crank;
      const int nt = tile_blocks<kCausal>(qb, p.nblk);  // key blocks this tile needs
      // key blocks the pair computes (M = 256 MMAs cover both tiles): the
      // longer tile's; this tile's blocks j >= nt are fully masked (P = 0)
      const int n = max(tile_blocks<kCausal>(2 * u, p.nblk), tile_blocks<kCausal>(2 * u + 1, p.nblk));
      const int last_blk = p.nblk - 1;
      const int tail_lim = p.N - last_blk * kBlockN - 1;  // last block: local key k visible iff k <= tail_lim
      for (int j = 0; j < n; ++j, ++g) {
        if ((g & 1u) != wg) continue;  // the other warpgroup's block
        ATTN_CYC_START();
        ptx::mbar_wait(&ctrl->s_full[wg], (g >> 1) & 1);
        ATTN_CYC_ADD(0);
        ATTN_CYC_COUNT(7);
        ptx::tc_fence_after();
        uint32_t r[kBlockN];
        ptx::tmem_ld128(trow + 128u * wg, r);
        // S(g) is in registers: the MMA warp may compute S(g+2) into S_wg
        ptx::tc_fence_before();
        __syncwarp();
        if (lane == 0) ptx::mbar_arrive_cluster_relaxed(ptx::mapa_shared(ptx::smem_u32(&ctrl->s_free[wg]), 0));
        // visible local keys are k <= lim: causal diagonal block (key <= query)
        // and/or the ragged last key block (key < N)
        int lim = kBlockN;
        if (kCausal && j == qb) lim = row;
        if (j == last_blk && tail_lim < lim) lim = tail_lim;
        if (j >= nt) lim = -1;  // a block only the other tile needs: m, l and O unchanged
        const bool diag = __any_sync(0xffffffffu, lim < kBlockN - 1);
        if (diag) {
#pragma unroll
          for (int k = 0; k < kBlockN; ++k)
            if (k > lim) r[k] = 0xff800000u;
        }
        float mq[4] = {-INFINITY, -INFINITY, -INFINITY, -INFINITY};
#pragma unroll
        for (int k = 0; k < kBlockN; k += 8) {
#pragma unroll
          for (int g4 = 0; g4 < 4; ++g4)
            mq[g4] = fmaxf(mq[g4], fmaxf(__uint_as_float(r[k + 2 * g4]), __uint_as_float(r[k + 2 * g4 + 1])));
        }
        const float mx = fmaxf(fmaxf(mq[0], mq[1]), fmaxf(mq[2], mq[3]));
        // the previous block's m (the other warpgroup's), also waited for at
        // j == 0 so that its reader has consumed mrow[g & 1] before it is rewritten
        float m = -INFINITY;
        ATTN_CYC_ADD(1);
        if (g > 0) {
          ptx::mbar_wait(&ctrl->m_ready[(g - 1) & 1], ((g - 1) >> 1) & 1);
          m = rs->mrow[(g - 1) & 1][row];
        }
        float m_use, alpha;
        bool rescale = false;
        if (j == 0) {
          m_use = mx;
          alpha = 0.f;
        } else if ((mx - m) * c > kRescaleThreshold) {
          m_use = mx;
          alpha = ptx::ex2((m - mx) * c);
          rescale = true;
        } else {
          m_use = m;
          alpha = 1.f;
        }
        ATTN_CYC_ADD(2);
        rs->mrow[g & 1][row] = m_use;
        __syncwarp();
        if (lane == 0) ptx::mbar_arrive(&ctrl->m_ready[g & 1]);
        if (__any_sync(0xffffffffu, rescale)) {
          // fix-up: O *= exp2((m_old - m_new) c) once O += P V
          // of the previous block is complete.  pv_done[(g-1) & 3] has
          // completed (g-1) >> 2 or (g-1) >> 2 + 1 phases: block g-5 is done
          // (the other warpgroup waited for it before storing P(g-3), and it
          // published m(g-1) after that), and P(g) is not out yet.
          const uint32_t g1 = g - 1;
          ptx::mbar_wait(&ctrl->pv_done[g1 & 3], (g1 >> 2) & 1);
          ptx::tc_fence_after();
#pragma unroll
          for (int cc = 0; cc < D; cc += 32) {
            uint32_t o[32];
            ptx::tmem_ld32(trow + kColO + cc, o);
#pragma unroll
            for (int k = 0; k < 32; ++k) o[k] = __float_as_uint(__uint_as_float(o[k]) * alpha);
            ptx::tmem_st32(trow + kColO + cc, o);
          }
        }
        const float neg = -m_use * c;
        // P = exp2(S c - m c): MUFU.EX2 for most pairs, the FMA-pipe polynomial
        // for every kEmuPeriod-th pair; published in two halves so O += P V
        // starts on the first while the second is computed.
        float2 sq[4] = {make_float2(0.f, 0.f), make_float2(0.f, 0.f), make_float2(0.f, 0.f),
                        make_float2(0.f, 0.f)};
        auto exp_block = [&](auto mask_tag) {
#pragma unroll
          for (int h = 0; h < 2; ++h) {
#pragma unroll
            for (int k = h * 64; k < (h + 1) * 64; k += 2) {
              const float2 x = ptx::ffma2(make_float2(__uint_as_float(r[k]), __uint_as_float(r[k + 1])), c, neg);
              float2 pr;
              constexpr int kEP = emu_period<D>();
              if (kEP > 0 && ((k >> 1) % (kEP > 0 ? kEP : 1)) == kEP - 1) {
                pr = ptx::ex2_poly2(x);
              } else {
                pr.x = ptx::ex2(x.x);
                pr.y = ptx::ex2(x.y);
              }
              if constexpr (decltype(mask_tag)::value) {
                pr.x = (k <= lim) ? pr.x : 0.f;
                pr.y = (k + 1 <= lim) ? pr.y : 0.f;
              }
              sq[(k >> 1) & 3] = ptx::fadd2(sq[(k >> 1) & 3], pr);
              r[k >> 1] = ptx::pack_bf16(pr.x, pr.y);
            }
#ifdef ATTN_CYCLES_EXP
            ATTN_CYC_ADD(3);
#endif
            if (h == 0 && g >= 2) {
              // P_wg is free once O += P(g-2) V is done (pv_done[(g-2) & 3]:
              // block g-6 is done, this warpgroup waited for it before P(g-4))
              const uint32_t g2 = g - 2;
              ptx::mbar_wait(&ctrl->pv_done[g2 & 3], (g2 >> 2) & 1);
              ptx::tc_fence_after();
            }
            ptx::tmem_st32(trow + kColP + 64u * wg + h * 32, r + h * 32);
            ptx::tmem_wait_st();
#ifdef ATTN_CYCLES_EXP
            ATTN_CYC_ADD(5);
#endif
            ptx::tc_fence_before();
            __syncwarp();
            if (lane == 0) ptx::mbar_arrive_cluster_relaxed(ptx::mapa_shared(ptx::smem_u32(&ctrl->p_full[wg][h]), 0));
#ifdef ATTN_CYCLES_EXP
            ATTN_CYC_ADD(6);
#endif
          }
        };
        if (diag) exp_block(std::true_type{});
        else exp_block(std::false_type{});
        const float2 s01 = ptx::fadd2(sq[0], sq[1]), s23 = ptx::fadd2(sq[2], sq[3]);
        const float2 s4 = ptx::fadd2(s01, s23);
        const float sum = s4.x + s4.y;
        // this warpgroup's partial row sum, relative to m_use (rescaled when
        // m moved since its previous block of the unit)
        ATTN_CYC_ADD(3);
        if (j < 2) {
          l_w = sum;
        } else if (m_use != m_w) {
          l_w = fmaf(l_w, ptx::ex2((m_w - m_use) * c), sum);
        } else {
          l_w += sum;
        }
        m_w = m_use;
        if (j == n - 2) {  // this warpgroup's last block of the unit: hand its partial to the other
          rs->lpart[un & 1][0][row] = l_w;
          rs->lpart[un & 1][1][row] = m_w;
          __syncwarp();
          if (lane == 0) ptx::mbar_arrive(&ctrl->lpart_ready[un & 1]);
        }
        ATTN_CYC_ADD(4);
        if (j != n - 1) continue;
        float l = l_w;  // merge the other warpgroup's partial (l_o, m_o <= m_use)
        if (n > 1) {
          ptx::mbar_wait(&ctrl->lpart_ready[un & 1], (un >> 1) & 1);
          const float l_o = rs->lpart[un & 1][0][row], m_o = rs->lpart[un & 1][1][row];
          l = (m_o == m_use) ? l_w + l_o : fmaf(l_o, ptx::ex2((m_o - m_use) * c), l_w);
        }
        // ---- epilogue (the unit's last block is this warpgroup's): O / l -> bf16 -> global
        ATTN_CYC_TIMED(6, ptx::mbar_wait(&ctrl->o_full, o_phase));
        ptx::tc_fence_after();
        const float inv_l = 1.f / l;
        const int hh = e.y;
        if (p.lse != nullptr && nt > 0 && qb * kBlockM + row < p.N)  // lse = scale*m + ln(l)
          p.lse[(long long)(e.x * p.Hq + hh) * p.N + qb * kBlockM + row] =
              (m_use * c + __log2f(l)) * 0.6931471805599453f;
        const long long orow =
            ((long long)(e.x * p.Hq_out + p.h_off + hh) * p.N + (long long)qb * kBlockM + row) * p.d_real;
        // rows >= N (ragged last query block) store nothing but still join the
        // warp-wide TMEM loads; padded head-dim columns are not stored
        const int ncol = (nt > 0 && qb * kBlockM + row < p.N) ? p.d_real : 0;
#pragma unroll
        for (int cc = 0; cc < D; cc += 32) {
          uint32_t o[32];
          ptx::tmem_ld32(trow + kColO + cc, o);
          uint32_t pk[16];
#pragma unroll
          for (int k = 0; k < 16; ++k)
            pk[k] = ptx::pack_bf16(__uint_as_float(o[2 * k]) * inv_l, __uint_as_float(o[2 * k + 1]) * inv_l);
          if (cc == D - 32) {  // every column of O is in registers: the next unit may overwrite it
            ptx::tc_fence_before();
            __syncwarp();
            if (lane == 0) ptx::mbar_arrive_cluster_relaxed(ptx::mapa_shared(ptx::smem_u32(&ctrl->o_empty), 0));
          }
          for (int di = 0; di < p.n_dst; ++di) {  // replicated output: one store per destination
            uint4* dst = reinterpret_cast<uint4*>(p.o_dst[di] + orow);
#pragma unroll
            for (int k = 0; k < 4; ++k) {
              if (cc + 8 * k >= ncol) break;
              dst[cc / 8 + k] = make_uint4(pk[4 * k], pk[4 * k + 1], pk[4 * k + 2], pk[4 * k + 3]);
            }
          }
        }
        ATTN_CYC_ADD(5);
      }
      // both warpgroups count the o_full phases of every unit, and the
      // partial-sum hand-overs (units of two or more blocks)
      o_phase ^= 1;
      if (n > 1) ++un;
      if (ATTN_PAIR_UNIT_SYNC) ptx::named_bar_sync(1, 32 * 4 * ATTN_PAIR_WGS);
    }
    ATTN_CYC_WRITE12(p.trace, warp)
  }

  ptx::tc_fence_before();
  __syncthreads();
  ptx::cluster_sync();  // no remote SMEM access / pair MMA may target an exited CTA
  if (warp == 2) {
    ptx::tc_fence_after();
    ptx::tmem_dealloc_2(*reinterpret_cast<volatile uint32_t*>(&ctrl->tmem_base), kTmemCols);
  }
}

}  // namespace pairk
}  // namespace attn
