// attn_fwd_n256_sm100.cuh -- head dim 128 forward with 256-key blocks, one
// 128-row query tile at a time and P in its own TMEM columns.
//
// Same math as attn_fwd_sm100.cuh (PAPER.md eq:fa, lines 149-155; the online
// softmax fix-up) and the same scheduler, units and mappings
// (a unit is still two 128-row query blocks; this kernel runs them one after
// the other).  What changes is the pipeline ("256-key
// kernel"):
//
//   TMEM (512 columns): S [0,256) fp32 | O [256,384) fp32 | P [384,512) bf16 pairs
//
// Because P does not alias S, the MMA warp issues S(j+1) = Q K_{j+1}^T as soon
// as every softmax warp has loaded S(j) into registers (s_free), so the softmax
// warps run block after block without waiting for the PV -> S -> softmax round
// trip that bounds the two-tile kernel.  Eight softmax warps cover 128 rows x
// 256 keys: warps 4-7 keys [0,128), warps 8-11 keys [128,256) of the same rows
// (warp w and w+4 share TMEM lane quarter w%4 and exchange row maxima through
// shared memory).  K/V stream through separate rings of 128-key slots (K runs
// one block ahead of V).
//
// Warp roles (384 threads, one CTA per SM, persistent):
//   warp 0  TMA producer     warp 1  MMA issuer     warp 2  scheduler + TMEM
//   warp 3  idle             warps 4-11  softmax / fix-up / epilogue
#pragma once
#include "attn_fwd_sm100.cuh"

namespace attn {
namespace n256 {

constexpr int kD = 128;
constexpr int kBN = 256;       // keys per block
constexpr int kSlotKeys = 128; // keys per K/V ring slot
#ifndef N256_K_STAGES
#define N256_K_STAGES 4
#endif
#ifndef N256_EMU_PERIOD
#define N256_EMU_PERIOD 8
#endif
#ifndef N256_MAX_CHAINS
#define N256_MAX_CHAINS 4
#endif
constexpr int kKStages = N256_K_STAGES;  // K ring slots (128 keys each): K(j+1) loads while S(j) runs
constexpr int kVStages = 2;    // V ring slots
constexpr int kTileBytes = 128 * kD * 2;  // a 128-row Q tile or a 128-key K/V slot (32 KB)
constexpr int kOffQ = 0;
constexpr int kOffK = kOffQ + kTileBytes;
constexpr int kOffV = kOffK + kKStages * kTileBytes;
constexpr int kOffCtrl = kOffV + kVStages * kTileBytes;
constexpr uint32_t kColS = 0, kColO = 256, kColP = 384;

struct __align__(16) Ctrl {
  uint64_t sched_full[kSchedRing];
  uint64_t sched_empty[kSchedRing];
  uint64_t q_full, q_empty;
  uint64_t k_full[kKStages], k_empty[kKStages];
  uint64_t v_full[kVStages], v_empty[kVStages];
  uint64_t s_ready, s_free;   // MMA -> softmax: S(j) in TMEM; softmax -> MMA: S(j) in registers
  uint64_t p_ready[2];        // softmax -> MMA: [0] P keys 0-127 stored and O fixed up by all 8 warps; [1] P keys 128-255
  uint64_t p_free, o_ready;   // MMA -> softmax: PV(j) complete (not the tile's last) / the tile's last PV complete
  int4 entry[kSchedRing];
  uint32_t tmem_base;
};
struct Red {
  float mx[4][2][2][32];  // [quarter][key half][parity][lane] partial row max (and, after a tile, row sum)
};
constexpr int kCtrlBytes = 1024;
// With four K slots the tiles fill 224 KB and ctrl + Red the last 3 KB of the
// 227 KB limit: no slack for aligning the dynamic SMEM base, which the kernel
// then requires to be 1024-byte aligned (it traps otherwise).
constexpr int kSlack = (kOffCtrl + kCtrlBytes + (int)sizeof(Red) + 1024 <= 232448) ? 1024 : 0;
constexpr int kSmemBytes = kOffCtrl + kCtrlBytes + (int)sizeof(Red) + kSlack;

template <bool kCausal>
__device__ __forceinline__ int tile_blocks(int qb, int nblk256) {
  return kCausal ? (qb >> 1) + 1 : nblk256;  // key block j holds keys [256j, 256j+256)
}

template <bool kCausal>
__global__ void __launch_bounds__(kThreads, 1)
    attn_fwd_n256_kernel(const __grid_constant__ CUtensorMap tm_q, const __grid_constant__ CUtensorMap tm_k,
                         const __grid_constant__ CUtensorMap tm_v, const KernelParams p) {
  static_assert(kSplit == 1, "the 256-key kernel assumes 8 softmax warps");
  static_assert(sizeof(Ctrl) <= kCtrlBytes, "control block exceeds 1 KB");
  static_assert(kSmemBytes <= 232448, "shared memory exceeds 227 KB");
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  if (kSlack == 0 && smem != smem_raw) __trap();
  uint8_t* q_smem = smem + kOffQ;
  uint8_t* k_smem = smem + kOffK;
  uint8_t* v_smem = smem + kOffV;
  Ctrl* ctrl = reinterpret_cast<Ctrl*>(smem + kOffCtrl);
  Red* red = reinterpret_cast<Red*>(smem + kOffCtrl + kCtrlBytes);
  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;
  const int nblk256 = (p.N + kBN - 1) / kBN;

  if (threadIdx.x == 0) {
    for (int i = 0; i < kSchedRing; ++i) {
      ptx::mbar_init(&ctrl->sched_full[i], 1);
      ptx::mbar_init(&ctrl->sched_empty[i], 2 + 8);  // TMA + MMA + 8 softmax warps
    }
    ptx::mbar_init(&ctrl->q_full, 1);
    ptx::mbar_init(&ctrl->q_empty, 1);
    for (int i = 0; i < kKStages; ++i) { ptx::mbar_init(&ctrl->k_full[i], 1); ptx::mbar_init(&ctrl->k_empty[i], 1); }
    for (int i = 0; i < kVStages; ++i) { ptx::mbar_init(&ctrl->v_full[i], 1); ptx::mbar_init(&ctrl->v_empty[i], 1); }
    ptx::mbar_init(&ctrl->s_ready, 1);
    ptx::mbar_init(&ctrl->s_free, 8);
    ptx::mbar_init(&ctrl->p_ready[0], 8);
    ptx::mbar_init(&ctrl->p_ready[1], 4);
    ptx::mbar_init(&ctrl->p_free, 1);
    ptx::mbar_init(&ctrl->o_ready, 1);
    ptx::fence_barrier_init();
  }
  if (warp == 0 && lane == 0) {
    ptx::tma_prefetch_desc(&tm_q);
    ptx::tma_prefetch_desc(&tm_k);
    ptx::tma_prefetch_desc(&tm_v);
  }
  if (warp == 2) {
    ptx::tmem_alloc(&ctrl->tmem_base, kTmemCols);
    ptx::tmem_relinquish();
  }
  ptx::tc_fence_before();
  __syncthreads();
  ptx::tc_fence_after();

  if (warp == 0) {
    // ------------------------------------------------------------ TMA producer
    // Per tile: Q, then K(0), K(1), V(0), K(2), V(1), ... (K one block ahead of
    // V, across tile and unit boundaries), each block as two 128-key slots.
    if (ATTN_SETMAXNREG) ptx::setmaxnreg_dec<kOtherRegs>();
    if (lane == 0) {
      SchedReader<1, Ctrl> sr;
      const uint64_t pol_q = ptx::policy_evict_first();
      const uint64_t pol_kv = ptx::policy_evict_normal();
      uint32_t q_phase = 0;
      int ks = 0, vs = 0;
      uint32_t kph = 0, vph = 0;
      auto load_blk = [&](bool is_k, int kvbh, int j) {
#pragma unroll
        for (int hh = 0; hh < 2; ++hh) {
          int& st = is_k ? ks : vs;
          uint32_t& ph = is_k ? kph : vph;
          uint64_t* full = is_k ? &ctrl->k_full[st] : &ctrl->v_full[st];
          ptx::mbar_wait(is_k ? &ctrl->k_empty[st] : &ctrl->v_empty[st], ph ^ 1);
#ifdef N256_DEBUG_NO_KV
          if (j >= 1) {  // bandwidth probe: reuse whatever is in the slot (wrong numerics)
            ptx::mbar_arrive(full);
            if (++st == (is_k ? kKStages : kVStages)) { st = 0; ph ^= 1; }
            continue;
          }
#endif
          ptx::mbar_arrive_expect_tx(full, kTileBytes);
          uint8_t* dst = (is_k ? k_smem : v_smem) + st * kTileBytes;
#pragma unroll
          for (int c = 0; c < 2; ++c)
            ptx::tma_load_3d(dst + c * kSlotKeys * 128, is_k ? (const void*)&tm_k : (const void*)&tm_v, full, c * 64,
                             j * kBN + hh * kSlotKeys, kvbh, pol_kv);
          if (++st == (is_k ? kKStages : kVStages)) { st = 0; ph ^= 1; }
        }
      };
      bool pend = false;
      int pend_bh = 0, pend_j = 0;
      while (true) {
        const int4 e = sr.next(ctrl, true);
        if (!e.w) break;
        const int b = e.x, h = e.y, u = e.z;
        const int kvbh = b * p.Hkv + h / p.G;
        for (int t = 0; t < 2; ++t) {
          const int qb = 2 * u + t;
          if (qb >= p.nblk) break;
          const int n = tile_blocks<kCausal>(qb, nblk256);
          ptx::mbar_wait(&ctrl->q_empty, q_phase ^ 1);
          q_phase ^= 1;
          ptx::mbar_arrive_expect_tx(&ctrl->q_full, kTileBytes);
#pragma unroll
          for (int c = 0; c < 2; ++c)
            ptx::tma_load_3d(q_smem + c * 128 * 128, &tm_q, &ctrl->q_full, c * 64, qb * 128, b * p.Hq + h, pol_q);
          for (int j = 0; j < n; ++j) {
            load_blk(true, kvbh, j);
            if (pend) load_blk(false, pend_bh, pend_j);
            pend = true;
            pend_bh = kvbh;
            pend_j = j;
          }
        }
      }
      if (pend) load_blk(false, pend_bh, pend_j);
    }
  } else if (warp == 1) {
    // -------------------------------------------------------------- MMA issuer
    if (ATTN_SETMAXNREG) ptx::setmaxnreg_dec<kOtherRegs>();
    const uint32_t tmem = *reinterpret_cast<volatile uint32_t*>(&ctrl->tmem_base);
    SchedReader<1, Ctrl> sr;
    constexpr uint32_t idesc_s = ptx::idesc_bf16_f32(128, kSlotKeys, 0, 0);
    constexpr uint32_t idesc_o = ptx::idesc_bf16_f32(128, kD, 0, 1);
    const uint64_t dq = ptx::smem_desc_sw128(ptx::smem_u32(q_smem), 16, 1024);
    const uint64_t dk0 = ptx::smem_desc_sw128(ptx::smem_u32(k_smem), 16, 1024);
    const uint64_t dv0 = ptx::smem_desc_sw128(ptx::smem_u32(v_smem), kSlotKeys * 128, 1024);
    uint32_t q_phase = 0, sf_phase = 0, p_phase = 0;
    int s_used = 0;
    int ks = 0, vs = 0;
    uint32_t kph = 0, vph = 0;
    auto take_k = [&]() {
      const int s = ks;
      ptx::mbar_wait(&ctrl->k_full[s], kph);
      if (++ks == kKStages) { ks = 0; kph ^= 1; }
      return s;
    };
    auto take_v = [&]() {
      const int s = vs;
      ptx::mbar_wait(&ctrl->v_full[s], vph);
      if (++vs == kVStages) { vs = 0; vph ^= 1; }
      return s;
    };
    // S = Q K^T over the block's two 128-key slots, into S columns [0,128) and [128,256)
    auto issue_s = [&](int k0, int k1, bool q_last) {
      const int s0 = take_k(), s1 = take_k();
      (void)k0; (void)k1;
      if (s_used) {
        ptx::mbar_wait(&ctrl->s_free, sf_phase);
        sf_phase ^= 1;
      }
      s_used = 1;
      ptx::tc_fence_after();
      if (ptx::elect_one_sync()) {
#pragma unroll
        for (int hh = 0; hh < 2; ++hh) {
          const uint64_t dk = dk0 + (uint64_t)(((hh ? s1 : s0) * kTileBytes) >> 4);
#pragma unroll
          for (int k = 0; k < kD / 16; ++k) {
            const uint32_t oq = ((k >> 2) * (128 * 128) + (k & 3) * 32) >> 4;
            const uint32_t ok = ((k >> 2) * (kSlotKeys * 128) + (k & 3) * 32) >> 4;
            ptx::mma_ss(tmem + kColS + hh * kSlotKeys, dq + oq, dk + ok, idesc_s, k > 0 ? 1u : 0u);
          }
        }
        ptx::mma_commit(&ctrl->s_ready);
        ptx::mma_commit(&ctrl->k_empty[s0]);
        ptx::mma_commit(&ctrl->k_empty[s1]);
        if (q_last) ptx::mma_commit(&ctrl->q_empty);
      }
      __syncwarp();
    };
#ifdef N256_TIMELINE
    long long* tl = (p.trace && blockIdx.x == 0) ? reinterpret_cast<long long*>(p.trace) : nullptr;
    if (tl && lane == 0) tl[1000] = clock64();
    int tile_no = 0;
#define N256_MSTAMP(i) if (tl && lane == 0 && tile_no == 0 && j < 64) tl[j * 8 + (i)] = clock64();
#else
#define N256_MSTAMP(i)
#endif
    while (true) {
      const int4 e = sr.next(ctrl, false);
      __syncwarp();
      if (lane == 0) sr.release_prev(ctrl);
      if (!e.w) break;
      const int u = e.z;
      for (int t = 0; t < 2; ++t) {
        const int qb = 2 * u + t;
        if (qb >= p.nblk) break;
        const int n = tile_blocks<kCausal>(qb, nblk256);
        ptx::mbar_wait(&ctrl->q_full, q_phase);
        q_phase ^= 1;
        issue_s(0, 0, n == 1);
        for (int j = 0; j < n; ++j) {
          N256_MSTAMP(0);
          if (j + 1 < n) issue_s(0, 0, j + 2 == n);
          N256_MSTAMP(1);
          // O += P V(j): keys 0-127 once every warp has published (p_ready[0]),
          // keys 128-255 once the second key half is stored (p_ready[1])
#pragma unroll
          for (int hh = 0; hh < 2; ++hh) {
            const int sv = take_v();
            ptx::mbar_wait(&ctrl->p_ready[hh], p_phase);
            N256_MSTAMP(2 + hh);
            ptx::tc_fence_after();
            if (ptx::elect_one_sync()) {
              const uint64_t dv = dv0 + (uint64_t)((sv * kTileBytes) >> 4);
#pragma unroll
              for (int kk = 0; kk < kSlotKeys / 16; ++kk) {
                const int k = hh * (kSlotKeys / 16) + kk;
                ptx::mma_ts(tmem + kColO, tmem + kColP + k * 8, dv + (uint64_t)((kk * 16 * 128) >> 4), idesc_o,
                            (j > 0 || k > 0) ? 1u : 0u);
              }
              if (hh == 1) ptx::mma_commit(j + 1 < n ? &ctrl->p_free : &ctrl->o_ready);
              ptx::mma_commit(&ctrl->v_empty[sv]);
            }
            __syncwarp();
          }
          p_phase ^= 1;
        }
#ifdef N256_TIMELINE
        ++tile_no;
#endif
      }
    }
  } else if (warp == 2) {
    // --------------------------------------------------------------- scheduler
    if (ATTN_SETMAXNREG) ptx::setmaxnreg_dec<kOtherRegs>();
    if (lane == 0) run_scheduler<1>(p, ctrl);
  } else if (warp >= 4) {
    // ------------------------------------------------ softmax / fix-up / epilogue
    if (ATTN_SETMAXNREG) ptx::setmaxnreg_inc<kSoftmaxRegs>();
    const uint32_t tmem = *reinterpret_cast<volatile uint32_t*>(&ctrl->tmem_base);
    const int hf = (warp - 4) >> 2;    // key half of every block: keys [128 hf, 128 hf + 128)
    const int quarter = warp & 3;      // TMEM lane quarter
    const int row = quarter * 32 + lane;
    const uint32_t trow = tmem + ((uint32_t)(quarter * 32) << 16);
    const uint32_t colS = kColS + hf * 128, colP = kColP + hf * 64, colO = kColO + hf * 64;
    const uint32_t bar_id = 1 + quarter;  // named barrier of warps (quarter, quarter + 4)
    const float c = p.scale_log2;
    SchedReader<1, Ctrl> sr;
    uint32_t s_phase = 0, o_phase = 0, pf_phase = 0, blk = 0;
#ifdef N256_TIMELINE
    int tile_no = 0;
#define N256_SSTAMP(i) if (tls) tls[i] = clock64();
#else
#define N256_SSTAMP(i)
#endif
    while (true) {
      const int4 e = sr.next(ctrl, false);
      __syncwarp();
      if (lane == 0) sr.release_prev(ctrl);
      if (!e.w) break;
      const int b = e.x, hh = e.y, u = e.z;
      for (int t = 0; t < 2; ++t) {
        const int qb = 2 * u + t;
        if (qb >= p.nblk) break;
        const int n = tile_blocks<kCausal>(qb, nblk256);
        const int qrow = qb * 128 + row;
        float m = -INFINITY, l = 0.f;
        for (int j = 0; j < n; ++j, ++blk) {
          ptx::mbar_wait(&ctrl->s_ready, s_phase);
#ifdef N256_TIMELINE
          long long* tls = (p.trace && blockIdx.x == 0 && quarter == 0 && lane == 0 && tile_no == 0 && j < 64)
                               ? reinterpret_cast<long long*>(p.trace) + 4096 + hf * 512 + j * 8 : nullptr;
#endif
          N256_SSTAMP(0);
          s_phase ^= 1;
          ptx::tc_fence_after();
          uint32_t r[128];
          ptx::tmem_ld128(trow + colS, r);
#ifdef N256_TIMELINE
          if (tls) tls[1] = clock64() + (r[0] & 0) + (r[127] & 0);
#endif
          ptx::tc_fence_before();
          __syncwarp();
          if (lane == 0) ptx::mbar_arrive(&ctrl->s_free);  // S(j) is in registers
#ifdef N256_DEBUG_SKIP_SOFTMAX
          if (j > 0) { ptx::mbar_wait(&ctrl->p_free, pf_phase); pf_phase ^= 1; }
          __syncwarp();
          if (lane == 0) { ptx::mbar_arrive(&ctrl->p_ready[0]); if (hf == 1) ptx::mbar_arrive(&ctrl->p_ready[1]); }
          m = 0.f; l = 1.f;
          continue;
#endif
          // visible local keys k <= lim: causal (key <= query) and ragged N (key < N)
          const int k0 = j * kBN + hf * 128;
          int lim = 127;
          if (kCausal && qrow - k0 < lim) lim = qrow - k0;
          if (p.N - 1 - k0 < lim) lim = p.N - 1 - k0;
          const bool diag = __any_sync(0xffffffffu, lim < 127);
          if (diag) {
#pragma unroll
            for (int k = 0; k < 128; ++k)
              if (k > lim) r[k] = 0xff800000u;
          }
          constexpr int kCh = N256_MAX_CHAINS;  // independent FMNMX3 chains
          float mq[kCh];
#pragma unroll
          for (int g = 0; g < kCh; ++g) mq[g] = -INFINITY;
#pragma unroll
          for (int k = 0; k < 128; k += 2 * kCh) {
#pragma unroll
            for (int g = 0; g < kCh; ++g)
              mq[g] = fmaxf(mq[g], fmaxf(__uint_as_float(r[k + 2 * g]), __uint_as_float(r[k + 2 * g + 1])));
          }
#pragma unroll
          for (int w = kCh / 2; w >= 1; w /= 2)
#pragma unroll
            for (int g = 0; g < w; ++g) mq[g] = fmaxf(mq[g], mq[g + w]);
          float mx = mq[0];
#ifdef N256_TIMELINE
          if (tls) tls[2] = clock64() + (long long)(mx == 12345.f);
#endif
          red->mx[quarter][hf][blk & 1][lane] = mx;
          ptx::named_bar_sync(bar_id, 64);
          mx = fmaxf(mx, red->mx[quarter][hf ^ 1][blk & 1][lane]);
#ifdef N256_TIMELINE
          if (tls) tls[3] = clock64() + (long long)(mx == 12345.f);
#endif
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
          const bool any_rescale = __any_sync(0xffffffffu, rescale);
          const float neg = -m_use * c;
          float2 sq[4] = {make_float2(0.f, 0.f), make_float2(0.f, 0.f), make_float2(0.f, 0.f),
                          make_float2(0.f, 0.f)};
          auto exps = [&](auto mask_tag) {
#pragma unroll
            for (int k = 0; k < 128; k += 2) {
              const float2 x = ptx::ffma2(make_float2(__uint_as_float(r[k]), __uint_as_float(r[k + 1])), c, neg);
              float2 pr;
              constexpr int kEP = N256_EMU_PERIOD;
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
          };
          if (diag) exps(std::true_type{});
          else exps(std::false_type{});
#ifdef N256_TIMELINE
          if (tls) tls[4] = clock64() + (long long)(r[63] == 12345u);
#endif
          if (j > 0) {
            // PV(j-1) has finished reading P and adding into O: fix up O, then overwrite P
            ptx::mbar_wait(&ctrl->p_free, pf_phase);
            pf_phase ^= 1;
            ptx::tc_fence_after();
            if (any_rescale) {  // fix-up: O *= exp2((m_old - m_new) c), this warp's 64 columns
#pragma unroll
              for (int cc = 0; cc < 64; cc += 32) {
                uint32_t o[32];
                ptx::tmem_ld32(trow + colO + cc, o);
#pragma unroll
                for (int k = 0; k < 32; ++k) o[k] = __float_as_uint(__uint_as_float(o[k]) * alpha);
                ptx::tmem_st32(trow + colO + cc, o);
              }
            }
          }
          N256_SSTAMP(5);
          if (hf == 1) {  // O columns 64-127 are fixed up: the first PV half may start
            ptx::tmem_wait_st();
            ptx::tc_fence_before();
            __syncwarp();
            if (lane == 0) ptx::mbar_arrive(&ctrl->p_ready[0]);
          }
          ptx::tmem_st32(trow + colP, r);
          ptx::tmem_st32(trow + colP + 32, r + 32);
          ptx::tmem_wait_st();
          ptx::tc_fence_before();
          __syncwarp();
          if (lane == 0) ptx::mbar_arrive(&ctrl->p_ready[hf]);
          N256_SSTAMP(6);
          const float2 s01 = ptx::fadd2(sq[0], sq[1]), s23 = ptx::fadd2(sq[2], sq[3]);
          const float2 s4 = ptx::fadd2(s01, s23);
          const float sum = s4.x + s4.y;
          l = (j == 0) ? sum : fmaf(l, alpha, sum);
          m = m_use;
        }
        // ---- epilogue: O / l -> bf16 -> global (this warp's 64 columns)
        // row sum through the parity slot the last block did not use (its
        // previous contents were read before the last block's barrier)
        red->mx[quarter][hf][blk & 1][lane] = l;
        ptx::named_bar_sync(bar_id, 64);
        l += red->mx[quarter][hf ^ 1][blk & 1][lane];
        ++blk;  // the next block's maxima go to the other slot, so this one is not overwritten before it is read
        ptx::mbar_wait(&ctrl->o_ready, o_phase);
        o_phase ^= 1;
        ptx::tc_fence_after();
        const float inv_l = 1.f / l;
        const bool live = qrow < p.N;
        if (p.lse != nullptr && hf == 0 && live)  // lse = scale*m + ln(l)
          p.lse[(long long)(b * p.Hq + hh) * p.N + qrow] = (m * c + __log2f(l)) * 0.6931471805599453f;
        const long long orow = ((long long)(b * p.Hq_out + p.h_off + hh) * p.N + qrow) * p.d_real + hf * 64;
        const int ncol = live ? p.d_real - hf * 64 : 0;
#pragma unroll
        for (int cc = 0; cc < 64; cc += 32) {
          uint32_t o[32];
          ptx::tmem_ld32(trow + colO + cc, o);
          uint32_t pk[16];
#pragma unroll
          for (int k = 0; k < 16; ++k)
            pk[k] = ptx::pack_bf16(__uint_as_float(o[2 * k]) * inv_l, __uint_as_float(o[2 * k + 1]) * inv_l);
          for (int di = 0; di < p.n_dst; ++di) {
            uint4* dst = reinterpret_cast<uint4*>(p.o_dst[di] + orow);
#pragma unroll
            for (int k = 0; k < 4; ++k) {
              if (cc + 8 * k >= ncol) break;
              dst[cc / 8 + k] = make_uint4(pk[4 * k], pk[4 * k + 1], pk[4 * k + 2], pk[4 * k + 3]);
            }
          }
        }
        ptx::tc_fence_before();
#ifdef N256_TIMELINE
        ++tile_no;
#endif
      }
    }
  } else {
    if (ATTN_SETMAXNREG) ptx::setmaxnreg_dec<kOtherRegs>();  // warp 3: idle
  }

  ptx::tc_fence_before();
  __syncthreads();
  if (warp == 2) {
    ptx::tc_fence_after();
    ptx::tmem_dealloc(*reinterpret_cast<volatile uint32_t*>(&ctrl->tmem_base), kTmemCols);
  }
}

}  // namespace n256
}  // namespace attn
