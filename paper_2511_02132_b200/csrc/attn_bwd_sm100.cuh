// attn_bwd_sm100.cuh -- attention backward (eq:ba) on sm_100a.
//
//   P  = exp(scale * Q K^T - lse)            (lse from the forward, per query row)
//   dV = P^T dO            dP = dO V^T        dS = P o (dP - D),  D = rowsum(dO o O)
//   dQ = scale * dS K      dK = scale * dS^T Q
//
// Three kernels, all with the forward's persistent scheduler, so the paper's
// mappings apply to the backward's work units too ("each
// workgroup computing different row blocks of the gradients ... may share the
// same Q, K, V, and dO tensors within the same attention head"):
//   attn_bwd_prep_kernel  D[b,h,i] = sum_c dO * O per row, and per 128-row block
//                         the vectors -lse*log2(e), -D that the dK/dV kernel
//                         bulk-copies with each Q_i / dO_i (bandwidth)
//   attn_bwd_dq_kernel    unit = (b, h, 128-row query block); Q and dO copied
//                         to TMEM once per unit; loops over key blocks:
//                         S = Q K_j^T and dP = dO V_j^T (TS MMAs) ->
//                         P (registers), dS (8 elementwise warps: TMEM lane =
//                         query row, two key halves; bf16 into TMEM over dP)
//                         -> dQ += dS K_j (TS MMA).
//   attn_bwd_dkdv_kernel  unit = (b, kv group g, 128-key block j); loops over
//                         the group's query heads and query blocks i:
//                         S^T = K_j Q_i^T and dP^T = V_j dO_i^T (SS MMAs, one
//                         KEY row per TMEM lane) -> P^T, dS^T (bf16 into TMEM)
//                         -> dV += P^T dO_i and dK += dS^T Q_i (TS MMAs).
// Both compute kernels keep every accumulator in TMEM (dQ kernel: S, dP, dQ =
// 384 columns; dK/dV kernel: S^T, dP^T, dV, dK = 512 columns) and run one
// 128-row tile per CTA.  Both split the elementwise work into a P phase (from
// S) and a dS phase (from dP) interleaved with the MMAs (see the MMA warps),
// so the tensor pipe keeps working while the exps run.
#pragma once
#include "attn_fwd_sm100.cuh"

namespace attn {
namespace bwd {

constexpr int kBM = 128;       // rows of a query block / keys of a key block

// Every ATTN_BWD_EMU_PERIOD-th exp2 of the P phases runs as a polynomial on the
// FMA pipe instead of MUFU (0 = all on MUFU); see ptx::ex2_poly.
#ifndef ATTN_BWD_EMU_PERIOD
#define ATTN_BWD_EMU_PERIOD 8
#endif
// k: the element's index in a fully unrolled loop (the test folds away).
__device__ __forceinline__ float bwd_ex2(float x, int k) {
  constexpr int P = ATTN_BWD_EMU_PERIOD > 0 ? ATTN_BWD_EMU_PERIOD : 1;
  if (ATTN_BWD_EMU_PERIOD > 0 && k % P == P - 1) return ptx::ex2_poly(x);
  return ptx::ex2(x);
}
constexpr int kThreadsKV = 384;  // warps 0 TMA, 1 MMA, 2 scheduler + TMEM, 3 idle, 4-11 elementwise (two column halves)

template <int D>
struct BCfg {
  static constexpr int kChunks = D / 64;
  static constexpr int kTile = kBM * D * 2;  // one 128 x D bf16 tile
  static constexpr int kStages = 2;          // ring depth of the streamed operand pairs
  // Control block and staged vectors first, then the 1024-B aligned tiles; the
  // dynamic SMEM base is 1024-B aligned (checked in-kernel), which lets the
  // dK/dV kernel use the full 227 KB at D = 128.
  static constexpr int kOffCtrl = 0;          // BCtrl (<= 1 KB)
  static constexpr int kOffVec = 1024;        // dKdV: -lse2 / -D of each ring stage's query block (kStages x 1 KB)
  static constexpr int kVecBytes = 2 * kBM * 4;
  static constexpr int kOffA = 3072;          // resident pair (dQ: Q, dO;  dKdV: K, V)
  static_assert(kOffVec + kStages * kVecBytes <= kOffA, "ring-stage vectors overlap the K/V tiles");
  static constexpr int kOffRing = kOffA + 2 * kTile;  // ring of streamed pairs (dQ: K, V;  dKdV: Q, dO)
  static constexpr int kOffPT = kOffRing + kStages * 2 * kTile;  // dKdV: P^T, 128 x 128 bf16 (SW128 K-major)
  static constexpr int kSmemBytesKV = kOffPT + kBM * kBM * 2;    // dK/dV kernel
  // dQ kernel: Q / dO go to TMEM, so its ring holds single K or V tiles
  static constexpr int kQSlots = 5;
  static constexpr int kSmemBytesQ = kOffRing + kQSlots * kTile;
  static_assert(kSmemBytesQ <= 232448, "dQ SMEM over the 227 KB opt-in limit");
  static_assert(kSmemBytesKV <= 232448, "dK/dV SMEM over the 227 KB opt-in limit");
};

struct BwdParams {
  int B, Hq, Hkv, N, G, nblk, d_real;
  float scale, scale_log2;
  const float* lse;    // [B][Hq][N], natural log
  const float* dvec;   // [B][Hq][N], rowsum(dO o O)
  const float* vecb;   // two-pass dK/dV: attn_bwd_prep_kernel's blocks (-lse2 | -D per 128 query rows)
  __nv_bfloat16* dq;   // [B][Hq][N][d]
  __nv_bfloat16* dk;   // [B][Hkv][N][d]
  __nv_bfloat16* dv;   // [B][Hkv][N][d]
  SchedParams sched;
  int U;               // units per "head" of the schedule (query or key blocks)
  int* counters;
  const signed char* domain_of_smid;
  int n_smid;
  long long* dbg;      // -D ATTN_BWD_TIMELINE: per-block stamps of CTA 0 (the trace buffer), else unused
};

struct __align__(16) BCtrl {
  uint64_t sched_full[kSchedRing];
  uint64_t sched_empty[kSchedRing];
  uint64_t a_full, a_empty;             // resident pair
  uint64_t ring_full[5], ring_empty[5]; // streamed pairs (dKdV) / single tiles (dQ)
  uint64_t s_ready, p_ready, o_ready;
  uint64_t dp_ready, ds_ready;          // dP in TMEM, dS stored (bf16, TMEM)
  uint64_t q_ready;                     // dQ: Q and dO copied into TMEM
  uint64_t s_free, dv_done;             // dKdV: S^T read into registers; dV MMA done (P^T SMEM free)
  uint64_t dk_done;                     // fused: dK and dQ MMAs done (dS^T SMEM free)
  uint64_t dq_full[2], dq_empty[2];     // fused: dQ TMEM buffers (MMA -> drain -> MMA)
  int4 entry[kSchedRing];
  uint32_t tmem_base;
};
static_assert(sizeof(BCtrl) <= 1024, "BCtrl must fit its 1 KB slot");

// The scheduler warp: identical pop / steal / broadcast protocol as the forward.
__device__ __forceinline__ void bwd_scheduler(const BwdParams& p, BCtrl* ctrl, int Hsched) {
  const int sm = (int)ptx::smid();
  int dom = (sm < p.n_smid) ? (int)p.domain_of_smid[sm] : 0;
  if (dom < 0) dom = 0;
  const int nq = p.sched.n_queues;
  const int q0 = (nq > 1) ? p.sched.queue_of_domain[dom] : 0;
  uint32_t exhausted = 0;
  int stage = 0;
  uint32_t phase = 0;
  while (true) {
    int b = 0, h = 0, u = 0, qi = -1;
    for (int t = 0; t < nq; ++t) {
      if (t > 0 && !p.sched.steal) break;
      const int qq = (q0 + t) % nq;
      if (exhausted & (1u << qq)) continue;
      const int pos = atomicAdd(&p.counters[qq * 32], 1);
      if (pos < p.sched.q[qq].len) {
        decode_unit(p.sched, qq, pos, Hsched, p.U, b, h, u);
        if ((p.sched.descending >> qq) & 1) u = p.U - 1 - u;
        qi = qq;
        break;
      }
      exhausted |= 1u << qq;
    }
    ptx::mbar_wait(&ctrl->sched_empty[stage], phase ^ 1);
    ctrl->entry[stage] = make_int4(b, h, u, qi >= 0 ? 1 : 0);
    ptx::mbar_arrive(&ctrl->sched_full[stage]);
    if (qi < 0) break;
    if (++stage == kSchedRing) { stage = 0; phase ^= 1; }
  }
  __threadfence();
  if (atomicAdd(&p.counters[kDoneCounter], 1) == (int)gridDim.x - 1) {
    for (int q = 0; q < nq; ++q) atomicExch(&p.counters[q * 32], 0);
    atomicExch(&p.counters[kDoneCounter], 0);
    __threadfence();
  }
}

struct BSchedReader {
  int stage = 0;
  uint32_t phase = 0;
  // warp_wide: all 32 lanes call next(); otherwise only the calling lane does.
  __device__ __forceinline__ int4 next(BCtrl* c, bool warp_wide = true) {
    ptx::mbar_wait(&c->sched_full[stage], phase);
    const volatile int* ve = reinterpret_cast<const volatile int*>(&c->entry[stage]);
    const int4 e = make_int4(ve[0], ve[1], ve[2], ve[3]);
    if (warp_wide) __syncwarp();
    if (!warp_wide || (threadIdx.x & 31) == 0) ptx::mbar_arrive(&c->sched_empty[stage]);
    if (++stage == kSchedRing) { stage = 0; phase ^= 1; }
    return e;
  }
};

// Causal: query block i needs key blocks 0..i;  key block j is needed by query
// blocks j..nblk-1.  Non-causal: all blocks.
template <bool kCausal>
__device__ __forceinline__ int dq_nblocks(int i, int nblk) { return kCausal ? i + 1 : nblk; }
template <bool kCausal>
__device__ __forceinline__ int dkdv_first_qblock(int j) { return kCausal ? j : 0; }

// =========================================================================== dQ
template <int D, bool kCausal>
__global__ void __launch_bounds__(kThreadsKV, 1)
    attn_bwd_dq_kernel(const __grid_constant__ CUtensorMap tm_q, const __grid_constant__ CUtensorMap tm_do,
                       const __grid_constant__ CUtensorMap tm_k, const __grid_constant__ CUtensorMap tm_v,
                       const BwdParams p) {
  using C = BCfg<D>;
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = smem_raw;
  if (ptx::smem_u32(smem_raw) & 1023) __trap();  // layout relies on a 1024-B aligned base
  uint8_t* sq = smem + C::kOffA;             // Q tile, then dO tile
  uint8_t* ring = smem + C::kOffRing;        // kQSlots single-tile slots: K_0, V_0, K_1, V_1, ...
  BCtrl* ctrl = reinterpret_cast<BCtrl*>(smem + C::kOffCtrl);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  // TMEM: S [0,128), dP [128,256), dQ [256, 256+D), Q [384, 384+D/2), dO [448, 448+D/2)
  // (Q and dO as bf16 pairs: the A operands of the S and dP MMAs come from TMEM,
  // so those MMAs read only K / V from SMEM)
  constexpr uint32_t kColS = 0, kColDP = 128, kColDQ = 256, kColQ = 384, kColDO = 448;
  constexpr int kEw = 8;  // elementwise warps

  if (threadIdx.x == 0) {
    for (int i = 0; i < kSchedRing; ++i) {
      ptx::mbar_init(&ctrl->sched_full[i], 1);
      ptx::mbar_init(&ctrl->sched_empty[i], 2 + kEw);
    }
    ptx::mbar_init(&ctrl->a_full, 1);
    ptx::mbar_init(&ctrl->a_empty, kEw);   // Q / dO SMEM copied into TMEM
    for (int i = 0; i < C::kQSlots; ++i) {
      ptx::mbar_init(&ctrl->ring_full[i], 1);
      ptx::mbar_init(&ctrl->ring_empty[i], 1);
    }
    ptx::mbar_init(&ctrl->q_ready, kEw);
    ptx::mbar_init(&ctrl->s_ready, 1);
    ptx::mbar_init(&ctrl->dp_ready, 1);
    ptx::mbar_init(&ctrl->p_ready, kEw);   // S consumed (P held in registers)
    ptx::mbar_init(&ctrl->ds_ready, kEw);
    ptx::mbar_init(&ctrl->o_ready, 1);
    ptx::fence_barrier_init();
  }
  if (warp == 2) {
    ptx::tmem_alloc(&ctrl->tmem_base, 512);
    ptx::tmem_relinquish();
  }
  ptx::tc_fence_before();
  __syncthreads();
  ptx::tc_fence_after();
  const uint32_t tmem = *reinterpret_cast<volatile uint32_t*>(&ctrl->tmem_base);

  if (warp == 0) {
    if (lane == 0) {
      BSchedReader sr;
      const uint64_t pol_first = ptx::policy_evict_first();
      const uint64_t pol_kv = ptx::policy_evict_normal();
      uint32_t a_phase = 0, r_phase = 0;
      int stage = 0;
      while (true) {
        const int4 e = sr.next(ctrl, false);
        if (!e.w) break;
        const int b = e.x, h = e.y, i = e.z;
        const int bh = b * p.Hq + h, kvbh = b * p.Hkv + h / p.G;
        ptx::mbar_wait(&ctrl->a_empty, a_phase ^ 1);
        a_phase ^= 1;
        ptx::mbar_arrive_expect_tx(&ctrl->a_full, 2 * C::kTile);
#pragma unroll
        for (int c = 0; c < C::kChunks; ++c) {
          ptx::tma_load_3d(sq + c * kBM * 128, &tm_q, &ctrl->a_full, c * 64, i * kBM, bh, pol_first);
          ptx::tma_load_3d(sq + C::kTile + c * kBM * 128, &tm_do, &ctrl->a_full, c * 64, i * kBM, bh, pol_first);
        }
        const int n = dq_nblocks<kCausal>(i, p.nblk);
        for (int j = 0; j < n; ++j) {
#pragma unroll
          for (int which = 0; which < 2; ++which) {  // K_j, then V_j, one slot each
            ptx::mbar_wait(&ctrl->ring_empty[stage], r_phase ^ 1);
            ptx::mbar_arrive_expect_tx(&ctrl->ring_full[stage], C::kTile);
            uint8_t* dst = ring + stage * C::kTile;
#pragma unroll
            for (int c = 0; c < C::kChunks; ++c)
              ptx::tma_load_3d(dst + c * kBM * 128, which == 0 ? (const void*)&tm_k : (const void*)&tm_v,
                               &ctrl->ring_full[stage], c * 64, j * kBM, kvbh, pol_kv);
            if (++stage == C::kQSlots) { stage = 0; r_phase ^= 1; }
          }
        }
      }
    }
  } else if (warp == 1) {
    // Per block j the tensor pipe runs  S(j+1) . dQ(j) . dP(j+1):  S(j+1) is
    // issued as soon as the elementwise warps have read S(j) (P stays in their
    // registers), so the exps of block j+1 overlap dQ(j) and dP(j+1).  Ring
    // slots are taken in the producer's order (K_j+1, then V_j+1); V_j is
    // released after dP(j), K_j after dQ(j).
    BSchedReader sr;
    constexpr uint32_t idesc_s = ptx::idesc_bf16_f32(kBM, kBM, 0, 0);  // S, dP: K-major A and B
    constexpr uint32_t idesc_q = ptx::idesc_bf16_f32(kBM, D, 0, 1);    // dQ: A = dS (TMEM), B = K MN-major
    const uint64_t dr0 = ptx::smem_desc_sw128(ptx::smem_u32(ring), 16, 1024);
    const uint64_t drm0 = ptx::smem_desc_sw128(ptx::smem_u32(ring), kBM * 128, 1024);
    uint32_t a_phase = 0, r_phase = 0, p_phase = 0;
    int slot = 0;
    auto take = [&]() {
      const int sl = slot;
      ptx::mbar_wait(&ctrl->ring_full[sl], r_phase);
      if (++slot == C::kQSlots) { slot = 0; r_phase ^= 1; }
      return sl;
    };
    auto ts_mma = [&](uint32_t d_col, uint32_t a_col, uint64_t b) {  // [128 x 128] = A[128 x D] (TMEM) B[128 x D]^T
#pragma unroll
      for (int k = 0; k < D / 16; ++k) {
        const uint32_t off = ((k >> 2) * (kBM * 128) + (k & 3) * 32) >> 4;
        ptx::mma_ts(tmem + d_col, tmem + a_col + k * 8, b + off, idesc_s, k > 0 ? 1u : 0u);
      }
    };
    auto kmaj = [&](int sl) { return dr0 + (uint64_t)((sl * C::kTile) >> 4); };
#ifdef ATTN_BWD_TIMELINE
    int unit_no = 0;
#define BWD_STAMP(j, i) if (p.dbg && blockIdx.x == 0 && lane == 0 && unit_no == 1 && (j) < 64) p.dbg[(j) * 16 + (i)] = clock64();
#else
#define BWD_STAMP(j, i)
#endif
    while (true) {
      const int4 e = sr.next(ctrl);
      if (!e.w) break;
      const int n = dq_nblocks<kCausal>(e.z, p.nblk);
#ifdef ATTN_BWD_TIMELINE
      ++unit_no;
#endif
      ptx::mbar_wait(&ctrl->q_ready, a_phase);
      a_phase ^= 1;
      int sK = take();
      const int sV0 = take();
      ptx::tc_fence_after();
      if (ptx::elect_one_sync()) {
        ts_mma(kColS, kColQ, kmaj(sK));                             // S  = Q  K_0^T
        ptx::mma_commit(&ctrl->s_ready);
        ts_mma(kColDP, kColDO, kmaj(sV0));                          // dP = dO V_0^T
        ptx::mma_commit(&ctrl->dp_ready);
        ptx::mma_commit(&ctrl->ring_empty[sV0]);
      }
      __syncwarp();
      for (int j = 0; j < n; ++j) {
        const bool nxt = j + 1 < n;
        ptx::mbar_wait(&ctrl->p_ready, p_phase);   // S(j) read
        BWD_STAMP(j, 0);
        ptx::tc_fence_after();
        int sK1 = sK;
        if (nxt) {
          sK1 = take();
          ptx::tc_fence_after();
          if (ptx::elect_one_sync()) {
            ts_mma(kColS, kColQ, kmaj(sK1));        // S(j+1)
            ptx::mma_commit(&ctrl->s_ready);
          }
          __syncwarp();
        }
        BWD_STAMP(j, 1);
        ptx::mbar_wait(&ctrl->ds_ready, p_phase);
        BWD_STAMP(j, 2);
        p_phase ^= 1;
        ptx::tc_fence_after();
        int sV1 = -1;
        if (nxt) sV1 = take();
        ptx::tc_fence_after();
        if (ptx::elect_one_sync()) {
          // dQ += dS K_j: A = dS (bf16 in TMEM over dP; queries' keys 0-63 in
          // columns [0,32), keys 64-127 in [64,96) of the region), B = K_j as
          // [keys x D] (MN-major)
          const uint64_t km = drm0 + (uint64_t)((sK * C::kTile) >> 4);
#pragma unroll
          for (int k = 0; k < kBM / 16; ++k)
            ptx::mma_ts(tmem + kColDQ, tmem + kColDP + k * 8 + (k >= 4 ? 32 : 0),
                        km + (uint64_t)((k * 16 * 128) >> 4), idesc_q, (j > 0 || k > 0) ? 1u : 0u);
          ptx::mma_commit(&ctrl->ring_empty[sK]);
          if (nxt) {
            ts_mma(kColDP, kColDO, kmaj(sV1));      // dP(j+1)
            ptx::mma_commit(&ctrl->dp_ready);
            ptx::mma_commit(&ctrl->ring_empty[sV1]);
          } else {
            ptx::mma_commit(&ctrl->o_ready);
          }
        }
        __syncwarp();
        BWD_STAMP(j, 3);
        sK = sK1;
      }
    }
#undef BWD_STAMP
  } else if (warp == 2) {
    if (lane == 0) bwd_scheduler(p, ctrl, p.Hq);
  } else if (warp >= 4) {
    // 256 threads: TMEM lane = query row (warp & 3), column half `half` =
    // keys [64*half, 64*half+64) of each block.
    const int quarter = warp & 3, row = quarter * 32 + lane;
    const int half = (warp - 4) >> 2, k0c = half * 64;
    const uint32_t trow = tmem + ((uint32_t)(quarter * 32) << 16);
    const float c = p.scale_log2;
    BSchedReader sr;
    uint32_t s_phase = 0, o_phase = 0, a_phase = 0;
#ifdef ATTN_BWD_TIMELINE
    int unit_no = 0;
#endif
    while (true) {
      const int4 e = sr.next(ctrl);
      if (!e.w) break;
      const int b = e.x, h = e.y, i = e.z;
      {
        // Q, dO (SW128 K-major SMEM, 64-column chunks) -> TMEM as bf16 pairs;
        // column half `half` copies chunks half, half + 2, ...
        ptx::mbar_wait(&ctrl->a_full, a_phase);
        a_phase ^= 1;
#pragma unroll
        for (int ch = half; ch < 2 * C::kChunks; ch += 2) {
          const int t = ch / C::kChunks, cc = ch % C::kChunks;
          const uint8_t* rowp = sq + t * C::kTile + cc * (kBM * 128) + row * 128;
          uint32_t v[32];
#pragma unroll
          for (int u = 0; u < 8; ++u) {
            const uint4 x = *reinterpret_cast<const uint4*>(rowp + ((u ^ (row & 7)) << 4));
            v[4 * u] = x.x; v[4 * u + 1] = x.y; v[4 * u + 2] = x.z; v[4 * u + 3] = x.w;
          }
          ptx::tmem_st32(trow + (t ? kColDO : kColQ) + cc * 32, v);
        }
        ptx::tmem_wait_st();
        ptx::tc_fence_before();
        __syncwarp();
        if (lane == 0) {
          ptx::mbar_arrive(&ctrl->q_ready);
          ptx::mbar_arrive(&ctrl->a_empty);
        }
      }
      const int qrow = i * kBM + row;
      const bool valid = qrow < p.N;
      const long long ridx = (long long)(b * p.Hq + h) * p.N + (valid ? qrow : 0);
      const float lse2 = valid ? p.lse[ridx] * 1.4426950408889634f : 0.f;
      const float dd = valid ? p.dvec[ridx] : 0.f;
      const int n = dq_nblocks<kCausal>(i, p.nblk);
#ifdef ATTN_BWD_TIMELINE
      ++unit_no;
#define BWD_ESTAMP(j, i) if (p.dbg && blockIdx.x == 0 && lane == 0 && quarter == 0 && unit_no == 1 && (j) < 64) \
    p.dbg[(j) * 16 + 4 + 5 * half + (i)] = clock64();
#else
#define BWD_ESTAMP(j, i)
#endif
      for (int j = 0; j < n; ++j) {
        // visible keys of this row in block j: k <= lim (causal diagonal, ragged tail)
        int lim = kBM - 1;
        if (kCausal && j == i) lim = row;
        if (j == p.nblk - 1) lim = min(lim, p.N - 1 - j * kBM);
        if (!valid) lim = -1;
        float pv[64];
        ptx::mbar_wait(&ctrl->s_ready, s_phase);
        BWD_ESTAMP(j, 0);
        ptx::tc_fence_after();
        // S -> registers, then release the S region (S(j+1) is issued at once)
        ptx::tmem_ld64(trow + kColS + k0c, reinterpret_cast<uint32_t*>(pv));   // one wait for 64 columns
        ptx::tc_fence_before();
        __syncwarp();
        if (lane == 0) ptx::mbar_arrive(&ctrl->p_ready);
        BWD_ESTAMP(j, 1);
        // masking (causal diagonal, ragged tail, rows past N) only where some
        // lane of the warp needs it: a warp-uniform branch, no per-element
        // compare + select on the common path
        // x = S * c - lse2, two columns per FFMA2 (the same rounding as fmaf)
        const float nl2 = -lse2;
        if (__any_sync(0xffffffffu, lim < k0c + 63)) {
#pragma unroll
          for (int k = 0; k < 64; k += 2) {
            const float2 x = ptx::ffma2(make_float2(pv[k], pv[k + 1]), c, nl2);
            const float p0 = bwd_ex2(x.x, k), p1 = bwd_ex2(x.y, k + 1);
            pv[k] = (k0c + k <= lim) ? p0 : 0.f;
            pv[k + 1] = (k0c + k + 1 <= lim) ? p1 : 0.f;
          }
        } else {
#pragma unroll
          for (int k = 0; k < 64; k += 2) {
            const float2 x = ptx::ffma2(make_float2(pv[k], pv[k + 1]), c, nl2);
            pv[k] = bwd_ex2(x.x, k);
            pv[k + 1] = bwd_ex2(x.y, k + 1);
          }
        }
        BWD_ESTAMP(j, 2);
        ptx::mbar_wait(&ctrl->dp_ready, s_phase);
        BWD_ESTAMP(j, 3);
        s_phase ^= 1;
        ptx::tc_fence_after();
        {
          uint32_t dp[64];
          ptx::tmem_ld64(trow + kColDP + k0c, dp);   // one wait for 64 columns
#pragma unroll
          for (int cc = 0; cc < 64; cc += 32) {
            uint32_t pk[16];
#pragma unroll
            for (int k = 0; k < 32; k += 2) {  // dS = P o (dP - D), packed (same rounding per lane)
              const float2 t = ptx::fadd2(make_float2(__uint_as_float(dp[cc + k]), __uint_as_float(dp[cc + k + 1])),
                                          make_float2(-dd, -dd));
              const float2 r = ptx::fmul2(make_float2(pv[cc + k], pv[cc + k + 1]), t);
              pk[k >> 1] = ptx::pack_bf16(r.x, r.y);
            }
            ptx::tmem_st16(trow + kColDP + k0c + cc / 2, pk);  // dS (bf16 pairs) over dP columns this half read
          }
        }
        ptx::tmem_wait_st();
        ptx::tc_fence_before();
        __syncwarp();
        if (lane == 0) ptx::mbar_arrive(&ctrl->ds_ready);
        BWD_ESTAMP(j, 4);
      }
#undef BWD_ESTAMP
      ptx::mbar_wait(&ctrl->o_ready, o_phase);
      o_phase ^= 1;
      ptx::tc_fence_after();
      __nv_bfloat16* dst = p.dq + ((long long)(b * p.Hq + h) * p.N + (valid ? qrow : 0)) * p.d_real;
#pragma unroll
      for (int cc = half * (D / 2); cc < (half + 1) * (D / 2); cc += 32) {  // each half stores D/2 columns
        uint32_t o[32];
        ptx::tmem_ld32(trow + kColDQ + cc, o);
        uint32_t pk[16];
#pragma unroll
        for (int k = 0; k < 16; ++k)
          pk[k] = ptx::pack_bf16(__uint_as_float(o[2 * k]) * p.scale, __uint_as_float(o[2 * k + 1]) * p.scale);
        if (valid) {
#pragma unroll
          for (int k = 0; k < 4; ++k)
            if (cc + 8 * k < p.d_real)
              reinterpret_cast<uint4*>(dst)[cc / 8 + k] = make_uint4(pk[4 * k], pk[4 * k + 1], pk[4 * k + 2], pk[4 * k + 3]);
        }
      }
      ptx::tc_fence_before();
    }
  }
  ptx::tc_fence_before();
  __syncthreads();
  if (warp == 2) {
    ptx::tc_fence_after();
    ptx::tmem_dealloc(tmem, 512);
  }
}

// ======================================================================== dK, dV
template <int D, bool kCausal>
__global__ void __launch_bounds__(kThreadsKV, 1)
    attn_bwd_dkdv_kernel(const __grid_constant__ CUtensorMap tm_q, const __grid_constant__ CUtensorMap tm_do,
                         const __grid_constant__ CUtensorMap tm_k, const __grid_constant__ CUtensorMap tm_v,
                         const BwdParams p) {
  using C = BCfg<D>;
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = smem_raw;
  if (ptx::smem_u32(smem_raw) & 1023) __trap();  // layout relies on a 1024-B aligned base
  uint8_t* skv = smem + C::kOffA;            // K tile, then V tile
  uint8_t* ring = smem + C::kOffRing;        // stage s: Q at 2s, dO at 2s+1
  uint8_t* spt = smem + C::kOffPT;           // P^T (bf16) as the A operand of dV
  BCtrl* ctrl = reinterpret_cast<BCtrl*>(smem + C::kOffCtrl);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  // TMEM: S^T [0,128), dP^T [128,256), dV [256, 256+D), dK [384, 384+D)
  constexpr uint32_t kColS = 0, kColDP = 128, kColDV = 256, kColDK = 384;
  constexpr int kEw = 8;  // elementwise warps

  if (threadIdx.x == 0) {
    for (int i = 0; i < kSchedRing; ++i) {
      ptx::mbar_init(&ctrl->sched_full[i], 1);
      ptx::mbar_init(&ctrl->sched_empty[i], 2 + kEw);
    }
    ptx::mbar_init(&ctrl->a_full, 1);
    ptx::mbar_init(&ctrl->a_empty, 1);
    for (int i = 0; i < C::kStages; ++i) {
      ptx::mbar_init(&ctrl->ring_full[i], 1);
      ptx::mbar_init(&ctrl->ring_empty[i], 1);
    }
    ptx::mbar_init(&ctrl->s_ready, 1);
    ptx::mbar_init(&ctrl->dp_ready, 1);
    ptx::mbar_init(&ctrl->p_ready, kEw);
    ptx::mbar_init(&ctrl->ds_ready, kEw);
    ptx::mbar_init(&ctrl->s_free, kEw);
    ptx::mbar_init(&ctrl->dv_done, 1);
    ptx::mbar_init(&ctrl->o_ready, 1);
    ptx::fence_barrier_init();
  }
  if (warp == 2) {
    ptx::tmem_alloc(&ctrl->tmem_base, 512);
    ptx::tmem_relinquish();
  }
  ptx::tc_fence_before();
  __syncthreads();
  ptx::tc_fence_after();
  const uint32_t tmem = *reinterpret_cast<volatile uint32_t*>(&ctrl->tmem_base);

  if (warp == 0) {
    if (lane == 0) {
      BSchedReader sr;
      const uint64_t pol_kv = ptx::policy_evict_first();
      const uint64_t pol_q = ptx::policy_evict_normal();
      uint32_t a_phase = 0, r_phase = 0;
      int stage = 0;
      while (true) {
        const int4 e = sr.next(ctrl, false);
        if (!e.w) break;
        const int b = e.x, g = e.y, j = e.z;
        const int kvbh = b * p.Hkv + g;
        ptx::mbar_wait(&ctrl->a_empty, a_phase ^ 1);
        a_phase ^= 1;
        ptx::mbar_arrive_expect_tx(&ctrl->a_full, 2 * C::kTile);
#pragma unroll
        for (int c = 0; c < C::kChunks; ++c) {
          ptx::tma_load_3d(skv + c * kBM * 128, &tm_k, &ctrl->a_full, c * 64, j * kBM, kvbh, pol_kv);
          ptx::tma_load_3d(skv + C::kTile + c * kBM * 128, &tm_v, &ctrl->a_full, c * 64, j * kBM, kvbh, pol_kv);
        }
        for (int hh = 0; hh < p.G; ++hh) {
          const int bh = b * p.Hq + g * p.G + hh;
          for (int i = dkdv_first_qblock<kCausal>(j); i < p.nblk; ++i) {
            ptx::mbar_wait(&ctrl->ring_empty[stage], r_phase ^ 1);
            ptx::mbar_arrive_expect_tx(&ctrl->ring_full[stage], 2 * C::kTile + C::kVecBytes);
            uint8_t* dst = ring + stage * 2 * C::kTile;
#pragma unroll
            for (int c = 0; c < C::kChunks; ++c) {
              ptx::tma_load_3d(dst + c * kBM * 128, &tm_q, &ctrl->ring_full[stage], c * 64, i * kBM, bh, pol_q);
              ptx::tma_load_3d(dst + C::kTile + c * kBM * 128, &tm_do, &ctrl->ring_full[stage], c * 64, i * kBM, bh,
                               pol_q);
            }
            // the block's -lse2 / -D (attn_bwd_prep_kernel) with the same barrier
            ptx::bulk_load(smem + C::kOffVec + stage * C::kVecBytes, p.vecb + ((long long)bh * p.nblk + i) * (2 * kBM),
                           C::kVecBytes, &ctrl->ring_full[stage], pol_q);
            if (++stage == C::kStages) { stage = 0; r_phase ^= 1; }
          }
        }
      }
    }
  } else if (warp == 1) {
    // Per block `it` the tensor pipe runs  S^T(it+1) . dV(it) . dK(it) . dP^T(it+1):
    // S^T(it+1) is issued as soon as the elementwise warps hold S^T(it) in
    // registers (s_free), dV(it) once they have written P^T(it) to SMEM, dK(it)
    // once dS^T(it) is in TMEM over dP^T(it) -- the exps of block it+1 overlap
    // dV(it), dK(it) and dP^T(it+1).
    BSchedReader sr;
    constexpr uint32_t idesc_s = ptx::idesc_bf16_f32(kBM, kBM, 0, 0);  // S^T, dP^T
    constexpr uint32_t idesc_g = ptx::idesc_bf16_f32(kBM, D, 0, 1);    // dV, dK: A K-major, B MN-major
    const uint64_t dkv0 = ptx::smem_desc_sw128(ptx::smem_u32(skv), 16, 1024);
    const uint64_t dr0 = ptx::smem_desc_sw128(ptx::smem_u32(ring), 16, 1024);
    const uint64_t drm0 = ptx::smem_desc_sw128(ptx::smem_u32(ring), kBM * 128, 1024);
    const uint64_t dpt0 = ptx::smem_desc_sw128(ptx::smem_u32(spt), 16, 1024);
    uint32_t a_phase = 0, r_phase = 0, p_phase = 0;
    int stage = 0;
    auto ss_mma = [&](uint32_t d_col, uint64_t a, uint64_t b) {
#pragma unroll
      for (int k = 0; k < D / 16; ++k) {
        const uint32_t off = ((k >> 2) * (kBM * 128) + (k & 3) * 32) >> 4;
        ptx::mma_ss(tmem + d_col, a + off, b + off, idesc_s, k > 0 ? 1u : 0u);
      }
    };
    while (true) {
      const int4 e = sr.next(ctrl);
      if (!e.w) break;
      const int n = p.G * (p.nblk - dkdv_first_qblock<kCausal>(e.z));
      ptx::mbar_wait(&ctrl->a_full, a_phase);
      a_phase ^= 1;
      int st = stage;
      ptx::mbar_wait(&ctrl->ring_full[st], r_phase);
      ptx::tc_fence_after();
      if (ptx::elect_one_sync()) {
        const uint64_t qd = dr0 + (uint64_t)((st * 2 * C::kTile) >> 4);
        ss_mma(kColS, dkv0, qd);                                                            // S^T  = K Q_i^T
        ptx::mma_commit(&ctrl->s_ready);
        ss_mma(kColDP, dkv0 + (uint64_t)(C::kTile >> 4), qd + (uint64_t)(C::kTile >> 4));   // dP^T = V dO_i^T
        ptx::mma_commit(&ctrl->dp_ready);
      }
      __syncwarp();
      for (int it = 0; it < n; ++it) {
        const int cur = st;
        const bool nxt = it + 1 < n;
        int nst = cur, nph = r_phase;
        if (nxt) {
          nst = cur + 1 == C::kStages ? 0 : cur + 1;
          nph = cur + 1 == C::kStages ? r_phase ^ 1 : r_phase;
        }
        const uint64_t qm = drm0 + (uint64_t)((cur * 2 * C::kTile) >> 4);  // Q_i as [queries x D] MN-major
        const uint64_t dom = qm + (uint64_t)(C::kTile >> 4);               // dO_i likewise
        const uint64_t qd = dr0 + (uint64_t)((nst * 2 * C::kTile) >> 4);
        ptx::mbar_wait(&ctrl->s_free, p_phase);
        ptx::tc_fence_after();
        if (nxt) {
          ptx::mbar_wait(&ctrl->ring_full[nst], nph);
          ptx::tc_fence_after();
          if (ptx::elect_one_sync()) {
            ss_mma(kColS, dkv0, qd);                         // S^T(it+1)
            ptx::mma_commit(&ctrl->s_ready);
          }
          __syncwarp();
        }
        ptx::mbar_wait(&ctrl->p_ready, p_phase);
        ptx::tc_fence_after();
        if (ptx::elect_one_sync()) {
#pragma unroll
          for (int k = 0; k < kBM / 16; ++k)                // dV += P^T dO_i  (A = P^T from SMEM)
            ptx::mma_ss(tmem + kColDV, dpt0 + (uint64_t)((((k >> 2) * (kBM * 128)) + (k & 3) * 32) >> 4),
                        dom + (uint64_t)((k * 16 * 128) >> 4), idesc_g, (it > 0 || k > 0) ? 1u : 0u);
          ptx::mma_commit(&ctrl->dv_done);
        }
        __syncwarp();
        ptx::mbar_wait(&ctrl->ds_ready, p_phase);
        p_phase ^= 1;
        ptx::tc_fence_after();
        if (ptx::elect_one_sync()) {
          // dK += dS^T Q_i: A = dS^T (bf16 in TMEM over dP^T; queries 0-63 packed
          // in columns [0,32) of the region, 64-127 in [64,96) -- each column half
          // of the elementwise warps overwrites only columns it has itself read)
#pragma unroll
          for (int k = 0; k < kBM / 16; ++k)
            ptx::mma_ts(tmem + kColDK, tmem + kColDP + k * 8 + (k >= 4 ? 32 : 0),
                        qm + (uint64_t)((k * 16 * 128) >> 4), idesc_g, (it > 0 || k > 0) ? 1u : 0u);
          ptx::mma_commit(&ctrl->ring_empty[cur]);
          if (nxt) {
            ss_mma(kColDP, dkv0 + (uint64_t)(C::kTile >> 4), qd + (uint64_t)(C::kTile >> 4));  // dP^T(it+1)
            ptx::mma_commit(&ctrl->dp_ready);
          } else {
            ptx::mma_commit(&ctrl->a_empty);
            ptx::mma_commit(&ctrl->o_ready);
          }
        }
        __syncwarp();
        st = nst;
        r_phase = nph;
      }
      stage = st + 1 == C::kStages ? 0 : st + 1;
      if (st + 1 == C::kStages) r_phase ^= 1;
    }
  } else if (warp == 2) {
    if (lane == 0) bwd_scheduler(p, ctrl, p.Hkv);
  } else if (warp >= 4) {
    // 256 threads: TMEM lane = key row (warp & 3), column half `half` = queries
    // [64*half, 64*half+64) of each block.  Phase A: P^T = exp2(S^T*c - lse2)
    // kept in registers (fp32) and stored bf16 to SMEM for the dV MMA; phase B:
    // dS^T = P^T o (dP^T - D) stored bf16 over dP^T.
    const int quarter = warp & 3, krow = quarter * 32 + lane;  // key row of the block
    const int half = (warp - 4) >> 2, q0c = half * 64;
    const uint32_t trow = tmem + ((uint32_t)(quarter * 32) << 16);
    const float c = p.scale_log2;
    BSchedReader sr;
    uint32_t s_phase = 0, o_phase = 0, blk = 0, pt_phase = 0;
    ATTN_CYC_DECL()
    while (true) {
      const int4 e = sr.next(ctrl);
      if (!e.w) break;
      const int b = e.x, g = e.y, j = e.z;
      const int kglob = j * kBM + krow;
      const int i0 = dkdv_first_qblock<kCausal>(j);
      for (int hh = 0; hh < p.G; ++hh) {
        for (int i = i0; i < p.nblk; ++i) {
          ATTN_CYC_START();
          // this block's -lse2 / -D: bulk-copied with Q_i, dO_i into ring stage blk % kStages
          const int rs = (int)(blk % C::kStages);
          ptx::mbar_wait(&ctrl->ring_full[rs], (blk / C::kStages) & 1);
          const float* sv = reinterpret_cast<const float*>(smem + C::kOffVec + rs * C::kVecBytes);
          ++blk;
          // visible queries of this key: q >= k (causal), q < N; local query index
          int qlo = 0, qhi = kBM - 1;
          if (kCausal && i == j) qlo = krow;           // query >= key
          if (i == p.nblk - 1) qhi = p.N - 1 - i * kBM;  // ragged tail
          float pv[64];
          ATTN_CYC_ADD(0);
          ptx::mbar_wait(&ctrl->s_ready, s_phase);
          ATTN_CYC_ADD(1);
          ptx::tc_fence_after();
          ptx::tmem_ld64(trow + kColS + q0c, reinterpret_cast<uint32_t*>(pv));   // one wait for 64 columns
          ptx::tc_fence_before();
          __syncwarp();
          if (lane == 0) ptx::mbar_arrive(&ctrl->s_free);   // S^T region may be overwritten
          // masking only where some lane needs it (warp-uniform branch)
          if (__any_sync(0xffffffffu, qlo > q0c || qhi < q0c + 63)) {
#pragma unroll
            for (int k = 0; k < 64; k += 4) {
              const float4 l4 = *reinterpret_cast<const float4*>(sv + q0c + k);  // -lse2
              const float2 x0 = ptx::ffma2(make_float2(pv[k], pv[k + 1]), make_float2(c, c), make_float2(l4.x, l4.y));
              const float2 x1 = ptx::ffma2(make_float2(pv[k + 2], pv[k + 3]), make_float2(c, c), make_float2(l4.z, l4.w));
              const float xs[4] = {x0.x, x0.y, x1.x, x1.y};
#pragma unroll
              for (int u = 0; u < 4; ++u) {
                const int q = q0c + k + u;
                const float pe = bwd_ex2(xs[u], k + u);
                pv[k + u] = (q >= qlo && q <= qhi) ? pe : 0.f;
              }
            }
          } else {
#pragma unroll
            for (int k = 0; k < 64; k += 4) {  // x = S^T c - lse2, two columns per FFMA2 (same rounding as fmaf)
              const float4 l4 = *reinterpret_cast<const float4*>(sv + q0c + k);
              const float2 x0 = ptx::ffma2(make_float2(pv[k], pv[k + 1]), make_float2(c, c), make_float2(l4.x, l4.y));
              const float2 x1 = ptx::ffma2(make_float2(pv[k + 2], pv[k + 3]), make_float2(c, c), make_float2(l4.z, l4.w));
              pv[k] = bwd_ex2(x0.x, k);
              pv[k + 1] = bwd_ex2(x0.y, k + 1);
              pv[k + 2] = bwd_ex2(x1.x, k + 2);
              pv[k + 3] = bwd_ex2(x1.y, k + 3);
            }
          }
          ATTN_CYC_ADD(2);
          // P^T -> SMEM (SW128 K-major: key row krow, 16-B unit u at (u ^ (krow & 7)))
          // once dV of the previous block has read the buffer
          ptx::mbar_wait(&ctrl->dv_done, pt_phase ^ 1);
          ATTN_CYC_ADD(6);
          pt_phase ^= 1;
          {
            uint8_t* rowp = spt + half * (kBM * 128) + krow * 128;
#pragma unroll
            for (int u = 0; u < 8; ++u)
              *reinterpret_cast<uint4*>(rowp + ((u ^ (krow & 7)) << 4)) =
                  make_uint4(ptx::pack_bf16(pv[8 * u + 0], pv[8 * u + 1]), ptx::pack_bf16(pv[8 * u + 2], pv[8 * u + 3]),
                             ptx::pack_bf16(pv[8 * u + 4], pv[8 * u + 5]), ptx::pack_bf16(pv[8 * u + 6], pv[8 * u + 7]));
          }
          ptx::fence_proxy_async_smem();
          __syncwarp();
          if (lane == 0) ptx::mbar_arrive(&ctrl->p_ready);
          ATTN_CYC_ADD(3);
          ptx::mbar_wait(&ctrl->dp_ready, s_phase);
          ATTN_CYC_ADD(4);
          s_phase ^= 1;
          ptx::tc_fence_after();
          uint32_t dp[64];
          ptx::tmem_ld64(trow + kColDP + q0c, dp);   // one wait for 64 columns
#pragma unroll
          for (int cc = 0; cc < 64; cc += 32) {
            uint32_t pd[16];
#pragma unroll
            for (int k = 0; k < 32; k += 4) {
              const float4 d4 = *reinterpret_cast<const float4*>(sv + kBM + q0c + cc + k);
              const float dvv[4] = {d4.x, d4.y, d4.z, d4.w};
#pragma unroll
              for (int u = 0; u < 4; u += 2) {  // dS^T = P^T o (dP^T - D), packed; dvv = -D
                const float2 t = ptx::fadd2(
                    make_float2(__uint_as_float(dp[cc + k + u]), __uint_as_float(dp[cc + k + u + 1])),
                    make_float2(dvv[u], dvv[u + 1]));
                const float2 r = ptx::fmul2(make_float2(pv[cc + k + u], pv[cc + k + u + 1]), t);
                pd[(k + u) >> 1] = ptx::pack_bf16(r.x, r.y);
              }
            }
            ptx::tmem_st16(trow + kColDP + q0c + cc / 2, pd);  // dS^T over consumed dP^T columns
          }
          ptx::tmem_wait_st();
          ptx::tc_fence_before();
          __syncwarp();
          if (lane == 0) ptx::mbar_arrive(&ctrl->ds_ready);
          ATTN_CYC_ADD(5);
          ATTN_CYC_COUNT(7);
        }
      }
      ptx::mbar_wait(&ctrl->o_ready, o_phase);
      o_phase ^= 1;
      ptx::tc_fence_after();
      const bool valid = kglob < p.N;
      const long long ro = ((long long)(b * p.Hkv + g) * p.N + (valid ? kglob : 0)) * p.d_real;
      {
        const int which = half;  // column half 0 writes dV, half 1 writes dK
        __nv_bfloat16* dst = (which == 0 ? p.dv : p.dk) + ro;
        const float f = which == 0 ? 1.f : p.scale;
        const uint32_t col = which == 0 ? kColDV : kColDK;
#pragma unroll
        for (int cc = 0; cc < D; cc += 32) {
          uint32_t o[32];
          ptx::tmem_ld32(trow + col + cc, o);
          uint32_t pk[16];
#pragma unroll
          for (int k = 0; k < 16; ++k)
            pk[k] = ptx::pack_bf16(__uint_as_float(o[2 * k]) * f, __uint_as_float(o[2 * k + 1]) * f);
          if (valid) {
#pragma unroll
            for (int k = 0; k < 4; ++k)
              if (cc + 8 * k < p.d_real)
                reinterpret_cast<uint4*>(dst)[cc / 8 + k] =
                    make_uint4(pk[4 * k], pk[4 * k + 1], pk[4 * k + 2], pk[4 * k + 3]);
          }
        }
      }
      ptx::tc_fence_before();
    }
    ATTN_CYC_WRITE(p.dbg, warp - 4)
  }
  ptx::tc_fence_before();
  __syncthreads();
  if (warp == 2) {
    ptx::tc_fence_after();
    ptx::tmem_dealloc(tmem, 512);
  }
}

}  // namespace bwd
}  // namespace attn
