// attn_bwd_fused_sm100.cuh -- single-pass attention backward (PAPER.md:157-165,
// eq:ba) for head dims up to 64 on sm_100a.
//
// The two-kernel backward (attn_bwd_sm100.cuh) computes P and dS twice: once
// in the dQ kernel (query-parallel) and once in the dK/dV kernel
// (key-parallel), 7 matmuls executed for the 5 of eq:ba.  This kernel is the
// dK/dV kernel extended with dQ: per (key block j, query block i) it also
// runs dQ_i += dS K_j and ADDS that 128 x D fp32 tile into a global fp32
// accumulator with a TMA tensor reduce (cp.reduce.async.bulk.tensor .add), so
// P and dS are computed once and 5 matmuls execute.  A small kernel then
// writes dq = bf16(scale * acc).
//
// The fp32 adds of different key blocks land in L2 in whatever order the
// CTAs reach them, so dq may differ in the last bits between runs (dk and dv
// are accumulated in TMEM in a fixed order and stay bit-reproducible); the
// two-kernel path remains for callers that need bit-identical dq
// (ATTN_BWD_DETERMINISTIC).
//
// At D = 64 an SS MMA with N = 64 reads 6 KB of SMEM per 32 tensor cycles,
// more than SMEM delivers, so every operand that can come from TMEM does:
//   S^T  = K Q_i^T       SS   (K resident, Q_i streamed)
//   dP^T = V dO_i^T      SS
//   dV  += P^T dO_i      TS   (P^T bf16 in TMEM, written by the elementwise warps)
//   dK  += dS^T Q_i      TS   (dS^T bf16 in TMEM over dP^T)
//   dQ_i = dS K_j        SS   (dS^T from SMEM read MN-major: the transpose is a
//                              descriptor bit; no TMEM layout has query rows)
// Roles (512 threads): warp 0 TMA, 1 MMA, 2 scheduler + TMEM allocation,
// 3 idle, 4-11 elementwise (TMEM lane = key row, two query halves), 12-15 dQ
// drain (TMEM lane = query row).
//   TMEM: S^T [0,128) | dP^T, then dS^T [128,256) | dV [256,320) | dK [320,384)
//         | dQ [384,448) | P^T bf16 [448,512)
//   SMEM: K, V (resident per unit) | 2-stage ring of (Q_i, dO_i, -lse2 / -D of
//         the block's 128 queries) | dS^T | two fp32 dQ staging tiles.
// MMA order per block:  S^T(i+1) . dV(i) . dK(i) . dQ(i) . dP^T(i+1).
#pragma once
#include "attn_bwd_sm100.cuh"
#include "instrument.cuh"

namespace attn {
namespace bwd {

constexpr int kThreadsF = 512;
constexpr int kDrainWarps = 4;
// setmaxnreg split of the 512 x 128 register pool (the MMA warp keeps ~100
// registers of descriptors live; the drain needs 32 values + addresses)
constexpr int kFOtherRegs = 104, kFDrainRegs = 48, kFEwRegs = 176;
static_assert(128 * (128 - kFOtherRegs) + 128 * (128 - kFDrainRegs) >= 256 * (kFEwRegs - 128),
              "fused backward setmaxnreg budget exceeds the register pool");

template <int D>
struct FCfg {
  static constexpr int kChunks = D / 64;
  static constexpr int kTile = kBM * D * 2;
  static constexpr int kStages = 2;
  static constexpr int kVecBytes = 2 * kBM * 4;                  // -lse2 | -D of one query block
  static constexpr int kStage = 2 * kTile + 1024;                // Q_i | dO_i | vectors (1024-B aligned stages)
  static constexpr int kOffCtrl = 0;
  static constexpr int kOffA = 1024;                             // K, V
  static constexpr int kOffRing = kOffA + 2 * kTile;
  static constexpr int kOffDS = kOffRing + kStages * kStage;     // dS^T bf16 (two 64-query SW128 chunks)
  static constexpr int kStgBytes = kBM * D * 4;                  // one fp32 dQ tile
  static constexpr int kStg = 2;
  static constexpr int kOffStg = kOffDS + kBM * kBM * 2;
  static constexpr int kSmemBytes = kOffStg + kStg * kStgBytes;
  static_assert(kSmemBytes <= 232448, "fused backward SMEM over the 227 KB opt-in limit");
};

// Walks the blocks of a dK/dV unit (key block j) in order: query head hh of
// the group, query block i.  Non-causal units start at query block j and
// wrap, so the CTAs working on one head add into different dQ tiles at any
// moment; causal units start at j anyway.  Incremental: no integer division
// (which would take MUFU.RCP slots from the exps) on the elementwise path.
template <bool kCausal>
struct BlockWalk {
  int j, i0, nblk, hh, i;
  __device__ __forceinline__ BlockWalk(int j_, int nblk_)
      : j(j_), i0(dkdv_first_qblock<kCausal>(j_)), nblk(nblk_), hh(0), i(j_) {}
  __device__ __forceinline__ int count(int G) const { return G * (nblk - i0); }
  __device__ __forceinline__ void next() {
    if (++i == nblk) i = i0;
    if (i == j) ++hh;
  }
};

// Per-row inputs of the fused kernel, in blocks of 128 query rows so one bulk
// copy brings a block's: vec[(bh*nblk + i)*256 + r] = -lse[row]*log2(e) and
// vec[... + 128 + r] = -rowsum(dO o O)[row] for row = i*128 + r < N, 0 past N.
// One warp per (padded) row.
// drow (optional): rowsum(dO o O) per row as well (the two-pass dQ kernel's input).
__global__ void attn_bwd_prep_kernel(const __nv_bfloat16* __restrict__ o, const __nv_bfloat16* __restrict__ dout,
                                     const float* __restrict__ lse, float* __restrict__ vec, long long bh_count, int N,
                                     int nblk, int d, float* __restrict__ drow = nullptr) {
  const long long prow = (long long)blockIdx.x * (blockDim.x / 32) + threadIdx.x / 32;
  const int lane = threadIdx.x & 31;
  const long long npad = (long long)nblk * kBM;
  if (prow >= bh_count * npad) return;
  const long long bh = prow / npad;
  const int n = (int)(prow - bh * npad);
  float acc = 0.f, l2 = 0.f;
  if (n < N) {
    const long long row = bh * N + n;
    const __nv_bfloat162* a = reinterpret_cast<const __nv_bfloat162*>(o + row * d);
    const __nv_bfloat162* b = reinterpret_cast<const __nv_bfloat162*>(dout + row * d);
    for (int c = lane; c < d / 2; c += 32) {
      const float2 x = __bfloat1622float2(a[c]), y = __bfloat1622float2(b[c]);
      acc = fmaf(x.x, y.x, fmaf(x.y, y.y, acc));
    }
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, off);
    l2 = lse[row] * 1.4426950408889634f;
  }
  if (lane == 0) {
    float* blk = vec + (bh * nblk + n / kBM) * (2 * kBM);
    blk[n % kBM] = -l2;
    blk[kBM + n % kBM] = -acc;
    if (drow != nullptr && n < N) drow[bh * N + n] = acc;
  }
}

// dq[b,h,n,c] = bf16(scale * acc[b,h,n,c]) for c < d (acc rows are dpad wide)
__global__ void attn_bwd_dq_convert_kernel(const float* __restrict__ acc, __nv_bfloat16* __restrict__ dq,
                                           long long rows, int d, int dpad, float scale) {
  const long long t = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  const int per_row = d / 8;
  if (t >= rows * per_row) return;
  const long long r = t / per_row;
  const int c = (int)(t - r * per_row) * 8;
  const float4 a = *reinterpret_cast<const float4*>(acc + r * dpad + c);
  const float4 b = *reinterpret_cast<const float4*>(acc + r * dpad + c + 4);
  *reinterpret_cast<uint4*>(dq + r * d + c) =
      make_uint4(ptx::pack_bf16(a.x * scale, a.y * scale), ptx::pack_bf16(a.z * scale, a.w * scale),
                 ptx::pack_bf16(b.x * scale, b.y * scale), ptx::pack_bf16(b.z * scale, b.w * scale));
}

template <int D, bool kCausal>
__global__ void __launch_bounds__(kThreadsF, 1)
    attn_bwd_fused_kernel(const __grid_constant__ CUtensorMap tm_q, const __grid_constant__ CUtensorMap tm_do,
                          const __grid_constant__ CUtensorMap tm_k, const __grid_constant__ CUtensorMap tm_v,
                          const __grid_constant__ CUtensorMap tm_acc, const BwdParams p) {
  static_assert(D == 64, "TMEM holds S^T, dP^T, dV, dK, dQ and P^T only for D <= 64");
  using C = FCfg<D>;
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = smem_raw;
  if (ptx::smem_u32(smem_raw) & 1023) __trap();  // layout relies on a 1024-B aligned base
  uint8_t* skv = smem + C::kOffA;
  uint8_t* ring = smem + C::kOffRing;
  uint8_t* sds = smem + C::kOffDS;
  uint8_t* stg = smem + C::kOffStg;
  BCtrl* ctrl = reinterpret_cast<BCtrl*>(smem + C::kOffCtrl);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  constexpr uint32_t kColS = 0, kColDP = 128, kColDV = 256, kColDK = 320, kColDQ = 384, kColPT = 448;
  constexpr int kEw = 8;
  const float* vec = p.dvec;  // attn_bwd_prep_kernel's blocks

  if (threadIdx.x == 0) {
    for (int i = 0; i < kSchedRing; ++i) {
      ptx::mbar_init(&ctrl->sched_full[i], 1);
      ptx::mbar_init(&ctrl->sched_empty[i], 2 + kEw + kDrainWarps);
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
    ptx::mbar_init(&ctrl->dk_done, 1);
    ptx::mbar_init(&ctrl->o_ready, 1);
    ptx::mbar_init(&ctrl->dq_full[0], 1);
    ptx::mbar_init(&ctrl->dq_empty[0], kDrainWarps);
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

  if (warp < 4) {
    ptx::setmaxnreg_dec<kFOtherRegs>();
    if (warp == 0 && lane == 0) {
      // ------------------------------------------------------------ TMA producer
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
        BlockWalk<kCausal> w(j, p.nblk);
        const int n = w.count(p.G);
        for (int it = 0; it < n; ++it, w.next()) {
          const int i = w.i, bh = b * p.Hq + g * p.G + w.hh;
          ptx::mbar_wait(&ctrl->ring_empty[stage], r_phase ^ 1);
          ptx::mbar_arrive_expect_tx(&ctrl->ring_full[stage], 2 * C::kTile + C::kVecBytes);
          uint8_t* dst = ring + stage * C::kStage;
#pragma unroll
          for (int c = 0; c < C::kChunks; ++c) {
            ptx::tma_load_3d(dst + c * kBM * 128, &tm_q, &ctrl->ring_full[stage], c * 64, i * kBM, bh, pol_q);
            ptx::tma_load_3d(dst + C::kTile + c * kBM * 128, &tm_do, &ctrl->ring_full[stage], c * 64, i * kBM, bh,
                             pol_q);
          }
          ptx::bulk_load(dst + 2 * C::kTile, vec + ((long long)bh * p.nblk + i) * (2 * kBM), C::kVecBytes,
                         &ctrl->ring_full[stage], pol_q);
          if (++stage == C::kStages) { stage = 0; r_phase ^= 1; }
        }
      }
    } else if (warp == 1) {
      // ------------------------------------------------------------------- MMA
      BSchedReader sr;
      constexpr uint32_t idesc_s = ptx::idesc_bf16_f32(kBM, kBM, 0, 0);  // S^T, dP^T: K-major A and B
      constexpr uint32_t idesc_g = ptx::idesc_bf16_f32(kBM, D, 0, 1);    // dV, dK: A (TMEM), B MN-major
      constexpr uint32_t idesc_q = ptx::idesc_bf16_f32(kBM, D, 1, 1);    // dQ: A = dS MN-major, B = K MN-major
      const uint64_t dkv0 = ptx::smem_desc_sw128(ptx::smem_u32(skv), 16, 1024);
      const uint64_t dkm = ptx::smem_desc_sw128(ptx::smem_u32(skv), kBM * 128, 1024);  // K_j as [keys x D]
      const uint64_t dr0 = ptx::smem_desc_sw128(ptx::smem_u32(ring), 16, 1024);
      const uint64_t drm0 = ptx::smem_desc_sw128(ptx::smem_u32(ring), kBM * 128, 1024);
      const uint64_t ddsm = ptx::smem_desc_sw128(ptx::smem_u32(sds), kBM * 128, 1024);  // dS, MN-major
      uint32_t a_phase = 0, r_phase = 0, p_phase = 0;
      int stage = 0;
      auto ss_mma = [&](uint32_t d_col, uint64_t a, uint64_t b) {  // [128 x 128] = A[128 x D] B[128 x D]^T
#pragma unroll
        for (int k = 0; k < D / 16; ++k) {
          const uint32_t off = ((k >> 2) * (kBM * 128) + (k & 3) * 32) >> 4;
          ptx::mma_ss(tmem + d_col, a + off, b + off, idesc_s, k > 0 ? 1u : 0u);
        }
      };
      auto rows16 = [](uint64_t base, int k) { return base + (uint64_t)((k * 16 * 128) >> 4); };  // MN-major k-step
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
          const uint64_t qd = dr0 + (uint64_t)((st * C::kStage) >> 4);
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
          const uint64_t qm = drm0 + (uint64_t)((cur * C::kStage) >> 4);  // Q_i as [queries x D] MN-major
          const uint64_t dom = qm + (uint64_t)(C::kTile >> 4);            // dO_i likewise
          const uint64_t qd = dr0 + (uint64_t)((nst * C::kStage) >> 4);
          ptx::mbar_wait(&ctrl->s_free, p_phase);
          ptx::tc_fence_after();
          if (nxt) {
            ptx::mbar_wait(&ctrl->ring_full[nst], nph);
            ptx::tc_fence_after();
            if (ptx::elect_one_sync()) {
              ss_mma(kColS, dkv0, qd);  // S^T(it+1)
              ptx::mma_commit(&ctrl->s_ready);
            }
            __syncwarp();
          }
          ptx::mbar_wait(&ctrl->p_ready, p_phase);
          ptx::tc_fence_after();
          if (ptx::elect_one_sync()) {
#pragma unroll
            for (int k = 0; k < kBM / 16; ++k)  // dV += P^T dO_i  (A = P^T bf16 pairs in TMEM)
              ptx::mma_ts(tmem + kColDV, tmem + kColPT + k * 8, rows16(dom, k), idesc_g, (it > 0 || k > 0) ? 1u : 0u);
            ptx::mma_commit(&ctrl->dv_done);
          }
          __syncwarp();
          ptx::mbar_wait(&ctrl->ds_ready, p_phase);
          ptx::mbar_wait(&ctrl->dq_empty[0], p_phase ^ 1);  // drain of the previous dQ tile has read TMEM
          p_phase ^= 1;
          ptx::tc_fence_after();
          if (ptx::elect_one_sync()) {
            // dK += dS^T Q_i: A = dS^T bf16 in TMEM over dP^T (queries 0-63 in
            // columns [0,32) of the region, 64-127 in [64,96): each column half
            // of the elementwise warps overwrote only columns it had read)
#pragma unroll
            for (int k = 0; k < kBM / 16; ++k)
              ptx::mma_ts(tmem + kColDK, tmem + kColDP + k * 8 + (k >= 4 ? 32 : 0), rows16(qm, k), idesc_g,
                          (it > 0 || k > 0) ? 1u : 0u);
#pragma unroll
            for (int k = 0; k < kBM / 16; ++k)  // dQ_i (this key block's part) = dS K_j
              ptx::mma_ss(tmem + kColDQ, rows16(ddsm, k), rows16(dkm, k), idesc_q, k > 0 ? 1u : 0u);
            ptx::mma_commit(&ctrl->dq_full[0]);
            ptx::mma_commit(&ctrl->dk_done);  // dS^T SMEM free
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
    }
  } else if (warp < 12) {
    // ------------------------------------------------------------ elementwise
    // TMEM lane = key row (warp & 3), column half `half` = queries
    // [64*half, 64*half+64).  Phase A: P^T = exp2(S^T*c - lse2) (registers;
    // bf16 pairs to TMEM for dV); phase B: dS^T = P^T o (dP^T - D), bf16
    // pairs to TMEM over dP^T (dK) and to SMEM (dQ).
    ptx::setmaxnreg_inc<kFEwRegs>();
    const int quarter = warp & 3, krow = quarter * 32 + lane;
    const int half = (warp - 4) >> 2, q0c = half * 64;
    const uint32_t trow = tmem + ((uint32_t)(quarter * 32) << 16);
    const float c = p.scale_log2;
    BSchedReader sr;
    uint32_t s_phase = 0, o_phase = 0, blk = 0, pt_phase = 0, ds_phase = 0;
    const int swz = (krow & 7) << 4;
    uint8_t* dsrow = sds + half * (kBM * 128) + krow * 128;
    ATTN_CYC_DECL()
    while (true) {
      const int4 e = sr.next(ctrl);
      if (!e.w) break;
      const int b = e.x, g = e.y, j = e.z;
      const int kglob = j * kBM + krow;
      BlockWalk<kCausal> w(j, p.nblk);
      const int n = w.count(p.G);
      for (int it = 0; it < n; ++it, ++blk, w.next()) {
        ATTN_CYC_START();
        const int i = w.i;
        // this block's -lse2 / -D (bulk-copied with Q_i, dO_i into ring stage blk % 2)
        const int rs = (int)(blk % C::kStages);
        ptx::mbar_wait(&ctrl->ring_full[rs], (blk / C::kStages) & 1);
        const float* sv = reinterpret_cast<const float*>(ring + rs * C::kStage + 2 * C::kTile);
        int qlo = 0, qhi = kBM - 1;
        if (kCausal && i == j) qlo = krow;             // query >= key
        if (i == p.nblk - 1) qhi = p.N - 1 - i * kBM;  // ragged tail
        float pv[64];
        ATTN_CYC_ADD(0);
        ptx::mbar_wait(&ctrl->s_ready, s_phase);
        ATTN_CYC_ADD(1);
        ptx::tc_fence_after();
        ptx::tmem_ld64(trow + kColS + q0c, reinterpret_cast<uint32_t*>(pv));
        ptx::tc_fence_before();
        __syncwarp();
        if (lane == 0) ptx::mbar_arrive(&ctrl->s_free);
        // x = S^T * c - lse2, two columns per FFMA2 (same rounding as fmaf)
#pragma unroll
        for (int k = 0; k < 64; k += 4) {
          const float4 l4 = *reinterpret_cast<const float4*>(sv + q0c + k);
          const float2 x0 = ptx::ffma2(make_float2(pv[k], pv[k + 1]), make_float2(c, c), make_float2(l4.x, l4.y));
          const float2 x1 = ptx::ffma2(make_float2(pv[k + 2], pv[k + 3]), make_float2(c, c), make_float2(l4.z, l4.w));
          pv[k] = bwd_ex2(x0.x, k);
          pv[k + 1] = bwd_ex2(x0.y, k + 1);
          pv[k + 2] = bwd_ex2(x1.x, k + 2);
          pv[k + 3] = bwd_ex2(x1.y, k + 3);
        }
        if (__any_sync(0xffffffffu, qlo > q0c || qhi < q0c + 63)) {  // masking only where some lane needs it
#pragma unroll
          for (int k = 0; k < 64; ++k)
            if (q0c + k < qlo || q0c + k > qhi) pv[k] = 0.f;
        }
        ATTN_CYC_ADD(2);
        // P^T -> TMEM (bf16 pairs, columns [32*half, 32*half+32) of the P^T
        // region) once dV of the previous block has read it
        ptx::mbar_wait(&ctrl->dv_done, pt_phase ^ 1);
        pt_phase ^= 1;
        ptx::tc_fence_after();
        {
          uint32_t pk[32];
#pragma unroll
          for (int k = 0; k < 32; ++k) pk[k] = ptx::pack_bf16(pv[2 * k], pv[2 * k + 1]);
          ptx::tmem_st32(trow + kColPT + 32 * half, pk);
        }
        ptx::tmem_wait_st();
        ptx::tc_fence_before();
        __syncwarp();
        if (lane == 0) ptx::mbar_arrive(&ctrl->p_ready);
        ATTN_CYC_ADD(3);
        ptx::mbar_wait(&ctrl->dp_ready, s_phase);
        ATTN_CYC_ADD(4);
        s_phase ^= 1;
        ptx::tc_fence_after();
        {
          uint32_t dp[64];
          ptx::tmem_ld64(trow + kColDP + q0c, dp);
#pragma unroll
          for (int k = 0; k < 64; k += 4) {  // dS^T = P^T o (dP^T - D), two columns per FADD2 / FMUL2
            const float4 d4 = *reinterpret_cast<const float4*>(sv + kBM + q0c + k);
            const float2 t0 = ptx::fadd2(make_float2(__uint_as_float(dp[k]), __uint_as_float(dp[k + 1])),
                                         make_float2(d4.x, d4.y));
            const float2 t1 = ptx::fadd2(make_float2(__uint_as_float(dp[k + 2]), __uint_as_float(dp[k + 3])),
                                         make_float2(d4.z, d4.w));
            const float2 s0 = ptx::fmul2(make_float2(pv[k], pv[k + 1]), t0);
            const float2 s1 = ptx::fmul2(make_float2(pv[k + 2], pv[k + 3]), t1);
            pv[k] = s0.x; pv[k + 1] = s0.y; pv[k + 2] = s1.x; pv[k + 3] = s1.y;
          }
        }
        uint32_t pk[32];
#pragma unroll
        for (int k = 0; k < 32; ++k) pk[k] = ptx::pack_bf16(pv[2 * k], pv[2 * k + 1]);
        ptx::tmem_st32(trow + kColDP + (half ? 64 : 0), pk);  // dS^T over the dP^T columns this half read
        ATTN_CYC_ADD(5);
        // dS^T -> SMEM (dQ's A operand) once dQ of the previous block has read it
        ptx::mbar_wait(&ctrl->dk_done, ds_phase ^ 1);
        ds_phase ^= 1;
#pragma unroll
        for (int u = 0; u < 8; ++u)
          *reinterpret_cast<uint4*>(dsrow + ((u << 4) ^ swz)) =
              make_uint4(pk[4 * u], pk[4 * u + 1], pk[4 * u + 2], pk[4 * u + 3]);
        ptx::fence_proxy_async_smem();
        ptx::tmem_wait_st();
        ptx::tc_fence_before();
        __syncwarp();
        if (lane == 0) ptx::mbar_arrive(&ctrl->ds_ready);
        ATTN_CYC_ADD(6);
        ATTN_CYC_COUNT(7);
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
  } else {
    // -------------------------------------------------------------- dQ drain
    // TMEM lane = query row of the block; each finished dQ tile goes TMEM ->
    // registers -> SMEM (SW128 fp32 boxes of 128 rows x 32) -> TMA tensor
    // reduce-add into the fp32 accumulator [B*Hq][N][D] (rows past N are out
    // of bounds: skipped).
    ptx::setmaxnreg_dec<kFDrainRegs>();
    const int quarter = warp & 3, row = quarter * 32 + lane;
    const uint32_t trow = tmem + ((uint32_t)(quarter * 32) << 16);
    const bool leader = threadIdx.x == 12 * 32;
    const int swz = (row & 7) << 4;
    BSchedReader sr;
    uint32_t nq_tiles = 0;
    while (true) {
      const int4 e = sr.next(ctrl);
      if (!e.w) break;
      const int b = e.x, g = e.y, j = e.z;
      BlockWalk<kCausal> w(j, p.nblk);
      const int n = w.count(p.G);
      for (int it = 0; it < n; ++it, w.next()) {
        const int i = w.i, bh = b * p.Hq + g * p.G + w.hh;
        uint8_t* sbuf = stg + (nq_tiles & 1) * C::kStgBytes;
        if (leader) ptx::bulk_wait_group_read<1>();  // the reduce that last used sbuf has read it
        ptx::named_bar_sync(2, 32 * kDrainWarps);
        ptx::mbar_wait(&ctrl->dq_full[0], nq_tiles & 1);
        ptx::tc_fence_after();
#pragma unroll
        for (int cb = 0; cb < D / 32; ++cb) {
          uint32_t v[32];
          ptx::tmem_ld32(trow + kColDQ + cb * 32, v);
          uint8_t* rowp = sbuf + cb * (kBM * 128) + row * 128;
#pragma unroll
          for (int u = 0; u < 8; ++u)
            *reinterpret_cast<uint4*>(rowp + ((u << 4) ^ swz)) = make_uint4(v[4 * u], v[4 * u + 1], v[4 * u + 2], v[4 * u + 3]);
        }
        ptx::tc_fence_before();
        __syncwarp();
        if (lane == 0) ptx::mbar_arrive(&ctrl->dq_empty[0]);
        ptx::fence_proxy_async_smem();
        ptx::named_bar_sync(2, 32 * kDrainWarps);
        if (leader) {
#pragma unroll
          for (int cb = 0; cb < D / 32; ++cb) ptx::tma_reduce_add_3d(&tm_acc, sbuf + cb * (kBM * 128), cb * 32, i * kBM, bh);
          ptx::bulk_commit_group();
        }
        ++nq_tiles;
      }
    }
    if (leader) ptx::bulk_wait_group<0>();
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
