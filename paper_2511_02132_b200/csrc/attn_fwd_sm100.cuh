// attn_fwd_sm100.cuh -- persistent, warp-specialised FlashAttention-2-style
// forward kernel for sm_100a (tcgen05 + TMEM + TMA), with the paper's
// mapping-selectable work scheduler.
//
// Math (PAPER.md eq:fa, lines 149-155, and the FA online softmax with its
// cross-tile "fix-up"): for every query row i of a 128-row
// block, over key blocks j of 128 keys
//     S_j  = Q K_j^T                           (tcgen05.mma, fp32 in TMEM)
//     m'   = max(m, rowmax(S_j))  (kept stale unless it grows by > 8 in log2)
//     P_j  = exp2(S_j*c - m'*c),  c = scale*log2(e)   (bf16, written to TMEM)
//     l    = l*exp2((m-m')c) + rowsum(P_j);   O = O*exp2((m-m')c) (fix-up)
//     O   += P_j V_j                           (tcgen05.mma, A from TMEM)
// and finally O / l in bf16.
//
// CTA layout (384 threads, one CTA per SM, persistent):
//   warp 0      TMA producer: Q pair, then K_j / V_j into a ring of slots
//   warp 1      MMA issuer (one elected lane): S0, S1, PV0, PV1 ... per key block
//   warp 2      TMEM allocator + work scheduler (atomic pops from the queues
//               of the active mapping, broadcast through a shared-memory ring)
//   warp 3      idle
//   warps 4-7   softmax + fix-up + epilogue of query tile 0 (one row/thread)
//   warps 8-11  same for query tile 1
// TMEM (512 columns): S0 [0,128) S1 [128,256) O0 [256,256+D) O1 [256+D,256+2D);
// P_i (bf16 pairs) aliases the first 64 columns of S_i.
#pragma once
#include <cuda.h>
#include <cuda_bf16.h>

#include <cstdint>
#include <type_traits>

#include "../../include/attn_numa.h"
#include "attn_sched.h"
#include "instrument.cuh"
#include "ptx.cuh"

namespace attn {

constexpr int kBlockM = 128;  // query rows per tile (the paper's BLOCK_M)
constexpr int kBlockN = 128;  // keys per K/V block
#ifndef ATTN_KV_EVICT_LAST
#define ATTN_KV_EVICT_LAST 0
#endif
#ifndef ATTN_O_EVICT_FIRST
#define ATTN_O_EVICT_FIRST 0
#endif
#ifndef ATTN_EXP_F16X2
#define ATTN_EXP_F16X2 0
#endif
#ifndef ATTN_SPLIT
#define ATTN_SPLIT 1
#endif
// P is published to the MMA warp in kPParts column slices (O += P V starts on
// the first slice while the softmax computes the rest; 4 slices measured slower).
#ifndef ATTN_P_PARTS
#define ATTN_P_PARTS 2
#endif
constexpr int kPParts = ATTN_P_PARTS;
// Head dim <= 64 (plain CTAs): P gets its own TMEM columns (the 128 that
// S0 S1 O0 O1 leave free) instead of aliasing S, so S_t(j+1) is issued as soon
// as the softmax has loaded S_t(j) into registers and each tile's softmax runs
// back to back instead of waiting for the PV -> S -> softmax round trip.
#ifndef ATTN_SEP_P
#define ATTN_SEP_P 1
#endif
// softmax warps per (tile, TMEM lane quarter): each handles kBlockN / kSplit
// columns of its 32 rows, so two warps share each SMSP's MUFU per tile.
constexpr int kSplit = ATTN_SPLIT;
constexpr int kSoftmaxWarps = 8 * kSplit;
constexpr int kThreads = 128 + 32 * kSoftmaxWarps;
static_assert(kPParts == 2 || (kPParts == 4 && kSplit == 1), "P slices: 2, or 4 with one warp per row");
constexpr int kSchedRing = 2;
constexpr int kTmemCols = 512;
constexpr int kDoneCounter = kMaxQueues * 32;  // counters[] index of the CTA-done count
constexpr float kRescaleThreshold = 8.0f;  // log2 units; see DESIGN.md "fix-up"
#ifndef ATTN_EMU_PERIOD
#define ATTN_EMU_PERIOD 8
#endif
#ifndef ATTN_SETMAXNREG
#define ATTN_SETMAXNREG 1
#endif

constexpr int kEmuPeriod = ATTN_EMU_PERIOD;  // every kEmuPeriod-th exp2 pair runs on the FMA pipe (0: none)
// Head dim <= 64: half the tensor work per exp, so the exps bound the kernel
// (MUFU alone would cap it near 57% of the tensor peak) and a larger share
// goes to the FMA-pipe polynomial.
#ifndef ATTN_EMU_PERIOD_D64
#define ATTN_EMU_PERIOD_D64 8
#endif
template <int D>
constexpr int emu_period() { return D <= 64 ? ATTN_EMU_PERIOD_D64 : kEmuPeriod; }
// Register split (setmaxnreg).  The CTA's register pool is what the launch
// allocated: kThreads * kInitRegs (ptxas caps a thread at 65536 / kThreads,
// rounded down to a multiple of 8).  Warps 0-3 release registers that the
// softmax warps then claim; .inc blocks forever if the pool is short, so the
// budget is checked at compile time.
constexpr int kInitRegs = ((65536 / kThreads) / 8) * 8;
constexpr int kOtherRegs = (kSplit == 1) ? 80 : 64;
constexpr int kSoftmaxRegs = (kSplit == 1) ? 208 : 104;
static_assert(128 * (kInitRegs - kOtherRegs) >= 32 * kSoftmaxWarps * (kSoftmaxRegs - kInitRegs),
              "setmaxnreg budget exceeds the CTA register pool");

template <int D>
struct Cfg {
  static constexpr int kChunks = D / 64;                  // 128-byte swizzle atoms per row
  static constexpr int kQTileBytes = kBlockM * D * 2;     // one 128-row Q tile
  static constexpr int kKVBytes = kBlockN * D * 2;        // one K or V block
#ifndef ATTN_KV_STAGES
#define ATTN_KV_STAGES 4
#endif
#ifndef ATTN_KV_STAGES_D64
#define ATTN_KV_STAGES_D64 8
#endif
  static constexpr int kStages = (D == 128) ? ATTN_KV_STAGES : ATTN_KV_STAGES_D64;  // K/V ring slots
  static constexpr int kOffQ = 0;
  static constexpr int kOffKV = 2 * kQTileBytes;
  static constexpr int kOffCtrl = kOffKV + kStages * kKVBytes;
  static constexpr int kCtrlBytes = (kSplit == 1) ? 1024 : 8192;
  static constexpr int kSmemBytes = kOffCtrl + kCtrlBytes + 1024;  // + alignment slack
  // TMEM columns: S_t at 128*t, O_t at 256 + D*t
  static __device__ __forceinline__ uint32_t col_s(int t) { return 128u * t; }
  static __device__ __forceinline__ uint32_t col_o(int t) { return 256u + (uint32_t)D * t; }
  // separate-P layout (D <= 64): P_t (bf16 pairs, 64 columns) after O1
  static __device__ __forceinline__ uint32_t col_p(int t) { return 256u + 2u * D + 64u * t; }
};

constexpr int kMaxDst = 8;  // ATTN_MAX_DST

struct KernelParams {
  int B, Hq, Hkv, N, G, U, nblk;
  int Usched;        // units per head in the queues: U, or ceil(U/2) cluster units (kCl == 2, adjacent mode)
  int Hsched;        // heads in the queues: Hq, or Hq/2 head pairs (kCl == 2, head-pair mode)
  int pair_heads;    // kCl == 2: 1 = the pair takes unit u of query heads 2h', 2h'+1 (one KV group);
                     //           0 = the pair takes units 2u', 2u'+1 of one head
  int d_real;        // head dim of the tensors (<= D; TMA zero-fills columns d_real..D-1)
  float scale_log2;  // scale * log2(e), >= 0
  __nv_bfloat16* o;   // == o_dst[0]
  // Output destinations (replicated output, SURVEY §8(e) fused alternative):
  // every finished O tile is stored into each o_dst[i], a [B][Hq_out][N][d]
  // buffer, at head h_off + h.  Plain call: n_dst = 1, Hq_out = Hq, h_off = 0.
  // Peer destinations are NVLink-mapped buffers of other GPUs (P2P stores).
  __nv_bfloat16* o_dst[kMaxDst];
  int n_dst, Hq_out, h_off;
  float* lse;        // optional [B][Hq][N] natural-log row LSE (backward input), may be null
  int kv_tx_bytes;   // bytes one K or V block lands in a CTA (kKVBytes, or 128 * d_real * 2 with kOnesL)
  SchedParams sched;
  int* counters;                 // one int per queue, 32 ints apart, then the done count
  const signed char* domain_of_smid;
  int n_smid;
  attn_trace_rec_t* trace;
  long long trace_cap;
};

struct __align__(16) Ctrl {
  uint64_t sched_full[kSchedRing];
  uint64_t sched_empty[kSchedRing];
  uint64_t q_full, q_empty;
  uint64_t kv_full[16];
  uint64_t kv_empty[16];
  uint64_t s_ready[2];
  uint64_t p_ready[2][4];   // [tile][slice of P]  softmax -> MMA
  uint64_t o_ready[2];
  uint64_t s_free[2];       // separate-P layout: softmax loaded S_t -> MMA may overwrite it
  uint64_t p_free[2];       // separate-P layout: PV_t done reading P_t (and adding into O_t)
  int4 entry[kSchedRing];  // (b, h, u, valid)
  uint32_t tmem_base;
};
// cross-warp row reductions of the kSplit == 2 softmax (after Ctrl in SMEM)
struct SplitRed {
  float red[2][4][2][2][32];   // [tile][quarter][half][parity][lane] partial row max
  float lsum[2][4][2][32];     // [tile][quarter][half][lane] partial row sum (epilogue)
};

// Key blocks each tile of unit (u) needs: n0 for block 2u, n1 for block 2u+1.
template <bool kCausal>
__device__ __forceinline__ void unit_blocks(int u, int nblk, int& n0, int& n1) {
  const bool has1 = (2 * u + 1) < nblk;
  if (kCausal) {  // kBlockN == kBlockM: block qb needs key blocks 0..qb
    n0 = 2 * u + 1;
    n1 = has1 ? 2 * u + 2 : 0;
  } else {
    n0 = nblk;
    n1 = has1 ? nblk : 0;
  }
}

// Consumer side of the scheduler ring.  kCl == 2 (CTA-pair clusters): the
// entries are written by the leader CTA's scheduler into both CTAs, and every
// consumer of both CTAs releases the slot on the LEADER's sched_empty.
template <int kCl, class CT = Ctrl>
struct SchedReader {
  int stage = 0;
  uint32_t phase = 0;
  __device__ __forceinline__ void release(CT* c, int st) {
    if constexpr (kCl == 1) ptx::mbar_arrive(&c->sched_empty[st]);
    // relaxed: the entry is already in registers, and a cluster-scope release
    // here would wait for every outstanding global store (MEMBAR.ALL.GPU)
    else ptx::mbar_arrive_cluster_relaxed(ptx::mapa_shared(ptx::smem_u32(&c->sched_empty[st]), 0));
  }
  __device__ __forceinline__ int4 next(CT* c, bool arrive) {
    if constexpr (kCl == 1) ptx::mbar_wait(&c->sched_full[stage], phase);
    else ptx::mbar_wait_cluster(&c->sched_full[stage], phase);
    const volatile int* ve = reinterpret_cast<const volatile int*>(&c->entry[stage]);
    const int4 e = make_int4(ve[0], ve[1], ve[2], ve[3]);
    if (arrive) release(c, stage);
    if (++stage == kSchedRing) { stage = 0; phase ^= 1; }
    return e;
  }
  __device__ __forceinline__ void release_prev(CT* c) { release(c, (stage + kSchedRing - 1) % kSchedRing); }
};

// This CTA's (head, unit) of a scheduler entry (b, h, u, w).  kCl == 1: (h, u).
// kCl == 2, head pairs: (2h + rank, u) -- both query heads of one KV group, so
// the pair needs exactly the same K/V blocks; adjacent units: (h, 2u + rank),
// unit -1 when the pair has only one unit.
template <int kCl>
__device__ __forceinline__ int own_unit(const int4& e, uint32_t crank, int U, int pair_heads, int& head) {
  if constexpr (kCl == 1) {
    head = e.y;
    return e.z;
  }
  if (pair_heads) {
    head = 2 * e.y + (int)crank;
    return e.z;
  }
  head = e.y;
  const int u = 2 * e.z + (int)crank;
  return u < U ? u : -1;
}
// K/V blocks the cluster streams for entry e: the longer unit of the pair.
template <bool kCausal>
__device__ __forceinline__ int pair_kv_blocks(const int4& e, const KernelParams& p);
template <bool kCausal>
__device__ __forceinline__ int unit_kv_blocks(int u, int nblk) {
  if (u < 0) return 0;
  int n0, n1;
  unit_blocks<kCausal>(u, nblk, n0, n1);
  return n0 > n1 ? n0 : n1;
}
template <bool kCausal>
__device__ __forceinline__ int pair_kv_blocks(const int4& e, const KernelParams& p) {
  if (p.pair_heads) return unit_kv_blocks<kCausal>(e.z, p.nblk);
  return max(unit_kv_blocks<kCausal>(2 * e.z, p.nblk),
             unit_kv_blocks<kCausal>(2 * e.z + 1 < p.U ? 2 * e.z + 1 : -1, p.nblk));
}

// The scheduler warp (lane 0): pop this SM's die queue (or the shared one),
// steal from the others when it runs dry, and broadcast (b, h, unit) to the
// CTA's consumers through the 2-entry SMEM ring; kCl == 2: the leader CTA
// serves both CTAs of the pair.
template <int kCl, class CT>
__device__ __forceinline__ void run_scheduler(const KernelParams& p, CT* ctrl) {
  const int sm = (int)ptx::smid();
  int dom = (sm < p.n_smid) ? (int)p.domain_of_smid[sm] : 0;
  if (dom < 0) dom = 0;
  const int nq = p.sched.n_queues;
  const int q0 = (nq > 1) ? p.sched.queue_of_domain[dom] : 0;
  uint32_t exhausted = 0;
  int stage = 0;
  uint32_t phase = 0;
  int seq = 0;
  while (true) {
    int b = 0, h = 0, u = 0, qi = -1, stolen = 0;
    for (int t = 0; t < nq; ++t) {
      if (t > 0 && !p.sched.steal) break;
      const int qq = (q0 + t) % nq;
      if (exhausted & (1u << qq)) continue;
      const int pos = atomicAdd(&p.counters[qq * 32], 1);
      if (pos < p.sched.q[qq].len) {
        decode_unit(p.sched, qq, pos, p.Hsched, p.Usched, b, h, u);
        if ((p.sched.descending >> qq) & 1) u = p.Usched - 1 - u;
        qi = qq;
        stolen = t > 0;
        break;
      }
      exhausted |= 1u << qq;
    }
    if constexpr (kCl == 1) {
      ptx::mbar_wait(&ctrl->sched_empty[stage], phase ^ 1);
      ctrl->entry[stage] = make_int4(b, h, u, qi >= 0 ? 1 : 0);
      ptx::mbar_arrive(&ctrl->sched_full[stage]);
    } else {
      // both CTAs' consumers released the slot on this (leader) CTA's barrier;
      // w packs valid | queue << 1 | stolen << 7 for the peers' trace records
      ptx::mbar_wait_cluster(&ctrl->sched_empty[stage], phase ^ 1);
      const int4 ent = make_int4(b, h, u, qi >= 0 ? (1 | (qi << 1) | (stolen << 7)) : 0);
      ctrl->entry[stage] = ent;
      ptx::st_cluster_v4(ptx::mapa_shared(ptx::smem_u32(&ctrl->entry[stage]), 1), ent);
      ptx::mbar_arrive(&ctrl->sched_full[stage]);
      ptx::mbar_arrive_cluster(ptx::mapa_shared(ptx::smem_u32(&ctrl->sched_full[stage]), 1));
    }
    if (qi < 0) break;
    if (kCl == 1 && p.trace && !ATTN_INSTRUMENTED) {  // instrumented builds reuse p.trace
      const long long id = ((long long)b * p.Hq + h) * p.U + u;
      if (id < p.trace_cap) {
        attn_trace_rec_t r;
        r.b = b; r.h = h; r.unit = u; r.smid = sm; r.domain = dom; r.queue = qi;
        r.stolen = stolen; r.seq = seq; r.t_pop_ns = ptx::globaltimer();
        p.trace[id] = r;
      }
    }
    ++seq;
    if (++stage == kSchedRing) { stage = 0; phase ^= 1; }
  }
  // Self-resetting counters: the last CTA to finish popping zeroes the
  // queue counters for the next launch on this slot (no host memset).
  __threadfence();
  if (atomicAdd(&p.counters[kDoneCounter], 1) == (int)gridDim.x / kCl - 1) {
    for (int q = 0; q < nq; ++q) atomicExch(&p.counters[q * 32], 0);
    atomicExch(&p.counters[kDoneCounter], 0);
    __threadfence();
  }
}

// kCl == 2: CTA-pair clusters (NEXT-4).  The pair works on the two halves of
// one cluster unit (units 2cu, 2cu+1 of the same head) and streams the SAME K/V
// blocks: each CTA TMA-loads half the rows of every block and multicasts them
// to both, and each MMA warp releases a ring slot to both CTAs' kv_empty.  The
// pair iterates over the longer unit's key blocks; the CTA whose own unit is
// shorter (causal) only releases the extra slots.
// kOnesL (D = 64, d_real < 64): the row sum l is not accumulated by the
// softmax but by the tensor core: K/V are loaded d_real columns wide, the
// ring slots' column d_real holds 1.0 (columns beyond it 0, written once per
// launch), so O += P V also accumulates O[:, d_real] = sum_k bf16(P_k) -- the
// same P the numerator uses -- and the fix-up rescales it with O.
template <int D, bool kCausal, int kCl, bool kOnesL>
__global__ void __launch_bounds__(kThreads, 1)
    attn_fwd_sm100_kernel(const __grid_constant__ CUtensorMap tm_q, const __grid_constant__ CUtensorMap tm_k,
                          const __grid_constant__ CUtensorMap tm_v, const KernelParams p) {
  using C = Cfg<D>;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* q_smem = smem + C::kOffQ;
  uint8_t* kv_smem = smem + C::kOffKV;
  Ctrl* ctrl = reinterpret_cast<Ctrl*>(smem + C::kOffCtrl);
  [[maybe_unused]] SplitRed* sred = reinterpret_cast<SplitRed*>(smem + C::kOffCtrl + 1024);
  static_assert(sizeof(Ctrl) <= 1024, "control block exceeds 1 KB");
  static_assert(C::kStages <= 16, "K/V ring deeper than the Ctrl barrier arrays");
  static_assert(kSplit == 1 || C::kCtrlBytes >= 1024 + (int)sizeof(SplitRed), "split reductions do not fit");
  static_assert(C::kSmemBytes <= 232448, "shared memory exceeds 227 KB");

  static_assert(kCl == 1 || kCl == 2, "cluster size 1 or 2");
  constexpr bool kSepP = ATTN_SEP_P && D <= 64 && kCl == 1;
  static_assert(!kSepP || 256 + 2 * D + 128 <= kTmemCols, "separate P does not fit in TMEM");
  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;
  const uint32_t crank = (kCl > 1) ? ptx::cluster_ctarank() : 0u;
  constexpr uint16_t kMask = (1u << kCl) - 1;

  if (threadIdx.x == 0) {
    for (int i = 0; i < kSchedRing; ++i) {
      ptx::mbar_init(&ctrl->sched_full[i], 1);
      // TMA + MMA + softmax warps (one arrive each), of every CTA of the cluster
      ptx::mbar_init(&ctrl->sched_empty[i], kCl * (2 + kSoftmaxWarps));
    }
    ptx::mbar_init(&ctrl->q_full, 1);
    ptx::mbar_init(&ctrl->q_empty, 1);
    for (int i = 0; i < C::kStages; ++i) {
      ptx::mbar_init(&ctrl->kv_full[i], 1);
      ptx::mbar_init(&ctrl->kv_empty[i], kCl);  // released by the MMA warp of every CTA of the cluster
    }
    for (int i = 0; i < 2; ++i) {
      ptx::mbar_init(&ctrl->s_ready[i], 1);
      for (int h = 0; h < kPParts; ++h)
        ptx::mbar_init(&ctrl->p_ready[i][h], 4 * kSplit);  // one arrive per softmax warp of the tile
      ptx::mbar_init(&ctrl->o_ready[i], 1);
      ptx::mbar_init(&ctrl->s_free[i], 4 * kSplit);
      ptx::mbar_init(&ctrl->p_free[i], 1);
    }
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
  if constexpr (kOnesL) {
    // K/V land d_real columns wide; logical column d_real of every ring slot
    // row is 1.0 and the columns after it 0 (16-byte chunks d_real/8 .. 7 of
    // each 128-byte row, at their 128B-swizzled positions).  Q keeps its
    // zero-filled padding, so the 1.0 in K's column d_real adds nothing to S.
    static_assert(!kOnesL || C::kChunks == 1, "ones column needs one swizzle atom per row");
    const int c0 = p.d_real / 8;
    for (int i = threadIdx.x; i < C::kStages * kBlockN * 8; i += kThreads) {
      const int chunk = i & 7, rrow = i >> 3;  // rrow = slot * 128 + row
      if (chunk < c0) continue;
      uint4 val = make_uint4(0u, 0u, 0u, 0u);
      if (chunk == c0) val.x = 0x3F80u;  // bf16 1.0 in the first element of the chunk
      const int phys = chunk ^ (rrow & 7);
      *reinterpret_cast<uint4*>(kv_smem + rrow * 128 + phys * 16) = val;
    }
    ptx::fence_proxy_async_smem();  // generic SMEM writes -> visible to TMA / tensor core
  }
  ptx::tc_fence_before();
  __syncthreads();
  if constexpr (kCl > 1) ptx::cluster_sync();  // peer barriers initialised before any remote arrive / multicast
  ptx::tc_fence_after();

  if (warp == 0) {
    // ------------------------------------------------------------ TMA producer
    if (ATTN_SETMAXNREG) ptx::setmaxnreg_dec<kOtherRegs>();
    if (lane == 0) {
      SchedReader<kCl> sr;
      const uint64_t pol_q = ptx::policy_evict_first();
#if ATTN_KV_EVICT_LAST
      const uint64_t pol_kv = ptx::policy_evict_last();
#else
      const uint64_t pol_kv = ptx::policy_evict_normal();
#endif
      uint32_t q_phase = 0;
      int kv_stage = 0;
      uint32_t kv_phase = 0;
      [[maybe_unused]] int seq = 0;
      while (true) {
        const int4 e = sr.next(ctrl, true);
        if (!e.w) break;
        int h;
        const int b = e.x, u = own_unit<kCl>(e, crank, p.U, p.pair_heads, h);
        int n0 = 0, n1 = 0;
        if (u >= 0) unit_blocks<kCausal>(u, p.nblk, n0, n1);
        const int n_own = n0 > n1 ? n0 : n1;
        // key blocks the cluster streams: the longer of the pair's units
        const int n = (kCl == 1) ? n_own : pair_kv_blocks<kCausal>(e, p);
        if constexpr (kCl > 1) {
          if (p.trace && u >= 0) {
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
        }
        if (n_own > 0) {
        ptx::mbar_wait(&ctrl->q_empty, q_phase ^ 1);
        q_phase ^= 1;
        const int ntile = n1 > 0 ? 2 : 1;
        ptx::mbar_arrive_expect_tx(&ctrl->q_full, ntile * C::kQTileBytes);
        for (int t = 0; t < ntile; ++t) {
          // 3-D view [B*Hq][N][d]: rows >= N of this head are out of bounds (zero-filled)
          const int bh = b * p.Hq + h, row = (2 * u + t) * kBlockM;
#pragma unroll
          for (int c = 0; c < C::kChunks; ++c)
            ptx::tma_load_3d(q_smem + t * C::kQTileBytes + c * kBlockM * 128, &tm_q, &ctrl->q_full, c * 64, row, bh,
                             pol_q);
        }
        }
        const int kvbh = b * p.Hkv + h / p.G;
        for (int jj = 0; jj < n; ++jj) {
#pragma unroll
          for (int ww = 0; ww < 2; ++ww) {
            // ring order K0 V0 K1 V1 ...; separate-P layout: K one block ahead,
            // K0 K1 V0 K2 V1 ... K(n-1) V(n-2) V(n-1), so the MMA warp can issue
            // S(j+1) before it needs V(j)
            int j = jj, which = ww;
            if constexpr (kSepP) {
              const int i = 2 * jj + ww;
              if (i == 0) { j = 0; which = 0; }
              else if (i == 2 * n - 1) { j = n - 1; which = 1; }
              else if (i & 1) { j = (i + 1) / 2; which = 0; }
              else { j = i / 2 - 1; which = 1; }
            }
            ptx::mbar_wait(&ctrl->kv_empty[kv_stage], kv_phase ^ 1);
            if constexpr (kCl > 1) {
              // this CTA's half of the block's rows, multicast into both CTAs
              ptx::mbar_arrive_expect_tx(&ctrl->kv_full[kv_stage], p.kv_tx_bytes);
              uint8_t* dst = kv_smem + kv_stage * C::kKVBytes + crank * (kBlockN / 2) * 128;
#pragma unroll
              for (int c = 0; c < C::kChunks; ++c)
                ptx::tma_load_3d_mc(dst + c * kBlockN * 128, which == 0 ? (const void*)&tm_k : (const void*)&tm_v,
                                    &ctrl->kv_full[kv_stage], c * 64, j * kBlockN + (int)crank * (kBlockN / 2), kvbh,
                                    kMask, pol_kv);
              if (++kv_stage == C::kStages) { kv_stage = 0; kv_phase ^= 1; }
              continue;
            }
            ptx::mbar_arrive_expect_tx(&ctrl->kv_full[kv_stage], p.kv_tx_bytes);
            uint8_t* dst = kv_smem + kv_stage * C::kKVBytes;
#pragma unroll
            for (int c = 0; c < C::kChunks; ++c)
              ptx::tma_load_3d(dst + c * kBlockN * 128, which == 0 ? (const void*)&tm_k : (const void*)&tm_v,
                               &ctrl->kv_full[kv_stage], c * 64, j * kBlockN, kvbh, pol_kv);
            if (++kv_stage == C::kStages) { kv_stage = 0; kv_phase ^= 1; }
          }
        }
      }
      if constexpr (kCl > 1) {
        // drain: every slot's last fill released by both CTAs, so no remote
        // commit is still in flight towards this CTA when it exits
        for (int i = 0; i < C::kStages; ++i) {
          ptx::mbar_wait(&ctrl->kv_empty[kv_stage], kv_phase ^ 1);
          if (++kv_stage == C::kStages) { kv_stage = 0; kv_phase ^= 1; }
        }
      }
    }
  } else if (warp == 1) {
    // -------------------------------------------------------------- MMA issuer
    // The whole warp runs the control flow (warp-uniform values stay in
    // uniform registers); one elected lane issues tcgen05.mma / commit.
    if (ATTN_SETMAXNREG) ptx::setmaxnreg_dec<kOtherRegs>();
    const uint32_t tmem = *reinterpret_cast<volatile uint32_t*>(&ctrl->tmem_base);
    SchedReader<kCl> sr;
    constexpr uint32_t idesc_s = ptx::idesc_bf16_f32(kBlockM, kBlockN, 0, 0);
    constexpr uint32_t idesc_o = ptx::idesc_bf16_f32(kBlockM, D, 0, 1);
    // descriptors at k = 0; advancing K by 16 elements adds 32 B (2 in the
    // >>4 address field) inside a 128-byte swizzle atom, and one atom
    // (rows * 128 B) every 4 steps.
    const uint64_t dq0 = ptx::smem_desc_sw128(ptx::smem_u32(q_smem), 16, 1024);
    const uint64_t dkv0 = ptx::smem_desc_sw128(ptx::smem_u32(kv_smem), 16, 1024);
    const uint64_t dv0 = ptx::smem_desc_sw128(ptx::smem_u32(kv_smem), kBlockN * 128, 1024);
    uint32_t q_phase = 0, p_phase0 = 0, p_phase1 = 0;
    [[maybe_unused]] int extra_blocks = 0;
    int kv_stage = 0;
    uint32_t kv_phase = 0;
    [[maybe_unused]] int s_used0 = 0, s_used1 = 0;
    [[maybe_unused]] uint32_t sf_phase0 = 0, sf_phase1 = 0;

    auto issue_s = [&](int t, int slot) {
      const uint64_t dq = dq0 + (uint64_t)((t * C::kQTileBytes) >> 4);
      const uint64_t dk = dkv0 + (uint64_t)((slot * C::kKVBytes) >> 4);
      const uint32_t d_tmem = tmem + C::col_s(t);
#pragma unroll
      for (int k = 0; k < D / 16; ++k) {
        const uint32_t oq = ((k >> 2) * (kBlockM * 128) + (k & 3) * 32) >> 4;
        const uint32_t ok = ((k >> 2) * (kBlockN * 128) + (k & 3) * 32) >> 4;
        ptx::mma_ss(d_tmem, dq + oq, dk + ok, idesc_s, k > 0 ? 1u : 0u);
      }
    };
    // O_t += P_t V: K = 128 keys in 8 steps of 16; the steps of slice h read
    // the part of P the softmax publishes separately (p_ready[t][h]).
    auto issue_pv_half = [&](int t, int slot, bool acc, int h) {
      const uint64_t dv = dv0 + (uint64_t)((slot * C::kKVBytes) >> 4);
      const uint32_t d_tmem = tmem + C::col_o(t);
      const uint32_t a_tmem = tmem + (kSepP ? C::col_p(t) : C::col_s(t));
#pragma unroll
      for (int k = h * (8 / kPParts); k < (h + 1) * (8 / kPParts); ++k)
        ptx::mma_ts(d_tmem, a_tmem + k * 8, dv + (uint64_t)((k * 16 * 128) >> 4), idesc_o,
                    (acc || k > 0) ? 1u : 0u);
    };
    auto take_slot = [&]() {
      const int s = kv_stage;
      ptx::mbar_wait(&ctrl->kv_full[s], kv_phase);
      if (++kv_stage == C::kStages) { kv_stage = 0; kv_phase ^= 1; }
      return s;
    };
    // release a K/V ring slot (to every CTA of the cluster) once the MMAs
    // issued so far have completed
    auto kv_release = [&](int s) {
      if constexpr (kCl == 1) ptx::mma_commit(&ctrl->kv_empty[s]);
      else ptx::mma_commit_mc(&ctrl->kv_empty[s], kMask);
    };

    while (true) {
      const int4 e = sr.next(ctrl, false);
      __syncwarp();
      if (lane == 0) sr.release_prev(ctrl);
      if (!e.w) break;
      int hu;
      const int u = own_unit<kCl>(e, crank, p.U, p.pair_heads, hu);
      int n0 = 0, n1 = 0;
      if (u >= 0) unit_blocks<kCausal>(u, p.nblk, n0, n1);
      const int n = n0 > n1 ? n0 : n1;
      if constexpr (kCl > 1) {
        // blocks the pair streams beyond this CTA's own unit: take and release
        const int n_all = pair_kv_blocks<kCausal>(e, p);
        if (n == 0) {
          for (int j = 0; j < n_all; ++j) {
            const int a = take_slot(), b2 = take_slot();
            if (ptx::elect_one_sync()) { kv_release(a); kv_release(b2); }
            __syncwarp();
          }
          continue;
        }
        extra_blocks = n_all - n;
      }
      if constexpr (kSepP) {
        // Separate-P order: S_t(j+1) as soon as the softmax has S_t(j) in
        // registers (s_free), PV_t(j) when P_t(j) is published; p_free / o_ready
        // tell the softmax when P_t may be overwritten and O_t rescaled / read.
        ptx::mbar_wait(&ctrl->q_full, q_phase);
        q_phase ^= 1;
        // S_t(j+1) once the softmax holds S_t(j) (s_free; not before a tile's
        // first block).  Each elected group also carries the commits and ring
        // releases that follow its MMAs in the stream (fewer elect / branch
        // round trips in this warp, whose own loop bounds the pipeline at
        // d <= 64: DESIGN.md section 6).
        auto issue_s_sep = [&](int t, int slot, bool last, bool q_done) {
          int& used = (t == 0) ? s_used0 : s_used1;
          uint32_t& sfp = (t == 0) ? sf_phase0 : sf_phase1;
          if (used) {
            ptx::mbar_wait(&ctrl->s_free[t], sfp);
            sfp ^= 1;
          }
          used = 1;
          ptx::tc_fence_after();
          if (ptx::elect_one_sync()) {
            issue_s(t, slot);
            ptx::mma_commit(&ctrl->s_ready[t]);
            if (last) {
              kv_release(slot);
              if (q_done) ptx::mma_commit(&ctrl->q_empty);
            }
          }
          __syncwarp();
        };
        int sK = take_slot();
        // n >= 1, n0 >= 1; tile 1 absent when n1 == 0
        issue_s_sep(0, sK, n1 == 0, n == 1);
        if (n1 > 0) issue_s_sep(1, sK, true, n == 1);
        for (int j = 0; j < n; ++j) {
          if (j + 1 < n) {
            sK = take_slot();
            const bool a0 = j + 1 < n0, a1 = j + 1 < n1;  // a0 || a1
            if (a0) issue_s_sep(0, sK, !a1, j + 2 == n);
            if (a1) issue_s_sep(1, sK, true, j + 2 == n);
          }
          const int sV = take_slot();
          const bool v1 = j < n1;  // tile 1 uses V(j); tile 0 does whenever tile 1 does not
#pragma unroll
          for (int t = 0; t < 2; ++t) {
            const int nt = (t == 0) ? n0 : n1;
            if (j < nt) {
              const uint32_t ph = (t == 0) ? p_phase0 : p_phase1;
#pragma unroll
              for (int h = 0; h < kPParts; ++h) {
                ptx::mbar_wait(&ctrl->p_ready[t][h], ph);
                ptx::tc_fence_after();
                if (ptx::elect_one_sync()) {
                  issue_pv_half(t, sV, j > 0, h);
                  if (h == kPParts - 1) {
                    ptx::mma_commit(j + 1 < nt ? &ctrl->p_free[t] : &ctrl->o_ready[t]);
                    if (t == 1 || !v1) kv_release(sV);
                  }
                }
                __syncwarp();
              }
              if (t == 0) p_phase0 ^= 1; else p_phase1 ^= 1;
            }
          }
        }
        continue;
      }
      ptx::mbar_wait(&ctrl->q_full, q_phase);
      q_phase ^= 1;
      int sK = take_slot();
      ptx::tc_fence_after();
      if (ptx::elect_one_sync()) {
        if (n0 > 0) {
          issue_s(0, sK);
          ptx::mma_commit(&ctrl->s_ready[0]);
        }
        if (n1 > 0) {
          issue_s(1, sK);
          ptx::mma_commit(&ctrl->s_ready[1]);
        }
        kv_release(sK);
        if (n == 1) ptx::mma_commit(&ctrl->q_empty);
      }
      __syncwarp();
      for (int j = 0; j < n; ++j) {
        const int sV = take_slot();
        const bool nxt = j + 1 < n;
        if (nxt) sK = take_slot();
        ptx::tc_fence_after();
#pragma unroll
        for (int t = 0; t < 2; ++t) {
          const int nt = (t == 0) ? n0 : n1;
          if (j < nt) {
            const uint32_t ph = (t == 0) ? p_phase0 : p_phase1;
            // the last slice's group also issues S_t(j+1) (or commits O_t) and,
            // for the last tile using this block, releases the ring slots
            const bool last_tile = (t == 1) || (j >= n1);
#pragma unroll
            for (int h = 0; h < kPParts; ++h) {
              ptx::mbar_wait(&ctrl->p_ready[t][h], ph);
              ptx::tc_fence_after();
              if (ptx::elect_one_sync()) {
                issue_pv_half(t, sV, j > 0, h);
                if (h == kPParts - 1) {
                  if (j + 1 < nt) {
                    issue_s(t, sK);
                    ptx::mma_commit(&ctrl->s_ready[t]);
                  } else {
                    ptx::mma_commit(&ctrl->o_ready[t]);
                  }
                  if (last_tile) {
                    kv_release(sV);
                    if (nxt) {
                      kv_release(sK);
                      if (j + 2 == n) ptx::mma_commit(&ctrl->q_empty);
                    }
                  }
                }
              }
              __syncwarp();
            }
            if (t == 0) p_phase0 ^= 1; else p_phase1 ^= 1;
          }
        }
      }
      if constexpr (kCl > 1) {
        for (int j = 0; j < extra_blocks; ++j) {
          const int a = take_slot(), b2 = take_slot();
          if (ptx::elect_one_sync()) { kv_release(a); kv_release(b2); }
          __syncwarp();
        }
        extra_blocks = 0;
      }
    }
  } else if (warp == 2) {
    // --------------------------------------------------------------- scheduler
    if (ATTN_SETMAXNREG) ptx::setmaxnreg_dec<kOtherRegs>();
    if (lane == 0 && crank == 0) run_scheduler<kCl>(p, ctrl);  // clusters: the leader schedules for the pair
  } else if (warp >= 4) {
    // ------------------------------------------------ softmax / fix-up / epilogue
    if (ATTN_SETMAXNREG) ptx::setmaxnreg_inc<kSoftmaxRegs>();
    const uint32_t tmem = *reinterpret_cast<volatile uint32_t*>(&ctrl->tmem_base);
    constexpr int kCols = kBlockN / kSplit;  // S columns per thread
    constexpr int kOCols = D / kSplit;       // O columns per thread (fix-up, epilogue)
    const int sw = warp - 4;
    const int t = sw / (4 * kSplit);         // query tile of the unit
    const int hf = (sw >> 2) % kSplit;       // which column slice of the row
    const int quarter = warp & 3;            // TMEM lane quarter this warp may access
    const int row = quarter * 32 + lane;     // row within the 128-row tile
    const int cbase = hf * kCols;            // first key column of this thread's slice
    const uint32_t trow = tmem + ((uint32_t)(quarter * 32) << 16);
    const uint32_t colS = C::col_s(t) + cbase;
    const uint32_t colP = (kSepP ? C::col_p(t) : C::col_s(t)) + cbase / 2;
    const uint32_t colO = C::col_o(t) + hf * kOCols;
    [[maybe_unused]] const uint32_t bar_id = 1 + t * 4 + quarter;  // named barrier of the row group's warps
    const float c = p.scale_log2;
#if ATTN_O_EVICT_FIRST
    const uint64_t pol_o = ptx::policy_evict_first();
#endif
    SchedReader<kCl> sr;
    uint32_t s_phase = 0, o_phase = 0, gblk = 0;
    ATTN_CYC_DECL()
    [[maybe_unused]] uint32_t pf_phase = 0;
    while (true) {
      const int4 e = sr.next(ctrl, false);
      __syncwarp();
      if (lane == 0) sr.release_prev(ctrl);
      if (!e.w) break;
      int hh;
      const int u = own_unit<kCl>(e, crank, p.U, p.pair_heads, hh);
      int n0 = 0, n1 = 0;
      if (u >= 0) unit_blocks<kCausal>(u, p.nblk, n0, n1);
      const int nt = (t == 0) ? n0 : n1;
      if (nt == 0) continue;
      const int qb = 2 * u + t;
      // keys of the last key block that exist (ragged N): local key k < tail_keys
      const int last_blk = p.nblk - 1;
      const int tail_lim = (p.N - last_blk * kBlockN - 1) - cbase;  // last block: local k visible iff k <= tail_lim
      float m = -INFINITY, l = 0.f;
      for (int j = 0; j < nt; ++j, ++gblk) {
        ATTN_CYC_START();
        ptx::mbar_wait(&ctrl->s_ready[t], s_phase);
        ATTN_CYC_ADD(0);
        s_phase ^= 1;
        ptx::tc_fence_after();
#ifdef ATTN_ABL_SKIPSM  // timing ablation only (wrong results): the softmax keeps only its barrier protocol
        {
          if constexpr (kSepP) {
            ptx::tc_fence_before();
            __syncwarp();
            if (lane == 0) ptx::mbar_arrive(&ctrl->s_free[t]);
          }
          for (int h = 0; h < kPParts; ++h) {
            if (kSepP && h == 0 && j > 0) {
              ptx::mbar_wait(&ctrl->p_free[t], pf_phase);
              pf_phase ^= 1;
            }
            ptx::tc_fence_before();
            __syncwarp();
            if (lane == 0) ptx::mbar_arrive(&ctrl->p_ready[t][h]);
          }
          l = 1.f;
          m = 0.f;
          continue;
        }
#endif
        uint32_t r[kCols];
        if constexpr (kCols == 128) ptx::tmem_ld128(trow + colS, r);
        else ptx::tmem_ld64(trow + colS, r);
        if constexpr (kSepP) {  // S_t is in registers: the MMA warp may compute S_t(j+1) over it
          ptx::tc_fence_before();
          __syncwarp();
          if (lane == 0) ptx::mbar_arrive(&ctrl->s_free[t]);
        }
        // visible local keys are k <= lim: causal diagonal block (key <= query)
        // and/or the ragged last key block (key < N)
        int lim = kCols;
        if (kCausal && j == qb) lim = row - cbase;
        if (j == last_blk && tail_lim < lim) lim = tail_lim;
        // warp-uniform choice between the masked and the unmasked loop bodies
        const bool diag = __any_sync(0xffffffffu, lim < kCols - 1);
        if (diag) {  // masked keys -> -inf
#pragma unroll
          for (int k = 0; k < kCols; ++k)
            if (k > lim) r[k] = 0xff800000u;
        }
        ATTN_CYC_ADD(1);
        // row max: four independent FMNMX3 chains, then across the kSplit warps
        float mq[4] = {-INFINITY, -INFINITY, -INFINITY, -INFINITY};
#pragma unroll
        for (int k = 0; k < kCols; k += 8) {
#pragma unroll
          for (int g4 = 0; g4 < 4; ++g4)
            mq[g4] = fmaxf(mq[g4], fmaxf(__uint_as_float(r[k + 2 * g4]), __uint_as_float(r[k + 2 * g4 + 1])));
        }
        float mx = fmaxf(fmaxf(mq[0], mq[1]), fmaxf(mq[2], mq[3]));
        if constexpr (kSplit == 2) {
          sred->red[t][quarter][hf][gblk & 1][lane] = mx;
          ptx::named_bar_sync(bar_id, 64);
          mx = fmaxf(mx, sred->red[t][quarter][hf ^ 1][gblk & 1][lane]);
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
        const bool any_rescale = __any_sync(0xffffffffu, rescale);
        // fix-up: O *= exp2((m_old - m_new) c) for this row,
        // once PV_t(j-1) is complete: it precedes S_t(j) in the MMA stream, or
        // (separate-P layout) p_free says so, just before P_t(j) is stored.
        auto fixup = [&]() {
#pragma unroll
          for (int cc = 0; cc < kOCols; cc += 32) {
            uint32_t o[32];
            ptx::tmem_ld32(trow + colO + cc, o);
#pragma unroll
            for (int k = 0; k < 32; ++k) o[k] = __float_as_uint(__uint_as_float(o[k]) * alpha);
            ptx::tmem_st32(trow + colO + cc, o);
          }
        };
        if (!kSepP && any_rescale) fixup();
        const float neg = -m_use * c;
        // P = exp2(S c - m c) on (even, odd) pairs with packed f32x2 math:
        // MUFU.EX2 for most pairs, the FMA-pipe polynomial for every
        // kEmuPeriod-th pair.  P is published in two halves so the tensor
        // core starts O += P V on the first half while the second is computed.
        float2 sq[4] = {make_float2(0.f, 0.f), make_float2(0.f, 0.f), make_float2(0.f, 0.f),
                        make_float2(0.f, 0.f)};
        auto exp_block = [&](auto mask_tag) {
#pragma unroll
        for (int h = 0; h < kPParts; ++h) {
#pragma unroll
          for (int k = h * kCols / kPParts; k < (h + 1) * kCols / kPParts; k += 2) {
            const float2 x = ptx::ffma2(make_float2(__uint_as_float(r[k]), __uint_as_float(r[k + 1])), c, neg);
            float2 pr;
            constexpr int kEP = emu_period<D>();
#ifdef ATTN_ABL_NOEXP  // timing ablation only (wrong results): no exp2
            if (true) {
              pr = x;
            } else
#endif
            if (kEP > 0 && ((k >> 1) % (kEP > 0 ? kEP : 1)) == kEP - 1) {
              pr = ptx::ex2_poly2(x);
            } else {
#if ATTN_EXP_F16X2
              pr = ptx::ex2_f16x2(x);
#else
              pr.x = ptx::ex2(x.x);
              pr.y = ptx::ex2(x.y);
#endif
            }
            if constexpr (decltype(mask_tag)::value) {
              pr.x = (k <= lim) ? pr.x : 0.f;
              pr.y = (k + 1 <= lim) ? pr.y : 0.f;
            }
            if constexpr (!kOnesL) sq[(k >> 1) & 3] = ptx::fadd2(sq[(k >> 1) & 3], pr);
            r[k >> 1] = ptx::pack_bf16(pr.x, pr.y);
          }
          ATTN_CYC_ADD(3);
          if constexpr (kSepP) {
            if (h == 0 && j > 0) {  // PV_t(j-1) has finished reading P_t and adding into O_t
              ptx::mbar_wait(&ctrl->p_free[t], pf_phase);
              ATTN_CYC_ADD(4);
              pf_phase ^= 1;
              ptx::tc_fence_after();
              if (any_rescale) fixup();
              ATTN_CYC_ADD(9);
            }
          }
          constexpr int kPc = kCols / kPParts / 2;  // packed P columns per slice
          if constexpr (kPc == 32) ptx::tmem_st32(trow + colP + h * 32, r + h * 32);
          else ptx::tmem_st16(trow + colP + h * 16, r + h * 16);
          ptx::tmem_wait_st();
          ptx::tc_fence_before();
          __syncwarp();
          if (lane == 0) ptx::mbar_arrive(&ctrl->p_ready[t][h]);
          ATTN_CYC_ADD(8);
        }
        };
        ATTN_CYC_ADD(2);
        if (diag) exp_block(std::true_type{});
        else exp_block(std::false_type{});
        if constexpr (!kOnesL) {
          const float2 s01 = ptx::fadd2(sq[0], sq[1]), s23 = ptx::fadd2(sq[2], sq[3]);
          const float2 s4 = ptx::fadd2(s01, s23);
          const float sum = s4.x + s4.y;
          l = (j == 0) ? sum : fmaf(l, alpha, sum);
        }
        m = m_use;
        ATTN_CYC_ADD(3);
        ATTN_CYC_COUNT(7);
      }
      ATTN_CYC_START();
      // ---- epilogue: O / l -> bf16 -> global
      if constexpr (kSplit == 2 && !kOnesL) {
        sred->lsum[t][quarter][hf][lane] = l;
        ptx::named_bar_sync(bar_id, 64);
        l += sred->lsum[t][quarter][hf ^ 1][lane];
      }
      ATTN_CYC_TIMED(6, ptx::mbar_wait(&ctrl->o_ready[t], o_phase));
      o_phase ^= 1;
      ptx::tc_fence_after();
      if constexpr (kOnesL) l = __uint_as_float(ptx::tmem_ld1(trow + C::col_o(t) + p.d_real));
      const float inv_l = 1.f / l;
      if (p.lse != nullptr && hf == 0 && qb * kBlockM + row < p.N)  // lse = scale*m + ln(l)
        p.lse[(long long)(e.x * p.Hq + hh) * p.N + qb * kBlockM + row] = (m * c + __log2f(l)) * 0.6931471805599453f;
      const long long orow =
          ((long long)(e.x * p.Hq_out + p.h_off + hh) * p.N + (long long)qb * kBlockM + row) * p.d_real + hf * kOCols;
      // real columns of this thread's slice (multiple of 8); rows >= N (ragged
      // last query block) store nothing but still join the warp-wide TMEM loads
      const int ncol = (qb * kBlockM + row < p.N) ? p.d_real - hf * kOCols : 0;
#pragma unroll
      for (int cc = 0; cc < kOCols; cc += 32) {
        uint32_t o[32];
        ptx::tmem_ld32(trow + colO + cc, o);
        uint32_t pk[16];
#pragma unroll
        for (int k = 0; k < 16; ++k)
          pk[k] = ptx::pack_bf16(__uint_as_float(o[2 * k]) * inv_l, __uint_as_float(o[2 * k + 1]) * inv_l);
        for (int di = 0; di < p.n_dst; ++di) {  // replicated output: one store per destination
          uint4* dst = reinterpret_cast<uint4*>(p.o_dst[di] + orow);
#pragma unroll
          for (int k = 0; k < 4; ++k) {
            if (cc + 8 * k >= ncol) break;  // padded head dim: the zero columns are not stored
#if ATTN_O_EVICT_FIRST
            ptx::st_global_v4_evict_first(dst + cc / 8 + k, make_uint4(pk[4 * k], pk[4 * k + 1], pk[4 * k + 2], pk[4 * k + 3]), pol_o);
#else
            dst[cc / 8 + k] = make_uint4(pk[4 * k], pk[4 * k + 1], pk[4 * k + 2], pk[4 * k + 3]);
#endif
          }
        }
      }
      ptx::tc_fence_before();
      ATTN_CYC_ADD(5);
    }
    ATTN_CYC_WRITE16(p.trace, warp - 4)
  } else {
    if (ATTN_SETMAXNREG) ptx::setmaxnreg_dec<kOtherRegs>();  // warp 3: idle
  }

  ptx::tc_fence_before();
  __syncthreads();
  if constexpr (kCl > 1) ptx::cluster_sync();  // no remote SMEM access may target an exited CTA
  if (warp == 2) {
    ptx::tc_fence_after();
    ptx::tmem_dealloc(*reinterpret_cast<volatile uint32_t*>(&ctrl->tmem_base), kTmemCols);
  }
}

}  // namespace attn
