// attn_sched.h -- work-unit queues for the three mappings (host + device).
//
// A work unit is a pair of adjacent 128-row query blocks of one (b, h)
// (rows [256u, 256u + 256)); the kernel computes both blocks against one K/V
// stream.  units_per_head U = ceil(N / 256).
//
// The paper's mappings become orders over units:
//   kind 0  block-major range  (Naive Block-first):
//           pos -> b = pos / (U*Hq), u = (pos % (U*Hq)) / Hq, h = pos % Hq
//   kind 1  head-major range   (Naive Head-first; also SHF queues cut
//           over the global (b, ACC) list or at unit granularity):
//           hm = start + pos -> b = hm / (Hq*U), h = (hm / U) % Hq, u = hm % U
//   kind 2  per-batch head range (Swizzled Head-first, Fig. 7 with
//           batch outermost): queue d holds, for every b, heads
//           [h_lo, h_lo + h_cnt) (whole ACCs) in head-major order.
//   kind 3  strided groups, block-major (Swizzled Block-first, P:236-243,
//           S:172): queue d holds the KV groups g = h_lo + i*stride
//           (i < n_groups) in order for b, for u, for g, for the G heads of g.
// Block-first and head-first use ONE queue popped by every SM of every die;
// swizzled head-first uses one queue per die (reading R8), or, when
// its ACCs are shared by all dies (R23), the one head-major queue of a single
// capacity domain.
#pragma once
#include <cstdint>

#ifndef ATTN_HD
#ifdef __CUDACC__
#define ATTN_HD __host__ __device__ __forceinline__
#else
#define ATTN_HD inline
#endif
#endif

namespace attn {

constexpr int kMaxQueues = 8;

struct QueueDesc {
  int kind;    // 0 block-major range, 1 head-major range, 2 per-batch head range, 3 strided groups
  int start;   // first position (kinds 0, 1)
  int len;     // number of units in the queue
  int h_lo;    // kind 2: first query head; kind 3: first KV group
  int h_cnt;   // kind 2: query heads per batch item; kind 3: number of KV groups
  int stride;  // kind 3: KV-group stride (= number of dies)
  int G;       // kind 3: query heads per KV group
};

struct SchedParams {
  int n_queues;
  int steal;                           // pop other queues when the own one is empty
  int descending;                      // bit q set: queue q visits each head's units in descending order
  int queue_of_domain[kMaxQueues];     // die -> queue popped first
  QueueDesc q[kMaxQueues];
};

ATTN_HD void decode_unit(const SchedParams& sp, int qi, int pos, int Hq, int U, int& b, int& h, int& u) {
  const QueueDesc& qd = sp.q[qi];
  if (qd.kind == 0) {
    const int p = qd.start + pos;
    b = p / (U * Hq);
    const int r = p % (U * Hq);
    u = r / Hq;
    h = r % Hq;
  } else if (qd.kind == 1) {
    const int hm = qd.start + pos;
    b = hm / (Hq * U);
    h = (hm / U) % Hq;
    u = hm % U;
  } else if (qd.kind == 2) {
    const int per_b = qd.h_cnt * U;
    b = pos / per_b;
    const int r = pos % per_b;
    h = qd.h_lo + r / U;
    u = r % U;
  } else {
    const int per_u = qd.h_cnt * qd.G;  // units of one (b, u) row of the queue
    b = pos / (per_u * U);
    const int r = pos % (per_u * U);
    u = r / per_u;
    const int i = r % per_u;
    h = (qd.h_lo + (i / qd.G) * qd.stride) * qd.G + i % qd.G;
  }
}

// Proportional contiguous cut of [0, total) by die sizes (rounded to nearest).
inline int prop_cut(long long total, const int* sizes, int n, int d) {
  long long S = 0, acc = 0;
  for (int e = 0; e < n; ++e) S += sizes[e];
  for (int e = 0; e < d; ++e) acc += sizes[e];
  if (d >= n) return (int)total;
  return (int)((total * acc + S / 2) / S);
}

// Mapping argument: low byte = mapping (0 BF, 1 HF, 2 SHF, 3 SBF); bit 8 =
// descending unit order inside every (b, h) (applied identically to every
// mapping; the paper's order is ascending); bit 10 = alternate the unit
// direction per queue (queue d descending iff d is odd; single-queue
// mappings are unaffected) -- see include/attn_numa.h ATTN_ORDER_ALTERNATE;
// bit 11 = SHF with every ACC shared by all dies (one head-major queue: the
// dies form one capacity domain), bit 12 = SHF with one die per ACC even
// where the library would share it (R23).
constexpr int kMapMask = 0xff;
constexpr int kOrderDescending = 0x100;
constexpr int kOrderAlternate = 0x400;
constexpr int kShfAccShared = 0x800;
constexpr int kShfAccPerDie = 0x1000;

// DESIGN.md R23 (B200 reading of P:259-270): the dies share ONE L2 (lines
// homed by address, far lines not replicated near: the probe's
// far_lines_cached_near = 0), so "each die serves one ACC at a time" keeps
// n_domains ACC K/V footprints live in that one L2.  When those footprints
// exceed half of it (the capacity sweep: SHF's DRAM
// bytes leave head-first's between 2 x 32 and 2 x 48 MiB per ACC on the
// 126 MiB L2), swizzled head-first shares each ACC among the dies instead:
// the whole GPU is one capacity domain, and SHF over one domain is the
// head-major order.
ATTN_HD bool shf_acc_shared(int n_domains, long long N, int d, long long l2_bytes) {
  const long long kv_acc = 2ll * N * d * 2;  // K and V of one KV head, bf16
  return n_domains > 1 && l2_bytes > 0 && (long long)n_domains * kv_acc > l2_bytes / 2;
}

// Per-queue direction mask of an order argument for n_queues queues.
ATTN_HD int direction_mask(int mapping_arg, int n_queues) {
  const int all = (1 << n_queues) - 1;
  int m = (mapping_arg & kOrderDescending) ? all : 0;
  if (mapping_arg & kOrderAlternate) m ^= (0xAA & all);
  return m;
}

// Build the queues of `mapping` for n_domains dies.  Returns false on bad arguments.
inline bool build_queues(int mapping_arg, int B, int Hq, int Hkv, int U, int n_domains, const int* sms_per_domain,
                         SchedParams& sp) {
  sp = SchedParams{};
  if (mapping_arg & ~(kMapMask | kOrderDescending | kOrderAlternate | kShfAccShared | kShfAccPerDie)) return false;
  const int mapping = mapping_arg & kMapMask;
  if (B <= 0 || Hq <= 0 || Hkv <= 0 || U <= 0 || Hq % Hkv != 0) return false;
  if (n_domains < 1 || n_domains > kMaxQueues) return false;
  const int G = Hq / Hkv;
  const int total = B * Hq * U;
  if (mapping < 0 || mapping > 3) return false;
  // R23: SHF with shared ACCs = SHF over ONE capacity domain = head-first order
  const bool one_domain = n_domains == 1 || (mapping == 2 && (mapping_arg & kShfAccShared));
  if (mapping == 0 || mapping == 1 || one_domain) {
    const bool block_major = (mapping == 0 || mapping == 3);  // SBF on one die == BF
    sp.n_queues = 1;
    sp.steal = 0;
    sp.q[0] = QueueDesc{block_major ? 0 : 1, 0, total, 0, Hq, 0, 0};
    return true;
  }
  const int D = n_domains;
  sp.n_queues = D;
  sp.steal = 1;
  for (int d = 0; d < D; ++d) sp.queue_of_domain[d] = d;
  if (mapping == 3) {
    for (int d = 0; d < D; ++d) {
      const int ng = (Hkv > d) ? (Hkv - d + D - 1) / D : 0;  // groups g = d, d + D, ...
      sp.q[d] = QueueDesc{3, 0, B * U * ng * G, d, ng, D, G};
    }
    return true;
  }
  if (Hkv >= D) {
    for (int d = 0; d < D; ++d) {
      const int a0 = prop_cut(Hkv, sms_per_domain, D, d), a1 = prop_cut(Hkv, sms_per_domain, D, d + 1);
      sp.q[d] = QueueDesc{2, 0, B * (a1 - a0) * G * U, a0 * G, (a1 - a0) * G, 0, 0};
    }
  } else if ((long long)B * Hkv >= D) {
    const int A = B * Hkv;
    for (int d = 0; d < D; ++d) {
      const int a0 = prop_cut(A, sms_per_domain, D, d), a1 = prop_cut(A, sms_per_domain, D, d + 1);
      sp.q[d] = QueueDesc{1, a0 * G * U, (a1 - a0) * G * U, 0, Hq, 0, 0};
    }
  } else {
    for (int d = 0; d < D; ++d) {
      const int t0 = prop_cut(total, sms_per_domain, D, d), t1 = prop_cut(total, sms_per_domain, D, d + 1);
      sp.q[d] = QueueDesc{1, t0, t1 - t0, 0, Hq, 0, 0};
    }
  }
  return true;
}

inline bool build_sched(int mapping_arg, int B, int Hq, int Hkv, int U, int n_domains, const int* sms_per_domain,
                        SchedParams& sp) {
  if (!build_queues(mapping_arg, B, Hq, Hkv, U, n_domains, sms_per_domain, sp)) return false;
  sp.descending = direction_mask(mapping_arg, sp.n_queues);
  return true;
}

}  // namespace attn
