// topology.cuh -- startup microbenchmark that discovers the SM -> die split.
//
// the dispatch of work-groups to dies is "implemented in the
// driver and subject to change ... kernels must incorporate mutable,
// algorithmic mapping logic".  On B200 the CTA -> SM placement is not
// documented and %smid is a virtual id, so the die of every SM is MEASURED:
//
//   1. census kernel: which %smid values exist (%nsmid bounds them);
//   2. latency kernel: one thread on every SM warms L probe lines (4 KiB
//      apart, so they hash to different L2 slices) and then pointer-chases
//      them R times with ld.global.cg, timing every hop with clock64;
//      lat[smid][line] = min over rounds (an L2-hit latency);
//   3. host: 1-D 2-means over all latencies -> near/far threshold; an SM's
//      near set is {lines below threshold}; SMs whose near set agrees with
//      SM s0's on more than half of the lines are die 0, the rest die 1.
// If the two clusters are not separated (margin < 8 cycles) or a die comes
// out empty, the probe is "inconclusive" and the library uses ONE domain
// (source = 2), in which case swizzled head-first equals head-first.
#pragma once
#include <cstdint>

namespace attn {

constexpr int kProbeLines = 128;
constexpr int kProbeStrideBytes = 4096;
constexpr int kProbeRounds = 8;

__global__ void topo_census_kernel(int* smid_seen, int* nsmid_out) {
  if (threadIdx.x == 0) {
    uint32_t s, n;
    asm volatile("mov.u32 %0, %%smid;" : "=r"(s));
    asm volatile("mov.u32 %0, %%nsmid;" : "=r"(n));
    if (s < 1024) atomicExch(&smid_seen[s], 1);
    atomicMax(nsmid_out, (int)n);
  }
}

// probe: kProbeLines lines, line l at byte offset l*kProbeStrideBytes; each
// line's first word holds its OWN byte offset, so `off = load(base + off)`
// chases the same line kChain times with every address depending on the
// previous load (the clock difference then spans the whole dependent chain).
constexpr int kChain = 8;
__global__ void topo_latency_kernel(const uint32_t* probe, int* claimed, uint32_t* lat, int max_smid) {
  if (threadIdx.x != 0) return;
  uint32_t s;
  asm volatile("mov.u32 %0, %%smid;" : "=r"(s));
  if ((int)s >= max_smid) return;
  if (atomicCAS(&claimed[s], 0, 1) != 0) return;
  const char* base = reinterpret_cast<const char*>(probe);
  uint32_t sink = 0;
  // warm: touch every line once (brings it into L2)
  for (int i = 0; i < kProbeLines; ++i) {
    uint32_t x;
    asm volatile("ld.volatile.global.u32 %0, [%1];" : "=r"(x) : "l"(base + (size_t)i * kProbeStrideBytes) : "memory");
    sink += x;
  }
  for (int i = 0; i < kProbeLines; ++i) {
    uint32_t best = 0xFFFFFFFFu;
    for (int r = 0; r < kProbeRounds; ++r) {
      uint32_t off = (uint32_t)i * kProbeStrideBytes;
      const long long t0 = clock64();
#pragma unroll
      for (int c = 0; c < kChain; ++c)
        asm volatile("ld.volatile.global.u32 %0, [%1];" : "=r"(off) : "l"(base + off) : "memory");
      sink += off;
      const long long t1 = clock64();
      const uint32_t dt = (uint32_t)((t1 - t0) / kChain);
      if (dt < best) best = dt;
    }
    lat[(size_t)s * kProbeLines + i] = best;
  }
  if (sink == 0xFFFFFFFFu) lat[0] = 0;  // keep the chain alive
}

// Re-read probe: does a FAR line, once read by an
// SM, become a near L2 hit for that SM (a near-die copy), or does it stay at
// its home die?  After the host flushes L2, the one thread on SM `target`
// reads each line once (a DRAM miss that fills L2 the way the attention
// kernel's loads do), then times kChain dependent re-reads of the same line,
// kProbeRounds times, with the same ld.volatile.global as topo_latency_kernel
// (so the two latencies are comparable): reread[line] = min cycles per
// re-read.  A far line whose re-read comes back at the near latency was
// cached near.
__global__ void topo_reread_kernel(const uint32_t* probe, int* claimed, int target, uint32_t* reread) {
  if (threadIdx.x != 0) return;
  uint32_t s;
  asm volatile("mov.u32 %0, %%smid;" : "=r"(s));
  if ((int)s != target || atomicCAS(claimed, 0, 1) != 0) return;
  const char* base = reinterpret_cast<const char*>(probe);
  uint32_t sink = 0;
  for (int i = 0; i < kProbeLines; ++i) {
    uint32_t x;
    asm volatile("ld.volatile.global.u32 %0, [%1];" : "=r"(x) : "l"(base + (size_t)i * kProbeStrideBytes) : "memory");
    sink += x;  // first touch
    uint32_t best = 0xFFFFFFFFu;
    for (int r = 0; r < kProbeRounds; ++r) {
      uint32_t off = (uint32_t)i * kProbeStrideBytes;
      const long long t0 = clock64();
#pragma unroll
      for (int c = 0; c < kChain; ++c)
        asm volatile("ld.volatile.global.u32 %0, [%1];" : "=r"(off) : "l"(base + off) : "memory");
      sink += off;
      const uint32_t dt = (uint32_t)((clock64() - t0) / kChain);
      if (dt < best) best = dt;
    }
    reread[i] = best;
  }
  if (sink == 0xFFFFFFFFu) reread[0] = 0;  // keep the chain alive
}

}  // namespace attn
