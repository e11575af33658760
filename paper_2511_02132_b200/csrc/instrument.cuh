// instrument.cuh -- opt-in cycle account of the forward kernel's softmax
// chain (build with -D ATTN_CYCLES; read out by scripts/cycles.py).  Every
// macro expands to nothing (or to its bare statement) in the product build,
// so the hot loops carry one-word markers instead of #ifdef blocks.
//
// Per softmax warp, cycles are summed in registers into 8 buckets and written
// once at exit to the schedule-trace buffer: [0] S wait, [1] TMEM load + mask,
// [2] row max, [3] exps + P stores, [4] p_free wait, [5] epilogue (incl. the
// o_ready wait), [6] o_ready wait, [7] key blocks processed.
// (The finer timeline / wait-profile builds of round 1 live in commit 2845b57.)
#pragma once

#ifdef ATTN_CYCLES
#define ATTN_CYC_DECL() \
  long long cyc_[16] = {0, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0}; \
  long long cyc_t_ = 0;
#define ATTN_CYC_START() cyc_t_ = clock64();
#define ATTN_CYC_ADD(i)                 \
  {                                     \
    const long long cyc_n_ = clock64(); \
    cyc_[i] += cyc_n_ - cyc_t_;         \
    cyc_t_ = cyc_n_;                    \
  }
#define ATTN_CYC_COUNT(i) cyc_[i] += 1;
#define ATTN_CYC_TIMED(i, stmt)         \
  {                                     \
    const long long cyc_w_ = clock64(); \
    stmt;                               \
    cyc_[i] += clock64() - cyc_w_;      \
  }
// one record of 8 counters per (CTA < 64, softmax warp)
#define ATTN_CYC_WRITE(trace, warp_index)                                                                   \
  if ((trace) && (threadIdx.x & 31) == 0 && blockIdx.x < 64) {                                             \
    long long* cyc_out_ = reinterpret_cast<long long*>(trace) + (blockIdx.x * 8 + (warp_index)) * 8;    \
    for (int cyc_i_ = 0; cyc_i_ < 8; ++cyc_i_) cyc_out_[cyc_i_] = cyc_[cyc_i_];                          \
  }
// forward kernel: one record of 16 counters per (CTA < 64, softmax warp); [8]
// P stores (tcgen05.st + wait + publish), [9] O fix-up
#define ATTN_CYC_WRITE16(trace, warp_index)                                                                \
  if ((trace) && (threadIdx.x & 31) == 0 && blockIdx.x < 64) {                                             \
    long long* cyc_out_ = reinterpret_cast<long long*>(trace) + (blockIdx.x * 8 + (warp_index)) * 16;   \
    for (int cyc_i_ = 0; cyc_i_ < 16; ++cyc_i_) cyc_out_[cyc_i_] = cyc_[cyc_i_];                         \
  }
// pair kernel: one record of 8 counters per (CTA < 64, warp 0..11)
#define ATTN_CYC_WRITE12(trace, warp_index)                                                                \
  if ((trace) && (threadIdx.x & 31) == 0 && blockIdx.x < 64) {                                             \
    long long* cyc_out_ = reinterpret_cast<long long*>(trace) + (blockIdx.x * 12 + (warp_index)) * 8;   \
    for (int cyc_i_ = 0; cyc_i_ < 8; ++cyc_i_) cyc_out_[cyc_i_] = cyc_[cyc_i_];                          \
  }
#define ATTN_INSTRUMENTED 1
#else
#define ATTN_CYC_WRITE12(trace, warp_index)
#define ATTN_CYC_WRITE16(trace, warp_index)
#define ATTN_CYC_DECL()
#define ATTN_CYC_START()
#define ATTN_CYC_ADD(i)
#define ATTN_CYC_COUNT(i)
#define ATTN_CYC_TIMED(i, stmt) stmt;
#define ATTN_CYC_WRITE(trace, warp_index)
#define ATTN_INSTRUMENTED 0
#endif
