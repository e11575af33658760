/*
 * attn_numa.h -- C-ABI boundary of the B200 attention hot path (forward,
 * and the backward of NEXT-3).
 *
 * The library computes the FlashAttention-2-style forward pass of
 * PAPER.md eq:fa (lines 149-155),
 *
 *     S = Q K^T,   P = softmax(scale * S) (row-wise),   O = P V,
 *
 * for multi-head (Hq == Hkv) and grouped-query (Hkv < Hq) attention
 * (PAPER.md:167), tiled into work units of query-row blocks (PAPER.md:174,
 * fig:fa2), and hands those units to SMs in one of four orders (the
 * paper's "mappings"):
 *
 *   ATTN_MAP_BLOCK_FIRST          Naive Block-first
 *   ATTN_MAP_HEAD_FIRST           Naive Head-first
 *   ATTN_MAP_SWIZZLED_HEAD_FIRST  Swizzled Head-first:
 *        every unit of one Attention Compute Cluster (a head, or a GQA
 *        group) is processed on SMs of one die, each die
 *        serving its ACCs one at a time.
 *   ATTN_MAP_SWIZZLED_BLOCK_FIRST Swizzled Block-first   (PAPER.md:236-243,
 *        SPEC.md:172): block-first order with KV group g pinned to die
 *        g mod n_dies (co-locates ACCs only when #groups is a multiple of
 *        the die count).
 *
 * The result does not depend on the mapping, bit for bit.
 *
 * Conventions shared by every entry point:
 *  - Tensors are row-major contiguous [B][H][N][d] (PAPER.md:187,
 *    fig:attn-grid): q and o are [B][Hq][N][d], k and v are [B][Hkv][N][d],
 *    all bf16 (raw 16-bit storage, passed as void*).  Accumulation is fp32.
 *  - GQA grouping: query head h reads K/V head h / (Hq / Hkv).
 *  - causal != 0 masks key j from query i when j > i (N_q == N_k).
 *  - Any N >= 1: a ragged last block is handled with TMA out-of-bounds
 *    zero fill, key masking and row-guarded stores.
 *  - Head dim d: any multiple of 8 up to 128 (DeepSeek-V3's 56, PAPER.md:417,
 *    included).  The kernel runs at 64 or 128 columns; TMA zero-fills the
 *    padding columns on load and they are never stored.
 *  - Pointers of attn_fwd / attn_fwd_stream are DEVICE pointers on the
 *    calling thread's current CUDA device; the caller owns them.  The
 *    library never frees or retains them beyond the enqueued kernel; q, k, v
 *    are read-only; every element of o is written.  Base pointers must be
 *    16-byte aligned; o must not overlap q, k or v.
 *  - All calls return an attn_status_t synchronously, before any launch.
 *    Nothing throws, aborts or prints.  A failed call leaves o untouched.
 *    attn_last_error() gives a thread-local detail string.
 *  - The library owns per-device workspace (die table, scheduler counters,
 *    probe buffers), created lazily under a mutex and released by
 *    attn_shutdown().
 *  - Concurrency: launches are asynchronous on the caller's stream.  Each
 *    stream gets its own slot of scheduler queue counters (the persistent
 *    grid pops work with atomics on them and its last CTA re-zeroes them), so
 *    any number of calls may be queued on one stream, and calls on up to 64
 *    DIFFERENT streams of one device may be in flight at the same time.
 *    Beyond 64 concurrently busy streams, or when a CUDA graph that captured
 *    a launch is replayed on another stream while eager launches run on the
 *    capture stream, two grids can share counters and skip or repeat work
 *    units: serialise such launches.  attn_bwd's rowsum(dO o O) workspace is
 *    allocated per call in stream order (cudaMallocAsync), so concurrent
 *    backward calls on different streams are safe.
 */
#ifndef ATTN_NUMA_H
#define ATTN_NUMA_H

#include <stdint.h>

#if defined(__GNUC__)
#define ATTN_API __attribute__((visibility("default")))
#else
#define ATTN_API
#endif

#ifdef __cplusplus
extern "C" {
#endif

typedef enum {
  ATTN_MAP_BLOCK_FIRST = 0,
  ATTN_MAP_HEAD_FIRST = 1,
  ATTN_MAP_SWIZZLED_HEAD_FIRST = 2,
  ATTN_MAP_SWIZZLED_BLOCK_FIRST = 3
} attn_mapping_t;

/* OR into `mapping`: visit the work units of every (b, h) in DESCENDING
 * order (longest causal unit first) instead of the paper's ascending order
 * (PAPER.md:226, :246).  Applied identically under every mapping; it changes
 * only the schedule, never the result bits. */
#define ATTN_ORDER_DESCENDING 0x100

/* OR into `mapping`: alternate the unit direction per die queue -- queue d
 * visits each (b, h)'s units ascending if d is even, descending if d is odd
 * (XOR-combined with ATTN_ORDER_DESCENDING).  Only the swizzled mappings have
 * more than one queue; block-first / head-first are unaffected.  Purpose
 * (B200 reading, R22): under swizzled head-first the two dies each
 * stream one causal head, and a causal head's live K/V prefix grows with the
 * unit index; running the dies in opposite directions keeps the SUM of the
 * two live prefixes -- what the dies' shared L2 must hold -- near one head's
 * K/V instead of two.  Schedule only: never changes the result bits. */
#define ATTN_ORDER_ALTERNATE 0x400

/* OR into `mapping` (forward only): run CTA pairs as thread-block clusters
 * (NEXT-4, the ACC idea one level down: "CTAs that share K/V
 * should run together").  The two CTAs of a cluster take adjacent work units
 * that need the same K/V blocks -- the same unit of two query heads of one
 * KV group when Hq/Hkv is even, else two adjacent units of one head -- and
 * stream them once: each CTA TMA-loads half of every block and multicasts it
 * to both, so a K/V block is read from L2 once per pair.  The mapping then
 * orders the pairs ("cluster units").  Bit-identical results to the
 * non-cluster path. */
#define ATTN_CLUSTER_MULTICAST 0x200

/* OR into `mapping` with ATTN_MAP_SWIZZLED_HEAD_FIRST: the grain of "one
 * ACC per die".  B200 reading R23: the two
 * dies share ONE L2 (lines homed by address; the probe measures that a far
 * line is not replicated near, far_lines_cached_near = 0), so serving one ACC
 * per die keeps n_domains ACC K/V footprints live in that L2 at once.
 *   ATTN_SHF_ACC_SHARED   every ACC is served by all dies together: the dies
 *                         form ONE capacity domain, and swizzled head-first
 *                         over one domain is the head-major order (one queue
 *                         popped by every SM);
 *   ATTN_SHF_ACC_PER_DIE  the paper's literal grain (one die per ACC) always;
 *   neither               the library decides per call with
 *                         attn_shf_acc_shared(n_domains, N, d, l2_bytes).
 * Schedule only: never changes the result bits.  Exclusive with each other;
 * ignored by the other mappings. */
#define ATTN_SHF_ACC_SHARED 0x800
#define ATTN_SHF_ACC_PER_DIE 0x1000

/* OR into `mapping` (attn_bwd / attn_bwd_host; the forward ignores it): run
 * the two-pass backward whose dq is bit-reproducible.  Without it, head dims
 * d <= 64 use the single-pass kernel (csrc/attn_bwd_fused_sm100.cuh), which
 * computes P and dS once and accumulates dq with fp32 reduce-adds in L2 in
 * arrival order: dq may then differ in the last bits between runs and
 * between mappings (dk and dv stay bit-identical).  d > 64 always runs the
 * two-pass backward. */
#define ATTN_BWD_DETERMINISTIC 0x2000

typedef enum {
  ATTN_OK = 0,
  ATTN_ERR_INVALID_VALUE = 1, /* null pointer, size <= 0, Hq % Hkv != 0, bad mapping value,
                                 non-finite scale, overlap, not device memory */
  ATTN_ERR_UNSUPPORTED = 2,   /* d > 128 or d % 8 != 0; misaligned; scale < 0;
                                 device is not sm_100 */
  ATTN_ERR_CUDA = 3,          /* CUDA runtime / driver failure (see attn_last_error) */
  ATTN_ERR_TOPOLOGY = 4       /* the die probe itself failed (an inconclusive probe is
                                 NOT an error: it falls back to one domain) */
} attn_status_t;

/* Per-device die topology, measured once per process by a startup
 * microbenchmark (%smid census + per-SM L2 hit latency matrix), or injected
 * with attn_set_topology_override.  PAPER.md:100-109 ("kernels must
 * incorporate mutable, algorithmic mapping logic"), :317-323 (per-die L2). */
#define ATTN_MAX_DOMAINS 8
#define ATTN_MAX_SMID 512
typedef struct {
  int num_sms;                              /* cudaDevAttrMultiProcessorCount */
  int nsmid;                                /* %nsmid: upper bound of %smid values */
  int n_domains;                            /* 1 or 2 on B200 */
  int sms_per_domain[ATTN_MAX_DOMAINS];
  signed char domain_of_smid[ATTN_MAX_SMID];/* -1 for ids never observed */
  float lat_near_cyc;                       /* median L2-hit latency, near lines */
  float lat_far_cyc;                        /* median L2-hit latency, far lines */
  int far_lines_cached_near;                /* measured: 1 if a far line re-read after its first
                                               (ld.global.cg) access comes back at the near
                                               latency, i.e. the reading die keeps a copy */
  long long l2_bytes;                       /* cudaDevAttrL2CacheSize */
  int source;                               /* 0 probe, 1 override, 2 fallback (1 domain) */
  int stable;                               /* 1 if two probe runs agreed */
  float lat_near_reread_cyc;                /* median re-read latency of near lines after a flush */
  float lat_far_reread_cyc;                 /* same for far lines (probe SM of each die) */
} attn_topology_t;

/* One record per work unit when a schedule trace buffer is installed. */
typedef struct {
  int32_t b, h, unit;   /* unit = pair of 128-row query blocks (rows [256u, 256u+256)) */
  int32_t smid;         /* %smid of the CTA that processed it */
  int32_t domain;       /* die of that SM per the active topology */
  int32_t queue;        /* queue it was popped from */
  int32_t stolen;       /* 1 if popped from another die's queue (tail balancing) */
  int32_t seq;          /* pop index within the CTA */
  uint64_t t_pop_ns;    /* %globaltimer at pop */
} attn_trace_rec_t;

/* Forward attention on the stream set by attn_set_stream (default: legacy
 * stream 0).  See the conventions above.  scale is typically 1/sqrt(d)
 * (eq:fa); any finite scale >= 0 is accepted, 0 gives uniform weights. */
ATTN_API int attn_fwd(const void* q, const void* k, const void* v, void* o, int B, int Hq, int Hkv, int N, int d,
             int causal, float scale, int mapping);

/* Same, on an explicit cudaStream_t (passed as void*; NULL = legacy stream). */
ATTN_API int attn_fwd_stream(const void* q, const void* k, const void* v, void* o, int B, int Hq, int Hkv, int N,
                    int d, int causal, float scale, int mapping, void* cuda_stream);

/* Same as attn_fwd_stream and also writes lse[B][Hq][N] (fp32, device
 * memory): lse[b,h,i] = log sum_j exp(scale * s_ij) over the visible keys
 * (natural log), the per-row statistic the backward pass needs. */
ATTN_API int attn_fwd_lse(const void* q, const void* k, const void* v, void* o, float* lse, int B, int Hq, int Hkv,
                          int N, int d, int causal, float scale, int mapping, void* cuda_stream);

/* Backward pass (eq:ba) on the stream `cuda_stream`:
 *   dV = P^T dO,  dP = dO V^T,  dS = P o (dP - rowsum(dO o O)),
 *   dQ = scale * dS K,  dK = scale * dS^T Q,   P = exp(scale * Q K^T - lse).
 * q, k, v, o, dout: device bf16 in the forward's layouts; lse: device fp32
 * [B][Hq][N] from attn_fwd_lse; dq [B][Hq][N][d], dk, dv [B][Hkv][N][d]: device
 * bf16 outputs, fully written (GQA: dk, dv sum over the group's query heads).
 * `mapping` orders the work units exactly as for the forward (dQ: query
 * blocks of a head; dK/dV: key blocks of a KV group).  Launches:
 * rowsum(dO o O) into per-call library workspace, then either the dQ kernel
 * and the dK/dV kernel (d > 64, or ATTN_BWD_DETERMINISTIC), or, for d <= 64,
 * a zero fill of a per-call fp32 dq accumulator [B][Hq][N][64] (4*B*Hq*N*64
 * bytes of workspace), the single-pass kernel and a dq conversion kernel.
 * Same validation and status codes as attn_fwd (ATTN_ORDER_DESCENDING
 * applies; ATTN_CLUSTER_MULTICAST returns ATTN_ERR_UNSUPPORTED: the
 * backward has no cluster variant); gradients must not overlap each other or
 * any input. */
ATTN_API int attn_bwd(const void* q, const void* k, const void* v, const void* o, const void* dout,
                      const float* lse, void* dq, void* dk, void* dv, int B, int Hq, int Hkv, int N, int d,
                      int causal, float scale, int mapping, void* cuda_stream);

/* End-to-end variant on HOST buffers (same layout): copies q/k/v host->device
 * into library-owned device buffers, runs the kernel, copies o device->host
 * and synchronises `cuda_stream` before returning.  Large problems are split
 * into chunks of whole KV groups (heads are independent, so the
 * result is bit-identical to one call) and pipelined on three library streams
 * ordered after `cuda_stream`: H2D of chunk i+1 overlaps the kernel of chunk i
 * and the D2H of chunk i-1.  Host buffers should be pinned (cudaHostAlloc /
 * torch pin_memory) for the copies to overlap; pageable memory works but is
 * slower.  Library buffers are reused across calls of equal or smaller size
 * and freed by attn_shutdown().  Not reentrant across threads on one device. */
ATTN_API int attn_fwd_host(const void* q_host, const void* k_host, const void* v_host, void* o_host, int B, int Hq,
                  int Hkv, int N, int d, int causal, float scale, int mapping, void* cuda_stream);

/* End-to-end backward on HOST buffers (layouts as attn_bwd; lse is fp32
 * [B][Hq][N]): copies q, k, v, o, dout, lse host->device into library-owned
 * device buffers, runs attn_bwd's kernels, copies dq, dk, dv device->host and
 * synchronises `cuda_stream` before returning.  Pipelined like attn_fwd_host
 * (chunks of whole KV groups of one batch item on three library streams:
 * H2D of chunk i+1 || backward of chunk i || D2H of chunk i-1); the gradients
 * of different KV groups are independent (eq:ba), so the
 * result is bit-identical to one attn_bwd call on device copies.  Host
 * buffers should be pinned.  Errors as attn_bwd (ATTN_CLUSTER_MULTICAST is
 * UNSUPPORTED); buffers are reused across calls and freed by attn_shutdown().
 * Not reentrant across threads on one device. */
ATTN_API int attn_bwd_host(const void* q_host, const void* k_host, const void* v_host, const void* o_host,
                           const void* dout_host, const float* lse_host, void* dq_host, void* dk_host, void* dv_host,
                           int B, int Hq, int Hkv, int N, int d, int causal, float scale, int mapping,
                           void* cuda_stream);

/* Head-sharded forward with REPLICATED output stored by the kernel itself
 * (the fused alternative to an all-gather of O; heads are
 * independent).  q, k, v are this rank's shard ([B][Hq][N][d],
 * [B][Hkv][N][d], device memory of the current device; B, Hq, Hkv are the
 * SHARD's sizes).  o_dst is a HOST array of n_dst (1..ATTN_MAX_DST) device
 * pointers, each a full output [B][Hq_out][N][d] bf16: this device's own
 * buffer, or a peer GPU's buffer mapped into this process (attn_ipc_open;
 * NVLink P2P).  The epilogue stores every finished O tile of head h into
 * every o_dst[i] at head head_offset + h, so after all ranks' kernels have
 * completed (the caller synchronises its stream and then the ranks, e.g. a
 * process-group barrier) each rank holds the whole [B][Hq_out][N][d] result.
 * Only the shard's heads are written; the values are bit-identical to
 * attn_fwd on the shard.  Needs 0 <= head_offset, head_offset + Hq <= Hq_out;
 * destinations must not overlap each other or the inputs.  Same status
 * codes as attn_fwd (ATTN_CLUSTER_MULTICAST and ATTN_ORDER_DESCENDING apply). */
#define ATTN_MAX_DST 8
ATTN_API int attn_fwd_replicated(const void* q, const void* k, const void* v, void* const* o_dst, int n_dst,
                                 int Hq_out, int head_offset, int B, int Hq, int Hkv, int N, int d, int causal,
                                 float scale, int mapping, void* cuda_stream);

/* CUDA IPC for attn_fwd_replicated's peer destinations.  attn_ipc_get_handle
 * exports the allocation containing dev_ptr (device memory of the current
 * device, from cudaMalloc, e.g. torch's caching allocator) and records
 * dev_ptr's offset in it; the 72-byte record is sent to the other ranks (any
 * byte transport).  attn_ipc_open, in ANOTHER process, maps it on the current
 * device (peer access enabled lazily) and returns the address of dev_ptr in
 * that mapping; attn_ipc_close unmaps a pointer attn_ipc_open returned.  The
 * exporting process must keep the allocation alive until every importer has
 * closed it.  Errors: ATTN_ERR_INVALID_VALUE (null / foreign pointer),
 * ATTN_ERR_CUDA (the CUDA IPC call failed, e.g. opening a handle in the
 * process that exported it). */
typedef struct {
  unsigned char handle[64]; /* cudaIpcMemHandle_t of the containing allocation */
  long long offset;         /* dev_ptr - allocation base */
} attn_ipc_handle_t;
ATTN_API int attn_ipc_get_handle(const void* dev_ptr, attn_ipc_handle_t* out);
ATTN_API int attn_ipc_open(const attn_ipc_handle_t* h, void** dev_ptr_out);
ATTN_API int attn_ipc_close(void* dev_ptr);

/* Thread-local default stream for attn_fwd. */
ATTN_API int attn_set_stream(void* cuda_stream);

/* Eager per-device init: runs the topology probe (normally done lazily on
 * the first call).  Benchmarks call it before timing. */
ATTN_API int attn_init(int device);

/* Copies the active topology of `device` into *out (probing if needed). */
ATTN_API int attn_topology(int device, attn_topology_t* out);

/* Replace the measured die table of `device` (tests / fakes): domain_of_smid
 * has n entries with values in [0, n_domains) or -1.  NULL restores the
 * measured table. */
ATTN_API int attn_set_topology_override(int device, const signed char* domain_of_smid, int n, int n_domains);

/* Install a device buffer of `capacity` attn_trace_rec_t records (indexed by
 * the unit's head-major id (b*Hq + h)*units_per_head + unit) that subsequent
 * launches on `device` fill; NULL disables.  Debug / evidence only. */
ATTN_API int attn_set_schedule_trace(int device, void* dev_buf, long long capacity);

/* Host-side view of the queues a launch would pop, for tests: writes, for
 * every queue q and position i, the unit (b, h, unit) into out[3*k..3*k+2]
 * in queue-major order and the queue lengths into queue_len[0..n_queues).
 * n_domains / sms_per_domain describe the dies (the active topology is not
 * consulted).  units_per_head = ceil(N / 256).  With ATTN_CLUSTER_MULTICAST
 * the entries are cluster units: if Hq/Hkv is even, (b, head pair p, unit u)
 * = unit u of query heads 2p and 2p+1 (Hq/2 "heads"); otherwise (b, h, c) =
 * units 2c and 2c+1 of head h (ceil(units_per_head / 2) per head).  Returns
 * INVALID_VALUE if capacity (in units) is too small. */
ATTN_API int attn_schedule_order(int B, int Hq, int Hkv, int N, int mapping, int n_domains, const int* sms_per_domain,
                        int32_t* out, long long capacity, int* n_queues, int* queue_len);

/* The rule swizzled head-first applies when neither ATTN_SHF_ACC_* flag is
 * given (R23): 1 (share every ACC among the dies) iff n_domains > 1,
 * l2_bytes > 0 and n_domains * (K + V bytes of one KV head = 4*N*d) >
 * l2_bytes / 2, else 0.  Pure function; no device access. */
ATTN_API int attn_shf_acc_shared(int n_domains, int N, int d, long long l2_bytes);

/* Launch geometry of the last successful attn_fwd* on this thread;
 * shf_acc_shared = 1 if swizzled head-first ran with ACCs shared by all dies. */
typedef struct {
  int grid, block, smem_bytes, units, n_queues, kernel_launches, shf_acc_shared;
} attn_launch_info_t;
ATTN_API int attn_last_launch_info(attn_launch_info_t* out);

ATTN_API const char* attn_status_string(int status);
ATTN_API const char* attn_last_error(void);
ATTN_API const char* attn_version(void);
ATTN_API void attn_shutdown(void);

#ifdef __cplusplus
}
#endif
#endif /* ATTN_NUMA_H */
