// api.cu -- the C-ABI boundary (include/attn_numa.h): argument validation,
// per-device state (die topology, scheduler counters), TMA descriptors and
// the launch of the sm_100a attention kernel.
#include <cuda.h>
#include <cuda_runtime.h>
#include <cudaTypedefs.h>

#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <mutex>
#include <string>
#include <vector>

#include "../../include/attn_numa.h"
#include "attn_bwd_sm100.cuh"
#include "attn_bwd_fused_sm100.cuh"
#include "attn_fwd_sm100.cuh"
#include "attn_fwd_pair.cuh"
#include "attn_sched.h"
#include "topology.cuh"

namespace {

using namespace attn;

constexpr int kMaxDevices = 16;
constexpr int kCounterSlots = 64;
#ifndef ATTN_E2E_CHUNKS
#define ATTN_E2E_CHUNKS 32
#endif
#ifndef ATTN_E2E_CHUNK_MB
#define ATTN_E2E_CHUNK_MB 48
#endif
constexpr int kE2EChunks = ATTN_E2E_CHUNKS;  // max chunks of the pipelined host-buffer path
constexpr int kCounterInts = (kMaxQueues + 1) * 32;  // one 128-byte line per queue + done count

thread_local std::string g_err;
thread_local cudaStream_t g_stream = nullptr;
thread_local attn_launch_info_t g_info = {};

int fail(int status, const std::string& msg) {
  g_err = msg;
  return status;
}
int cuda_fail(cudaError_t e, const char* what) {
  g_err = std::string(what) + ": " + cudaGetErrorString(e);
  return ATTN_ERR_CUDA;
}
#define ATTN_CUDA(call)                                  \
  do {                                                   \
    cudaError_t e__ = (call);                            \
    if (e__ != cudaSuccess) return cuda_fail(e__, #call); \
  } while (0)

struct DevState {
  std::mutex mu;
  bool init = false;
  int num_sms = 0;
  attn_topology_t measured{};
  attn_topology_t active{};
  signed char* d_domain = nullptr;
  int* d_counters = nullptr;
  // counter slot of each stream that launched recently (see counter_slot)
  cudaStream_t slot_stream[kCounterSlots] = {};
  unsigned long long slot_used[kCounterSlots] = {};
  unsigned long long slot_tick = 0;
  attn_trace_rec_t* trace = nullptr;
  long long trace_cap = 0;
  bool attr_done[16] = {};       // forward variants: [idx + 4 * cluster + 8 * ones-column row sum]
  int max_clusters[8] = {};       // co-resident CTA-pair clusters per forward variant [idx + 4 * ones]
  bool pattr_done[2] = {false, false};  // attn_fwd_pair_kernel<causal>
  int pmax_clusters[2] = {0, 0};
  // e2e host-buffer path
  void* hbuf[4] = {nullptr, nullptr, nullptr, nullptr};
  size_t hbuf_bytes[4] = {0, 0, 0, 0};
  // backward host-buffer path: q k v o dO lse dq dk dv
  void* bbuf[9] = {};
  size_t bbuf_bytes[9] = {};
  bool e2e_ready = false;
  bool battr_done[8] = {false, false, false, false, false, false, false, false};
  bool fattr_done[2] = {false, false};  // attn_bwd_fused_kernel<64, causal>
  // stream-ordered pool for per-call backward workspace (rowsum(dO o O), the
  // fp32 dQ accumulator); keeps freed blocks mapped (release threshold max)
  cudaMemPool_t ws_pool = nullptr;
  cudaStream_t e2e_stream[4] = {nullptr, nullptr, nullptr, nullptr};  // H2D, compute (even chunks), D2H, compute (odd)
  cudaEvent_t e2e_ev[2][kE2EChunks + 1] = {};
};

DevState g_dev[kMaxDevices];

PFN_cuTensorMapEncodeTiled_v12000 g_encode = nullptr;

int get_encode() {
  if (g_encode) return ATTN_OK;
  void* fn = nullptr;
  cudaDriverEntryPointQueryResult q;
  cudaError_t e = cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q);
  if (e != cudaSuccess || fn == nullptr || q != cudaDriverEntryPointSuccess)
    return fail(ATTN_ERR_CUDA, "cuTensorMapEncodeTiled entry point not found");
  g_encode = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(fn);
  return ATTN_OK;
}

// ---------------------------------------------------------------- topology
void fallback_topology(attn_topology_t& t) {
  t.n_domains = 1;
  for (int i = 0; i < ATTN_MAX_DOMAINS; ++i) t.sms_per_domain[i] = 0;
  int n = 0;
  for (int s = 0; s < ATTN_MAX_SMID; ++s) {
    if (t.domain_of_smid[s] >= 0) {
      t.domain_of_smid[s] = 0;
      ++n;
    }
  }
  t.sms_per_domain[0] = n > 0 ? n : t.num_sms;
  t.source = 2;
}

// One probe run: fills lat (nsmid x kProbeLines, 0xFFFFFFFF for absent SMs).
int probe_once(int nsmid, const uint32_t* d_probe, std::vector<uint32_t>& lat, int num_sms) {
  int* d_claimed = nullptr;
  uint32_t* d_lat = nullptr;
  ATTN_CUDA(cudaMalloc(&d_claimed, sizeof(int) * nsmid));
  ATTN_CUDA(cudaMalloc(&d_lat, sizeof(uint32_t) * nsmid * kProbeLines));
  ATTN_CUDA(cudaMemset(d_claimed, 0, sizeof(int) * nsmid));
  ATTN_CUDA(cudaMemset(d_lat, 0xFF, sizeof(uint32_t) * nsmid * kProbeLines));
  topo_latency_kernel<<<8 * num_sms, 32>>>(d_probe, d_claimed, d_lat, nsmid);
  ATTN_CUDA(cudaGetLastError());
  ATTN_CUDA(cudaDeviceSynchronize());
  lat.assign((size_t)nsmid * kProbeLines, 0);
  ATTN_CUDA(cudaMemcpy(lat.data(), d_lat, sizeof(uint32_t) * lat.size(), cudaMemcpyDeviceToHost));
  cudaFree(d_claimed);
  cudaFree(d_lat);
  return ATTN_OK;
}

// Classify SMs into dies from a latency matrix (returns false if inconclusive).
// Every SM's vector of per-line latencies is centred on its own mean; SMs of
// one die see the same lines as near/far, so their vectors are close.  Two
// centroids are seeded with SM s0 and the SM farthest from it, then refined
// by 2-means (Lloyd).  The split is accepted if the centroids differ by at
// least 8 cycles on average over the lines (near ~235 vs far ~265 cycles).
bool classify(const std::vector<uint32_t>& lat, const std::vector<int>& present, signed char* dom, float& near_c,
              float& far_c) {
  const int S = (int)present.size(), L = kProbeLines;
  if (S < 2) return false;
  std::vector<double> z((size_t)S * L);
  for (int i = 0; i < S; ++i) {
    double mean = 0;
    for (int l = 0; l < L; ++l) mean += lat[(size_t)present[i] * L + l];
    mean /= L;
    for (int l = 0; l < L; ++l) z[(size_t)i * L + l] = lat[(size_t)present[i] * L + l] - mean;
  }
  auto dist2 = [&](const double* a, const double* b) {
    double d = 0;
    for (int l = 0; l < L; ++l) d += (a[l] - b[l]) * (a[l] - b[l]);
    return d;
  };
  int far_i = 0;
  double best = -1;
  for (int i = 0; i < S; ++i) {
    const double d = dist2(&z[0], &z[(size_t)i * L]);
    if (d > best) { best = d; far_i = i; }
  }
  std::vector<double> c0(z.begin(), z.begin() + L), c1(z.begin() + (size_t)far_i * L, z.begin() + (size_t)far_i * L + L);
  std::vector<int> lab(S, 0);
  for (int it = 0; it < 30; ++it) {
    for (int i = 0; i < S; ++i) lab[i] = dist2(&z[(size_t)i * L], c1.data()) < dist2(&z[(size_t)i * L], c0.data());
    lab[0] = 0;  // s0 defines die 0
    std::vector<double> n0(L, 0), n1(L, 0);
    int k0 = 0, k1 = 0;
    for (int i = 0; i < S; ++i) {
      auto& c = lab[i] ? n1 : n0;
      for (int l = 0; l < L; ++l) c[l] += z[(size_t)i * L + l];
      (lab[i] ? k1 : k0)++;
    }
    if (k0 == 0 || k1 == 0) return false;
    for (int l = 0; l < L; ++l) { c0[l] = n0[l] / k0; c1[l] = n1[l] / k1; }
  }
  double sep = 0;
  for (int l = 0; l < L; ++l) sep += std::fabs(c0[l] - c1[l]);
  sep /= L;
  // near/far latency: per line, the lower / higher of the two clusters' raw means
  std::vector<double> nearv, farv;
  for (int l = 0; l < L; ++l) {
    double m0 = 0, m1 = 0;
    int k0 = 0, k1 = 0;
    for (int i = 0; i < S; ++i) {
      const double x = lat[(size_t)present[i] * L + l];
      if (lab[i]) { m1 += x; ++k1; } else { m0 += x; ++k0; }
    }
    m0 /= k0;
    m1 /= k1;
    nearv.push_back(std::min(m0, m1));
    farv.push_back(std::max(m0, m1));
  }
  std::sort(nearv.begin(), nearv.end());
  std::sort(farv.begin(), farv.end());
  near_c = (float)nearv[L / 2];
  far_c = (float)farv[L / 2];
  if (sep < 8.0) return false;
  for (int i = 0; i < S; ++i) dom[present[i]] = (signed char)lab[i];
  return true;
}

// SURVEY.md §8(a1) step 6, measured: for one SM of each die, flush L2, touch
// every probe line once and time its re-reads (topo_reread_kernel).  Which
// lines are far for an SM comes from the latency matrix: per line, the die
// whose SMs see the higher mean latency is the far one.  far_lines_cached_near
// = 1 if far lines re-read closer to the near than to the far latency.
int measure_reread(attn_topology_t& t, const std::vector<int>& present, const std::vector<uint32_t>& lat,
                   const uint32_t* d_probe) {
  const int L = kProbeLines;
  std::vector<double> mean[2] = {std::vector<double>(L, 0.0), std::vector<double>(L, 0.0)};
  int cnt[2] = {0, 0};
  for (int s : present) {
    const int dm = t.domain_of_smid[s];
    for (int l = 0; l < L; ++l) mean[dm][l] += lat[(size_t)s * L + l];
    ++cnt[dm];
  }
  if (cnt[0] == 0 || cnt[1] == 0) return ATTN_OK;
  for (int dm = 0; dm < 2; ++dm)
    for (int l = 0; l < L; ++l) mean[dm][l] /= cnt[dm];
  size_t l2 = (size_t)t.l2_bytes;
  void* flush = nullptr;
  int* d_claimed = nullptr;
  uint32_t* d_rr = nullptr;
  std::vector<double> near_rr, far_rr;
  // the scratch buffers are freed on every path out of the measurement
  auto measure = [&]() -> int {
    ATTN_CUDA(cudaMalloc(&flush, 2 * l2));
    ATTN_CUDA(cudaMalloc(&d_claimed, sizeof(int)));
    ATTN_CUDA(cudaMalloc(&d_rr, sizeof(uint32_t) * L));
    for (int dm = 0; dm < 2; ++dm) {
      int target = -1;
      for (int s : present)
        if (t.domain_of_smid[s] == dm) { target = s; break; }
      ATTN_CUDA(cudaMemset(flush, dm + 1, 2 * l2));  // evict the probe lines from L2
      ATTN_CUDA(cudaMemset(d_claimed, 0, sizeof(int)));
      ATTN_CUDA(cudaMemset(d_rr, 0xFF, sizeof(uint32_t) * L));
      topo_reread_kernel<<<8 * t.num_sms, 32>>>(d_probe, d_claimed, target, d_rr);
      ATTN_CUDA(cudaGetLastError());
      ATTN_CUDA(cudaDeviceSynchronize());
      std::vector<uint32_t> rr(L);
      ATTN_CUDA(cudaMemcpy(rr.data(), d_rr, sizeof(uint32_t) * L, cudaMemcpyDeviceToHost));
      for (int l = 0; l < L; ++l) {
        if (rr[l] == 0xFFFFFFFFu) continue;  // target SM never ran a CTA (cannot happen with 8 CTAs per SM)
        (mean[dm][l] > mean[1 - dm][l] ? far_rr : near_rr).push_back(rr[l]);
      }
    }
    return ATTN_OK;
  };
  const int mrc = measure();
  if (flush) cudaFree(flush);
  if (d_claimed) cudaFree(d_claimed);
  if (d_rr) cudaFree(d_rr);
  if (mrc != ATTN_OK) return mrc;
  if (near_rr.empty() || far_rr.empty()) return ATTN_OK;
  std::sort(near_rr.begin(), near_rr.end());
  std::sort(far_rr.begin(), far_rr.end());
  t.lat_near_reread_cyc = (float)near_rr[near_rr.size() / 2];
  t.lat_far_reread_cyc = (float)far_rr[far_rr.size() / 2];
  t.far_lines_cached_near =
      (t.lat_far_reread_cyc - t.lat_near_reread_cyc) < 0.5f * (t.lat_far_cyc - t.lat_near_cyc) ? 1 : 0;
  return ATTN_OK;
}

int run_probe(int dev, DevState& st) {
  attn_topology_t t{};
  memset(t.domain_of_smid, -1, sizeof(t.domain_of_smid));
  ATTN_CUDA(cudaDeviceGetAttribute(&t.num_sms, cudaDevAttrMultiProcessorCount, dev));
  int l2 = 0;
  ATTN_CUDA(cudaDeviceGetAttribute(&l2, cudaDevAttrL2CacheSize, dev));
  t.l2_bytes = l2;
  st.num_sms = t.num_sms;

  int *d_seen = nullptr, *d_n = nullptr;
  ATTN_CUDA(cudaMalloc(&d_seen, sizeof(int) * 1024));
  ATTN_CUDA(cudaMalloc(&d_n, sizeof(int)));
  ATTN_CUDA(cudaMemset(d_seen, 0, sizeof(int) * 1024));
  ATTN_CUDA(cudaMemset(d_n, 0, sizeof(int)));
  topo_census_kernel<<<8 * t.num_sms, 32>>>(d_seen, d_n);
  ATTN_CUDA(cudaGetLastError());
  ATTN_CUDA(cudaDeviceSynchronize());
  std::vector<int> seen(1024);
  int nsmid = 0;
  ATTN_CUDA(cudaMemcpy(seen.data(), d_seen, sizeof(int) * 1024, cudaMemcpyDeviceToHost));
  ATTN_CUDA(cudaMemcpy(&nsmid, d_n, sizeof(int), cudaMemcpyDeviceToHost));
  cudaFree(d_seen);
  cudaFree(d_n);
  std::vector<int> present;
  for (int s = 0; s < 1024; ++s)
    if (seen[s]) {
      if (s >= ATTN_MAX_SMID) return fail(ATTN_ERR_TOPOLOGY, "smid beyond ATTN_MAX_SMID");
      present.push_back(s);
      nsmid = std::max(nsmid, s + 1);
    }
  t.nsmid = nsmid;
  for (int s : present) t.domain_of_smid[s] = 0;

  const char* env = getenv("ATTN_NUMA_TOPOLOGY");
  if (env && strcmp(env, "fallback") == 0) {
    fallback_topology(t);
    t.stable = 1;
    st.measured = t;
    return ATTN_OK;
  }

  // probe buffer: every line's first word holds its own byte offset
  std::vector<uint32_t> host((size_t)kProbeLines * kProbeStrideBytes / 4, 0);
  for (int i = 0; i < kProbeLines; ++i) host[(size_t)i * kProbeStrideBytes / 4] = (uint32_t)i * kProbeStrideBytes;
  uint32_t* d_probe = nullptr;
  ATTN_CUDA(cudaMalloc(&d_probe, host.size() * 4));
  ATTN_CUDA(cudaMemcpy(d_probe, host.data(), host.size() * 4, cudaMemcpyHostToDevice));

  std::vector<uint32_t> lat_a, lat_b;
  int rc = probe_once(nsmid, d_probe, lat_a, t.num_sms);
  if (rc == ATTN_OK) rc = probe_once(nsmid, d_probe, lat_b, t.num_sms);
  if (rc != ATTN_OK) {
    cudaFree(d_probe);
    return rc;
  }
  if (const char* dump = getenv("ATTN_NUMA_PROBE_DUMP")) {
    if (FILE* f = fopen(dump, "w")) {
      for (int s : present) {
        fprintf(f, "%d", s);
        for (int l = 0; l < kProbeLines; ++l) fprintf(f, ",%u,%u", lat_a[(size_t)s * kProbeLines + l],
                                                     lat_b[(size_t)s * kProbeLines + l]);
        fprintf(f, "\n");
      }
      fclose(f);
    }
  }
  std::vector<int> measured_present;
  for (int s : present)
    if (lat_a[(size_t)s * kProbeLines] != 0xFFFFFFFFu && lat_b[(size_t)s * kProbeLines] != 0xFFFFFFFFu)
      measured_present.push_back(s);

  signed char dom_a[ATTN_MAX_SMID], dom_b[ATTN_MAX_SMID];
  memset(dom_a, -1, sizeof dom_a);
  memset(dom_b, -1, sizeof dom_b);
  float na = 0, fa = 0, nb = 0, fb = 0;
  const bool ok_a = measured_present.size() == present.size() &&
                    classify(lat_a, measured_present, dom_a, na, fa);
  const bool ok_b = ok_a && classify(lat_b, measured_present, dom_b, nb, fb);
  bool same = ok_a && ok_b;
  if (same) {
    // the reference SM defines die 0 in both runs, so the labels are comparable
    for (int s : present) same = same && (dom_a[s] == dom_b[s]);
  }
  t.lat_near_cyc = na;
  t.lat_far_cyc = fa;
  t.stable = same ? 1 : 0;
  if (!same) {
    cudaFree(d_probe);
    fallback_topology(t);
    st.measured = t;
    return ATTN_OK;
  }
  t.n_domains = 2;
  t.sms_per_domain[0] = t.sms_per_domain[1] = 0;
  for (int s : present) {
    t.domain_of_smid[s] = dom_a[s];
    ++t.sms_per_domain[(int)dom_a[s]];
  }
  rc = measure_reread(t, present, lat_a, d_probe);
  cudaFree(d_probe);
  if (rc != ATTN_OK) return rc;
  t.source = 0;
  st.measured = t;
  return ATTN_OK;
}

int upload_domain(DevState& st) {
  if (!st.d_domain) ATTN_CUDA(cudaMalloc(&st.d_domain, ATTN_MAX_SMID));
  ATTN_CUDA(cudaMemcpy(st.d_domain, st.active.domain_of_smid, ATTN_MAX_SMID, cudaMemcpyHostToDevice));
  return ATTN_OK;
}

// Caller holds st.mu and has set the current device.
int ensure_init(int dev, DevState& st) {
  if (st.init) return ATTN_OK;
  cudaDeviceProp prop;
  ATTN_CUDA(cudaGetDeviceProperties(&prop, dev));
  if (prop.major != 10 || prop.minor != 0)
    return fail(ATTN_ERR_UNSUPPORTED, "device is not sm_100 (compute capability " + std::to_string(prop.major) +
                                          "." + std::to_string(prop.minor) + ")");
  int rc = run_probe(dev, st);
  if (rc != ATTN_OK) return rc;
  st.active = st.measured;
  rc = upload_domain(st);
  if (rc != ATTN_OK) return rc;
  ATTN_CUDA(cudaMalloc(&st.d_counters, sizeof(int) * kCounterInts * kCounterSlots));
  ATTN_CUDA(cudaMemset(st.d_counters, 0, sizeof(int) * kCounterInts * kCounterSlots));
  st.init = true;
  return ATTN_OK;
}

// Scheduler counters of a launch on `s` (caller holds st.mu).  The kernels
// pop their queues with atomics on these counters and the last CTA zeroes
// them on exit, so two grids may share a slot only if they never run at the
// same time.  Every stream keeps its own slot (launches on one stream are
// serialised, so a slot is back at zero when the stream's next grid starts);
// with more than kCounterSlots streams the least recently used stream's slot
// is handed over.  Contract (include/attn_numa.h): at most kCounterSlots
// streams of one device may have attention launches in flight at once.
unsigned counter_slot(DevState& st, cudaStream_t s) {
  unsigned best = 0;
  for (unsigned i = 0; i < kCounterSlots; ++i) {
    if (st.slot_used[i] != 0 && st.slot_stream[i] == s) {
      st.slot_used[i] = ++st.slot_tick;
      return i;
    }
    if (st.slot_used[i] < st.slot_used[best]) best = i;
  }
  st.slot_stream[best] = s;
  st.slot_used[best] = ++st.slot_tick;
  return best;
}

int current_device(int& dev) {
  ATTN_CUDA(cudaGetDevice(&dev));
  if (dev < 0 || dev >= kMaxDevices) return fail(ATTN_ERR_UNSUPPORTED, "device index beyond kMaxDevices");
  return ATTN_OK;
}

// ----------------------------------------------------------------- launch
int check_dev_ptr(const void* p, int dev, const char* name) {
  cudaPointerAttributes a;
  cudaError_t e = cudaPointerGetAttributes(&a, p);
  if (e != cudaSuccess) {
    cudaGetLastError();
    return fail(ATTN_ERR_INVALID_VALUE, std::string(name) + " is not a CUDA pointer");
  }
  if (!(a.type == cudaMemoryTypeDevice || a.type == cudaMemoryTypeManaged) || a.device != dev)
    return fail(ATTN_ERR_INVALID_VALUE, std::string(name) + " is not device memory of the current device");
  return ATTN_OK;
}

bool overlaps(const void* a, size_t na, const void* b, size_t nb) {
  const uintptr_t x = reinterpret_cast<uintptr_t>(a), y = reinterpret_cast<uintptr_t>(b);
  return x < y + nb && y < x + na;
}

int validate(const void* q, const void* k, const void* v, void* o, int B, int Hq, int Hkv, int N, int d,
             float scale, int mapping) {
  if (!q || !k || !v || !o) return fail(ATTN_ERR_INVALID_VALUE, "null pointer");
  if (B <= 0 || Hq <= 0 || Hkv <= 0 || N <= 0 || d <= 0) return fail(ATTN_ERR_INVALID_VALUE, "size <= 0");
  if (Hq % Hkv != 0) return fail(ATTN_ERR_INVALID_VALUE, "Hq % Hkv != 0 (non-uniform GQA groups)");
  if ((mapping & ~(kMapMask | kOrderDescending | kOrderAlternate | ATTN_CLUSTER_MULTICAST | kShfAccShared |
                   kShfAccPerDie | ATTN_BWD_DETERMINISTIC)) || (mapping & kMapMask) > 3)
    return fail(ATTN_ERR_INVALID_VALUE,
                "mapping not in {0,1,2,3} (| ATTN_ORDER_DESCENDING | ATTN_ORDER_ALTERNATE | ATTN_CLUSTER_MULTICAST | "
                "ATTN_SHF_ACC_SHARED | ATTN_SHF_ACC_PER_DIE | ATTN_BWD_DETERMINISTIC)");
  if ((mapping & kShfAccShared) && (mapping & kShfAccPerDie))
    return fail(ATTN_ERR_INVALID_VALUE, "ATTN_SHF_ACC_SHARED and ATTN_SHF_ACC_PER_DIE are exclusive");
  if (!std::isfinite(scale)) return fail(ATTN_ERR_INVALID_VALUE, "non-finite scale");
  const size_t qb = (size_t)B * Hq * N * d * 2, kb = (size_t)B * Hkv * N * d * 2;
  if (overlaps(o, qb, q, qb) || overlaps(o, qb, k, kb) || overlaps(o, qb, v, kb))
    return fail(ATTN_ERR_INVALID_VALUE, "o overlaps an input");
  if (d > 128 || d % 8 != 0) return fail(ATTN_ERR_UNSUPPORTED, "head dim must be a multiple of 8 and <= 128");
  if (scale < 0.f) return fail(ATTN_ERR_UNSUPPORTED, "negative scale");
  if ((long long)B * Hq * N >= (1ll << 31) || (long long)B * Hkv * N >= (1ll << 31))
    return fail(ATTN_ERR_UNSUPPORTED, "B*H*N exceeds 2^31 rows");
  for (const void* p : {q, k, v, (const void*)o})
    if (reinterpret_cast<uintptr_t>(p) % 16 != 0) return fail(ATTN_ERR_UNSUPPORTED, "pointer not 16-byte aligned");
  return ATTN_OK;
}

// 3-D view [heads][N][d] of a [B][H][N][d] tensor: a box never crosses into
// the next head, and rows >= N are out of bounds (zero-filled by TMA).
// fp32 [heads][N][d] view with boxes of box_rows x 32 floats (one 128-B
// swizzle row): the dQ accumulator of the fused backward (TMA reduce-add).
int make_tmap_f32(CUtensorMap* m, void* base, long long heads, int N, int d, int box_rows) {
  cuuint64_t dims[3] = {(cuuint64_t)d, (cuuint64_t)N, (cuuint64_t)heads};
  cuuint64_t strides[2] = {(cuuint64_t)d * 4, (cuuint64_t)N * d * 4};
  cuuint32_t box[3] = {32, (cuuint32_t)box_rows, 1};
  cuuint32_t estr[3] = {1, 1, 1};
  CUresult r = g_encode(m, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 3, base, dims, strides, box, estr,
                        CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                        CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) return fail(ATTN_ERR_CUDA, "cuTensorMapEncodeTiled (fp32) failed (" + std::to_string((int)r) + ")");
  return ATTN_OK;
}

int make_tmap(CUtensorMap* m, const void* base, long long heads, int N, int d, int box_rows, int box_cols = 64) {
  cuuint64_t dims[3] = {(cuuint64_t)d, (cuuint64_t)N, (cuuint64_t)heads};
  cuuint64_t strides[2] = {(cuuint64_t)d * 2, (cuuint64_t)N * d * 2};
  cuuint32_t box[3] = {(cuuint32_t)box_cols, (cuuint32_t)box_rows, 1};
  cuuint32_t estr[3] = {1, 1, 1};
  CUresult r = g_encode(m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 3, const_cast<void*>(base), dims, strides, box, estr,
                        CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                        CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) return fail(ATTN_ERR_CUDA, "cuTensorMapEncodeTiled failed (" + std::to_string((int)r) + ")");
  return ATTN_OK;
}

template <int D, bool kCausal, bool kOnesL = false>
int launch_t(DevState& st, int attr_idx, const CUtensorMap& tq, const CUtensorMap& tk, const CUtensorMap& tv,
             const KernelParams& kp, int grid, cudaStream_t s, bool cluster, int cluster_units) {
  const int smem = Cfg<D>::kSmemBytes;
  const int ai = attr_idx + (kOnesL ? 8 : 0), ci = attr_idx + (kOnesL ? 4 : 0);
  if (!cluster) {
    auto* fn = attn_fwd_sm100_kernel<D, kCausal, 1, kOnesL>;
    if (!st.attr_done[ai]) {
      ATTN_CUDA(cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
      st.attr_done[ai] = true;
    }
    fn<<<grid, kThreads, smem, s>>>(tq, tk, tv, kp);
  } else {
    auto* fn = attn_fwd_sm100_kernel<D, kCausal, 2, kOnesL>;
    cudaLaunchConfig_t cfg = {};
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = 2;
    attr[0].val.clusterDim.y = 1;
    attr[0].val.clusterDim.z = 1;
    cfg.blockDim = dim3(kThreads);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = s;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    if (!st.attr_done[4 + ai]) {
      ATTN_CUDA(cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
      // persistent grid: as many pairs as can be co-resident (pairs need two
      // free SMs of one GPC, so this can be below num_sms / 2)
      cfg.gridDim = dim3(st.num_sms);
      int nc = 0;
      ATTN_CUDA(cudaOccupancyMaxActiveClusters(&nc, fn, &cfg));
      st.max_clusters[ci] = nc > 0 ? nc : st.num_sms / 2;
      st.attr_done[4 + ai] = true;
    }
    grid = 2 * std::min(st.max_clusters[ci], cluster_units);
    cfg.gridDim = dim3(grid);
    ATTN_CUDA(cudaLaunchKernelEx(&cfg, fn, tq, tk, tv, kp));
  }
  ATTN_CUDA(cudaGetLastError());
  g_info.grid = grid;
  g_info.block = kThreads;
  g_info.smem_bytes = smem;
  return ATTN_OK;
}

// d < 64 forward: the row sum rides in the PV MMA (a ones column of V);
// ATTN_ONES_L=0 in the environment keeps it on the softmax warps (comparison).
bool use_ones_column() {
  static const bool on = [] {
    const char* e = getenv("ATTN_ONES_L");
    return !(e && e[0] == '0');
  }();
  return on;
}

// d in (64, 128]: one query tile per SM, the unit's two tiles on a CTA pair
// (attn_fwd_pair.cuh) when ATTN_FWD_PAIR=1 in the environment (an
// experiment, slower than the default: DESIGN.md section 6); otherwise the
// two-tiles-per-CTA kernel.
bool use_pair_kernel() {
  static const bool on = [] {
    const char* e = getenv("ATTN_FWD_PAIR");
    return e && e[0] == '1';
  }();
  return on;
}

template <bool kCausal>
int launch_pair(DevState& st, const CUtensorMap& tq, const CUtensorMap& tk, const CUtensorMap& tv,
                const KernelParams& kp, cudaStream_t s, int units) {
  const int smem = pairk::kSmemBytes;
  auto* fn = pairk::attn_fwd_pair_kernel<kCausal>;
  cudaLaunchConfig_t cfg = {};
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = 2;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  cfg.blockDim = dim3(kThreads);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = s;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  const int idx = kCausal ? 1 : 0;
  if (!st.pattr_done[idx]) {
    ATTN_CUDA(cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
    cfg.gridDim = dim3(st.num_sms);
    int nc = 0;
    ATTN_CUDA(cudaOccupancyMaxActiveClusters(&nc, fn, &cfg));
    st.pmax_clusters[idx] = nc > 0 ? nc : st.num_sms / 2;
    st.pattr_done[idx] = true;
  }
  const int grid = 2 * std::min(st.pmax_clusters[idx], units);
  cfg.gridDim = dim3(grid);
  ATTN_CUDA(cudaLaunchKernelEx(&cfg, fn, tq, tk, tv, kp));
  ATTN_CUDA(cudaGetLastError());
  g_info.grid = grid;
  g_info.block = kThreads;
  g_info.smem_bytes = smem;
  return ATTN_OK;
}

// Where the epilogue stores O (attn_fwd_replicated): n destinations of
// [B][Hq_out][N][d], the shard's heads at h_off.
struct OutSpec {
  void* const* dst;
  int n, Hq_out, h_off;
};

// A destination must be device memory of this device or of a peer this
// device can access (NVLink P2P, e.g. an attn_ipc_open mapping).
int check_dst_ptr(const void* p, int dev, int i) {
  cudaPointerAttributes a;
  if (cudaPointerGetAttributes(&a, p) != cudaSuccess) {
    cudaGetLastError();
    return fail(ATTN_ERR_INVALID_VALUE, "o_dst[" + std::to_string(i) + "] is not a CUDA pointer");
  }
  if (a.type != cudaMemoryTypeDevice && a.type != cudaMemoryTypeManaged)
    return fail(ATTN_ERR_INVALID_VALUE, "o_dst[" + std::to_string(i) + "] is not device memory");
  if (a.type == cudaMemoryTypeDevice && a.device != dev) {
    int can = 0;
    if (cudaDeviceCanAccessPeer(&can, dev, a.device) != cudaSuccess || !can) {
      cudaGetLastError();
      return fail(ATTN_ERR_INVALID_VALUE, "o_dst[" + std::to_string(i) + "] is on a device without peer access");
    }
  }
  return ATTN_OK;
}

int validate_out(const OutSpec& out, const void* q, const void* k, const void* v, int B, int Hq, int Hkv, int N,
                 int d, int dev) {
  if (!out.dst || out.n < 1 || out.n > kMaxDst)
    return fail(ATTN_ERR_INVALID_VALUE, "n_dst must be in [1, ATTN_MAX_DST]");
  if (out.Hq_out < Hq || out.h_off < 0 || out.h_off > out.Hq_out - Hq)
    return fail(ATTN_ERR_INVALID_VALUE, "need 0 <= head_offset and head_offset + Hq <= Hq_out");
  if ((long long)B * out.Hq_out * N >= (1ll << 31)) return fail(ATTN_ERR_UNSUPPORTED, "B*Hq_out*N exceeds 2^31 rows");
  const size_t ob = (size_t)B * out.Hq_out * N * d * 2;
  const size_t qb = (size_t)B * Hq * N * d * 2, kb = (size_t)B * Hkv * N * d * 2;
  for (int i = 0; i < out.n; ++i) {
    const void* o = out.dst[i];
    if (!o) return fail(ATTN_ERR_INVALID_VALUE, "null o_dst[" + std::to_string(i) + "]");
    if (reinterpret_cast<uintptr_t>(o) % 16 != 0) return fail(ATTN_ERR_UNSUPPORTED, "o_dst pointer not 16-byte aligned");
    if (overlaps(o, ob, q, qb) || overlaps(o, ob, k, kb) || overlaps(o, ob, v, kb))
      return fail(ATTN_ERR_INVALID_VALUE, "o_dst[" + std::to_string(i) + "] overlaps an input");
    for (int j = 0; j < i; ++j)
      if (overlaps(o, ob, out.dst[j], ob)) return fail(ATTN_ERR_INVALID_VALUE, "o_dst buffers overlap");
    int rc = check_dst_ptr(o, dev, i);
    if (rc != ATTN_OK) return rc;
  }
  return ATTN_OK;
}

int fwd_impl(const void* q, const void* k, const void* v, void* o, int B, int Hq, int Hkv, int N, int d, int causal,
             float scale, int mapping, cudaStream_t stream, float* lse = nullptr, const OutSpec* out = nullptr) {
  int rc = validate(q, k, v, o, B, Hq, Hkv, N, d, scale, mapping);
  if (rc != ATTN_OK) return rc;
  int dev = 0;
  rc = current_device(dev);
  if (rc != ATTN_OK) return rc;
  if (out && (rc = validate_out(*out, q, k, v, B, Hq, Hkv, N, d, dev)) != ATTN_OK) return rc;
  for (auto pr : {std::make_pair(q, "q"), std::make_pair(k, "k"), std::make_pair(v, "v"),
                  std::make_pair((const void*)o, "o")}) {
    if (out && pr.first == o) continue;  // replicated output: checked by validate_out (may be a peer buffer)
    rc = check_dev_ptr(pr.first, dev, pr.second);
    if (rc != ATTN_OK) return rc;
  }
  if (lse && (rc = check_dev_ptr(lse, dev, "lse")) != ATTN_OK) return rc;
  rc = get_encode();
  if (rc != ATTN_OK) return rc;
  DevState& st = g_dev[dev];
  std::lock_guard<std::mutex> lk(st.mu);
  rc = ensure_init(dev, st);
  if (rc != ATTN_OK) return rc;

  const int nblk = (N + kBlockM - 1) / kBlockM;  // last block may be ragged
  const int U = (nblk + 1) / 2;
  // head dims > 64 run the CTA-pair kernel (attn_fwd_pair.cuh) over the plain
  // per-unit queues whether or not ATTN_CLUSTER_MULTICAST is given (it is a
  // CTA-pair kernel); head dims <= 64 honour the flag with the kCl = 2 path
  const bool pair = d > 64 && use_pair_kernel();
  const bool cluster = (mapping & ATTN_CLUSTER_MULTICAST) != 0 && !pair;
  mapping &= ~ATTN_CLUSTER_MULTICAST;
  // cluster units: with an even GQA group the pair takes the same unit of two
  // query heads of one KV group (identical K/V blocks); otherwise two adjacent
  // units of one head
  const bool pair_heads = cluster && (Hq / Hkv) % 2 == 0;
  const int Usched = (cluster && !pair_heads) ? (U + 1) / 2 : U;
  const int Hsched = pair_heads ? Hq / 2 : Hq;
  KernelParams kp{};
  kp.B = B; kp.Hq = Hq; kp.Hkv = Hkv; kp.N = N; kp.G = Hq / Hkv; kp.U = U; kp.nblk = nblk;
  kp.Usched = Usched;
  kp.Hsched = Hsched;
  kp.pair_heads = pair_heads ? 1 : 0;
  kp.d_real = d;
  const int dpad = d <= 64 ? 64 : 128;  // kernel head dim; TMA zero-fills columns d..dpad-1
  kp.scale_log2 = scale * 1.4426950408889634f;
  kp.o = reinterpret_cast<__nv_bfloat16*>(o);
  if (out) {
    for (int i = 0; i < out->n; ++i) kp.o_dst[i] = reinterpret_cast<__nv_bfloat16*>(out->dst[i]);
    kp.n_dst = out->n;
    kp.Hq_out = out->Hq_out;
    kp.h_off = out->h_off;
  } else {
    kp.o_dst[0] = kp.o;
    kp.n_dst = 1;
    kp.Hq_out = Hq;
    kp.h_off = 0;
  }
  kp.lse = lse;
  // R23: swizzled head-first shares each ACC among the dies when the dies'
  // ACC footprints would overflow the shared L2 (unless forced either way)
  if ((mapping & kMapMask) == ATTN_MAP_SWIZZLED_HEAD_FIRST && !(mapping & (kShfAccShared | kShfAccPerDie)) &&
      shf_acc_shared(st.active.n_domains, N, d, st.measured.l2_bytes))
    mapping |= kShfAccShared;
  if (!build_sched(mapping, B, Hsched, Hkv, Usched, st.active.n_domains, st.active.sms_per_domain, kp.sched))
    return fail(ATTN_ERR_INVALID_VALUE, "cannot build the schedule");
  kp.counters = st.d_counters + (size_t)counter_slot(st, stream) * kCounterInts;
  kp.domain_of_smid = st.d_domain;
  kp.n_smid = ATTN_MAX_SMID;
  kp.trace = st.trace;
  kp.trace_cap = st.trace_cap;

  CUtensorMap tq, tk, tv;
  if ((rc = make_tmap(&tq, q, (long long)B * Hq, N, d, kBlockM)) != ATTN_OK) return rc;
  // clusters: each CTA loads half the rows of every K/V block; CTA-pair MMA
  // (pair kernel): half the keys of K, half the head-dim columns of V
  const int k_box = (cluster || pair) ? kBlockN / 2 : kBlockN;
  const int v_box = cluster ? kBlockN / 2 : kBlockN;
  // d < 64: K and V land d columns wide and the tensor core sums P into the
  // spare column d of O (the row sum l; attn_fwd_sm100.cuh kOnesL).  That l
  // sums the bf16-rounded P (as the numerator does), within 2^-9 relative of
  // the fp32 sum; the backward's LSE input keeps the fp32 sum (attn_fwd_lse).
  const bool ones = dpad == 64 && d < 64 && lse == nullptr && use_ones_column();
  const int kv_cols = ones ? d : 64;
  kp.kv_tx_bytes = kBlockN * kv_cols * 2 * (dpad / 64);
  if ((rc = make_tmap(&tk, k, (long long)B * Hkv, N, d, k_box, kv_cols)) != ATTN_OK) return rc;
  if ((rc = make_tmap(&tv, v, (long long)B * Hkv, N, d, v_box, kv_cols)) != ATTN_OK) return rc;

  const int total = B * Hq * U;
  const int cunits = B * Hsched * Usched;
  const int grid = std::min(st.num_sms, total);
  if (pair)
    rc = causal ? launch_pair<true>(st, tq, tk, tv, kp, stream, total)
                : launch_pair<false>(st, tq, tk, tv, kp, stream, total);
  else if (dpad == 128 && causal) rc = launch_t<128, true>(st, 0, tq, tk, tv, kp, grid, stream, cluster, cunits);
  else if (dpad == 128) rc = launch_t<128, false>(st, 1, tq, tk, tv, kp, grid, stream, cluster, cunits);
  else if (causal && ones) rc = launch_t<64, true, true>(st, 2, tq, tk, tv, kp, grid, stream, cluster, cunits);
  else if (ones) rc = launch_t<64, false, true>(st, 3, tq, tk, tv, kp, grid, stream, cluster, cunits);
  else if (causal) rc = launch_t<64, true>(st, 2, tq, tk, tv, kp, grid, stream, cluster, cunits);
  else rc = launch_t<64, false>(st, 3, tq, tk, tv, kp, grid, stream, cluster, cunits);
  if (rc != ATTN_OK) return rc;
  g_info.units = total;
  g_info.n_queues = kp.sched.n_queues;
  g_info.shf_acc_shared = ((mapping & kMapMask) == ATTN_MAP_SWIZZLED_HEAD_FIRST && (mapping & kShfAccShared) &&
                           st.active.n_domains > 1) ? 1 : 0;
  g_info.kernel_launches = 1;
  return ATTN_OK;
}


template <int D, bool kCausal>
int launch_bwd_t(DevState& st, const CUtensorMap& tq, const CUtensorMap& tdo, const CUtensorMap& tk,
                 const CUtensorMap& tv, bwd::BwdParams pq, bwd::BwdParams pkv, int grid_q, int grid_kv,
                 cudaStream_t s) {
  const int idx = (D == 128 ? 0 : 2) + (kCausal ? 1 : 0);
  auto* kq = bwd::attn_bwd_dq_kernel<D, kCausal>;
  auto* kkv = bwd::attn_bwd_dkdv_kernel<D, kCausal>;
  const int smem_kv = bwd::BCfg<D>::kSmemBytesKV;
  if (!st.battr_done[idx]) {
    ATTN_CUDA(cudaFuncSetAttribute(kq, cudaFuncAttributeMaxDynamicSharedMemorySize, bwd::BCfg<D>::kSmemBytesQ));
    ATTN_CUDA(cudaFuncSetAttribute(kkv, cudaFuncAttributeMaxDynamicSharedMemorySize, smem_kv));
    st.battr_done[idx] = true;
  }
  kq<<<grid_q, bwd::kThreadsKV, bwd::BCfg<D>::kSmemBytesQ, s>>>(tq, tdo, tk, tv, pq);
  ATTN_CUDA(cudaGetLastError());
  kkv<<<grid_kv, bwd::kThreadsKV, smem_kv, s>>>(tq, tdo, tk, tv, pkv);
  ATTN_CUDA(cudaGetLastError());
  return ATTN_OK;
}

template <bool kCausal>
int launch_bwd_fused(DevState& st, const CUtensorMap& tq, const CUtensorMap& tdo, const CUtensorMap& tk,
                     const CUtensorMap& tv, const CUtensorMap& tacc, const bwd::BwdParams& pkv, int grid,
                     cudaStream_t s) {
  auto* fn = bwd::attn_bwd_fused_kernel<64, kCausal>;
  constexpr int smem = bwd::FCfg<64>::kSmemBytes;
  if (!st.fattr_done[kCausal ? 1 : 0]) {
    ATTN_CUDA(cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
    st.fattr_done[kCausal ? 1 : 0] = true;
  }
  fn<<<grid, bwd::kThreadsF, smem, s>>>(tq, tdo, tk, tv, tacc, pkv);
  ATTN_CUDA(cudaGetLastError());
  return ATTN_OK;
}

// The library's stream-ordered workspace pool on `dev` (created on first use).
int ws_pool(DevState& st, int dev, cudaMemPool_t* out) {
  if (!st.ws_pool) {
    cudaMemPoolProps props = {};
    props.allocType = cudaMemAllocationTypePinned;
    props.location.type = cudaMemLocationTypeDevice;
    props.location.id = dev;
    ATTN_CUDA(cudaMemPoolCreate(&st.ws_pool, &props));
    cuuint64_t thr = ~0ull;
    ATTN_CUDA(cudaMemPoolSetAttribute(st.ws_pool, cudaMemPoolAttrReleaseThreshold, &thr));
  }
  *out = st.ws_pool;
  return ATTN_OK;
}

int bwd_impl(const void* q, const void* k, const void* v, const void* o, const void* dout, const float* lse, void* dq,
             void* dk, void* dv, int B, int Hq, int Hkv, int N, int d, int causal, float scale, int mapping,
             cudaStream_t stream) {
  int rc = validate(q, k, v, dq, B, Hq, Hkv, N, d, scale, mapping);
  if (rc != ATTN_OK) return rc;
  if (mapping & ATTN_CLUSTER_MULTICAST) return fail(ATTN_ERR_UNSUPPORTED, "ATTN_CLUSTER_MULTICAST is forward-only");
  if (!o || !dout || !lse || !dk || !dv) return fail(ATTN_ERR_INVALID_VALUE, "null pointer");
  const size_t qb = (size_t)B * Hq * N * d * 2, kb = (size_t)B * Hkv * N * d * 2, lb = (size_t)B * Hq * N * 4;
  for (const void* out : {(const void*)dq, (const void*)dk, (const void*)dv}) {
    const size_t ob = (out == dq) ? qb : kb;
    for (auto in : {std::make_pair(q, qb), std::make_pair(k, kb), std::make_pair(v, kb), std::make_pair(o, qb),
                    std::make_pair(dout, qb), std::make_pair((const void*)lse, lb)})
      if (overlaps(out, ob, in.first, in.second)) return fail(ATTN_ERR_INVALID_VALUE, "a gradient overlaps an input");
  }
  if (overlaps(dq, qb, dk, kb) || overlaps(dq, qb, dv, kb) || overlaps(dk, kb, dv, kb))
    return fail(ATTN_ERR_INVALID_VALUE, "gradients overlap each other");
  for (const void* ptr : {o, dout, (const void*)dk, (const void*)dv})
    if (reinterpret_cast<uintptr_t>(ptr) % 16 != 0) return fail(ATTN_ERR_UNSUPPORTED, "pointer not 16-byte aligned");
  int dev = 0;
  if ((rc = current_device(dev)) != ATTN_OK) return rc;
  for (auto pr : {std::make_pair(q, "q"), std::make_pair(k, "k"), std::make_pair(v, "v"), std::make_pair(o, "o"),
                  std::make_pair(dout, "dout"), std::make_pair((const void*)lse, "lse"),
                  std::make_pair((const void*)dq, "dq"), std::make_pair((const void*)dk, "dk"),
                  std::make_pair((const void*)dv, "dv")})
    if ((rc = check_dev_ptr(pr.first, dev, pr.second)) != ATTN_OK) return rc;
  if ((rc = get_encode()) != ATTN_OK) return rc;
  DevState& st = g_dev[dev];
  std::lock_guard<std::mutex> lk(st.mu);
  if ((rc = ensure_init(dev, st)) != ATTN_OK) return rc;
  // rowsum(dO o O) workspace, private to this call: allocated and freed in
  // the order of `stream` (stream-ordered pool), so concurrent backward calls
  // on other streams never share it.
  const size_t rows = (size_t)B * Hq * N;
  const int dpad = d <= 64 ? 64 : 128;
  const bool fused = dpad == 64 && !(mapping & ATTN_BWD_DETERMINISTIC);
  mapping &= ~ATTN_BWD_DETERMINISTIC;
  cudaMemPool_t pool = nullptr;
  if ((rc = ws_pool(st, dev, &pool)) != ATTN_OK) return rc;
  float* dvec = nullptr;
  float* dq_acc = nullptr;  // fused path: fp32 [B*Hq][N][64]
  // two-pass: rowsum(dO o O) per row; fused: -lse2 / -D in blocks of 128 rows (attn_bwd_prep_kernel)
  // two-pass: both (dQ reads D per row, dK/dV the blocks), in one allocation
  const int nblk_ws = (N + bwd::kBM - 1) / bwd::kBM;
  const size_t blk_floats = (size_t)B * Hq * nblk_ws * 2 * bwd::kBM;
  const size_t rows_pad = (rows + 63) & ~(size_t)63;  // the blocks are bulk-copied: 16-B (here 256-B) aligned
  const size_t vec_floats = fused ? blk_floats : blk_floats + rows_pad;
  ATTN_CUDA(cudaMallocFromPoolAsync(reinterpret_cast<void**>(&dvec), vec_floats * sizeof(float), pool, stream));
  float* vecb = fused ? dvec : dvec + rows_pad;  // the blocked (-lse2 | -D) layout
  if (fused) {
    if (cudaError_t e = cudaMallocFromPoolAsync(reinterpret_cast<void**>(&dq_acc), rows * dpad * sizeof(float), pool,
                                                stream);
        e != cudaSuccess) {
      cudaFreeAsync(dvec, stream);
      return cuda_fail(e, "dq accumulator allocation");
    }
  }
  auto free_ws = [&]() {
    cudaFreeAsync(dvec, stream);
    if (dq_acc) cudaFreeAsync(dq_acc, stream);
  };
  const int nblk = (N + bwd::kBM - 1) / bwd::kBM;
  bwd::BwdParams pq{};
  pq.B = B; pq.Hq = Hq; pq.Hkv = Hkv; pq.N = N; pq.G = Hq / Hkv; pq.nblk = nblk; pq.d_real = d;
  pq.scale = scale; pq.scale_log2 = scale * 1.4426950408889634f;
  pq.lse = lse; pq.dvec = dvec; pq.vecb = vecb;
  pq.dq = reinterpret_cast<__nv_bfloat16*>(dq);
  pq.dk = reinterpret_cast<__nv_bfloat16*>(dk);
  pq.dv = reinterpret_cast<__nv_bfloat16*>(dv);
  pq.domain_of_smid = st.d_domain;
  pq.dbg = reinterpret_cast<long long*>(st.trace);  // ATTN_BWD_TIMELINE builds only
  pq.n_smid = ATTN_MAX_SMID;
  bwd::BwdParams pkv = pq;
  // dQ units: (b, query head, query block); dK/dV units: (b, KV group, key block)
  pq.U = nblk;
  pkv.U = nblk;
  if (!build_sched(mapping, B, Hq, Hkv, nblk, st.active.n_domains, st.active.sms_per_domain, pq.sched) ||
      !build_sched(mapping, B, Hkv, Hkv, nblk, st.active.n_domains, st.active.sms_per_domain, pkv.sched)) {
    free_ws();
    return fail(ATTN_ERR_INVALID_VALUE, "cannot build the schedule");
  }
  // the dQ and dK/dV grids run one after the other on `stream`: one slot
  pq.counters = pkv.counters = st.d_counters + (size_t)counter_slot(st, stream) * kCounterInts;
  CUtensorMap tq, tdo, tk, tv, tacc;
  if ((rc = make_tmap(&tq, q, (long long)B * Hq, N, d, bwd::kBM)) != ATTN_OK ||
      (rc = make_tmap(&tdo, dout, (long long)B * Hq, N, d, bwd::kBM)) != ATTN_OK ||
      (rc = make_tmap(&tk, k, (long long)B * Hkv, N, d, bwd::kBM)) != ATTN_OK ||
      (rc = make_tmap(&tv, v, (long long)B * Hkv, N, d, bwd::kBM)) != ATTN_OK ||
      (fused && (rc = make_tmap_f32(&tacc, dq_acc, (long long)B * Hq, N, dpad, bwd::kBM)) != ATTN_OK)) {
    free_ws();
    return rc;
  }
  if (fused) {
    const long long prows = (long long)B * Hq * nblk * bwd::kBM;
    bwd::attn_bwd_prep_kernel<<<(unsigned)((prows + 7) / 8), 256, 0, stream>>>(
        reinterpret_cast<const __nv_bfloat16*>(o), reinterpret_cast<const __nv_bfloat16*>(dout), lse, dvec,
        (long long)B * Hq, N, nblk, d);
  } else {  // D per row (dQ kernel) and the blocked -lse2 / -D (dK/dV kernel) in one pass
    const long long prows = (long long)B * Hq * nblk * bwd::kBM;
    bwd::attn_bwd_prep_kernel<<<(unsigned)((prows + 7) / 8), 256, 0, stream>>>(
        reinterpret_cast<const __nv_bfloat16*>(o), reinterpret_cast<const __nv_bfloat16*>(dout), lse, vecb,
        (long long)B * Hq, N, nblk, d, dvec);
  }
  if (cudaError_t e = cudaGetLastError(); e != cudaSuccess) {
    free_ws();
    return cuda_fail(e, "attn_bwd_prep_kernel launch");
  }
  const int grid_q = std::min(st.num_sms, B * Hq * nblk), grid_kv = std::min(st.num_sms, B * Hkv * nblk);
  if (fused) {
    if (cudaError_t e = cudaMemsetAsync(dq_acc, 0, rows * dpad * sizeof(float), stream); e != cudaSuccess) {
      free_ws();
      return cuda_fail(e, "dq accumulator zero fill");
    }
    rc = causal ? launch_bwd_fused<true>(st, tq, tdo, tk, tv, tacc, pkv, grid_kv, stream)
                : launch_bwd_fused<false>(st, tq, tdo, tk, tv, tacc, pkv, grid_kv, stream);
    if (rc == ATTN_OK) {
      const long long work = (long long)rows * (d / 8);
      bwd::attn_bwd_dq_convert_kernel<<<(unsigned)((work + 255) / 256), 256, 0, stream>>>(
          dq_acc, reinterpret_cast<__nv_bfloat16*>(dq), (long long)rows, d, dpad, scale);
      if (cudaError_t e = cudaGetLastError(); e != cudaSuccess) rc = cuda_fail(e, "attn_bwd_dq_convert_kernel launch");
    }
  } else if (dpad == 128 && causal) {
    rc = launch_bwd_t<128, true>(st, tq, tdo, tk, tv, pq, pkv, grid_q, grid_kv, stream);
  } else if (dpad == 128) {
    rc = launch_bwd_t<128, false>(st, tq, tdo, tk, tv, pq, pkv, grid_q, grid_kv, stream);
  } else if (causal) {
    rc = launch_bwd_t<64, true>(st, tq, tdo, tk, tv, pq, pkv, grid_q, grid_kv, stream);
  } else {
    rc = launch_bwd_t<64, false>(st, tq, tdo, tk, tv, pq, pkv, grid_q, grid_kv, stream);
  }
  free_ws();  // after the kernels in stream order
  if (rc != ATTN_OK) return rc;
  g_info.kernel_launches = 3;  // D, then fused + dq convert (after a memset) or dQ + dK/dV
  g_info.units = fused ? B * Hkv * nblk : B * Hq * nblk + B * Hkv * nblk;
  return ATTN_OK;
}

}  // namespace

extern "C" {

int attn_fwd(const void* q, const void* k, const void* v, void* o, int B, int Hq, int Hkv, int N, int d, int causal,
             float scale, int mapping) {
  return fwd_impl(q, k, v, o, B, Hq, Hkv, N, d, causal, scale, mapping, g_stream);
}

int attn_fwd_stream(const void* q, const void* k, const void* v, void* o, int B, int Hq, int Hkv, int N, int d,
                    int causal, float scale, int mapping, void* cuda_stream) {
  return fwd_impl(q, k, v, o, B, Hq, Hkv, N, d, causal, scale, mapping, reinterpret_cast<cudaStream_t>(cuda_stream));
}

int attn_fwd_lse(const void* q, const void* k, const void* v, void* o, float* lse, int B, int Hq, int Hkv, int N,
                 int d, int causal, float scale, int mapping, void* cuda_stream) {
  if (!lse) return fail(ATTN_ERR_INVALID_VALUE, "null lse");
  if (B > 0 && Hq > 0 && N > 0 &&
      (overlaps(lse, (size_t)B * Hq * N * 4, o, (size_t)B * Hq * N * (d > 0 ? d : 0) * 2) ||
       reinterpret_cast<uintptr_t>(lse) % 4 != 0))
    return fail(ATTN_ERR_INVALID_VALUE, "lse overlaps o or is misaligned");
  return fwd_impl(q, k, v, o, B, Hq, Hkv, N, d, causal, scale, mapping, reinterpret_cast<cudaStream_t>(cuda_stream),
                  lse);
}

int attn_fwd_replicated(const void* q, const void* k, const void* v, void* const* o_dst, int n_dst, int Hq_out,
                        int head_offset, int B, int Hq, int Hkv, int N, int d, int causal, float scale, int mapping,
                        void* cuda_stream) {
  if (!o_dst || n_dst < 1 || n_dst > kMaxDst) return fail(ATTN_ERR_INVALID_VALUE, "n_dst must be in [1, ATTN_MAX_DST]");
  const OutSpec out{o_dst, n_dst, Hq_out, head_offset};
  return fwd_impl(q, k, v, o_dst[0], B, Hq, Hkv, N, d, causal, scale, mapping,
                  reinterpret_cast<cudaStream_t>(cuda_stream), nullptr, &out);
}

int attn_ipc_get_handle(const void* dev_ptr, attn_ipc_handle_t* out) {
  if (!dev_ptr || !out) return fail(ATTN_ERR_INVALID_VALUE, "null pointer");
  void* fn = nullptr;
  cudaDriverEntryPointQueryResult qr;
  if (cudaGetDriverEntryPoint("cuMemGetAddressRange", &fn, cudaEnableDefault, &qr) != cudaSuccess || !fn)
    return fail(ATTN_ERR_CUDA, "cuMemGetAddressRange unavailable");
  CUdeviceptr base = 0;
  size_t size = 0;
  if (reinterpret_cast<PFN_cuMemGetAddressRange_v3020>(fn)(&base, &size, (CUdeviceptr)dev_ptr) != CUDA_SUCCESS)
    return fail(ATTN_ERR_INVALID_VALUE, "dev_ptr is not inside a device allocation");
  cudaIpcMemHandle_t h;
  ATTN_CUDA(cudaIpcGetMemHandle(&h, reinterpret_cast<void*>(base)));
  static_assert(sizeof(h) == sizeof(out->handle), "cudaIpcMemHandle_t size");
  std::memcpy(out->handle, &h, sizeof(h));
  out->offset = (long long)((CUdeviceptr)dev_ptr - base);
  return ATTN_OK;
}

namespace {
std::mutex g_ipc_mu;
std::vector<std::pair<void*, void*>> g_ipc_open;  // (returned pointer, mapped base)
}  // namespace

int attn_ipc_open(const attn_ipc_handle_t* h, void** dev_ptr_out) {
  if (!h || !dev_ptr_out || h->offset < 0) return fail(ATTN_ERR_INVALID_VALUE, "bad handle or null output");
  cudaIpcMemHandle_t ch;
  std::memcpy(&ch, h->handle, sizeof(ch));
  void* base = nullptr;
  ATTN_CUDA(cudaIpcOpenMemHandle(&base, ch, cudaIpcMemLazyEnablePeerAccess));
  void* p = static_cast<char*>(base) + h->offset;
  std::lock_guard<std::mutex> lk(g_ipc_mu);
  g_ipc_open.emplace_back(p, base);
  *dev_ptr_out = p;
  return ATTN_OK;
}

int attn_ipc_close(void* dev_ptr) {
  void* base = nullptr;
  {
    std::lock_guard<std::mutex> lk(g_ipc_mu);
    for (size_t i = 0; i < g_ipc_open.size(); ++i)
      if (g_ipc_open[i].first == dev_ptr) {
        base = g_ipc_open[i].second;
        g_ipc_open.erase(g_ipc_open.begin() + i);
        break;
      }
  }
  if (!base) return fail(ATTN_ERR_INVALID_VALUE, "pointer was not returned by attn_ipc_open");
  ATTN_CUDA(cudaIpcCloseMemHandle(base));
  return ATTN_OK;
}

int attn_bwd(const void* q, const void* k, const void* v, const void* o, const void* dout, const float* lse, void* dq,
             void* dk, void* dv, int B, int Hq, int Hkv, int N, int d, int causal, float scale, int mapping,
             void* cuda_stream) {
  return bwd_impl(q, k, v, o, dout, lse, dq, dk, dv, B, Hq, Hkv, N, d, causal, scale, mapping,
                  reinterpret_cast<cudaStream_t>(cuda_stream));
}

int attn_fwd_host(const void* q_host, const void* k_host, const void* v_host, void* o_host, int B, int Hq, int Hkv,
                  int N, int d, int causal, float scale, int mapping, void* cuda_stream) {
  if (!q_host || !k_host || !v_host || !o_host) return fail(ATTN_ERR_INVALID_VALUE, "null pointer");
  if (B <= 0 || Hq <= 0 || Hkv <= 0 || N <= 0 || d <= 0) return fail(ATTN_ERR_INVALID_VALUE, "size <= 0");
  if (Hq % Hkv != 0) return fail(ATTN_ERR_INVALID_VALUE, "Hq % Hkv != 0 (non-uniform GQA groups)");
  int dev = 0;
  int rc = current_device(dev);
  if (rc != ATTN_OK) return rc;
  DevState& st = g_dev[dev];
  cudaStream_t s = reinterpret_cast<cudaStream_t>(cuda_stream);
  const int G = Hq / Hkv;
  const size_t row_bytes = (size_t)N * d * 2;  // one head of one batch item
  const size_t nq = (size_t)B * Hq * row_bytes, nk = (size_t)B * Hkv * row_bytes;
  const size_t need[4] = {nq, nk, nk, nq};
  {
    std::lock_guard<std::mutex> lk(st.mu);
    for (int i = 0; i < 4; ++i) {
      if (st.hbuf_bytes[i] < need[i]) {
        if (st.hbuf[i]) cudaFree(st.hbuf[i]);
        st.hbuf[i] = nullptr;
        st.hbuf_bytes[i] = 0;
        ATTN_CUDA(cudaMalloc(&st.hbuf[i], need[i]));
        st.hbuf_bytes[i] = need[i];
      }
    }
    if (!st.e2e_ready) {
      for (int i = 0; i < 4; ++i) ATTN_CUDA(cudaStreamCreateWithFlags(&st.e2e_stream[i], cudaStreamNonBlocking));
      for (int i = 0; i < kE2EChunks + 1; ++i)
        for (int j = 0; j < 2; ++j) ATTN_CUDA(cudaEventCreateWithFlags(&st.e2e_ev[j][i], cudaEventDisableTiming));
      st.e2e_ready = true;
    }
  }
  // Chunks of whole KV groups inside one batch item (contiguous sub-tensors;
  // heads are independent, so the result is bit-identical to one call).
  // Three-stage pipeline: H2D chunk i+1 || kernel chunk i || D2H chunk i-1.
  const size_t total = 2 * nq + 2 * nk;
  int target = (int)std::min<size_t>(kE2EChunks, std::max<size_t>(1, total / ((size_t)ATTN_E2E_CHUNK_MB << 20)));
  const int tg = B * Hkv;
  target = std::min(target, tg);
  int gpc = (tg + target - 1) / target;  // KV groups per chunk
  gpc = std::min(gpc, Hkv);
  // consecutive chunks compute on two streams, so chunk i+1's persistent CTAs
  // take the SMs chunk i's tail leaves idle (heads are independent)
  cudaStream_t cin = st.e2e_stream[0], cout = st.e2e_stream[2];
  const cudaStream_t comps[2] = {st.e2e_stream[1], st.e2e_stream[3]};
  cudaEvent_t* ev_in = st.e2e_ev[0];
  cudaEvent_t* ev_k = st.e2e_ev[1];
  ATTN_CUDA(cudaEventRecord(ev_in[kE2EChunks], s));  // order after the caller's prior work
  for (cudaStream_t x : {cin, comps[0], comps[1], cout}) ATTN_CUDA(cudaStreamWaitEvent(x, ev_in[kE2EChunks], 0));
  char* dq = static_cast<char*>(st.hbuf[0]);
  char* dk = static_cast<char*>(st.hbuf[1]);
  char* dv = static_cast<char*>(st.hbuf[2]);
  char* dout = static_cast<char*>(st.hbuf[3]);
  int c = 0;
  for (int b = 0; b < B; ++b) {
    for (int g0 = 0; g0 < Hkv; g0 += gpc, ++c) {
      const int gn = std::min(gpc, Hkv - g0);
      const size_t qoff = ((size_t)b * Hq + (size_t)g0 * G) * row_bytes, qlen = (size_t)gn * G * row_bytes;
      const size_t koff = ((size_t)b * Hkv + g0) * row_bytes, klen = (size_t)gn * row_bytes;
      const int e = c % kE2EChunks;
      const cudaStream_t comp = comps[c & 1];
      if (c >= kE2EChunks) ATTN_CUDA(cudaStreamWaitEvent(cin, ev_k[e], 0));  // slot's previous chunk consumed
      ATTN_CUDA(cudaMemcpyAsync(dq + qoff, static_cast<const char*>(q_host) + qoff, qlen, cudaMemcpyHostToDevice, cin));
      ATTN_CUDA(cudaMemcpyAsync(dk + koff, static_cast<const char*>(k_host) + koff, klen, cudaMemcpyHostToDevice, cin));
      ATTN_CUDA(cudaMemcpyAsync(dv + koff, static_cast<const char*>(v_host) + koff, klen, cudaMemcpyHostToDevice, cin));
      ATTN_CUDA(cudaEventRecord(ev_in[e], cin));
      ATTN_CUDA(cudaStreamWaitEvent(comp, ev_in[e], 0));
      rc = fwd_impl(dq + qoff, dk + koff, dv + koff, dout + qoff, 1, gn * G, gn, N, d, causal, scale, mapping, comp);
      if (rc != ATTN_OK) return rc;
      ATTN_CUDA(cudaEventRecord(ev_k[e], comp));
      ATTN_CUDA(cudaStreamWaitEvent(cout, ev_k[e], 0));
      ATTN_CUDA(cudaMemcpyAsync(static_cast<char*>(o_host) + qoff, dout + qoff, qlen, cudaMemcpyDeviceToHost, cout));
    }
  }
  ATTN_CUDA(cudaEventRecord(ev_k[kE2EChunks], cout));
  ATTN_CUDA(cudaStreamWaitEvent(s, ev_k[kE2EChunks], 0));
  ATTN_CUDA(cudaStreamSynchronize(s));
  g_info.kernel_launches = c;
  return ATTN_OK;
}

int attn_bwd_host(const void* q_host, const void* k_host, const void* v_host, const void* o_host,
                  const void* dout_host, const float* lse_host, void* dq_host, void* dk_host, void* dv_host, int B,
                  int Hq, int Hkv, int N, int d, int causal, float scale, int mapping, void* cuda_stream) {
  if (!q_host || !k_host || !v_host || !o_host || !dout_host || !lse_host || !dq_host || !dk_host || !dv_host)
    return fail(ATTN_ERR_INVALID_VALUE, "null pointer");
  if (B <= 0 || Hq <= 0 || Hkv <= 0 || N <= 0 || d <= 0) return fail(ATTN_ERR_INVALID_VALUE, "size <= 0");
  if (Hq % Hkv != 0) return fail(ATTN_ERR_INVALID_VALUE, "Hq % Hkv != 0 (non-uniform GQA groups)");
  if (mapping & ATTN_CLUSTER_MULTICAST) return fail(ATTN_ERR_UNSUPPORTED, "ATTN_CLUSTER_MULTICAST is forward-only");
  int dev = 0;
  int rc = current_device(dev);
  if (rc != ATTN_OK) return rc;
  DevState& st = g_dev[dev];
  cudaStream_t s = reinterpret_cast<cudaStream_t>(cuda_stream);
  const int G = Hq / Hkv;
  const size_t row_bytes = (size_t)N * d * 2, lrow_bytes = (size_t)N * 4;
  const size_t nq = (size_t)B * Hq * row_bytes, nk = (size_t)B * Hkv * row_bytes, nl = (size_t)B * Hq * lrow_bytes;
  const size_t need[9] = {nq, nk, nk, nq, nq, nl, nq, nk, nk};
  {
    std::lock_guard<std::mutex> lk(st.mu);
    for (int i = 0; i < 9; ++i) {
      if (st.bbuf_bytes[i] < need[i]) {
        if (st.bbuf[i]) cudaFree(st.bbuf[i]);
        st.bbuf[i] = nullptr;
        st.bbuf_bytes[i] = 0;
        ATTN_CUDA(cudaMalloc(&st.bbuf[i], need[i]));
        st.bbuf_bytes[i] = need[i];
      }
    }
    if (!st.e2e_ready) {
      for (int i = 0; i < 4; ++i) ATTN_CUDA(cudaStreamCreateWithFlags(&st.e2e_stream[i], cudaStreamNonBlocking));
      for (int i = 0; i < kE2EChunks + 1; ++i)
        for (int j = 0; j < 2; ++j) ATTN_CUDA(cudaEventCreateWithFlags(&st.e2e_ev[j][i], cudaEventDisableTiming));
      st.e2e_ready = true;
    }
  }
  // Same pipeline as attn_fwd_host: chunks of whole KV groups of one batch
  // item (the gradients of different KV groups are independent), H2D of chunk
  // i+1 || the three backward kernels of chunk i || D2H of chunk i-1.
  const size_t total = 4 * nq + 4 * nk + nl;
  int target = (int)std::min<size_t>(kE2EChunks, std::max<size_t>(1, total / ((size_t)ATTN_E2E_CHUNK_MB << 20)));
  const int tg = B * Hkv;
  target = std::min(target, tg);
  int gpc = (tg + target - 1) / target;  // KV groups per chunk
  gpc = std::min(gpc, Hkv);
  // consecutive chunks compute on two streams, so chunk i+1's persistent CTAs
  // take the SMs chunk i's tail leaves idle (heads are independent)
  cudaStream_t cin = st.e2e_stream[0], cout = st.e2e_stream[2];
  const cudaStream_t comps[2] = {st.e2e_stream[1], st.e2e_stream[3]};
  cudaEvent_t* ev_in = st.e2e_ev[0];
  cudaEvent_t* ev_k = st.e2e_ev[1];
  ATTN_CUDA(cudaEventRecord(ev_in[kE2EChunks], s));  // order after the caller's prior work
  for (cudaStream_t x : {cin, comps[0], comps[1], cout}) ATTN_CUDA(cudaStreamWaitEvent(x, ev_in[kE2EChunks], 0));
  char* b[9];
  for (int i = 0; i < 9; ++i) b[i] = static_cast<char*>(st.bbuf[i]);
  const char* hin[6] = {static_cast<const char*>(q_host), static_cast<const char*>(k_host),
                        static_cast<const char*>(v_host), static_cast<const char*>(o_host),
                        static_cast<const char*>(dout_host), reinterpret_cast<const char*>(lse_host)};
  char* hout[3] = {static_cast<char*>(dq_host), static_cast<char*>(dk_host), static_cast<char*>(dv_host)};
  int c = 0;
  for (int bi = 0; bi < B; ++bi) {
    for (int g0 = 0; g0 < Hkv; g0 += gpc, ++c) {
      const int gn = std::min(gpc, Hkv - g0);
      const size_t qoff = ((size_t)bi * Hq + (size_t)g0 * G) * row_bytes, qlen = (size_t)gn * G * row_bytes;
      const size_t koff = ((size_t)bi * Hkv + g0) * row_bytes, klen = (size_t)gn * row_bytes;
      const size_t loff = ((size_t)bi * Hq + (size_t)g0 * G) * lrow_bytes, llen = (size_t)gn * G * lrow_bytes;
      const size_t off[6] = {qoff, koff, koff, qoff, qoff, loff}, len[6] = {qlen, klen, klen, qlen, qlen, llen};
      const int e = c % kE2EChunks;
      const cudaStream_t comp = comps[c & 1];
      if (c >= kE2EChunks) ATTN_CUDA(cudaStreamWaitEvent(cin, ev_k[e], 0));  // the event slot's previous chunk ran
      for (int i = 0; i < 6; ++i)
        ATTN_CUDA(cudaMemcpyAsync(b[i] + off[i], hin[i] + off[i], len[i], cudaMemcpyHostToDevice, cin));
      ATTN_CUDA(cudaEventRecord(ev_in[e], cin));
      ATTN_CUDA(cudaStreamWaitEvent(comp, ev_in[e], 0));
      rc = bwd_impl(b[0] + qoff, b[1] + koff, b[2] + koff, b[3] + qoff, b[4] + qoff,
                    reinterpret_cast<const float*>(b[5] + loff), b[6] + qoff, b[7] + koff, b[8] + koff, 1, gn * G, gn,
                    N, d, causal, scale, mapping, comp);
      if (rc != ATTN_OK) return rc;
      ATTN_CUDA(cudaEventRecord(ev_k[e], comp));
      ATTN_CUDA(cudaStreamWaitEvent(cout, ev_k[e], 0));
      ATTN_CUDA(cudaMemcpyAsync(hout[0] + qoff, b[6] + qoff, qlen, cudaMemcpyDeviceToHost, cout));
      ATTN_CUDA(cudaMemcpyAsync(hout[1] + koff, b[7] + koff, klen, cudaMemcpyDeviceToHost, cout));
      ATTN_CUDA(cudaMemcpyAsync(hout[2] + koff, b[8] + koff, klen, cudaMemcpyDeviceToHost, cout));
    }
  }
  ATTN_CUDA(cudaEventRecord(ev_k[kE2EChunks], cout));
  ATTN_CUDA(cudaStreamWaitEvent(s, ev_k[kE2EChunks], 0));
  ATTN_CUDA(cudaStreamSynchronize(s));
  g_info.kernel_launches = 3 * c;  // D, dQ and dK/dV kernels per chunk
  return ATTN_OK;
}

int attn_set_stream(void* cuda_stream) {
  g_stream = reinterpret_cast<cudaStream_t>(cuda_stream);
  return ATTN_OK;
}

int attn_init(int device) {
  if (device < 0 || device >= kMaxDevices) return fail(ATTN_ERR_INVALID_VALUE, "bad device index");
  int prev = 0;
  ATTN_CUDA(cudaGetDevice(&prev));
  ATTN_CUDA(cudaSetDevice(device));
  DevState& st = g_dev[device];
  int rc;
  {
    std::lock_guard<std::mutex> lk(st.mu);
    rc = ensure_init(device, st);
  }
  cudaSetDevice(prev);
  return rc;
}

int attn_topology(int device, attn_topology_t* out) {
  if (!out) return fail(ATTN_ERR_INVALID_VALUE, "null out");
  int rc = attn_init(device);
  if (rc != ATTN_OK) return rc;
  DevState& st = g_dev[device];
  std::lock_guard<std::mutex> lk(st.mu);
  *out = st.active;
  return ATTN_OK;
}

int attn_set_topology_override(int device, const signed char* domain_of_smid, int n, int n_domains) {
  int rc = attn_init(device);
  if (rc != ATTN_OK) return rc;
  DevState& st = g_dev[device];
  std::lock_guard<std::mutex> lk(st.mu);
  if (!domain_of_smid) {
    st.active = st.measured;
  } else {
    if (n <= 0 || n > ATTN_MAX_SMID || n_domains < 1 || n_domains > ATTN_MAX_DOMAINS)
      return fail(ATTN_ERR_INVALID_VALUE, "bad override table size");
    attn_topology_t t = st.measured;
    memset(t.domain_of_smid, -1, sizeof t.domain_of_smid);
    for (int i = 0; i < ATTN_MAX_DOMAINS; ++i) t.sms_per_domain[i] = 0;
    for (int s = 0; s < n; ++s) {
      const int d = domain_of_smid[s];
      if (d < -1 || d >= n_domains) return fail(ATTN_ERR_INVALID_VALUE, "domain id out of range");
      t.domain_of_smid[s] = (signed char)d;
      if (d >= 0) ++t.sms_per_domain[d];
    }
    for (int d = 0; d < n_domains; ++d)
      if (t.sms_per_domain[d] == 0) t.sms_per_domain[d] = 1;  // keep the proportional cut defined
    t.n_domains = n_domains;
    t.source = 1;
    st.active = t;
  }
  int prev = 0;
  ATTN_CUDA(cudaGetDevice(&prev));
  ATTN_CUDA(cudaSetDevice(device));
  rc = upload_domain(st);
  cudaSetDevice(prev);
  return rc;
}

int attn_set_schedule_trace(int device, void* dev_buf, long long capacity) {
  if (device < 0 || device >= kMaxDevices) return fail(ATTN_ERR_INVALID_VALUE, "bad device index");
  if (dev_buf && capacity <= 0) return fail(ATTN_ERR_INVALID_VALUE, "capacity <= 0");
  DevState& st = g_dev[device];
  std::lock_guard<std::mutex> lk(st.mu);
  st.trace = reinterpret_cast<attn_trace_rec_t*>(dev_buf);
  st.trace_cap = dev_buf ? capacity : 0;
  return ATTN_OK;
}

int attn_schedule_order(int B, int Hq, int Hkv, int N, int mapping, int n_domains, const int* sms_per_domain,
                        int32_t* out, long long capacity, int* n_queues, int* queue_len) {
  if (!out || !n_queues || !queue_len || !sms_per_domain) return fail(ATTN_ERR_INVALID_VALUE, "null pointer");
  if (B <= 0 || Hq <= 0 || Hkv <= 0 || N <= 0 || Hq % Hkv) return fail(ATTN_ERR_INVALID_VALUE, "bad sizes");
  // ATTN_CLUSTER_MULTICAST: the queues hold cluster units -- (b, head pair,
  // unit) when Hq/Hkv is even, else (b, head, pair of adjacent units)
  const bool cl = (mapping & ATTN_CLUSTER_MULTICAST) != 0, pair_heads = cl && (Hq / Hkv) % 2 == 0;
  const int U = (cl && !pair_heads) ? ((N + 255) / 256 + 1) / 2 : (N + 255) / 256;
  if (pair_heads) Hq /= 2;
  mapping &= ~ATTN_CLUSTER_MULTICAST;
  SchedParams sp;
  if (!build_sched(mapping, B, Hq, Hkv, U, n_domains, sms_per_domain, sp))
    return fail(ATTN_ERR_INVALID_VALUE, "bad mapping or domains");
  long long total = 0;
  for (int qi = 0; qi < sp.n_queues; ++qi) total += sp.q[qi].len;
  if (total > capacity) return fail(ATTN_ERR_INVALID_VALUE, "capacity too small");
  long long w = 0;
  for (int qi = 0; qi < sp.n_queues; ++qi) {
    queue_len[qi] = sp.q[qi].len;
    for (int pos = 0; pos < sp.q[qi].len; ++pos) {
      int b, h, u;
      decode_unit(sp, qi, pos, Hq, U, b, h, u);
      if ((sp.descending >> qi) & 1) u = U - 1 - u;
      out[3 * w] = b;
      out[3 * w + 1] = h;
      out[3 * w + 2] = u;
      ++w;
    }
  }
  *n_queues = sp.n_queues;
  return ATTN_OK;
}

int attn_shf_acc_shared(int n_domains, int N, int d, long long l2_bytes) {
  return shf_acc_shared(n_domains, N, d, l2_bytes) ? 1 : 0;
}

int attn_last_launch_info(attn_launch_info_t* out) {
  if (!out) return fail(ATTN_ERR_INVALID_VALUE, "null out");
  *out = g_info;
  return ATTN_OK;
}

const char* attn_status_string(int status) {
  switch (status) {
    case ATTN_OK: return "ATTN_OK";
    case ATTN_ERR_INVALID_VALUE: return "ATTN_ERR_INVALID_VALUE";
    case ATTN_ERR_UNSUPPORTED: return "ATTN_ERR_UNSUPPORTED";
    case ATTN_ERR_CUDA: return "ATTN_ERR_CUDA";
    case ATTN_ERR_TOPOLOGY: return "ATTN_ERR_TOPOLOGY";
    default: return "ATTN_ERR_UNKNOWN";
  }
}

const char* attn_last_error(void) { return g_err.c_str(); }

const char* attn_version(void) { return "attn-numa-b200 0.1 (sm_100a tcgen05)"; }

void attn_shutdown(void) {
  for (int dv = 0; dv < kMaxDevices; ++dv) {
    DevState& st = g_dev[dv];
    std::lock_guard<std::mutex> lk(st.mu);
    if (!st.init && !st.hbuf[0] && !st.bbuf[0]) continue;
    int prev = 0;
    cudaGetDevice(&prev);
    cudaSetDevice(dv);
    if (st.d_domain) cudaFree(st.d_domain);
    if (st.d_counters) cudaFree(st.d_counters);
    for (bool& a : st.battr_done) a = false;
    for (bool& a : st.fattr_done) a = false;
    if (st.ws_pool) {
      cudaDeviceSynchronize();  // per-call workspace is freed in stream order
      cudaMemPoolDestroy(st.ws_pool);
      st.ws_pool = nullptr;
    }
    for (int i = 0; i < 4; ++i)
      if (st.hbuf[i]) cudaFree(st.hbuf[i]);
    cudaSetDevice(prev);
    st.d_domain = nullptr;
    st.d_counters = nullptr;
    for (int i = 0; i < 4; ++i) { st.hbuf[i] = nullptr; st.hbuf_bytes[i] = 0; }
    for (int i = 0; i < 9; ++i) {
      if (st.bbuf[i]) cudaFree(st.bbuf[i]);
      st.bbuf[i] = nullptr;
      st.bbuf_bytes[i] = 0;
    }
    if (st.e2e_ready) {
      for (int i = 0; i < 4; ++i) cudaStreamDestroy(st.e2e_stream[i]);
      for (int j = 0; j < 2; ++j)
        for (int i = 0; i < kE2EChunks + 1; ++i) cudaEventDestroy(st.e2e_ev[j][i]);
      st.e2e_ready = false;
    }
    st.init = false;
    for (bool& a : st.attr_done) a = false;
    for (int i = 0; i < kCounterSlots; ++i) { st.slot_stream[i] = nullptr; st.slot_used[i] = 0; }
  }
}

}  // extern "C"
