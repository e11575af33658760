// tcgen05.mma issue back-pressure probe (not part of the library).
// One CTA per SM; one thread issues `n` MMAs (M128 N128 K16, SS or TS) back to
// back and records clock64() after each issue.  If the tensor pipe's
// instruction queue is bounded, the issue timestamps settle to the execution
// rate (64 cycles/MMA) after the first `depth` instructions.
#include <cstdio>
#include <cstdint>
#include <vector>
#include "../../paper_2511_02132_b200/csrc/ptx.cuh"
using namespace attn;

constexpr int kN = 48;

template <bool TS, int NN, int BMN>
__global__ void __launch_bounds__(128, 1) issue(long long* out) {
  extern __shared__ __align__(1024) uint8_t smem[];
  __shared__ uint64_t bar;
  __shared__ uint32_t tbase;
  const int warp = threadIdx.x / 32;
  for (int i = threadIdx.x; i < 65536 / 4; i += blockDim.x) reinterpret_cast<uint32_t*>(smem)[i] = 0;
  if (threadIdx.x == 0) { ptx::mbar_init(&bar, 1); ptx::fence_barrier_init(); }
  if (warp == 0) { ptx::tmem_alloc(&tbase, 512); ptx::tmem_relinquish(); }
  asm volatile("fence.proxy.async.shared::cta;");
  ptx::tc_fence_before(); __syncthreads(); ptx::tc_fence_after();
  const uint32_t tmem = tbase;
  if (warp == 0) {
    const uint64_t da = ptx::smem_desc_sw128(ptx::smem_u32(smem), 16, 1024);
    // BMN: B operand MN-major (the PV layout: V rows = keys, 128-B swizzled d columns)
    const uint64_t db = ptx::smem_desc_sw128(ptx::smem_u32(smem + 32768), BMN ? 128 * 128 : 16, 1024);
    constexpr uint32_t idesc = ptx::idesc_bf16_f32(128, NN, 0, BMN);
    long long t[kN + 2];
    if (ptx::elect_one_sync()) {
      t[0] = clock64();
#pragma unroll
      for (int i = 0; i < kN; ++i) {
        if (TS) ptx::mma_ts(tmem + 256, tmem + (i & 7) * 8, db + (BMN ? (uint64_t)(((i & 7) * 16 * 128) >> 4) : 0), idesc, 1);
        else ptx::mma_ss(tmem, da + ((i & 3) * 2), db + ((i & 3) * 2), idesc, 1);
        t[i + 1] = clock64();
      }
      ptx::mma_commit(&bar);
      ptx::mbar_wait(&bar, 0);
      t[kN + 1] = clock64();
      if (blockIdx.x == 0)
        for (int i = 0; i < kN + 2; ++i) out[i] = t[i] - t[0];
    }
    __syncwarp();
  }
  ptx::tc_fence_before(); __syncthreads();
  if (warp == 0) { ptx::tc_fence_after(); ptx::tmem_dealloc(tmem, 512); }
}

template <bool TS, int NN = 128, int BMN = 0>
void run(const char* name) {
  long long* d; cudaMalloc(&d, sizeof(long long) * (kN + 2));
  auto k = issue<TS, NN, BMN>;
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 65536 + 1024);
  for (int r = 0; r < 3; ++r) k<<<148, 128, 65536 + 1024>>>(d);
  cudaError_t e = cudaDeviceSynchronize();
  std::vector<long long> h(kN + 2); cudaMemcpy(h.data(), d, sizeof(long long) * (kN + 2), cudaMemcpyDeviceToHost);
  printf("%s %s\n  issue-done cycle after MMA i:", name, e == cudaSuccess ? "" : cudaGetErrorString(e));
  for (int i = 1; i <= kN; ++i) printf(" %lld", h[i]);
  printf("\n  all complete: %lld\n", h[kN + 1]);
  cudaFree(d);
}

int main() {
  run<false>("SS M128 N128 K16");
  run<true>("TS M128 N128 K16");
  run<true, 128, 1>("TS M128 N128 K16, B MN-major (PV at d = 128)");
  run<true, 64, 1>("TS M128 N64 K16, B MN-major (PV at d = 64)");
  run<false, 64, 0>("SS M128 N64 K16");
  return 0;
}
