// Standalone tcgen05.mma throughput probe (not part of the library).
// One CTA per SM issues `iters` MMAs of one shape back to back into one TMEM
// accumulator; reports cycles per MMA (median over CTAs).
#include <cstdio>
#include <cstdint>
#include <vector>
#include <algorithm>
#include "../../paper_2511_02132_b200/csrc/ptx.cuh"
using namespace attn;

template <int N, bool TS, int COMMIT_EVERY = 0>
__global__ void __launch_bounds__(128, 1) mma_rate(long long* out, int iters) {
  extern __shared__ __align__(1024) uint8_t smem[];
  __shared__ uint64_t bar;
  __shared__ uint64_t bar2[4];
  __shared__ uint32_t tbase;
  const int warp = threadIdx.x / 32;
  for (int i = threadIdx.x; i < 65536 / 4; i += blockDim.x) reinterpret_cast<uint32_t*>(smem)[i] = 0;
  if (threadIdx.x == 0) { ptx::mbar_init(&bar, 1); for (int i = 0; i < 4; ++i) ptx::mbar_init(&bar2[i], 1); ptx::fence_barrier_init(); }
  if (warp == 0) { ptx::tmem_alloc(&tbase, 512); ptx::tmem_relinquish(); }
  asm volatile("fence.proxy.async.shared::cta;");
  ptx::tc_fence_before(); __syncthreads(); ptx::tc_fence_after();
  const uint32_t tmem = tbase;
  if (warp == 0) {
    const uint64_t da = ptx::smem_desc_sw128(ptx::smem_u32(smem), 16, 1024);
    const uint64_t db = ptx::smem_desc_sw128(ptx::smem_u32(smem + 32768), 16, 1024);
    constexpr uint32_t idesc = ptx::idesc_bf16_f32(128, N, 0, 0);
    long long t0 = clock64();
    if (ptx::elect_one_sync()) {
      for (int i = 0; i < iters; ++i) {
        if (TS) ptx::mma_ts(tmem + 256, tmem + (i & 7) * 8, db, idesc, 1);
        else ptx::mma_ss(tmem, da + ((i & 3) * 2), db + ((i & 3) * 2), idesc, 1);
        if (COMMIT_EVERY > 0 && (i % COMMIT_EVERY) == COMMIT_EVERY - 1) ptx::mma_commit(&bar2[(i / COMMIT_EVERY) & 3]);
      }
      ptx::mma_commit(&bar);
    }
    __syncwarp();
    ptx::mbar_wait(&bar, 0);
    long long t1 = clock64();
    if (threadIdx.x == 0) out[blockIdx.x] = t1 - t0;
  }
  ptx::tc_fence_before(); __syncthreads();
  if (warp == 0) { ptx::tc_fence_after(); ptx::tmem_dealloc(tmem, 512); }
}

template <int N, bool TS, int CE = 0>
void run(const char* name, int grid) {
  long long* d; cudaMalloc(&d, sizeof(long long) * grid);
  auto k = mma_rate<N, TS, CE>;
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 65536 + 1024);
  const int iters = 4096;
  k<<<grid, 128, 65536 + 1024>>>(d, iters);
  k<<<grid, 128, 65536 + 1024>>>(d, iters);
  cudaError_t e = cudaDeviceSynchronize();
  std::vector<long long> h(grid); cudaMemcpy(h.data(), d, sizeof(long long) * grid, cudaMemcpyDeviceToHost);
  std::sort(h.begin(), h.end());
  double cyc = (double)h[grid / 2] / iters;
  double flops = 2.0 * 128 * N * 16;
  printf("%-18s grid %3d: %6.1f cycles/MMA  -> %6.0f flop/clk/SM (peak 8192) %s\n", name, grid, cyc, flops / cyc,
         e == cudaSuccess ? "" : cudaGetErrorString(e));
  cudaFree(d);
}

int main() {
  for (int g : {148}) {
    run<64, false>("SS M128 N64", g);
    run<128, false>("SS M128 N128", g);
    run<128, true>("TS M128 N128", g);
    run<128, false, 8>("SS N128 commit/8", g);
    run<128, false, 4>("SS N128 commit/4", g);
    run<128, true, 8>("TS N128 commit/8", g);
  }
  return 0;
}
