// Latency of: issue K MMAs (M128 N128 K16) + tcgen05.commit -> mbarrier wait returns,
// (a) waiter in the issuing warp, (b) round trip through a second warp that
// waits on the commit barrier and arrives on a barrier the first warp waits on.
#include <cstdio>
#include <cstdint>
#include "../../paper_2511_02132_b200/csrc/ptx.cuh"
using namespace attn;

__global__ void __launch_bounds__(128, 1) lat(long long* out, int kmma) {
  extern __shared__ __align__(1024) uint8_t smem[];
  __shared__ uint64_t barA, barB, barC;
  __shared__ uint32_t tbase;
  const int warp = threadIdx.x / 32;
  for (int i = threadIdx.x; i < 65536 / 4; i += blockDim.x) reinterpret_cast<uint32_t*>(smem)[i] = 0;
  if (threadIdx.x == 0) {
    ptx::mbar_init(&barA, 1); ptx::mbar_init(&barB, 1); ptx::mbar_init(&barC, 1);
    ptx::fence_barrier_init();
  }
  if (warp == 0) { ptx::tmem_alloc(&tbase, 512); ptx::tmem_relinquish(); }
  asm volatile("fence.proxy.async.shared::cta;");
  ptx::tc_fence_before(); __syncthreads(); ptx::tc_fence_after();
  const uint32_t tmem = tbase;
  const uint64_t da = ptx::smem_desc_sw128(ptx::smem_u32(smem), 16, 1024);
  const uint64_t db = ptx::smem_desc_sw128(ptx::smem_u32(smem + 32768), 16, 1024);
  constexpr uint32_t idesc = ptx::idesc_bf16_f32(128, 128, 0, 0);
  long long same = 0, cross = 0;
  const int R = 64;
  for (int r = 0; r < R; ++r) {
    if (warp == 0) {
      long long t0 = clock64();
      if (ptx::elect_one_sync()) {
        for (int i = 0; i < kmma; ++i) ptx::mma_ss(tmem, da, db, idesc, 1);
        ptx::mma_commit(&barA);
      }
      __syncwarp();
      ptx::mbar_wait(&barA, r & 1);
      same += clock64() - t0;
    }
    __syncthreads();
    if (warp == 0) {
      long long t0 = clock64();
      if (ptx::elect_one_sync()) {
        for (int i = 0; i < kmma; ++i) ptx::mma_ss(tmem, da, db, idesc, 1);
        ptx::mma_commit(&barB);
      }
      __syncwarp();
      ptx::mbar_wait(&barC, r & 1);
      cross += clock64() - t0;
    } else if (warp == 1) {
      ptx::mbar_wait(&barB, r & 1);
      ptx::tc_fence_after();
      ptx::tc_fence_before();
      __syncwarp();
      if ((threadIdx.x & 31) == 0) ptx::mbar_arrive(&barC);
    }
    __syncthreads();
  }
  if (threadIdx.x == 0) { out[0] = same / R; out[1] = cross / R; }
  ptx::tc_fence_before(); __syncthreads();
  if (warp == 0) { ptx::tc_fence_after(); ptx::tmem_dealloc(tmem, 512); }
}

int main() {
  long long* d; cudaMalloc(&d, 16);
  cudaFuncSetAttribute(lat, cudaFuncAttributeMaxDynamicSharedMemorySize, 65536 + 1024);
  for (int k : {1, 4, 8, 16}) {
    lat<<<1, 128, 65536 + 1024>>>(d, k);
    long long h[2];
    cudaError_t e = cudaMemcpy(h, d, 16, cudaMemcpyDeviceToHost);
    printf("%2d MMAs (%4d cyc of work): issue->commit->same-warp wake %5lld cyc; round trip via 2nd warp %5lld cyc %s\n",
           k, 64 * k, h[0], h[1], e == cudaSuccess ? "" : cudaGetErrorString(e));
  }
  return 0;
}
