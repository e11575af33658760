// Does tcgen05.mma kind::f16 accept A = f16 (TMEM) with B = bf16 (SMEM)?
// A = 1.5 (f16 0x3E00), B = 2.0 (bf16 0x4000), K = 16  ->  D = 48 expected.
#include <cstdio>
#include <cstdint>
#include "../../paper_2511_02132_b200/csrc/ptx.cuh"
using namespace attn;

__global__ void __launch_bounds__(128, 1) k(float* out, uint32_t a_fmt) {
  extern __shared__ __align__(1024) uint8_t smem[];
  __shared__ uint64_t bar;
  __shared__ uint32_t tbase;
  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  for (int i = threadIdx.x; i < 16384 / 2; i += blockDim.x) reinterpret_cast<uint16_t*>(smem)[i] = 0x4000;
  if (threadIdx.x == 0) { ptx::mbar_init(&bar, 1); ptx::fence_barrier_init(); }
  if (warp == 0) { ptx::tmem_alloc(&tbase, 256); ptx::tmem_relinquish(); }
  asm volatile("fence.proxy.async.shared::cta;");
  ptx::tc_fence_before(); __syncthreads(); ptx::tc_fence_after();
  const uint32_t tmem = tbase;
  uint32_t r[32];
  for (int i = 0; i < 32; ++i) r[i] = 0x3E003E00u;  // f16 pair (1.5, 1.5)
  ptx::tmem_st32(tmem + ((uint32_t)(warp * 32) << 16), r);
  ptx::tmem_wait_st();
  ptx::tc_fence_before(); __syncthreads(); ptx::tc_fence_after();
  if (warp == 0) {
    const uint64_t db = ptx::smem_desc_sw128(ptx::smem_u32(smem), 128 * 128, 1024);
    const uint32_t idesc = (1u << 4) | (a_fmt << 7) | (1u << 10) | (0u << 15) | (1u << 16) | ((128u >> 3) << 17) |
                           ((128u >> 4) << 24);
    if (ptx::elect_one_sync()) {
      ptx::mma_ts(tmem + 128, tmem, db, idesc, 0);
      ptx::mma_commit(&bar);
    }
    __syncwarp();
    ptx::mbar_wait(&bar, 0);
  }
  ptx::tc_fence_before(); __syncthreads(); ptx::tc_fence_after();
  ptx::tmem_ld32(tmem + ((uint32_t)(warp * 32) << 16) + 128, r);
  out[threadIdx.x] = __uint_as_float(r[0]);
  ptx::tc_fence_before(); __syncthreads();
  if (warp == 0) { ptx::tc_fence_after(); ptx::tmem_dealloc(tmem, 256); }
}

int main() {
  float* d; cudaMalloc(&d, 128 * 4);
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 16384 + 1024);
  for (uint32_t fmt : {0u, 1u}) {
    k<<<1, 128, 16384 + 1024>>>(d, fmt);
    float h[128];
    cudaError_t e = cudaMemcpy(h, d, sizeof h, cudaMemcpyDeviceToHost);
    printf("A format %s: D[0]=%g D[127]=%g (expect 48 if A read as f16) %s\n", fmt ? "bf16" : "f16", h[0], h[127],
           e == cudaSuccess ? "" : cudaGetErrorString(e));
  }
  return 0;
}
