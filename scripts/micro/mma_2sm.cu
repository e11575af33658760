// CTA-pair (cta_group::2) tcgen05.mma probe (not part of the library;
// groundwork for a CTA-pair forward / dK-dV backward).
// A cluster of two CTAs allocates TMEM with cta_group::2; the leader's elected
// thread issues kN back-to-back M256 x N x K16 bf16 SS MMAs (each CTA supplies
// its own 128 rows of A and half of B from its SMEM) and stamps clock64()
// after each issue; one multicast commit signals both CTAs.  Steady-state
// cycles per MMA give the pair's rate (M256 N256 K16 at full rate = 128
// cycles, i.e. 8192 flop/clk per SM, the same as M128 N256 on one SM, with
// half the B operand read per SM).
#include <cstdint>
#include <cstdio>
#include <vector>

#include "../../paper_2511_02132_b200/csrc/ptx.cuh"
using namespace attn;

constexpr int kN = 48;

__device__ __forceinline__ void mma_ss_2cta(uint32_t d_tmem, uint64_t a_desc, uint64_t b_desc, uint32_t idesc,
                                            uint32_t acc) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::2.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(d_tmem),
      "l"(a_desc), "l"(b_desc), "r"(idesc), "r"(acc)
      : "memory");
}

template <int NN>
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(128, 1) pair(long long* out) {
  extern __shared__ __align__(1024) uint8_t smem[];
  __shared__ uint64_t bar;
  __shared__ uint32_t tbase;
  const int warp = threadIdx.x / 32;
  const uint32_t rank = ptx::cluster_ctarank();
  for (int i = threadIdx.x; i < 65536 / 4; i += blockDim.x) reinterpret_cast<uint32_t*>(smem)[i] = 0;
  if (threadIdx.x == 0) {
    ptx::mbar_init(&bar, 1);
    ptx::fence_barrier_init();
  }
  asm volatile("fence.proxy.async.shared::cta;");
  ptx::cluster_sync();
  if (warp == 0) {  // one warp of each CTA of the pair
    asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(ptx::smem_u32(&tbase)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;");
  }
  ptx::tc_fence_before();
  __syncthreads();
  ptx::cluster_sync();
  ptx::tc_fence_after();
  const uint32_t tmem = tbase;
  if (warp == 0 && rank == 0) {
    const uint64_t da = ptx::smem_desc_sw128(ptx::smem_u32(smem), 16, 1024);
    const uint64_t db = ptx::smem_desc_sw128(ptx::smem_u32(smem + 32768), 16, 1024);
    constexpr uint32_t idesc = ptx::idesc_bf16_f32(256, NN, 0, 0);
    long long t[kN + 2];
    if (ptx::elect_one_sync()) {
      t[0] = clock64();
#pragma unroll
      for (int i = 0; i < kN; ++i) {
        mma_ss_2cta(tmem, da + ((i & 3) * 2), db + ((i & 3) * 2), idesc, 1);
        t[i + 1] = clock64();
      }
      asm volatile(
          "tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;" ::"r"(
              ptx::smem_u32(&bar)),
          "h"((uint16_t)3)
          : "memory");
      ptx::mbar_wait(&bar, 0);
      t[kN + 1] = clock64();
      if (blockIdx.x == 0)
        for (int i = 0; i < kN + 2; ++i) out[i] = t[i] - t[0];
    }
    __syncwarp();
  }
  if (rank == 1 && threadIdx.x == 0) ptx::mbar_wait(&bar, 0);  // the peer sees the multicast commit too
  ptx::tc_fence_before();
  __syncthreads();
  ptx::cluster_sync();
  if (warp == 0) {
    ptx::tc_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, 512;" ::"r"(tmem));
  }
}

template <int NN>
void run(const char* name) {
  long long* d;
  cudaMalloc(&d, sizeof(long long) * (kN + 2));
  cudaMemset(d, 0, sizeof(long long) * (kN + 2));
  auto k = pair<NN>;
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 65536 + 1024);
  for (int r = 0; r < 3; ++r) k<<<148, 128, 65536 + 1024>>>(d);
  cudaError_t e = cudaDeviceSynchronize();
  std::vector<long long> h(kN + 2);
  cudaMemcpy(h.data(), d, sizeof(long long) * (kN + 2), cudaMemcpyDeviceToHost);
  printf("%s %s\n  issue-done cycle after MMA i:", name, e == cudaSuccess ? "ok" : cudaGetErrorString(e));
  for (int i = 1; i <= kN; ++i) printf(" %lld", h[i]);
  printf("\n  all complete: %lld  -> steady cycles/MMA %.1f\n", h[kN + 1],
         (double)(h[kN] - h[kN / 2]) / (kN / 2));
  cudaFree(d);
}

int main() {
  run<256>("2-CTA SS M256 N256 K16");
  run<128>("2-CTA SS M256 N128 K16");
  return 0;
}
