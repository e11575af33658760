// Latency of a wait on an ALREADY-COMPLETED mbarrier phase (try_wait vs
// test_wait), alone and with 8 warps keeping the SMSPs busy with MUFU.EX2 /
// FMA work (the softmax's mix).  Not part of the library.
#include <cstdint>
#include <cstdio>

#include "../../paper_2511_02132_b200/csrc/ptx.cuh"
using namespace attn;

__device__ __forceinline__ bool test_wait(uint64_t* bar, uint32_t parity) {
  uint32_t ok;
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "mbarrier.test_wait.parity.acquire.cta.shared::cta.b64 p, [%1], %2;\n\t"
      "selp.u32 %0, 1, 0, p;\n\t}"
      : "=r"(ok)
      : "r"(ptx::smem_u32(bar)), "r"(parity)
      : "memory");
  return ok != 0;
}

template <bool kTest, bool kLoad>
__global__ void __launch_bounds__(384, 1) probe(long long* out, float* sink) {
  __shared__ uint64_t bar;
  __shared__ volatile int stop;
  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  if (threadIdx.x == 0) {
    ptx::mbar_init(&bar, 1);
    ptx::fence_barrier_init();
    stop = 0;
  }
  __syncthreads();
  if (threadIdx.x == 0) ptx::mbar_arrive(&bar);  // phase 0 completes
  __syncthreads();
  if (warp == 1) {
    long long tot = 0;
    int okc = 0;
    for (int i = 0; i < 2000; ++i) {
      const long long t0 = clock64();
      const bool ok = kTest ? test_wait(&bar, 0) : ptx::mbar_try_wait(&bar, 0);
      if (!ok) break;  // the branch resolves on the predicate before the clock read
      const long long t1 = clock64();
      okc += ok;
      tot += t1 - t0;
    }
    if (lane == 0 && blockIdx.x == 0) { out[0] = tot / 2000; out[1] = okc; }
    if (lane == 0) stop = 1;
  } else if (warp >= 4 && kLoad) {
    float x = threadIdx.x * 1e-3f, y = 0.f;
    while (!stop) {
#pragma unroll 16
      for (int k = 0; k < 64; ++k) {
        x = ptx::ex2(x * 0.999f - 1.0f);
        y = fmaf(x, 1.0001f, y);
      }
    }
    if (y == 12345.f) sink[threadIdx.x] = y;
  }
}

template <bool kTest, bool kLoad>
void run(const char* name) {
  long long* d;
  float* s;
  cudaMalloc(&d, 16);
  cudaMalloc(&s, 4096);
  probe<kTest, kLoad><<<148, 384>>>(d, s);
  probe<kTest, kLoad><<<148, 384>>>(d, s);
  cudaError_t e = cudaDeviceSynchronize();
  long long h[2];
  cudaMemcpy(h, d, 16, cudaMemcpyDeviceToHost);
  printf("%-44s %s cycles per completed-phase wait: %lld (ok %lld/2000)\n", name,
         e == cudaSuccess ? "" : cudaGetErrorString(e), h[0], h[1]);
  cudaFree(d);
  cudaFree(s);
}

int main() {
  run<false, false>("try_wait, idle SM");
  run<true, false>("test_wait, idle SM");
  run<false, true>("try_wait, 8 warps of MUFU/FMA load");
  run<true, true>("test_wait, 8 warps of MUFU/FMA load");
  return 0;
}
