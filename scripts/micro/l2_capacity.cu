// l2_capacity.cu -- does one die of B200 see the whole 126 MB L2, or only
// its own half?  (The paper's premise is a private L2 per chiplet, PAPER.md
// :100-105 and Table 1 :317-323.)  Analysis tooling only.
//
// A persistent grid of one CTA per SM streams a buffer of S bytes `passes`
// times with 16-byte ld.global.cg loads (L2-cached, L1 bypassed).  Only the
// SMs of the dies in `die_mask` take part (die of every SM from the
// library's probe, passed in as domain_of_smid).  Modes:
//   0 split : every line of the buffer is read once per pass by ONE of the
//             participating SMs (the participants split the buffer);
//   1 each  : every participating DIE reads the whole buffer once per pass
//             (split among that die's SMs) -- two dies read every line.
// If the buffer fits in the L2 that the readers can use, passes 2..n hit:
// DRAM bytes ~ S instead of passes * S (ncu), and time per pass drops.
//
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -shared -Xcompiler -fPIC
//        -o scripts/micro/libl2cap.so scripts/micro/l2_capacity.cu
#include <cuda_runtime.h>

#include <cstdint>

__global__ void __launch_bounds__(1024, 1)
    l2cap_kernel(const int4* __restrict__ buf, long long n16, const signed char* dom, int die_mask, int mode,
                 int passes, const int* die_rank_base, int parts_total, const int* parts_die, int* ctr,
                 unsigned long long* sink) {
  extern __shared__ int smem_pad[];  // large dynamic SMEM: one CTA per SM
  __shared__ int rank_s;
  uint32_t sm;
  asm volatile("mov.u32 %0, %%smid;" : "=r"(sm));
  const int die = dom[sm] < 0 ? 0 : dom[sm];
  if (!((die_mask >> die) & 1)) return;
  if (threadIdx.x == 0) rank_s = atomicAdd(&ctr[mode == 1 ? die : 0], 1);
  __syncthreads();
  const int rank = rank_s;
  const int parts = (mode == 1) ? parts_die[die] : parts_total;
  if (rank >= parts) return;  // more CTAs than SMs landed on these dies
  unsigned long long acc = 0;
  for (int p = 0; p < passes; ++p) {
    for (long long i = (long long)rank * blockDim.x + threadIdx.x; i < n16; i += (long long)parts * blockDim.x) {
      int4 x;
      asm volatile("ld.global.cg.v4.s32 {%0,%1,%2,%3}, [%4];"
                   : "=r"(x.x), "=r"(x.y), "=r"(x.z), "=r"(x.w)
                   : "l"(buf + i));
      acc += (unsigned)(x.x ^ x.y ^ x.z ^ x.w);
    }
  }
  if (acc == 0x123456789ull) sink[0] = acc + (unsigned long long)smem_pad[0];
}

extern "C" {
// Returns elapsed ms (device events) of the launch, or a negative CUDA error.
float l2cap_run(const void* buf, long long bytes, const signed char* d_dom, int die_mask, int mode, int passes,
                int num_sms, const int* sms_per_die) {
  int* d_ctr = nullptr;
  int* d_parts = nullptr;
  unsigned long long* d_sink = nullptr;
  cudaMalloc(&d_ctr, 8 * sizeof(int));
  cudaMalloc(&d_parts, 8 * sizeof(int));
  cudaMalloc(&d_sink, sizeof(unsigned long long));
  cudaMemset(d_ctr, 0, 8 * sizeof(int));
  int parts_total = 0;
  for (int d = 0; d < 2; ++d)
    if ((die_mask >> d) & 1) parts_total += sms_per_die[d];
  cudaMemcpy(d_parts, sms_per_die, 2 * sizeof(int), cudaMemcpyHostToDevice);
  const int smem = 150 * 1024;
  cudaFuncSetAttribute(l2cap_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  cudaEventRecord(e0);
  l2cap_kernel<<<num_sms, 1024, smem>>>(static_cast<const int4*>(buf), bytes / 16, d_dom, die_mask, mode, passes,
                                        nullptr, parts_total, d_parts, d_ctr, d_sink);
  cudaEventRecord(e1);
  cudaError_t e = cudaEventSynchronize(e1);
  float ms = -1.f;
  if (e == cudaSuccess && cudaGetLastError() == cudaSuccess) cudaEventElapsedTime(&ms, e0, e1);
  else ms = -(float)e;
  cudaEventDestroy(e0);
  cudaEventDestroy(e1);
  cudaFree(d_ctr);
  cudaFree(d_parts);
  cudaFree(d_sink);
  return ms;
}
}
