// MUFU.EX2 throughput per SM vs warps per SMSP (independent ex2 chains).
#include <cstdio>
#include <cstdint>
__global__ void k(float* out, int iters, long long* cyc) {
  float a[8];
  for (int i = 0; i < 8; ++i) a[i] = threadIdx.x * 1e-3f + i * 1e-4f;
  __syncthreads();
  long long t0 = clock64();
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < 8; ++i) asm volatile("ex2.approx.ftz.f32 %0, %0;" : "+f"(a[i]));
  }
  __syncthreads();
  long long t1 = clock64();
  float s = 0;
  for (int i = 0; i < 8; ++i) s += a[i];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
  if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
}
int main() {
  float* o; long long* c; cudaMalloc(&o, 148 * 1024 * 4); cudaMalloc(&c, 148 * 8);
  for (int warps : {4, 8, 16, 32}) {
    const int iters = 2048;
    k<<<148, warps * 32>>>(o, iters, c);
    k<<<148, warps * 32>>>(o, iters, c);
    long long h; cudaMemcpy(&h, c, 8, cudaMemcpyDeviceToHost);
    double ex2 = (double)warps * 32 * iters * 8;
    printf("%2d warps/SM (%d per SMSP): %.2f ex2/clk/SM\n", warps, warps / 4, ex2 / h);
  }
  return 0;
}
