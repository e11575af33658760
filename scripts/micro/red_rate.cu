// red_rate.cu -- how fast can 148 SMs reduce-add fp32 tiles into global
// memory (L2)?  Decides whether a fused backward that accumulates dQ with fp32
// reductions (one 128 x D tile per (key block, query block) pair) is
// bandwidth-feasible on B200.  Analysis only, not part of the product.
//
// Pattern (as the fused backward would issue it): persistent grid, one CTA per
// SM, 128 threads (thread = query row).  Work unit w = (head h, key block j);
// for it in 0..nblk-1 the CTA adds a 128 x D fp32 tile into
// acc[h][(j + it) % nblk] (rotated start, so CTAs of one head do not hit the
// same query block together).
//   mode 0: red.global.add.v4.f32 from registers, lane = row
//   mode 1: red.global.add.f32 (scalar) from registers
//   mode 2: registers -> SMEM (row-major, rotated 16-B chunks), then one
//           cp.reduce.async.bulk .add.f32 of the contiguous 128*D*4 bytes,
//           double-buffered
//   mode 3: mode 2 without the SMEM writes (bulk-reduce engine alone)
//
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o red_rate red_rate.cu
#include <cstdio>
#include <cstdint>
#include <cstdlib>
#include <cuda_runtime.h>

template <int D, int kMode>
__global__ void __launch_bounds__(128, 1) red_kernel(float* acc, int H, int nblk) {
  extern __shared__ __align__(128) uint8_t smem[];
  const int row = threadIdx.x;
  const int N = nblk * 128;
  float v[D];
#pragma unroll
  for (int c = 0; c < D; ++c) v[c] = 1.0f / (1 + ((row + c) & 7));
  int buf = 0;
  for (int w = blockIdx.x; w < H * nblk; w += gridDim.x) {
    const int h = w / nblk, j = w % nblk;
    for (int it = 0; it < nblk; ++it) {
      const int i = (j + it) % nblk;
      float* tile = acc + ((long long)h * N + (long long)i * 128) * D;
      if (kMode == 0) {
        float* dst = tile + row * D;
#pragma unroll
        for (int c = 0; c < D; c += 4)
          asm volatile("red.global.add.v4.f32 [%0], {%1, %2, %3, %4};" ::"l"(dst + c), "f"(v[c]), "f"(v[c + 1]),
                       "f"(v[c + 2]), "f"(v[c + 3])
                       : "memory");
      } else if (kMode == 1) {
        float* dst = tile + row * D;
#pragma unroll
        for (int c = 0; c < D; ++c) asm volatile("red.global.add.f32 [%0], %1;" ::"l"(dst + c), "f"(v[c]) : "memory");
      } else {
        uint8_t* sb = smem + buf * (128 * D * 4);
        if (threadIdx.x == 0) asm volatile("cp.async.bulk.wait_group.read 1;" ::: "memory");
        __syncthreads();
        if (kMode == 2) {
          float4* rp = reinterpret_cast<float4*>(sb + row * D * 4);
#pragma unroll
          for (int c = 0; c < D / 4; ++c) {
            const int cc = (c + row) & (D / 4 - 1);  // rotate: 8 lanes of a phase hit distinct banks
            rp[cc] = make_float4(v[4 * c], v[4 * c + 1], v[4 * c + 2], v[4 * c + 3]);
          }
        }
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        __syncthreads();
        if (threadIdx.x == 0) {
          asm volatile("cp.reduce.async.bulk.global.shared::cta.bulk_group.add.f32 [%0], [%1], %2;" ::"l"(tile),
                       "r"((uint32_t)__cvta_generic_to_shared(sb)), "r"(128 * D * 4)
                       : "memory");
          asm volatile("cp.async.bulk.commit_group;" ::: "memory");
        }
        buf ^= 1;
      }
    }
  }
  if (kMode >= 2 && threadIdx.x == 0) asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
}

template <int D, int kMode>
float run(float* acc, int H, int nblk, int sms, int reps) {
  auto k = red_kernel<D, kMode>;
  const int smem = kMode >= 2 ? 2 * 128 * D * 4 : 0;
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
  k<<<sms, 128, 200 * 1024>>>(acc, H, nblk);  // warm-up (200 KB: one CTA per SM)
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  cudaEventRecord(a);
  for (int r = 0; r < reps; ++r) k<<<sms, 128, 200 * 1024>>>(acc, H, nblk);
  cudaEventRecord(b);
  cudaEventSynchronize(b);
  float ms = 0;
  cudaEventElapsedTime(&ms, a, b);
  (void)smem;
  return ms / reps;
}

int main(int argc, char** argv) {
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  const int nblk = 64;  // N = 8192
  for (int H : {2, 8, 32}) {
    const long long N = nblk * 128LL;
    float* acc;
    cudaMalloc(&acc, (size_t)H * N * 128 * 4);
    cudaMemset(acc, 0, (size_t)H * N * 128 * 4);
    const double units = (double)H * nblk * nblk;
    const char* names[4] = {"red.v4 regs", "red scalar", "bulk + smem", "bulk only"};
    float t64[4] = {run<64, 0>(acc, H, nblk, sms, 5), run<64, 1>(acc, H, nblk, sms, 5),
                    run<64, 2>(acc, H, nblk, sms, 5), run<64, 3>(acc, H, nblk, sms, 5)};
    float t128[4] = {run<128, 0>(acc, H, nblk, sms, 5), run<128, 1>(acc, H, nblk, sms, 5),
                     run<128, 2>(acc, H, nblk, sms, 5), run<128, 3>(acc, H, nblk, sms, 5)};
    for (int m = 0; m < 4; ++m) {
      printf("H=%2d acc %5.0f MB  D=64 %-12s %7.3f ms %7.0f GB/s (%.2f us/tile/SM) | D=128 %7.3f ms %7.0f GB/s (%.2f us/tile/SM)\n",
             H, H * N * 64 * 4 / 1e6, names[m], t64[m], units * 128 * 64 * 4 / (t64[m] * 1e6),
             t64[m] * 1e3 / (units / sms), t128[m], units * 128 * 128 * 4 / (t128[m] * 1e6),
             t128[m] * 1e3 / (units / sms));
    }
    cudaError_t e = cudaDeviceSynchronize();
    if (e != cudaSuccess) printf("error %s\n", cudaGetErrorString(e));
    cudaFree(acc);
  }
  return 0;
}
