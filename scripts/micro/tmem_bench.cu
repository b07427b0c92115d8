// TMEM -> register read bandwidth (tcgen05.ld.32x32b.x32) per SM, with W warps
// (W/4 warps per 32-lane quarter) and C CTAs per SM.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -I../../paper_2210_03052_b200/csrc tmem_bench.cu -o tmem_bench
#include <cstdio>
#include <cuda_runtime.h>
#include <cuda_bf16.h>
#include "ptx.cuh"
using namespace bt;

__global__ void k(float* out, int iters, int cols) {
  __shared__ uint32_t holder;
  const int warp = threadIdx.x >> 5;
  if (warp == 0) { ptx::tmem_alloc(&holder, cols); ptx::tmem_relinquish(); }
  ptx::tc_fence_before();
  __syncthreads();
  ptx::tc_fence_after();
  const uint32_t base = holder + (static_cast<uint32_t>((warp & 3) * 32) << 16);
  const int nw = blockDim.x >> 5;
  float acc = 0.f;
  for (int i = 0; i < iters; ++i) {
    for (int c = (warp >> 2) * 32; c < cols; c += 32 * (nw >> 2)) {
      uint32_t r[32];
      ptx::tmem_ld32(base + c, r);
      ptx::tmem_wait_ld(r);
      acc += __uint_as_float(r[0]) + __uint_as_float(r[31]);
    }
  }
  out[blockIdx.x * blockDim.x + threadIdx.x] = acc;
  ptx::tc_fence_before();
  __syncthreads();
  if (warp == 0) { ptx::tc_fence_after(); ptx::tmem_dealloc(holder, cols); }
}

int main() {
  int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  int clk; cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
  float* out; cudaMalloc(&out, sizeof(float) * sms * 4 * 1024);
  const int cfgs[][3] = {{4, 1, 256}, {8, 1, 256}, {16, 1, 256}, {4, 2, 256}, {8, 2, 256}, {4, 1, 512}, {16, 1, 512}};
  for (auto& c : cfgs) {
    const int warps = c[0], ctas = c[1], cols = c[2];
    const int iters = 2000;
    k<<<sms * ctas, warps * 32>>>(out, 4, cols);
    cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
    cudaEventRecord(e0);
    k<<<sms * ctas, warps * 32>>>(out, iters, cols);
    cudaEventRecord(e1); cudaEventSynchronize(e1);
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    cudaError_t err = cudaGetLastError();
    double bytes = double(sms) * ctas * iters * 128.0 * cols * 4;
    printf("warps %2d ctas/SM %d cols %3d: %.3f ms  %.1f B/clk/SM  (%s)\n", warps, ctas, cols, ms,
           bytes / (ms * 1e-3) / sms / (clk * 1e3), cudaGetErrorString(err));
  }
  return 0;
}
