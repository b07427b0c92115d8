// TMEM -> register read bandwidth per SM, with U loads in flight per warp
// before tcgen05.wait::ld (separates latency from bandwidth), W warps per CTA
// (W/4 per 32-lane quarter), C CTAs per SM, and 32x32b.x32 vs .x64 shapes.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -I../../paper_2210_03052_b200/csrc tmem_bw.cu -o tmem_bw
#include <cstdio>
#include <cuda_runtime.h>
#include "ptx.cuh"
using namespace bt;

template <int U, int X>
__global__ void k(float* out, int iters, int cols) {
  __shared__ uint32_t holder;
  const int warp = threadIdx.x >> 5;
  if (warp == 0) { ptx::tmem_alloc(&holder, cols); ptx::tmem_relinquish(); }
  ptx::tc_fence_before();
  __syncthreads();
  ptx::tc_fence_after();
  const uint32_t base = holder + (static_cast<uint32_t>((warp & 3) * 32) << 16);
  const int nw = blockDim.x >> 5;
  const int colw = cols / (nw >> 2);  // columns owned by this warp
  const uint32_t mybase = base + (warp >> 2) * colw;
  float acc = 0.f;
  for (int i = 0; i < iters; ++i) {
    for (int c = 0; c + U * X <= colw; c += U * X) {
      uint32_t r[U][X];
#pragma unroll
      for (int u = 0; u < U; ++u) {
        if constexpr (X == 32) {
          asm volatile(
              "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16,%17,"
              "%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
              : "=r"(r[u][0]), "=r"(r[u][1]), "=r"(r[u][2]), "=r"(r[u][3]), "=r"(r[u][4]), "=r"(r[u][5]),
                "=r"(r[u][6]), "=r"(r[u][7]), "=r"(r[u][8]), "=r"(r[u][9]), "=r"(r[u][10]), "=r"(r[u][11]),
                "=r"(r[u][12]), "=r"(r[u][13]), "=r"(r[u][14]), "=r"(r[u][15]), "=r"(r[u][16]), "=r"(r[u][17]),
                "=r"(r[u][18]), "=r"(r[u][19]), "=r"(r[u][20]), "=r"(r[u][21]), "=r"(r[u][22]), "=r"(r[u][23]),
                "=r"(r[u][24]), "=r"(r[u][25]), "=r"(r[u][26]), "=r"(r[u][27]), "=r"(r[u][28]), "=r"(r[u][29]),
                "=r"(r[u][30]), "=r"(r[u][31])
              : "r"(mybase + c + u * X));
        } else {
          asm volatile("tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
                       : "=r"(r[u][0]), "=r"(r[u][1]), "=r"(r[u][2]), "=r"(r[u][3]), "=r"(r[u][4]), "=r"(r[u][5]),
                         "=r"(r[u][6]), "=r"(r[u][7]), "=r"(r[u][8]), "=r"(r[u][9]), "=r"(r[u][10]), "=r"(r[u][11]),
                         "=r"(r[u][12]), "=r"(r[u][13]), "=r"(r[u][14]), "=r"(r[u][15])
                       : "r"(mybase + c + u * X));
        }
      }
      asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
      for (int u = 0; u < U; ++u) acc += __uint_as_float(r[u][0]) + __uint_as_float(r[u][X - 1]);
    }
  }
  out[blockIdx.x * blockDim.x + threadIdx.x] = acc;
  ptx::tc_fence_before();
  __syncthreads();
  if (warp == 0) { ptx::tc_fence_after(); ptx::tmem_dealloc(holder, cols); }
}

template <int U, int X>
void run(int sms, int clk, float* out, int warps, int ctas, int cols) {
  const int iters = 2000;
  k<U, X><<<sms * ctas, warps * 32>>>(out, 4, cols);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  cudaEventRecord(e0);
  k<U, X><<<sms * ctas, warps * 32>>>(out, iters, cols);
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  float ms;
  cudaEventElapsedTime(&ms, e0, e1);
  cudaError_t err = cudaGetLastError();
  const int colw = cols / (warps / 4);
  const int used = colw / (U * X) * (U * X) * (warps / 4);
  double bytes = double(sms) * ctas * iters * 128.0 * used * 4;
  printf("U %d x%-2d warps %2d ctas/SM %d cols %3d: %.3f ms  %.1f B/clk/SM  (%s)\n", U, X, warps, ctas, cols, ms,
         bytes / (ms * 1e-3) / sms / (clk * 1e3), cudaGetErrorString(err));
}

int main() {
  int sms, clk;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
  float* out;
  cudaMalloc(&out, sizeof(float) * sms * 4 * 1024);
  for (int w : {4, 8, 16}) {
    run<1, 32>(sms, clk, out, w, 1, 256);
    run<2, 32>(sms, clk, out, w, 1, 256);
    run<4, 32>(sms, clk, out, w, 1, 256);
    run<4, 16>(sms, clk, out, w, 1, 256);
  }
  run<2, 32>(sms, clk, out, 8, 2, 256);
  run<4, 32>(sms, clk, out, 8, 2, 256);
  run<4, 32>(sms, clk, out, 4, 1, 512);
  run<4, 32>(sms, clk, out, 16, 1, 512);
  return 0;
}
