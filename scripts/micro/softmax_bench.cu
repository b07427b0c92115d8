// Cycles for the MHA softmax inner block (one 128-key block per row, values
// in registers) with W softmax warps per SM, as in mha_fwd_kernel: exp2 of
// 128 values per row (POLY of every 16 on the FMA pipe), bf16 pack, P stores
// to swizzled smem, row sum.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -I../../paper_2210_03052_b200/csrc softmax_bench.cu -o softmax_bench
#include <cstdio>
#include <cuda_runtime.h>
#include <cuda_bf16.h>
#include "ptx.cuh"
using namespace bt;

template <int POLY, int KEYS>
__global__ void __launch_bounds__(128) k(float* out, int iters, long long* cyc) {
  __shared__ __align__(1024) uint8_t sP[128 * KEYS * 2];
  const int row = threadIdx.x;
  float s[KEYS];
#pragma unroll
  for (int i = 0; i < KEYS; ++i) s[i] = (threadIdx.x * 7 + i * 13) % 97 * 0.01f - 0.5f;
  unsigned long long acc = 0;
  const float sl2 = 0.18f;
  long long t0 = clock64();
  for (int it = 0; it < iters; ++it) {
    const float msc = 0.3f + it * 1e-7f;
    const unsigned long long sl2x2 = ptx::f2(sl2, sl2), nm2 = ptx::f2(-msc, -msc);
    unsigned long long sum4[4] = {0, 0, 0, 0};
#pragma unroll
    for (int c = 0; c < KEYS / 32; ++c) {
      uint8_t* prow = sP + (c >> 1) * 128 * 128 + row * 128;
      float ev[32];
#pragma unroll
      for (int i = 0; i < 32; i += 2) {
        float x0, x1;
        ptx::unf2(ptx::fma2(ptx::f2(s[32 * c + i], s[32 * c + i + 1]), sl2x2, nm2), x0, x1);
        if ((i & 15) < POLY) {
          ptx::ex2_poly2(x0, x1, ev[i], ev[i + 1]);
        } else {
          ev[i] = ptx::ex2_approx(x0);
          ev[i + 1] = ptx::ex2_approx(x1);
        }
      }
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        uint32_t pk[4];
#pragma unroll
        for (int e = 0; e < 8; e += 2) {
          sum4[e / 2] = ptx::add2(sum4[e / 2], ptx::f2(ev[8 * q + e], ev[8 * q + e + 1]));
          pk[e / 2] = ptx::pack_bf16x2(ev[8 * q + e], ev[8 * q + e + 1]);
        }
        const int cb = (c & 1) * 4;
        *reinterpret_cast<uint4*>(prow + (((cb + q) ^ (row & 7)) << 4)) = make_uint4(pk[0], pk[1], pk[2], pk[3]);
      }
    }
    acc = ptx::add2(acc, ptx::add2(ptx::add2(sum4[0], sum4[1]), ptx::add2(sum4[2], sum4[3])));
    __syncwarp();
  }
  long long t1 = clock64();
  float a, b;
  ptx::unf2(acc, a, b);
  out[blockIdx.x * 128 + threadIdx.x] = a + b + sP[(threadIdx.x * 37) % sizeof(sP)];
  if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
}

template <int POLY, int KEYS>
void run(int sms, int ctas_per_sm, float* out, long long* cyc) {
  const int iters = 200;
  k<POLY, KEYS><<<sms * ctas_per_sm, 128>>>(out, 2, cyc);
  k<POLY, KEYS><<<sms * ctas_per_sm, 128>>>(out, iters, cyc);
  cudaDeviceSynchronize();
  long long h[1024];
  cudaMemcpy(h, cyc, sizeof(long long) * sms * ctas_per_sm, cudaMemcpyDeviceToHost);
  double m = 0;
  for (int i = 0; i < sms * ctas_per_sm; ++i) m += h[i];
  m /= sms * ctas_per_sm;
  printf("POLY %2d keys %3d  %d CTA(s) of 4 warps per SM: %.0f cycles per block-item (%s)\n", POLY, KEYS, ctas_per_sm,
         m / iters, cudaGetErrorString(cudaGetLastError()));
}

int main() {
  int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  float* out; long long* cyc;
  cudaMalloc(&out, sizeof(float) * sms * 8 * 128);
  cudaMalloc(&cyc, sizeof(long long) * sms * 8);
  for (int c = 1; c <= 4; c *= 2) {
    run<0, 128>(sms, c, out, cyc);
    run<6, 128>(sms, c, out, cyc);
    run<16, 128>(sms, c, out, cyc);
    run<0, 64>(sms, c, out, cyc);
    run<6, 64>(sms, c, out, cyc);
  }
  return 0;
}
