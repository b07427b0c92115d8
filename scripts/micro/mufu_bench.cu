// Throughput of the SFU (MUFU) ops the epilogues / softmax use, per SM per clock.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 mufu_bench.cu -o mufu_bench
#include <cstdio>
#include <cuda_runtime.h>

template <int OP>
__global__ void k(float* out, int iters) {
  float a0 = threadIdx.x * 1e-3f, a1 = a0 + 0.1f, a2 = a0 + 0.2f, a3 = a0 + 0.3f;
  float a4 = a0 + 0.4f, a5 = a0 + 0.5f, a6 = a0 + 0.6f, a7 = a0 + 0.7f;
  for (int i = 0; i < iters; ++i) {
#define OPX(x)                                                                   \
  if (OP == 0) asm volatile("tanh.approx.f32 %0, %0;" : "+f"(x));                \
  if (OP == 1) asm volatile("ex2.approx.ftz.f32 %0, %0;" : "+f"(x));             \
  if (OP == 2) asm volatile("rcp.approx.ftz.f32 %0, %0;" : "+f"(x));             \
  if (OP == 3) { unsigned r; asm volatile("cvt.rn.bf16x2.f32 %0, %1, %1;" : "=r"(r) : "f"(x)); x = __uint_as_float(r); } \
  if (OP == 4) asm volatile("fma.rn.f32 %0, %0, %0, %0;" : "+f"(x));                \
  if (OP == 5) asm volatile("ex2.approx.f16x2 %0, %0;" : "+r"(*reinterpret_cast<unsigned*>(&x))); \
  if (OP == 6) asm volatile("ex2.approx.ftz.bf16x2 %0, %0;" : "+r"(*reinterpret_cast<unsigned*>(&x)));
    OPX(a0) OPX(a1) OPX(a2) OPX(a3) OPX(a4) OPX(a5) OPX(a6) OPX(a7)
  }
  out[blockIdx.x * blockDim.x + threadIdx.x] = a0 + a1 + a2 + a3 + a4 + a5 + a6 + a7;
}

template <int OP>
void run(const char* name, float* out, int sms) {
  const int iters = 4096, threads = 512, blocks = sms * 2;
  k<OP><<<blocks, threads>>>(out, 16);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0); cudaEventCreate(&e1);
  cudaEventRecord(e0);
  k<OP><<<blocks, threads>>>(out, iters);
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  float ms; cudaEventElapsedTime(&ms, e0, e1);
  int clk; cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
  double ops = double(blocks) * threads * iters * 8;
  double per_sm_clk = ops / (ms * 1e-3) / sms / (clk * 1e3);
  printf("%-10s %.3f ms  %.2f ops/clk/SM (at %d MHz nominal)\n", name, ms, per_sm_clk, clk / 1000);
}

int main() {
  int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  float* out; cudaMalloc(&out, sizeof(float) * sms * 2 * 512);
  run<0>("tanh", out, sms);
  run<1>("ex2", out, sms);
  run<2>("rcp", out, sms);
  run<3>("cvt_bf16x2", out, sms);
  run<4>("ffma", out, sms);
  run<5>("ex2_f16x2 (ops = packed instrs; x2 for elements)", out, sms);
  run<6>("ex2_bf16x2 (ops = packed instrs; x2 for elements)", out, sms);
  return 0;
}
