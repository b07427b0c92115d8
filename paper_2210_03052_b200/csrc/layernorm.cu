// Fused add-bias + residual + LayerNorm (paper section III-C1, reference
// fusion.py:79-98):  z = (x + residual) + bias;  y = gamma * (z - mean) /
// sqrt(var + eps) + beta, population variance over the row.
//
// HBM-bound: one warp per row, each lane holds ceil(k/256) 16-byte chunks of
// x and residual in registers (k = 768 -> 3, k = 1024 -> 4), fp32 two-pass
// mean / centred variance with shuffle reductions, one global round trip.

#include "common.cuh"
#include "ptx.cuh"

namespace bt {

// One 8-column chunk of a LayerNorm output row: bf16 into out (packed rows),
// or -- the forward's last LayerNorm -- the same bf16-rounded values widened
// to fp32 straight into the final output row (row_map[row] of the padded
// output, or row itself when row_map is null), which replaces the unpack
// pass (packing.py:151-160) bit for bit.
__device__ __forceinline__ void store_row_chunk(const uint4& o, __nv_bfloat16* out, float* outf,
                                                const int32_t* row_map, int row, size_t base, int k, int c) {
  if (outf == nullptr) {
    reinterpret_cast<uint4*>(out + base)[c] = o;
    return;
  }
  const size_t orow = row_map ? static_cast<size_t>(__ldg(row_map + row)) : static_cast<size_t>(row);
  float4* d = reinterpret_cast<float4*>(outf + orow * k + 8 * c);
  d[0] = make_float4(__uint_as_float(o.x << 16), __uint_as_float(o.x & 0xffff0000u), __uint_as_float(o.y << 16),
                     __uint_as_float(o.y & 0xffff0000u));
  d[1] = make_float4(__uint_as_float(o.z << 16), __uint_as_float(o.z & 0xffff0000u), __uint_as_float(o.w << 16),
                     __uint_as_float(o.w & 0xffff0000u));
}

// Register-resident parameters: best while they fit with >= 2 CTAs per SM
// (k <= 768: 126 registers); wider rows use the shared-memory variant.
template <int NCH, bool HOIST>
__global__ void __launch_bounds__(256) ln_bias_residual_regs_kernel(const __nv_bfloat16* __restrict__ x,
                                                               const __nv_bfloat16* __restrict__ res,
                                                               const float* __restrict__ bias,
                                                               const float* __restrict__ gamma,
                                                               const float* __restrict__ beta, float eps,
                                                               __nv_bfloat16* __restrict__ out, int T, int k,
                                                               float* __restrict__ outf,
                                                               const int32_t* __restrict__ row_map) {
  const int lane = threadIdx.x & 31;
  const int wpb = blockDim.x >> 5;
  const int nchunk = k >> 3;
  const float inv_k = 1.0f / static_cast<float>(k);
  // Parameters do not depend on the previous kernel: fetch them into
  // registers before griddepcontrol.wait so their latency overlaps its tail.
  // (HOIST = false for very wide rows, where the parameters would not fit in
  // registers: they are then re-read per row from L1.)
  float bv[NCH][8], gv[NCH][8], ev[NCH][8];
  auto load_params = [&]() {
#pragma unroll
  for (int i = 0; i < NCH; ++i) {
    const int c = lane + 32 * i;
#pragma unroll
    for (int e = 0; e < 8; ++e) bv[i][e] = 0.f, gv[i][e] = 0.f, ev[i][e] = 0.f;
    if (c < nchunk) {
      const float4* g4 = reinterpret_cast<const float4*>(gamma) + 2 * c;
      const float4* e4 = reinterpret_cast<const float4*>(beta) + 2 * c;
      const float4 g0 = __ldg(g4), g1 = __ldg(g4 + 1), e0 = __ldg(e4), e1 = __ldg(e4 + 1);
      gv[i][0] = g0.x; gv[i][1] = g0.y; gv[i][2] = g0.z; gv[i][3] = g0.w;
      gv[i][4] = g1.x; gv[i][5] = g1.y; gv[i][6] = g1.z; gv[i][7] = g1.w;
      ev[i][0] = e0.x; ev[i][1] = e0.y; ev[i][2] = e0.z; ev[i][3] = e0.w;
      ev[i][4] = e1.x; ev[i][5] = e1.y; ev[i][6] = e1.z; ev[i][7] = e1.w;
      if (bias) {
        const float4* b4 = reinterpret_cast<const float4*>(bias) + 2 * c;
        const float4 b0 = __ldg(b4), b1 = __ldg(b4 + 1);
        bv[i][0] = b0.x; bv[i][1] = b0.y; bv[i][2] = b0.z; bv[i][3] = b0.w;
        bv[i][4] = b1.x; bv[i][5] = b1.y; bv[i][6] = b1.z; bv[i][7] = b1.w;
      }
    }
  }
  };
  if constexpr (HOIST) load_params();
  ptx::griddep_launch_dependents();
  ptx::griddep_wait();
  for (int row = blockIdx.x * wpb + (threadIdx.x >> 5); row < T; row += gridDim.x * wpb) {
    const size_t base = static_cast<size_t>(row) * k;
    if constexpr (!HOIST) load_params();
    uint4 xv[NCH], rv[NCH];
#pragma unroll
    for (int i = 0; i < NCH; ++i) {  // issue every load of the row before using any
      const int c = lane + 32 * i;
      xv[i] = make_uint4(0, 0, 0, 0);
      rv[i] = make_uint4(0, 0, 0, 0);
      if (c < nchunk) {
        xv[i] = __ldg(reinterpret_cast<const uint4*>(x + base) + c);
        if (res) rv[i] = __ldg(reinterpret_cast<const uint4*>(res + base) + c);
      }
    }
    float z[NCH][8];
    float sum = 0.f;
#pragma unroll
    for (int i = 0; i < NCH; ++i) {
      const __nv_bfloat162* xh = reinterpret_cast<const __nv_bfloat162*>(&xv[i]);
      const __nv_bfloat162* rh = reinterpret_cast<const __nv_bfloat162*>(&rv[i]);
#pragma unroll
      for (int e = 0; e < 4; ++e) {
        const float2 xf = __bfloat1622float2(xh[e]);
        const float2 rf = __bfloat1622float2(rh[e]);
        z[i][2 * e] = (xf.x + rf.x) + bv[i][2 * e];  // (x + residual) + bias, fusion.py:96
        z[i][2 * e + 1] = (xf.y + rf.y) + bv[i][2 * e + 1];
      }
      if (lane + 32 * i < nchunk) {
#pragma unroll
        for (int e = 0; e < 8; ++e) sum += z[i][e];
      }
    }
#pragma unroll
    for (int o = 16; o; o >>= 1) sum += __shfl_xor_sync(0xffffffffu, sum, o);
    const float mean = sum * inv_k;
    float sq = 0.f;
#pragma unroll
    for (int i = 0; i < NCH; ++i) {
      if (lane + 32 * i < nchunk) {
#pragma unroll
        for (int e = 0; e < 8; ++e) {
          const float d = z[i][e] - mean;
          sq += d * d;
        }
      }
    }
#pragma unroll
    for (int o = 16; o; o >>= 1) sq += __shfl_xor_sync(0xffffffffu, sq, o);
    const float rstd = 1.0f / sqrtf(sq * inv_k + eps);
#pragma unroll
    for (int i = 0; i < NCH; ++i) {
      const int c = lane + 32 * i;
      if (c < nchunk) {
        uint4 o;
        uint32_t* ow = reinterpret_cast<uint32_t*>(&o);
#pragma unroll
        for (int e = 0; e < 4; ++e) {
          const float y0 = gv[i][2 * e] * ((z[i][2 * e] - mean) * rstd) + ev[i][2 * e];
          const float y1 = gv[i][2 * e + 1] * ((z[i][2 * e + 1] - mean) * rstd) + ev[i][2 * e + 1];
          ow[e] = ptx::pack_bf16x2(y0, y1);
        }
        store_row_chunk(o, out, outf, row_map, row, base, k, c);
      }
    }
  }
}

// Parameters (bias, gamma, beta: 3 x k fp32) are staged in shared memory once
// per CTA -- before griddepcontrol.wait, so the copy overlaps the previous
// kernel's tail -- rather than held in registers: at k = 1024 holding them cost
// 162 registers per thread and left one 256-thread CTA (8 warps) per SM,
// too few loads in flight to cover HBM latency (C5: 0.40-0.54 of HBM).
template <int NCH>
__global__ void __launch_bounds__(256) ln_bias_residual_kernel(const __nv_bfloat16* __restrict__ x,
                                                               const __nv_bfloat16* __restrict__ res,
                                                               const float* __restrict__ bias,
                                                               const float* __restrict__ gamma,
                                                               const float* __restrict__ beta, float eps,
                                                               __nv_bfloat16* __restrict__ out, int T, int k,
                                                               float* __restrict__ outf,
                                                               const int32_t* __restrict__ row_map) {
  extern __shared__ float4 sparams[];  // [3][k / 4]: bias (0 if none), gamma, beta
  const int lane = threadIdx.x & 31;
  const int wpb = blockDim.x >> 5;
  const int nchunk = k >> 3;
  const int k4 = k >> 2;
  const float inv_k = 1.0f / static_cast<float>(k);
  for (int i = threadIdx.x; i < k4; i += blockDim.x) {
    sparams[i] = bias ? __ldg(reinterpret_cast<const float4*>(bias) + i) : make_float4(0.f, 0.f, 0.f, 0.f);
    sparams[k4 + i] = __ldg(reinterpret_cast<const float4*>(gamma) + i);
    sparams[2 * k4 + i] = __ldg(reinterpret_cast<const float4*>(beta) + i);
  }
  __syncthreads();
  ptx::griddep_launch_dependents();
  ptx::griddep_wait();
  for (int row = blockIdx.x * wpb + (threadIdx.x >> 5); row < T; row += gridDim.x * wpb) {
    const size_t base = static_cast<size_t>(row) * k;
    uint4 xv[NCH], rv[NCH];
#pragma unroll
    for (int i = 0; i < NCH; ++i) {  // issue every load of the row before using any
      const int c = lane + 32 * i;
      xv[i] = make_uint4(0, 0, 0, 0);
      rv[i] = make_uint4(0, 0, 0, 0);
      if (c < nchunk) {
        xv[i] = __ldg(reinterpret_cast<const uint4*>(x + base) + c);
        if (res) rv[i] = __ldg(reinterpret_cast<const uint4*>(res + base) + c);
      }
    }
    float z[NCH][8];
    float sum = 0.f;
#pragma unroll
    for (int i = 0; i < NCH; ++i) {
      const int c = lane + 32 * i;
      const __nv_bfloat162* xh = reinterpret_cast<const __nv_bfloat162*>(&xv[i]);
      const __nv_bfloat162* rh = reinterpret_cast<const __nv_bfloat162*>(&rv[i]);
      float4 b0 = make_float4(0.f, 0.f, 0.f, 0.f), b1 = b0;
      if (c < nchunk) {
        b0 = sparams[2 * c];
        b1 = sparams[2 * c + 1];
      }
      const float bb[8] = {b0.x, b0.y, b0.z, b0.w, b1.x, b1.y, b1.z, b1.w};
#pragma unroll
      for (int e = 0; e < 4; ++e) {
        const float2 xf = __bfloat1622float2(xh[e]);
        const float2 rf = __bfloat1622float2(rh[e]);
        z[i][2 * e] = (xf.x + rf.x) + bb[2 * e];  // (x + residual) + bias, fusion.py:96
        z[i][2 * e + 1] = (xf.y + rf.y) + bb[2 * e + 1];
      }
      if (c < nchunk) {
#pragma unroll
        for (int e = 0; e < 8; ++e) sum += z[i][e];
      }
    }
#pragma unroll
    for (int o = 16; o; o >>= 1) sum += __shfl_xor_sync(0xffffffffu, sum, o);
    const float mean = sum * inv_k;
    float sq = 0.f;
#pragma unroll
    for (int i = 0; i < NCH; ++i) {
      if (lane + 32 * i < nchunk) {
#pragma unroll
        for (int e = 0; e < 8; ++e) {
          const float d = z[i][e] - mean;
          sq += d * d;
        }
      }
    }
#pragma unroll
    for (int o = 16; o; o >>= 1) sq += __shfl_xor_sync(0xffffffffu, sq, o);
    const float rstd = 1.0f / sqrtf(sq * inv_k + eps);
#pragma unroll
    for (int i = 0; i < NCH; ++i) {
      const int c = lane + 32 * i;
      if (c < nchunk) {
        const float4 g0 = sparams[k4 + 2 * c], g1 = sparams[k4 + 2 * c + 1];
        const float4 e0 = sparams[2 * k4 + 2 * c], e1 = sparams[2 * k4 + 2 * c + 1];
        const float gg[8] = {g0.x, g0.y, g0.z, g0.w, g1.x, g1.y, g1.z, g1.w};
        const float ee[8] = {e0.x, e0.y, e0.z, e0.w, e1.x, e1.y, e1.z, e1.w};
        uint4 o;
        uint32_t* ow = reinterpret_cast<uint32_t*>(&o);
#pragma unroll
        for (int e = 0; e < 4; ++e) {
          const float y0 = gg[2 * e] * ((z[i][2 * e] - mean) * rstd) + ee[2 * e];
          const float y1 = gg[2 * e + 1] * ((z[i][2 * e + 1] - mean) * rstd) + ee[2 * e + 1];
          ow[e] = ptx::pack_bf16x2(y0, y1);
        }
        store_row_chunk(o, out, outf, row_map, row, base, k, c);
      }
    }
  }
}

template <int NCH>
static int launch_ln(const __nv_bfloat16* x, const __nv_bfloat16* r, const float* b, const float* g, const float* be,
                      float eps, __nv_bfloat16* out, int T, int k, cudaStream_t s, float* outf, const int32_t* row_map) {
  const int threads = 256, wpb = threads / 32;
  if constexpr (NCH <= 3) {
    const int sms0 = num_sms() > 0 ? num_sms() : 148;
    long long grid0 = (T + wpb - 1) / wpb;
    if (grid0 > sms0 * 8LL) grid0 = sms0 * 8LL;
    if (grid0 < 1) grid0 = 1;
    BT_LAUNCH((ln_bias_residual_regs_kernel<NCH, true>), dim3(static_cast<int>(grid0)), dim3(threads), 0, s, 1, x, r,
              b, g, be, eps, out, T, k, outf, row_map);
    return BT_OK;
  }
  const int sms = num_sms() > 0 ? num_sms() : 148;
  const size_t smem = static_cast<size_t>(3) * k * sizeof(float);
  auto kern = ln_bias_residual_kernel<NCH>;
  static bool attr_set = false;
  if (!attr_set) {
    BT_CUDA_CHECK(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, 3 * 4096 * 4));
    attr_set = true;
  }
  int per_sm = 0;
  BT_CUDA_CHECK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, threads, smem));
  long long grid = (T + wpb - 1) / wpb;
  const long long cap = static_cast<long long>(sms) * (per_sm > 0 ? per_sm : 1);
  if (grid > cap) grid = cap;  // resident grid, rows grid-strided
  if (grid < 1) grid = 1;
  BT_LAUNCH(kern, dim3(static_cast<int>(grid)), dim3(threads), smem, s, 1, x, r, b, g, be, eps, out, T, k, outf,
            row_map);
  return BT_OK;
}

}  // namespace bt

namespace bt {
// LayerNorm with an optional fp32 final-output destination (see
// store_row_chunk); out may be null when outf is given.
int ln_launch(const void* x, const void* residual, const float* bias, const float* gamma, const float* beta, float eps,
              void* out, int T, int k, cudaStream_t s, float* outf, const int32_t* row_map) {
  BT_REQUIRE(T >= 0 && k >= 8 && k % 8 == 0 && k <= 4096, BT_ESHAPE,
             "layernorm: need k %% 8 == 0 and 8 <= k <= 4096, got k=%d", k);
  BT_REQUIRE(eps > 0.f, BT_ESHAPE, "layernorm eps must be > 0, got %g", static_cast<double>(eps));
  BT_REQUIRE(x && gamma && beta && (out || outf), BT_ESHAPE, "layernorm: null pointer");
  if (T == 0) return BT_OK;
  const auto* xb = static_cast<const __nv_bfloat16*>(x);
  const auto* rb = static_cast<const __nv_bfloat16*>(residual);
  auto* ob = static_cast<__nv_bfloat16*>(out);
  const int nch = (k / 8 + 31) / 32;
  switch (nch) {
    case 1: return launch_ln<1>(xb, rb, bias, gamma, beta, eps, ob, T, k, s, outf, row_map);
    case 2: return launch_ln<2>(xb, rb, bias, gamma, beta, eps, ob, T, k, s, outf, row_map);
    case 3: return launch_ln<3>(xb, rb, bias, gamma, beta, eps, ob, T, k, s, outf, row_map);
    case 4: return launch_ln<4>(xb, rb, bias, gamma, beta, eps, ob, T, k, s, outf, row_map);
    case 5: case 6: return launch_ln<6>(xb, rb, bias, gamma, beta, eps, ob, T, k, s, outf, row_map);
    case 7: case 8: return launch_ln<8>(xb, rb, bias, gamma, beta, eps, ob, T, k, s, outf, row_map);
    default: return launch_ln<16>(xb, rb, bias, gamma, beta, eps, ob, T, k, s, outf, row_map);
  }
}
}  // namespace bt

extern "C" int bt_ln_bias_residual(const void* x, const void* residual, const float* bias, const float* gamma,
                                   const float* beta, float eps, void* out, int T, int k, bt_stream_t stream) {
  BT_REQUIRE(out, BT_ESHAPE, "layernorm: null pointer");
  return bt::ln_launch(x, residual, bias, gamma, beta, eps, out, T, k, bt::as_stream(stream), nullptr, nullptr);
}

extern "C" int bt_ln_bias_residual_out(const void* x, const void* residual, const float* bias, const float* gamma,
                                       const float* beta, float eps, float* out_f32, const int32_t* row_map, int T,
                                       int k, bt_stream_t stream) {
  BT_REQUIRE(out_f32, BT_ESHAPE, "layernorm: null pointer");
  return bt::ln_launch(x, residual, bias, gamma, beta, eps, nullptr, T, k, bt::as_stream(stream), out_f32, row_map);
}
