// Memory-bound element-wise passes used by the unfused ladder variants and the
// operator-level API (reference fusion.py:23-76):
//   bt_bias_act: out = act(x + bias[col])  (act = identity or tanh-GELU),
//                strided rows so it can write column slices of a wider tensor
//   bt_add:      out = x + y
// bf16 or fp32 in/out, 8 elements (16 B of bf16) per thread per step.

#include <type_traits>

#include "common.cuh"
#include "ptx.cuh"

namespace bt {

__device__ __forceinline__ void ld8(const float* p, float (&v)[8]) {
  const float4 a = __ldg(reinterpret_cast<const float4*>(p));
  const float4 b = __ldg(reinterpret_cast<const float4*>(p) + 1);
  v[0] = a.x; v[1] = a.y; v[2] = a.z; v[3] = a.w; v[4] = b.x; v[5] = b.y; v[6] = b.z; v[7] = b.w;
}
__device__ __forceinline__ void ld8(const __nv_bfloat16* p, float (&v)[8]) {
  const uint4 a = __ldg(reinterpret_cast<const uint4*>(p));
  const __nv_bfloat162* h = reinterpret_cast<const __nv_bfloat162*>(&a);
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    const float2 f = __bfloat1622float2(h[i]);
    v[2 * i] = f.x;
    v[2 * i + 1] = f.y;
  }
}
__device__ __forceinline__ void st8(float* p, const float (&v)[8]) {
  reinterpret_cast<float4*>(p)[0] = make_float4(v[0], v[1], v[2], v[3]);
  reinterpret_cast<float4*>(p)[1] = make_float4(v[4], v[5], v[6], v[7]);
}
__device__ __forceinline__ void st8(__nv_bfloat16* p, const float (&v)[8]) {
  uint4 o;
  o.x = ptx::pack_bf16x2(v[0], v[1]);
  o.y = ptx::pack_bf16x2(v[2], v[3]);
  o.z = ptx::pack_bf16x2(v[4], v[5]);
  o.w = ptx::pack_bf16x2(v[6], v[7]);
  *reinterpret_cast<uint4*>(p) = o;
}

template <typename Ti, typename To, bool GELU>
__global__ void bias_act_kernel(const Ti* __restrict__ x, int ldx, const float* __restrict__ bias, To* __restrict__ out,
                                int ldo, int rows, int cols) {
  ptx::griddep_launch_dependents();
  ptx::griddep_wait();
  const int chunks = cols / 8;
  const long long total = static_cast<long long>(rows) * chunks;
  for (long long i = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; i < total;
       i += static_cast<long long>(gridDim.x) * blockDim.x) {
    const int r = static_cast<int>(i / chunks);
    const int c = static_cast<int>(i - static_cast<long long>(r) * chunks) * 8;
    float v[8];
    ld8(x + static_cast<size_t>(r) * ldx + c, v);
    if (bias) {
      float b[8];
      ld8(bias + c, b);
#pragma unroll
      for (int e = 0; e < 8; ++e) v[e] += b[e];
    }
    if constexpr (GELU) {
#pragma unroll
      for (int e = 0; e < 8; ++e) v[e] = ptx::gelu_tanh(v[e]);
    }
    st8(out + static_cast<size_t>(r) * ldo + c, v);
  }
}

template <typename T>
__global__ void add_kernel(const T* __restrict__ x, const T* __restrict__ y, T* __restrict__ out, long long n8) {
  ptx::griddep_launch_dependents();
  ptx::griddep_wait();
  for (long long i = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; i < n8;
       i += static_cast<long long>(gridDim.x) * blockDim.x) {
    float a[8], b[8];
    ld8(x + 8 * i, a);
    ld8(y + 8 * i, b);
#pragma unroll
    for (int e = 0; e < 8; ++e) a[e] += b[e];
    st8(out + 8 * i, a);
  }
}

static int ew_grid(long long items) {
  const int sms = num_sms() > 0 ? num_sms() : 148;
  long long g = (items + 255) / 256;
  if (g > sms * 8LL) g = sms * 8LL;
  return g < 1 ? 1 : static_cast<int>(g);
}

template <typename Ti, typename To>
static int launch_bias_act(const void* x, int ldx, const float* bias, void* out, int ldo, int rows, int cols, int act,
                           cudaStream_t s) {
  const int g = ew_grid(static_cast<long long>(rows) * (cols / 8));
  if (act)
    BT_LAUNCH((bias_act_kernel<Ti, To, true>), dim3(g), dim3(256), 0, s, 1, static_cast<const Ti*>(x), ldx, bias,
              static_cast<To*>(out), ldo, rows, cols);
  else
    BT_LAUNCH((bias_act_kernel<Ti, To, false>), dim3(g), dim3(256), 0, s, 1, static_cast<const Ti*>(x), ldx, bias,
              static_cast<To*>(out), ldo, rows, cols);
  return BT_OK;
}

}  // namespace bt

extern "C" BT_API int bt_bias_act(const void* x, int in_dtype, int ldx, const float* bias, void* out, int out_dtype,
                                  int ldo, int rows, int cols, int act, bt_stream_t stream) {
  BT_REQUIRE(rows >= 0 && cols >= 8 && cols % 8 == 0 && ldx >= cols && ldo >= cols && ldx % 8 == 0 && ldo % 8 == 0,
             BT_ESHAPE, "bias_act: bad shape rows=%d cols=%d ldx=%d ldo=%d", rows, cols, ldx, ldo);
  BT_REQUIRE((in_dtype == BT_F32 || in_dtype == BT_BF16) && (out_dtype == BT_F32 || out_dtype == BT_BF16), BT_ECONFIG,
             "bias_act: bad dtypes");
  if (rows == 0) return BT_OK;
  cudaStream_t s = bt::as_stream(stream);
  if (in_dtype == BT_F32 && out_dtype == BT_F32)
    return bt::launch_bias_act<float, float>(x, ldx, bias, out, ldo, rows, cols, act, s);
  if (in_dtype == BT_F32) return bt::launch_bias_act<float, __nv_bfloat16>(x, ldx, bias, out, ldo, rows, cols, act, s);
  if (out_dtype == BT_F32) return bt::launch_bias_act<__nv_bfloat16, float>(x, ldx, bias, out, ldo, rows, cols, act, s);
  return bt::launch_bias_act<__nv_bfloat16, __nv_bfloat16>(x, ldx, bias, out, ldo, rows, cols, act, s);
}

extern "C" BT_API int bt_add(const void* x, const void* y, void* out, int dtype, long long n, bt_stream_t stream) {
  BT_REQUIRE(n >= 0 && n % 8 == 0, BT_ESHAPE, "add: element count %lld must be a multiple of 8", n);
  BT_REQUIRE(dtype == BT_F32 || dtype == BT_BF16, BT_ECONFIG, "add: bad dtype");
  if (n == 0) return BT_OK;
  cudaStream_t s = bt::as_stream(stream);
  const int g = bt::ew_grid(n / 8);
  if (dtype == BT_F32)
    BT_LAUNCH(bt::add_kernel<float>, dim3(g), dim3(256), 0, s, 1, static_cast<const float*>(x),
              static_cast<const float*>(y), static_cast<float*>(out), n / 8);
  else
    BT_LAUNCH(bt::add_kernel<__nv_bfloat16>, dim3(g), dim3(256), 0, s, 1, static_cast<const __nv_bfloat16*>(x),
              static_cast<const __nv_bfloat16*>(y), static_cast<__nv_bfloat16*>(out), n / 8);
  return BT_OK;
}
