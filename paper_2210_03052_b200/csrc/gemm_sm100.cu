// Persistent, warp-specialised tcgen05 GEMM for the encoder's four
// projections (reference encoder.py:356-404; paper Fig. 2(a) GEMM #0-#3):
//
//   C[M,N] = epilogue( A[M,K] * Bt[N,K]^T )     bf16 in, fp32 accumulate
//
//   warp 0      TMA producer: A/B tiles -> STAGES-deep smem ring (128B swizzle)
//   warp 1      TMEM allocator + single-thread tcgen05.mma issuer
//   warps 2..5  epilogue: tcgen05.ld (TMEM -> regs), bias / GELU / residual,
//               bf16 pack, 16-byte global stores
//
// The accumulator is double-buffered in TMEM (2 x BN fp32 columns) so the
// epilogue of tile i overlaps the mainloop of tile i+1.  Tiles are 128 x BN
// (BN in {64, 128, 256}) with BK = 64 (one 128-byte swizzle atom of bf16).
// Epilogue kinds mirror the reference EpilogueHook (tensor.py:74-106):
// none / add_bias / add_bias_gelu (fusion.py:30-35) / bias+residual.

#include "common.cuh"
#include "ptx.cuh"
#include "tma_host.cuh"

namespace bt {

struct GemmParams {
  int M, N, K;
  __nv_bfloat16* C;
  const float* bias;
  const __nv_bfloat16* residual;
  int num_m_blocks, num_n_blocks, num_tiles;
};

constexpr int GEMM_BM = 128;
constexpr int GEMM_BK = 64;
constexpr int GEMM_THREADS = 192;

template <int BN>
struct GemmCfg {
  static constexpr uint32_t A_BYTES = GEMM_BM * GEMM_BK * 2;
  static constexpr uint32_t B_BYTES = BN * GEMM_BK * 2;
  static constexpr uint32_t STAGE_BYTES = A_BYTES + B_BYTES;
  static constexpr int STAGES = (BN == 64) ? 8 : (BN == 128 ? 6 : 4);
  static constexpr uint32_t TMEM_COLS = 2 * BN;  // 128 / 256 / 512: powers of two >= 32
  static constexpr size_t SMEM = 1024 + static_cast<size_t>(STAGES) * STAGE_BYTES + 256;
};

template <int EPI>
__device__ __forceinline__ void epilogue_store(const uint32_t (&acc)[32], const GemmParams& p, int row, int col) {
  float v[32];
#pragma unroll
  for (int i = 0; i < 32; ++i) v[i] = __uint_as_float(acc[i]);
  if constexpr (EPI == BT_EPI_BIAS_RESIDUAL) {
    const uint4* r = reinterpret_cast<const uint4*>(p.residual + static_cast<size_t>(row) * p.N + col);
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      const uint4 rv = __ldg(r + q);
      const __nv_bfloat162* rh = reinterpret_cast<const __nv_bfloat162*>(&rv);
#pragma unroll
      for (int e = 0; e < 4; ++e) {
        const float2 f = __bfloat1622float2(rh[e]);
        v[q * 8 + 2 * e] += f.x;
        v[q * 8 + 2 * e + 1] += f.y;
      }
    }
  }
  if constexpr (EPI != BT_EPI_NONE) {
    const float4* b4 = reinterpret_cast<const float4*>(p.bias + col);
#pragma unroll
    for (int q = 0; q < 8; ++q) {
      const float4 b = __ldg(b4 + q);
      v[4 * q] += b.x;
      v[4 * q + 1] += b.y;
      v[4 * q + 2] += b.z;
      v[4 * q + 3] += b.w;
    }
  }
  if constexpr (EPI == BT_EPI_BIAS_GELU) {
#pragma unroll
    for (int i = 0; i < 32; ++i) v[i] = ptx::gelu_tanh(v[i]);
  }
  uint4* dst = reinterpret_cast<uint4*>(p.C + static_cast<size_t>(row) * p.N + col);
#pragma unroll
  for (int q = 0; q < 4; ++q) {
    uint4 o;
    o.x = ptx::pack_bf16x2(v[8 * q + 0], v[8 * q + 1]);
    o.y = ptx::pack_bf16x2(v[8 * q + 2], v[8 * q + 3]);
    o.z = ptx::pack_bf16x2(v[8 * q + 4], v[8 * q + 5]);
    o.w = ptx::pack_bf16x2(v[8 * q + 6], v[8 * q + 7]);
    dst[q] = o;
  }
}

template <int BN, int EPI>
__global__ void __launch_bounds__(GEMM_THREADS, 1)
    gemm_bf16_tcgen05_kernel(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB,
                             const GemmParams p) {
  using Cfg = GemmCfg<BN>;
  constexpr int STAGES = Cfg::STAGES;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* sA = smem;
  uint8_t* sB = smem + STAGES * Cfg::A_BYTES;
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + STAGES * Cfg::STAGE_BYTES);
  uint64_t* empty = full + STAGES;
  uint64_t* tfull = empty + STAGES;
  uint64_t* tempty = tfull + 2;
  uint32_t* tmem_holder = reinterpret_cast<uint32_t*>(tempty + 2);

  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;
  const int num_k = p.K / GEMM_BK;

  if (warp == 0 && lane == 0) {
    ptx::prefetch_tmap(&tmA);
    ptx::prefetch_tmap(&tmB);
    for (int s = 0; s < STAGES; ++s) {
      ptx::mbar_init(&full[s], 1);
      ptx::mbar_init(&empty[s], 1);
    }
    for (int a = 0; a < 2; ++a) {
      ptx::mbar_init(&tfull[a], 1);
      ptx::mbar_init(&tempty[a], 128);
    }
    ptx::fence_mbar_init();
  }
  if (warp == 1) {
    ptx::tmem_alloc(tmem_holder, Cfg::TMEM_COLS);
    ptx::tmem_relinquish();
  }
  ptx::tc_fence_before();
  __syncthreads();
  ptx::tc_fence_after();
  const uint32_t tmem_base = *tmem_holder;

  if (warp == 0) {
    if (lane == 0) {
      // ---------------- TMA producer
      int stage = 0;
      uint32_t phase = 0;
      for (int tile = blockIdx.x; tile < p.num_tiles; tile += gridDim.x) {
        const int mb = tile % p.num_m_blocks;
        const int nb = tile / p.num_m_blocks;
        for (int kb = 0; kb < num_k; ++kb) {
          ptx::mbar_wait(&empty[stage], phase ^ 1u);
          ptx::mbar_arrive_expect_tx(&full[stage], Cfg::STAGE_BYTES);
          ptx::tma_load_2d(sA + stage * Cfg::A_BYTES, &tmA, &full[stage], kb * GEMM_BK, mb * GEMM_BM);
          ptx::tma_load_2d(sB + stage * Cfg::B_BYTES, &tmB, &full[stage], kb * GEMM_BK, nb * BN);
          if (++stage == STAGES) {
            stage = 0;
            phase ^= 1u;
          }
        }
      }
    }
  } else if (warp == 1) {
    if (lane == 0) {
      // ---------------- MMA issuer (one thread)
      constexpr uint32_t idesc = ptx::idesc_bf16(GEMM_BM, BN, false, false);
      int stage = 0;
      uint32_t phase = 0;
      int it = 0;
      for (int tile = blockIdx.x; tile < p.num_tiles; tile += gridDim.x, ++it) {
        const int acc = it & 1;
        const uint32_t aphase = (it >> 1) & 1;
        ptx::mbar_wait(&tempty[acc], aphase ^ 1u);
        ptx::tc_fence_after();
        const uint32_t d_tmem = tmem_base + acc * BN;
        for (int kb = 0; kb < num_k; ++kb) {
          ptx::mbar_wait(&full[stage], phase);
          ptx::tc_fence_after();
          const uint32_t a0 = ptx::smem_u32(sA + stage * Cfg::A_BYTES);
          const uint32_t b0 = ptx::smem_u32(sB + stage * Cfg::B_BYTES);
#pragma unroll
          for (int k = 0; k < GEMM_BK / 16; ++k) {
            const uint64_t ad = ptx::sdesc_sw128(a0 + k * 32, 1024, 16);
            const uint64_t bd = ptx::sdesc_sw128(b0 + k * 32, 1024, 16);
            ptx::mma_bf16_ss(d_tmem, ad, bd, idesc, (kb | k) != 0);
          }
          ptx::mma_commit(&empty[stage]);  // frees the smem slot when these MMAs retire
          if (++stage == STAGES) {
            stage = 0;
            phase ^= 1u;
          }
        }
        ptx::mma_commit(&tfull[acc]);  // accumulator ready for the epilogue
      }
    }
  } else {
    // ---------------- epilogue warps 2..5; warp w owns TMEM lanes 32*(w%4)
    const int quarter = warp & 3;
    const int row_in_tile = quarter * 32 + lane;
    int it = 0;
    for (int tile = blockIdx.x; tile < p.num_tiles; tile += gridDim.x, ++it) {
      const int acc = it & 1;
      const uint32_t aphase = (it >> 1) & 1;
      const int mb = tile % p.num_m_blocks;
      const int nb = tile / p.num_m_blocks;
      ptx::mbar_wait(&tfull[acc], aphase);
      ptx::tc_fence_after();
      const int row = mb * GEMM_BM + row_in_tile;
      const uint32_t taddr = tmem_base + (static_cast<uint32_t>(quarter * 32) << 16) + acc * BN;
#pragma unroll 1
      for (int c = 0; c < BN; c += 32) {
        uint32_t r[32];
        ptx::tmem_ld32(taddr + c, r);
        ptx::tmem_wait_ld(r);
        if (row < p.M) epilogue_store<EPI>(r, p, row, nb * BN + c);
      }
      ptx::tc_fence_before();
      ptx::mbar_arrive(&tempty[acc]);
    }
  }

  ptx::tc_fence_before();
  __syncthreads();
  if (warp == 1) {
    ptx::tc_fence_after();
    ptx::tmem_dealloc(tmem_base, Cfg::TMEM_COLS);
  }
}

template <int BN, int EPI>
static int launch_gemm_t(const CUtensorMap& ta, const CUtensorMap& tb, const GemmParams& p, int grid,
                         cudaStream_t s) {
  using Cfg = GemmCfg<BN>;
  auto kern = gemm_bf16_tcgen05_kernel<BN, EPI>;
  static bool attr_set = false;  // one flag per instantiation
  if (!attr_set) {
    BT_CUDA_CHECK(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(Cfg::SMEM)));
    attr_set = true;
  }
  kern<<<grid, GEMM_THREADS, Cfg::SMEM, s>>>(ta, tb, p);
  BT_LAUNCH_CHECK();
  return BT_OK;
}

template <int BN>
static int dispatch_epi(int epi, const CUtensorMap& ta, const CUtensorMap& tb, const GemmParams& p, int grid,
                        cudaStream_t s) {
  switch (epi) {
    case BT_EPI_NONE: return launch_gemm_t<BN, BT_EPI_NONE>(ta, tb, p, grid, s);
    case BT_EPI_BIAS: return launch_gemm_t<BN, BT_EPI_BIAS>(ta, tb, p, grid, s);
    case BT_EPI_BIAS_GELU: return launch_gemm_t<BN, BT_EPI_BIAS_GELU>(ta, tb, p, grid, s);
    default: return launch_gemm_t<BN, BT_EPI_BIAS_RESIDUAL>(ta, tb, p, grid, s);
  }
}

// Pick BN to minimise (waves x per-tile mainloop cycles): small-M problems
// (T = 1-5k packed rows) otherwise leave most of the 148 SMs idle.
static int choose_bn(int M, int N, int K, int sms) {
  const int cands[3] = {256, 128, 64};
  int best = 64;
  double best_cost = 1e30;
  const int mblocks = (M + GEMM_BM - 1) / GEMM_BM;
  for (int bn : cands) {
    if (N % bn) continue;
    const long long tiles = static_cast<long long>(mblocks) * (N / bn);
    const long long waves = (tiles + sms - 1) / sms;
    const double cost = static_cast<double>(waves) * (bn * (K / 32.0) + 700.0);
    if (cost < best_cost - 1e-9) {
      best_cost = cost;
      best = bn;
    }
  }
  return best;
}

int gemm_launch(const void* A, const void* Bt, const float* bias, const void* residual, void* C, int M, int N,
                int K, int epi, int force_bn, cudaStream_t s) {
  BT_REQUIRE(M >= 0 && N > 0 && K > 0, BT_ESHAPE, "gemm: bad shape M=%d N=%d K=%d", M, N, K);
  BT_REQUIRE(K % GEMM_BK == 0, BT_ESHAPE, "gemm: K=%d must be a multiple of 64", K);
  BT_REQUIRE(N % 64 == 0, BT_ESHAPE, "gemm: N=%d must be a multiple of 64", N);
  BT_REQUIRE(epi >= BT_EPI_NONE && epi <= BT_EPI_BIAS_RESIDUAL, BT_ECONFIG, "gemm: unknown epilogue %d", epi);
  BT_REQUIRE(epi == BT_EPI_NONE || bias != nullptr, BT_ESHAPE, "gemm: epilogue %d needs a bias", epi);
  BT_REQUIRE(epi != BT_EPI_BIAS_RESIDUAL || residual != nullptr, BT_ESHAPE, "gemm: residual epilogue needs residual");
  if (M == 0) return BT_OK;
  const int sms = num_sms() > 0 ? num_sms() : 148;
  const int bn = force_bn ? force_bn : choose_bn(M, N, K, sms);
  BT_REQUIRE(N % bn == 0, BT_ESHAPE, "gemm: N=%d not a multiple of BN=%d", N, bn);
  CUtensorMap ta, tb;
  BT_TRY(make_tmap_bf16_2d(&ta, A, M, K, K, GEMM_BM, GEMM_BK));
  BT_TRY(make_tmap_bf16_2d(&tb, Bt, N, K, K, bn, GEMM_BK));
  GemmParams p;
  p.M = M;
  p.N = N;
  p.K = K;
  p.C = static_cast<__nv_bfloat16*>(C);
  p.bias = bias;
  p.residual = static_cast<const __nv_bfloat16*>(residual);
  p.num_m_blocks = (M + GEMM_BM - 1) / GEMM_BM;
  p.num_n_blocks = N / bn;
  p.num_tiles = p.num_m_blocks * p.num_n_blocks;
  const int grid = p.num_tiles < sms ? p.num_tiles : sms;
  switch (bn) {
    case 64: return dispatch_epi<64>(epi, ta, tb, p, grid, s);
    case 128: return dispatch_epi<128>(epi, ta, tb, p, grid, s);
    default: return dispatch_epi<256>(epi, ta, tb, p, grid, s);
  }
}

}  // namespace bt

extern "C" int bt_gemm(const void* A, const void* Bt, const float* bias, const void* residual, void* C, int M,
                       int N, int K, int epilogue, bt_stream_t stream) {
  return bt::gemm_launch(A, Bt, bias, residual, C, M, N, K, epilogue, 0, bt::as_stream(stream));
}

// Test hook: force a tile width (64/128/256) so every instantiation is covered.
extern "C" int bt_gemm_bn(const void* A, const void* Bt, const float* bias, const void* residual, void* C, int M,
                          int N, int K, int epilogue, int bn, bt_stream_t stream) {
  BT_REQUIRE(bn == 64 || bn == 128 || bn == 256, BT_ECONFIG, "bt_gemm_bn: bn must be 64/128/256, got %d", bn);
  return bt::gemm_launch(A, Bt, bias, residual, C, M, N, K, epilogue, bn, bt::as_stream(stream));
}
